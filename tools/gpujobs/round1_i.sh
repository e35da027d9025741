timeout 900 python bench.py --config C4 --warmup 1 > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 1 --warmup 1 --n 1024 --no-cpu-baseline --no-dense --dist-backend gloo > gpurun_out/bench_2rank.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2rank.log
timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -q -k "c3" > gpurun_out/pytest_c3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c3.log
timeout 300 python tools/tensor_profile.py > gpurun_out/tp_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 120 --csv --log-file gpurun_out/launches_tensor.csv python tools/tensor_profile.py > gpurun_out/ncu_launch.log 2>&1
tail -c 1500 gpurun_out/bench_c4.log; tail -c 800 gpurun_out/bench_2rank.log; tail -n 3 gpurun_out/pytest_c3.log
