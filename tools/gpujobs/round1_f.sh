timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_configs.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python -m pytest tests/test_gpu_configs.py -m gpu -q > gpurun_out/pytest_cfg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cfg.log
timeout 600 python tools/tensor_profile.py > gpurun_out/tensor_profile.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_c5e.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5e.log
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/pytest_cfg.log; cat gpurun_out/tensor_profile.log | tail -3; tail -c 1500 gpurun_out/bench_c5e.log
