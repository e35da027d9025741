timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 1 --warmup 1 --size 1024 --no-cpu-baseline --no-dense --dist-backend gloo > gpurun_out/bench_2rank.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2rank.log
timeout 300 python tools/profile_kernels.py --what op > gpurun_out/prof_op_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_ -s 2 -c 2 -o gpurun_out/prof_band python tools/profile_kernels.py --what op > gpurun_out/ncu_band.log 2>&1
timeout 300 python tools/profile_kernels.py --what msolve > gpurun_out/prof_ms_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16ref -s 6 -c 1 -o gpurun_out/prof_f16ref2 python tools/profile_kernels.py --what msolve > gpurun_out/ncu_f16ref2.log 2>&1
tail -c 1000 gpurun_out/bench_2rank.log; ls -la gpurun_out/*.ncu-rep
