timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5c.log
timeout 300 python tools/profile_kernels.py --what msolve_tc > gpurun_out/prof_tc_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16tc -s 2 -c 1 -o gpurun_out/prof_tc python tools/profile_kernels.py --what msolve_tc > gpurun_out/ncu_tc.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log; tail -c 600 gpurun_out/bench_c5c.log; cat gpurun_out/prof_tc_plain.log
