set -x
./tools/microbench/mb > gpurun_out/mb2.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_c5b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5b.log
timeout 300 python tools/profile_kernels.py --what op > gpurun_out/prof_op_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 1 -c 1 -o gpurun_out/prof_op python tools/profile_kernels.py --what op > gpurun_out/ncu_op.log 2>&1
timeout 300 python tools/profile_kernels.py --what msolve > gpurun_out/prof_ms_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16ref -s 2 -c 1 -o gpurun_out/prof_msolve python tools/profile_kernels.py --what msolve > gpurun_out/ncu_ms.log 2>&1
tail -3 gpurun_out/pytest_gpu.log gpurun_out/mb2.log
