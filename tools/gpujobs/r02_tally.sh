mkdir -p gpurun_out/r02tally
exec > gpurun_out/r02tally/log.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_lpblas.py tests/test_cpp_api.py tests/test_abi.py -q -x 2>&1 | tail -5
