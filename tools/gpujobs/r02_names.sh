mkdir -p gpurun_out/r02names
exec > gpurun_out/r02names/log.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cpp_api.py tests/test_abi.py tests/test_gpu_lpblas.py -q -x 2>&1 | tail -8
