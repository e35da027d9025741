mkdir -p gpurun_out/r02w
exec > gpurun_out/r02w/log.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_batch.py tests/test_gpu_problem_dev.py -m gpu -q 2>&1 | tail -6; echo "rc=$?"
