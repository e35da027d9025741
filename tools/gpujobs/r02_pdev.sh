mkdir -p gpurun_out/r02t
exec > gpurun_out/r02t/log.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_problem_dev.py -m gpu -q 2>&1 | tail -25; echo "rc=$?"
