timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_m.log 2>&1; echo "pytest rc=$?"
tail -n 5 gpurun_out/pytest_gpu_m.log
