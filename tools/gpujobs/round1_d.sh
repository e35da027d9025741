timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_configs.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python -m pytest tests/test_gpu_configs.py -m gpu -q -k "c1 or c2" > gpurun_out/pytest_cfg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cfg.log
timeout 900 python tools/c5_modes.py > gpurun_out/c5_modes.log 2>&1
tail -n 5 gpurun_out/pytest_gpu.log gpurun_out/pytest_cfg.log; cat gpurun_out/c5_modes.log | tail -20
