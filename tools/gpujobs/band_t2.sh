timeout 300 python tools/time_op.py 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"band_" --csv --log-file gpurun_out/launches_band3.csv python tools/time_op.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_band3.csv
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_configs.py -q -m gpu -x 2>&1 | tail -2
