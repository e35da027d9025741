timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"band_" --csv --log-file gpurun_out/lb_6.csv python tools/time_op.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/lb_6.csv
timeout 300 python tools/time_op.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -m gpu -x -k "band or operator or kronsum" 2>&1 | tail -2
