for a in 0 1; do KP_BAND_A=$a timeout 300 python tools/time_op.py > gpurun_out/to_$a.txt 2>&1; tail -n 1 gpurun_out/to_$a.txt; done
for a in 0 1; do KP_BAND_A=$a timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"band_" --csv --log-file gpurun_out/launches_band5_$a.csv python tools/time_op.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches_band5_$a.csv; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -m gpu -x -k "band or operator or kronsum" 2>&1 | tail -2
