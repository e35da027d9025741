# banded operator: timing, launch list, parity tests, one full capture of both passes
exec > gpurun_out/band/log.txt 2>&1
timeout 300 python tools/time_op.py 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"band_" --csv --log-file gpurun_out/band/spec.csv python tools/time_op.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/band/spec.csv
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_configs.py -q -m gpu -x -k "band or operator or kronsum" 2>&1 | tail -2



