for b in 1 2; do KP_BAND_B_BUF=$b timeout 300 python tools/time_op.py 2>&1 | tail -1; done
KP_BAND_B_BUF=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"band_" --csv --log-file gpurun_out/launches_band1.csv python tools/time_op.py > /dev/null 2>&1
KP_BAND_B_BUF=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"band_" --csv --log-file gpurun_out/launches_band2.csv python tools/time_op.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_band1.csv; python tools/launch_summary.py gpurun_out/launches_band2.csv
