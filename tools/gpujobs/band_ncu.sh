KP_BAND_A=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"band_cols_kernel|band_rows_kernel" -s 2 -c 2 -o gpurun_out/band_full python tools/time_op.py > gpurun_out/band_full.log 2>&1; echo rc=$?
tail -n 2 gpurun_out/band_full.log
