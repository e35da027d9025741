timeout 300 python tools/c4_one.py > gpurun_out/c4_one.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/c4_one.py > gpurun_out/ncu_c4.log 2>&1
tail -n 2 gpurun_out/c4_one.log gpurun_out/ncu_c4.log
