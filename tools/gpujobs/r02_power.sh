mkdir -p gpurun_out/r02m
exec > gpurun_out/r02m/log.txt 2>&1
timeout 600 python tools/power_probe.py
