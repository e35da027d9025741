mkdir -p gpurun_out/r02l
exec > gpurun_out/r02l/log.txt 2>&1
timeout 600 python tools/f16x_data_time.py
