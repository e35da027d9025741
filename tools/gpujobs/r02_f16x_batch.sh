mkdir -p gpurun_out/r02j
exec > gpurun_out/r02j/log.txt 2>&1
timeout 900 python tools/f16x_batch_time.py
