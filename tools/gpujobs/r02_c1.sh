mkdir -p gpurun_out/r02r
exec > gpurun_out/r02r/log.txt 2>&1
timeout 600 python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02r/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02r/c1.csv python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02r/ncu.log 2>&1; echo "rc=$?"
python tools/launch_summary.py gpurun_out/r02r/c1.csv | head -25
