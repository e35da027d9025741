# round-2 first check: GPU tests, smoke, C5 bench (f16x default), launch list
mkdir -p gpurun_out/r02a
exec > gpurun_out/r02a/log.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02a/bench_c5.json 2> gpurun_out/r02a/bench_c5.err; echo "bench rc=$?"
cut -c1-3000 gpurun_out/r02a/bench_c5.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kp::|gemm_|band_|pcg_|cgls_|cast_|copy_|weights_|spectral_|finish_|fill_|f16x" --csv --log-file gpurun_out/r02a/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02a/ncu_list.log 2>&1; echo "list rc=$?"
python tools/launch_summary.py gpurun_out/r02a/launches_c5.csv | head -30
