# bench (C5 default) + launch list of the same command + ncu full captures of the top kernels
timeout 900 python bench.py > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err; echo "bench rc=$?"
cat gpurun_out/bench_o.json | cut -c1-300
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_o.csv python bench.py --steps 1 --warmup 3 --no-tensor --no-dense --no-cpu-baseline > gpurun_out/ncu_bench_o.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16ref_kernel -s 20 -c 1 -o gpurun_out/r01_gemm_f16ref_n4096_v2 python bench.py --steps 1 --warmup 3 --no-tensor --no-dense --no-cpu-baseline > gpurun_out/ncu_full_f16ref.log 2>&1; echo "ncu f16ref rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"band_rows_kernel|band_cols_kernel|pcg_update_kernel" -s 6 -c 3 -o gpurun_out/r01_band_vec_n4096 python bench.py --steps 1 --warmup 3 --no-tensor --no-dense --no-cpu-baseline > gpurun_out/ncu_full_band.log 2>&1; echo "ncu band rc=$?"
tail -n 3 gpurun_out/ncu_full_f16ref.log gpurun_out/ncu_full_band.log
