# round-1 measurement set: bench lines (C5 default, C1-C4), reference arm, launch list, ncu captures
mkdir -p gpurun_out/measure
timeout 900 python bench.py > gpurun_out/measure/bench_c5.json 2> gpurun_out/measure/bench_c5.err; echo "c5 rc=$?"
for c in C1 C2 C3; do timeout 900 python bench.py --config $c > gpurun_out/measure/bench_$c.json 2> gpurun_out/measure/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --config C4 --workers 6 > gpurun_out/measure/bench_C4.json 2> gpurun_out/measure/bench_C4.err; echo "C4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/measure/bench_ref_c5.json 2> gpurun_out/measure/bench_ref_c5.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kp::|gemm_|band_|pcg_|cgls_|cast_|copy_|weights_|spectral_|finish_|fill_" --csv --log-file gpurun_out/measure/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs > gpurun_out/measure/ncu_list.log 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16ref_kernel -s 20 -c 1 -o gpurun_out/measure/r01_gemm_f16ref_u64_n4096 python bench.py --steps 1 --warmup 3 --no-tensor --no-dense --no-cpu-baseline --no-other-runs > gpurun_out/measure/ncu_f16ref.log 2>&1; echo "f16ref rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16tc_kernel -s 8 -c 4 -o gpurun_out/measure/r01_gemm_f16tc_solve_n4096 python bench.py --steps 1 --warmup 1 --no-dense --no-cpu-baseline --no-other-runs > gpurun_out/measure/ncu_f16tc.log 2>&1; echo "f16tc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"band_rows_kernel|band_cols_kernel|pcg_update_kernel|pcg_p_update_kernel" -s 8 -c 4 -o gpurun_out/measure/r01_band_vec_n4096 python bench.py --steps 1 --warmup 3 --no-tensor --no-dense --no-cpu-baseline --no-other-runs > gpurun_out/measure/ncu_band.log 2>&1; echo "band rc=$?"
ls -la gpurun_out/measure
