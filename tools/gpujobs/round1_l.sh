# vector kernels vectorised + f16tc F64 epilogue batching: tests, launch list, bench
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_l.log 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/pytest_gpu_l.log
timeout 300 python tools/tensor_solve.py > gpurun_out/ts_plain_l.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_f16tc|band_|pcg_|cast|copy" --csv --log-file gpurun_out/launches_tensor_l.csv python tools/tensor_solve.py > gpurun_out/ncu_ts_l.log 2>&1
tail -n 2 gpurun_out/ts_plain_l.log
timeout 900 python bench.py > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; echo "bench rc=$?"
cat gpurun_out/bench_l.json
