timeout 300 python tools/tensor_solve.py > gpurun_out/ts_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_f16tc|band_|pcg_|cast|copy" --csv --log-file gpurun_out/launches_tensor2.csv python tools/tensor_solve.py > gpurun_out/ncu_ts.log 2>&1
tail -2 gpurun_out/ts_plain.log gpurun_out/ncu_ts.log
