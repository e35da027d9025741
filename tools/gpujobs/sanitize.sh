export PYTHONPATH=$PWD
timeout 1500 compute-sanitizer --tool memcheck --leak-check none --print-limit 20 python -m pytest tests/test_gpu_edges.py tests/test_gpu_lpblas.py -q -m gpu -x -k "not ragged and not 64-64-64 and not 2-1000" > gpurun_out/memcheck1.log 2>&1; echo "rc=$?"
grep -E "ERROR SUMMARY|Invalid|passed|failed" gpurun_out/memcheck1.log | head -20
timeout 1500 compute-sanitizer --tool memcheck --leak-check none --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "kats or scalar_preconditioner or banded_normal or spectral_data or opt_wgcv or tensor_mode_precond_solve and 16" > gpurun_out/memcheck2.log 2>&1; echo "rc=$?"
grep -E "ERROR SUMMARY|Invalid|passed|failed" gpurun_out/memcheck2.log | head -20
