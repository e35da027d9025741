# reference-exact fp16 GEMM: bitwise + timing sweep (default config), then the parity subset
timeout 900 python tools/sweep_f16ref.py 0 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lpblas.py tests/test_gpu_edges.py -q -m gpu -x -k "bitwise or lp_matmul or ragged or lpblas" 2>&1 | tail -1
