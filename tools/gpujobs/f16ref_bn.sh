for bn in 64 32; do KP_F16REF_BN=$bn timeout 900 python tools/sweep_f16ref.py 0 2>&1 | tail -1; done
timeout 900 python tools/sweep_f16ref.py 0 2>&1 | tail -1
for c in C1 C2; do timeout 600 python bench.py --config $c --no-dense --no-cpu-baseline --no-tensor --no-other-runs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['metric'], d['value'], d['e2e']['value'])"; done
timeout 600 python bench.py --config C4 --workers 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['metric'][:30], d['value'])"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lpblas.py tests/test_gpu_edges.py -q -m gpu -x -k "bitwise or lp_matmul or ragged or lpblas" 2>&1 | tail -1
