mkdir -p gpurun_out/r02f64
exec > gpurun_out/r02f64/log.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "operator or kronsum or dense or fp64 or spectral or gcv or discrepancy or c5 or C5 or c3 or C3 or filtered or tma" 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/r02f64/bench_c5.json 2> gpurun_out/r02f64/bench_c5.err; echo "c5 rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/r02f64/bench_c5.json').read().strip().splitlines()[-1])
print('c5', d['value'], d['e2e']['value'], d['roofline']['frac'])
for k in ('dense_operator', 'other_runs', 'tensor_mode'):
    print(k, json.dumps(d.get(k))[:600])
PY
