mkdir -p gpurun_out/r02vec
exec > gpurun_out/r02vec/log.txt 2>&1
timeout 900 python -m pytest tests/test_bench_contract.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02vec/c5.json 2> gpurun_out/r02vec/c5.err; echo rc=$?
python - <<'PY'
import json
d = json.loads(open('gpurun_out/r02vec/c5.json').read().strip().splitlines()[-1])
print(d['value'], json.dumps(d['roofline_vector'], indent=1))
PY
