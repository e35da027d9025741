timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_q.log
timeout 900 python bench.py > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
timeout 600 python bench.py --config C1 --no-dense > gpurun_out/bench_q_c1.json 2> gpurun_out/bench_q_c1.err; echo "c1 rc=$?"
timeout 900 python bench.py --config C4 --workers 8 > gpurun_out/bench_q_c4_w8.json 2> gpurun_out/bench_q_c4.err; echo "c4 rc=$?"
for f in gpurun_out/bench_q*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d.get('e2e',{}) and d['e2e'].get('value'), (d.get('roofline') or {}).get('frac'), (d.get('tensor_mode') or {}).get('value'), (d.get('profiled_pass') or {}).get('value'), d.get('kernels') and {k:round(v['share'],3) for k,v in d['kernels'].items()})"; done
