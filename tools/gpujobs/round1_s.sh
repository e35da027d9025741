timeout 300 python tools/time_op.py > gpurun_out/time_op_s.txt 2>&1; cat gpurun_out/time_op_s.txt | tail -2
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py --config C2 --no-dense --no-cpu-baseline > gpurun_out/bench_s_c2a.json 2>&1
timeout 900 python bench.py --config C2 --no-dense --no-cpu-baseline > gpurun_out/bench_s_c2b.json 2>&1
timeout 900 python bench.py --no-dense --no-cpu-baseline > gpurun_out/bench_s_c5.json 2>&1
for f in gpurun_out/bench_s_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['profiled_pass']['value'], (d.get('tensor_mode') or {}).get('value'), d['roofline_other']['achieved'], d['roofline_other']['frac'])"; done
