# re-entry check of HEAD: GPU suite, smoke, bench lines (C5 default, C1-C4), N=2 multi-rank line on one GPU is NOT run
mkdir -p gpurun_out/r02head
exec > gpurun_out/r02head/log.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02head/bench_c5.json 2> gpurun_out/r02head/bench_c5.err; echo "c5 rc=$?"
for c in C1 C2 C3 C4; do timeout 900 python bench.py --config $c > gpurun_out/r02head/bench_$c.json 2> gpurun_out/r02head/bench_$c.err; echo "$c rc=$?"; done
for f in bench_c5 bench_C1 bench_C2 bench_C3 bench_C4; do python -c "
import json; d=json.loads(open('gpurun_out/r02head/$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value'],2), round(d.get('e2e',{}).get('value',0),2), (d.get('roofline') or {}).get('frac'), (d.get('roofline') or {}).get('ms_per_launch'), (d.get('cpu_baseline') or {}).get('value'), d.get('gpu_launches'))"; done
