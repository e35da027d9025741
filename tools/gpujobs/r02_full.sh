# full GPU suite + smoke + bench lines (C5 default, C4 batch) + reference arm
mkdir -p gpurun_out/r02g
exec > gpurun_out/r02g/log.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02g/bench_c5.json 2> gpurun_out/r02g/bench_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --config C4 > gpurun_out/r02g/bench_c4.json 2> gpurun_out/r02g/bench_c4.err; echo "bench c4 rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02g/bench_ref_c5.json 2> gpurun_out/r02g/bench_ref_c5.err; echo "ref rc=$?"
for f in bench_c5 bench_c4 bench_ref_c5; do python -c "
import json; d=json.load(open('gpurun_out/r02g/$f.json'))
print('$f', d['metric'][:40], d['value'], d.get('e2e',{}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('cpu_baseline') or {}).get('value'))"; done
