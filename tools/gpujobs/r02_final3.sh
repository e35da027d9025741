# round-2 measurement set: GPU suite, smoke, bench lines (C5 default, C1-C4), reference arm,
# launch lists for C5 and C2 (bench frac vs ncu cross-check)
mkdir -p gpurun_out/r02f3
exec > gpurun_out/r02f3/log.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02f3/bench_c5.json 2> gpurun_out/r02f3/bench_c5.err; echo "c5 rc=$?"
for c in C1 C2 C3 C4; do timeout 900 python bench.py --config $c > gpurun_out/r02f3/bench_$c.json 2> gpurun_out/r02f3/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02f3/bench_ref_c5.json 2> gpurun_out/r02f3/bench_ref_c5.err; echo "ref rc=$?"
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02f3/plain5.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f3/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02f3/ncu5.log 2>&1; echo "list5 rc=$?"
timeout 900 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02f3/plain2.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f3/launches_c2.csv python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02f3/ncu2.log 2>&1; echo "list2 rc=$?"
for f in bench_c5 bench_C1 bench_C2 bench_C3 bench_C4 bench_ref_c5; do python -c "
import json; d=json.load(open('gpurun_out/r02f3/$f.json'))
print('$f', round(d['value'],2), round(d.get('e2e',{}).get('value',0),2), (d.get('roofline') or {}).get('frac'), (d.get('roofline') or {}).get('ms_per_launch'), (d.get('cpu_baseline') or {}).get('value'))"; done
