# ncu evidence for round 2: launch list of the C5 bench step, a full capture of gemm_f16x in the
# C5 solve, and the other configs' bench lines
mkdir -p gpurun_out/r02h
exec > gpurun_out/r02h/log.txt 2>&1
for c in C1 C2 C3; do timeout 900 python bench.py --config $c > gpurun_out/r02h/bench_$c.json 2> gpurun_out/r02h/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02h/plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02h/ncu_list.log 2>&1; echo "list rc=$?"
python tools/launch_summary.py gpurun_out/r02h/launches_c5.csv | head -20
python tools/c5_solve_once.py 5 > gpurun_out/r02h/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x_kernel -s 8 -c 1 -o gpurun_out/r02h/f16x_c5 python tools/c5_solve_once.py 5 > gpurun_out/r02h/ncu_full.log 2>&1; echo "full rc=$?"
for c in C1 C2 C3; do python -c "
import json; d=json.load(open('gpurun_out/r02h/bench_$c.json'))
print('$c', d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline']['value'])"; done
