mkdir -p gpurun_out/r02p
exec > gpurun_out/r02p/log.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6; echo "pytest rc=$?"
for c in C1 C2; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-other-runs > gpurun_out/r02p/$c.json 2> gpurun_out/r02p/$c.err; python -c "
import json; d=json.load(open('gpurun_out/r02p/$c.json')); print('$c', d['value'], d['e2e']['value'], d['roofline']['frac'])"; done
