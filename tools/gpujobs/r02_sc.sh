mkdir -p gpurun_out/r02x
exec > gpurun_out/r02x/log.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4; echo "pytest rc=$?"
for c in C1 C2; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-other-runs --no-tensor > gpurun_out/r02x/$c.json 2> gpurun_out/r02x/$c.err; python -c "
import json; d=json.load(open('gpurun_out/r02x/$c.json')); print('$c', d['value'], d['e2e']['value'])"; done
timeout 900 python bench.py --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02x/c5.json 2> gpurun_out/r02x/c5.err; python -c "
import json; d=json.load(open('gpurun_out/r02x/c5.json')); print('C5', d['value'], d['e2e']['value'])"
