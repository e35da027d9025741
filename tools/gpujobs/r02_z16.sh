mkdir -p gpurun_out/r02o
exec > gpurun_out/r02o/log.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4; echo "pytest rc=$?"
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02o/c5.json 2> gpurun_out/r02o/c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config C4 --no-cpu-baseline > gpurun_out/r02o/c4.json 2> gpurun_out/r02o/c4.err; echo "c4 rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/r02o/c5.json')); print('C5', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['kernels'])
d=json.load(open('gpurun_out/r02o/c4.json')); print('C4', d['value'], d['roofline']['ms_per_launch'], 'tensor', d['tensor_mode']['value'])"
