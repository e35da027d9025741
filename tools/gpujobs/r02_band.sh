mkdir -p gpurun_out/r02y
exec > gpurun_out/r02y/log.txt 2>&1
for c in C5 C2 C1; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02y/$c.json 2> gpurun_out/r02y/$c.err; python -c "
import json; d=json.load(open('gpurun_out/r02y/$c.json')); o=d['roofline_other']; print('$c', round(d['value'],2), 'operator', o['kernel'][:20], round(o['achieved'],2), round(o['frac'],3))"; done
timeout 900 python bench.py --config C4 --no-cpu-baseline --no-tensor > gpurun_out/r02y/C4.json 2> gpurun_out/r02y/C4.err; python -c "
import json; d=json.load(open('gpurun_out/r02y/C4.json')); print('C4', d['value'])"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -x -k "band or operator or kronsum" 2>&1 | tail -2
