mkdir -p gpurun_out/r02z
exec > gpurun_out/r02z/log.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02z/c5.json 2> gpurun_out/r02z/c5.err; python -c "
import json; d=json.load(open('gpurun_out/r02z/c5.json')); print('C5', d['value'], d['e2e']['value'], d['kernels']['vector'])"
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02z/plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z/l5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02z/ncu.log 2>&1; echo "list rc=$?"
python tools/launch_summary.py gpurun_out/r02z/l5.csv | head -12
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x 2>&1 | tail -2
