mkdir -p gpurun_out/r02fold
exec > gpurun_out/r02fold/log.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fold.py tests/test_gpu_loop.py -q -x 2>&1 | tail -15
for c in C1 C1 C2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02fold/$c.json 2> gpurun_out/r02fold/$c.err
  python -c "
import json; d=json.load(open('gpurun_out/r02fold/$c.json')); print('$c', d['value'], d['e2e']['value'], d['gpu_launches'])"
done
KP_FOLD_SCALARS=0 timeout 900 python bench.py --config C1 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02fold/C1_nofold.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r02fold/C1_nofold.json')); print('C1 nofold', d['value'], d['e2e']['value'], d['gpu_launches'])"
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
