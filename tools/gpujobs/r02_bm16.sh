mkdir -p gpurun_out/r02bm
exec > gpurun_out/r02bm/log.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_loop.py tests/test_gpu_batch.py tests/test_gpu_parity.py tests/test_gpu_lpblas.py tests/test_gpu_parity_large.py -q -x 2>&1 | tail -4
for c in C1 C1 C2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02bm/$c.json 2> gpurun_out/r02bm/$c.err
  python -c "
import json; d=json.load(open('gpurun_out/r02bm/$c.json')); print('$c', d['value'], d['e2e']['value'], d['gpu_launches'], d['run_info'].get('iterations_per_solve'), d['kernels'])"
done
KP_F16REF_BM=32 timeout 900 python bench.py --config C1 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02bm/C1_bm32.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r02bm/C1_bm32.json')); print('C1 bm32', d['value'], d['e2e']['value'], d['kernels'])"
