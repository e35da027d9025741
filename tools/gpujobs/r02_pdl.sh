mkdir -p gpurun_out/r02pdl
exec > gpurun_out/r02pdl/log.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_loop.py tests/test_gpu_batch.py tests/test_gpu_parity.py -q -x 2>&1 | tail -4
for v in notrig trig; do
  cp _variants/$v.so paper_2311_15393_b200/_lib/libkronprec_b200.so
  for c in C1 C2 C5; do
    timeout 900 python bench.py --config $c --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02pdl/${c}_$v.json 2> gpurun_out/r02pdl/${c}_$v.err
    python -c "
import json; d=json.load(open('gpurun_out/r02pdl/${c}_$v.json')); print('$c $v', d['value'], d['e2e']['value'], d['gpu_launches'])"
  done
done
