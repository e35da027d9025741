mkdir -p gpurun_out/r02hash
exec > gpurun_out/r02hash/log2.txt 2>&1
timeout 600 python tools/f16x_quick.py 2>&1 | tail -1
for c in C5 C4 C2; do
  a=""; [ $c = C5 ] || a="--config $c"
  timeout 900 python bench.py $a --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02hash/$c.json 2> gpurun_out/r02hash/$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/r02hash/$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['e2e']['value'])"
done
timeout 1500 python -m pytest tests -m gpu -q -x -k "batch or large or lpblas or edges or fold or loop" 2>&1 | tail -3
