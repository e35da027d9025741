mkdir -p gpurun_out/r02b2
exec > gpurun_out/r02b2/log.txt 2>&1
for c in C5 C2 C1 C3 C4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02b2/$c.json 2> gpurun_out/r02b2/$c.err
  python -c "
import json; d=json.load(open('gpurun_out/r02b2/$c.json')); print('$c', d['value'], d['e2e']['value'], d.get('clocks'))"
done
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
