mkdir -p gpurun_out/r02lp
exec > gpurun_out/r02lp/log.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_loop.py -q -x 2>&1 | tail -15
timeout 600 python tools/solve_timeline.py C1 4 > gpurun_out/r02lp/c1_tl.txt 2>&1
for c in C1 C2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02lp/$c.json 2> gpurun_out/r02lp/$c.err
  python -c "
import json; d=json.load(open('gpurun_out/r02lp/$c.json')); print('$c', d['value'], d['e2e']['value'], d['gpu_launches'])"
done
KP_GRAPH_LOOP=0 timeout 900 python bench.py --config C1 --no-cpu-baseline --no-other-runs --no-tensor --no-dense > gpurun_out/r02lp/C1_poll.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r02lp/C1_poll.json')); print('C1 polled', d['value'], d['e2e']['value'], d['gpu_launches'])"
