for i in 1 2; do timeout 900 python bench.py --no-tensor --no-dense --no-cpu-baseline > gpurun_out/bench_r$i.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_r$i.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['profiled_pass']['value'])"; done
timeout 900 python bench.py --no-dense --no-cpu-baseline > gpurun_out/bench_r3.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_r3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['profiled_pass']['value'], d['tensor_mode']['value'])"
