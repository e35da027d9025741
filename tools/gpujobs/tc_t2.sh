timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tensor" 2>&1 | tail -1
timeout 900 python bench.py --no-dense --no-cpu-baseline > gpurun_out/bench_tc2.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_tc2.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['tensor_mode'])"
