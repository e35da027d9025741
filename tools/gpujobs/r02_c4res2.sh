mkdir -p gpurun_out/r02c4res
exec > gpurun_out/r02c4res/log2.txt 2>&1
timeout 900 python bench.py --config C4 --no-cpu-baseline --no-tensor > gpurun_out/r02c4res/C4b.json 2> gpurun_out/r02c4res/C4b.err; echo rc=$?; tail -3 gpurun_out/r02c4res/C4b.err
python -c "
import json; d=json.loads(open('gpurun_out/r02c4res/C4b.json').read().strip().splitlines()[-1]); print('C4 value', d['value'], 'e2e', d['e2e']['value'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29545 bench.py --gpus 2 --config C4 --size 256 --dist-backend gloo --no-cpu-baseline --no-tensor > gpurun_out/r02c4res/mr2.json 2> gpurun_out/r02c4res/mr2.err; echo "2-rank rc=$?"; cut -c1-200 gpurun_out/r02c4res/mr2.json
timeout 600 python -m pytest tests/test_bench_contract.py tests/test_multirank.py -q 2>&1 | tail -2
