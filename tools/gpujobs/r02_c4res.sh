mkdir -p gpurun_out/r02c4res
exec > gpurun_out/r02c4res/log.txt 2>&1
timeout 900 python bench.py --config C4 --no-cpu-baseline > gpurun_out/r02c4res/C4.json 2> gpurun_out/r02c4res/C4.err; echo rc=$?; tail -3 gpurun_out/r02c4res/C4.err
python -c "
import json; d=json.loads(open('gpurun_out/r02c4res/C4.json').read().strip().splitlines()[-1]); print('C4 value', d['value'], 'e2e', d['e2e']['value'], d['ms_per_step'], d['tensor_mode']['value'])"
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_abi.py tests/test_bench_contract.py -q -x 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 2 --config C4 --size 256 --dist-backend gloo --no-cpu-baseline --no-tensor > gpurun_out/r02c4res/mr.json 2> gpurun_out/r02c4res/mr.err; echo "2-rank rc=$?"; cut -c1-300 gpurun_out/r02c4res/mr.json
