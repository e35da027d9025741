mkdir -p gpurun_out/r02k
exec > gpurun_out/r02k/log.txt 2>&1
./tools/microbench/hsub
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py -m gpu -q -x -k "batch or tensor or fused" 2>&1 | tail -4; echo "tests rc=$?"
timeout 900 python bench.py --config C4 --no-cpu-baseline > gpurun_out/r02k/c4.json 2> gpurun_out/r02k/c4.err; echo "c4 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02k/c4.json')); print('C4', d['value'], 'tensor', d['tensor_mode']['value'], d['tensor_mode']['mean_iterations'])"
