mkdir -p gpurun_out/r02f
exec > gpurun_out/r02f/log.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py -m gpu -q -x 2>&1 | tail -15; echo "batch tests rc=$?"
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_parity_large.py -m gpu -q -x 2>&1 | tail -5; echo "parity tests rc=$?"
timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-tensor > gpurun_out/r02f/bench_c4_batch.json 2> gpurun_out/r02f/bench_c4_batch.err; echo "c4 batch rc=$?"
cut -c1-2800 gpurun_out/r02f/bench_c4_batch.json; tail -3 gpurun_out/r02f/bench_c4_batch.err
timeout 600 python tools/svd_time.py device host
KP_SVD_ALGO=gesvdj timeout 600 python tools/svd_time.py device
timeout 600 python tools/c4_batch_profile.py > gpurun_out/r02f/c4prof.txt 2>&1; tail -30 gpurun_out/r02f/c4prof.txt
