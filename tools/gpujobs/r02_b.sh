# new large-size parity tests, bench with the new accounting, full ncu capture of gemm_f16x
mkdir -p gpurun_out/r02b
exec > gpurun_out/r02b/log.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity_large.py tests/test_bench_contract.py "tests/test_gpu_configs.py::test_tensor_mode_at_config_scale" -m gpu -q -x 2>&1 | tail -15; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/r02b/bench_c5.json 2> gpurun_out/r02b/bench_c5.err; echo "bench rc=$?"
cut -c1-6000 gpurun_out/r02b/bench_c5.json
python tools/f16x_time.py 4096 tensor > gpurun_out/r02b/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x_kernel -s 2 -c 1 -o gpurun_out/r02b/f16x_n4096 python tools/f16x_time.py 4096 tensor > gpurun_out/r02b/ncu.log 2>&1; echo "ncu rc=$?"
