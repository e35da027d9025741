mkdir -p gpurun_out/r02e
exec > gpurun_out/r02e/log.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py -m gpu -q -x 2>&1 | tail -15; echo "batch tests rc=$?"
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "c4" 2>&1 | tail -5; echo "c4 tests rc=$?"
timeout 900 python bench.py --config C4 --steps 1 --warmup 1 --no-tensor > gpurun_out/r02e/bench_c4_batch.json 2> gpurun_out/r02e/bench_c4_batch.err; echo "c4 batch rc=$?"
cut -c1-2500 gpurun_out/r02e/bench_c4_batch.json; tail -3 gpurun_out/r02e/bench_c4_batch.err
timeout 900 python bench.py --config C4 --c4-mode streams --steps 1 --warmup 1 --no-tensor --no-cpu-baseline > gpurun_out/r02e/bench_c4_streams.json 2> gpurun_out/r02e/bench_c4_streams.err; echo "c4 streams rc=$?"
cut -c1-400 gpurun_out/r02e/bench_c4_streams.json
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC"
for v in "-DKP_F16X_REGLV=1" ""; do
  $NV $v -c paper_2311_15393_b200/csrc/gemm_f16x.cu -o paper_2311_15393_b200/_build/gemm_f16x.cu.o 2>/dev/null && python -c "from paper_2311_15393_b200 import build; build.build_library()"
  VARIANT="$v" timeout 300 python tools/f16x_quick.py 2>&1 | tail -1
done
