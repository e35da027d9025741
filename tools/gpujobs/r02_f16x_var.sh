# gemm_f16x: per-group N=128 MMAs; variants of stages / register counter levels; bitwise checks
mkdir -p gpurun_out/r02c
exec > gpurun_out/r02c/log.txt 2>&1
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC"
for v in "-DKP_F16X_NSTAGE=3 -DKP_F16X_REGLV=3" "-DKP_F16X_NSTAGE=2 -DKP_F16X_REGLV=3" ""; do
  echo "=== variant [$v]"
  $NV $v -c paper_2311_15393_b200/csrc/gemm_f16x.cu -o paper_2311_15393_b200/_build/gemm_f16x.cu.o && python -c "from paper_2311_15393_b200 import build; build.build_library()"
  timeout 600 python tools/f16x_check.py 2>&1 | tail -4
done
timeout 1200 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_lpblas.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --no-tensor --no-dense --no-other-runs > gpurun_out/r02c/bench_c5.json 2> gpurun_out/r02c/bench_c5.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02c/bench_c5.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'])"
python tools/f16x_time.py 4096 tensor > gpurun_out/r02c/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x_kernel -s 2 -c 1 -o gpurun_out/r02c/f16x_n4096 python tools/f16x_time.py 4096 tensor > gpurun_out/r02c/ncu.log 2>&1; echo "ncu rc=$?"
