# gemm_f16x: software-pipelined epilogue loads (bitwise check + time per n=4096 product), then the timeline
mkdir -p gpurun_out/r02swp
exec > gpurun_out/r02swp/log.txt 2>&1
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC"
for v in "-DKP_F16X_SWP=1" "-DKP_F16X_SWP=0" $EXTRA_VARIANTS; do
  $NV $v -c paper_2311_15393_b200/csrc/gemm_f16x.cu -o paper_2311_15393_b200/_build/gemm_f16x.cu.o 2>/dev/null && python -c "from paper_2311_15393_b200 import build; build.build_library()"
  VARIANT="$v" timeout 300 python tools/f16x_quick.py 2>&1 | tail -1
done
for v in "-DKP_F16X_SWP=1"; do
  $NV $v -DKP_F16X_TRACE=1 -c paper_2311_15393_b200/csrc/gemm_f16x.cu -o paper_2311_15393_b200/_build/gemm_f16x.cu.o 2>/dev/null && python -c "from paper_2311_15393_b200 import build; build.build_library()"
  echo "trace $v"; timeout 300 python tools/f16x_trace.py 2>&1 | tail -40
done
