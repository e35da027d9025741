# gemm_f16x: 8-warp software-pipelined epilogue vs the 16-warp kernel (bitwise check + time per n=4096 product)
# variants: one per line in $VARIANTS
mkdir -p gpurun_out/r02w8
exec > gpurun_out/r02w8/log.txt 2>&1
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC"
[ -z "$VARIANTS" ] && VARIANTS=$'-DKP_F16X_W8=1\n-DKP_F16X_W8=0'
while IFS= read -r v; do
  $NV $v -c paper_2311_15393_b200/csrc/gemm_f16x.cu -o paper_2311_15393_b200/_build/gemm_f16x.cu.o 2>/dev/null || { echo "compile failed: $v"; continue; }
  python -c "from paper_2311_15393_b200 import build; build.build_library()"
  VARIANT="$v" timeout 300 python tools/f16x_quick.py 2>&1 | tail -1
done <<< "$VARIANTS"
