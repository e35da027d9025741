mkdir -p gpurun_out/r02trace
exec > gpurun_out/r02trace/log.txt 2>&1
export KP_NVCC_EXTRA="-DKP_F16X_TRACE=1"
touch paper_2311_15393_b200/csrc/gemm_f16x.cu
python -c "from paper_2311_15393_b200 import build; build.build_library()"
timeout 600 python tools/f16x_trace.py
