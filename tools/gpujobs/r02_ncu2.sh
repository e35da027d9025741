# full ncu captures of the TMA-staged DMMA GEMM (dense operator, C5 size) and of gemm_f16x in the C5 solve
mkdir -p gpurun_out/r02ncu2
exec > gpurun_out/r02ncu2/log.txt 2>&1
timeout 600 python tools/f64_dense_once.py 3 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_tma_kernel -s 2 -c 2 -o gpurun_out/r02ncu2/gemm_f64_tma_c5 python tools/f64_dense_once.py 3 > gpurun_out/r02ncu2/ncu_f64.log 2>&1; echo "f64 rc=$?"
python tools/ncu_keys.py gpurun_out/r02ncu2/gemm_f64_tma_c5.ncu-rep
python tools/c5_solve_once.py 5 > gpurun_out/r02ncu2/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x_kernel -s 8 -c 1 -o gpurun_out/r02ncu2/gemm_f16x_c5 python tools/c5_solve_once.py 5 > gpurun_out/r02ncu2/ncu_f16x.log 2>&1; echo "f16x rc=$?"
python tools/ncu_keys.py gpurun_out/r02ncu2/gemm_f16x_c5.ncu-rep
