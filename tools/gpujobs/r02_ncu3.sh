# full ncu capture of gemm_f16x in the C5 solve (host-polled graph replays: ncu cannot profile
# kernel nodes of a graph with a conditional node)
mkdir -p gpurun_out/r02ncu2
exec > gpurun_out/r02ncu2/log3.txt 2>&1
export KP_GRAPH_LOOP=0
python tools/c5_solve_once.py 5 > gpurun_out/r02ncu2/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x_kernel -s 8 -c 1 -o gpurun_out/r02ncu2/gemm_f16x_c5 python tools/c5_solve_once.py 5 > gpurun_out/r02ncu2/ncu_f16x.log 2>&1; echo "f16x rc=$?"
python tools/ncu_keys.py gpurun_out/r02ncu2/gemm_f16x_c5.ncu-rep
