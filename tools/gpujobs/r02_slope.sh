mkdir -p gpurun_out/r02slope
exec > gpurun_out/r02slope/log.txt 2>&1
python tools/iter_slope.py C1 2>&1 | tail -2
python tools/iter_slope.py C1 KP_FOLD_SCALARS=0 2>&1 | tail -1
python tools/iter_slope.py C1 KP_GRAPH_LOOP=0 2>&1 | tail -1
python tools/iter_slope.py C1 KP_F16REF_BM=32 2>&1 | tail -1
python tools/iter_slope.py C2 2>&1 | tail -1
