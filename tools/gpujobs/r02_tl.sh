mkdir -p gpurun_out/r02tl
timeout 600 python tools/solve_timeline.py C1 4 > gpurun_out/r02tl/c1.txt 2>&1
timeout 600 python tools/solve_timeline.py C2 2 > gpurun_out/r02tl/c2.txt 2>&1
