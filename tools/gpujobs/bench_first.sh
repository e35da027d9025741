nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 600 python bench.py --n 1024 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_n1024.log 2>&1
echo "rc=$?" >> gpurun_out/bench_n1024.log
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_c5.log 2>&1
echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 300 python -c "
import sys,time; sys.path.insert(0,'.')
from paper_2311_15393_b200 import configs, problems as P
import numpy as np
a=np.random.default_rng(0).standard_normal((4096,4096)); a=np.asfortranarray(a)
t=time.time(); P.host_svd(a); print('host dgesdd 4096', time.time()-t)
" > gpurun_out/svd_time.log 2>&1
tail -5 gpurun_out/bench_n1024.log gpurun_out/bench_c5.log gpurun_out/svd_time.log
