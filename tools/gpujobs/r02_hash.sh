mkdir -p gpurun_out/r02hash
exec > gpurun_out/r02hash/log.txt 2>&1
timeout 600 python tools/f16x_quick.py 2>&1 | tail -5
for v in 1 0; do
  KP_HASH_SMEM=$v timeout 600 python - <<'PY'
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import _lib
from paper_2311_15393_b200.kronprec import SvdTriple
n = 4096
rng = np.random.default_rng(1)
v = rng.standard_normal((n, n)).astype(np.float16).astype(np.float64) / 64
trip = SvdTriple(v, np.linspace(1, 1e-3, n), v)
m = K.build_preconditioner_from_svd(trip, trip, 0.01, K.PrecisionFormat.fp16())
r = rng.standard_normal(n * n)
K.set_fp16_products("tensor")
L = _lib.lib()
K.precond_solve(m, r)
L.kp_profile_reset(); L.kp_profile_enable(1)
for _ in range(5): K.precond_solve(m, r)
t, c = C.c_double(), C.c_longlong()
L.kp_profile_read(4, C.byref(t), C.byref(c))
print("KP_HASH_SMEM", os.environ["KP_HASH_SMEM"], "precond_aux: %.1f us per launch (%d launches)" % (1e3 * t.value / c.value, c.value))
PY
done
timeout 900 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_lpblas.py tests/test_gpu_batch.py -q -x 2>&1 | tail -3
