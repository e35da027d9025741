"""Per-kernel-class device time of one C4 image's PCG solve (dev tool).

Prints the graph-replayed solve time, then the same solve with per-launch
events (kp_profile) split into operator / preconditioner / vector classes.
"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2311_15393_b200 import kronprec as K  # noqa: E402
from paper_2311_15393_b200._lib import check, lib  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard  # noqa: E402

L = lib()
check(L.kp_init(0))
sh = C4Shard(svd="gpu")
tp = sh.problem(0)
sd = K.make_spectral_data(sh.m0, tp.b)
lam = K.discrepancy(sd, float(np.linalg.norm(tp.noise)), sh.eta).lambda_
m = K.with_lambda(sh.m0, lam)
opts = K.SolverOptions(lambda_=lam, max_iterations=100, rel_residual_tol=sh.tol)
for _ in range(2):
    K.pcg(sh.a, tp.b, m, opts)
t = time.perf_counter()
for _ in range(5):
    r = K.pcg(sh.a, tp.b, m, opts)
dt = (time.perf_counter() - t) / 5
it = r.history.iterations_used
print(f"solve {dt * 1e3:.2f} ms, {it} iterations, {dt / it * 1e6:.1f} us/iteration (host wall, host buffers)")
check(L.kp_profile_reset())
check(L.kp_profile_enable(1))
K.pcg(sh.a, tp.b, m, opts)
check(L.kp_profile_enable(0))
tot = 0.0
for cls, name in enumerate(["operator", "precond", "vector", "spectral"]):
    tt, cc = C.c_double(), C.c_longlong()
    check(L.kp_profile_read(cls, C.byref(tt), C.byref(cc)))
    tot += tt.value
    print(f"{name:9s} {tt.value:8.2f} ms  {cc.value:6d} launches  {tt.value / it * 1e3:7.1f} us/iteration")
print(f"sum      {tot:8.2f} ms")
