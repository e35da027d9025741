"""Per-iteration and per-solve fixed device time of a config's solve: solves
capped at k iterations (tolerance 0), timed with events on the library
stream, median of repeats; slope = time per iteration.

    python tools/iter_slope.py C1 [env=value ...]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
for kv in sys.argv[2:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
import bench  # noqa: E402
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200._lib import check, kp_history, kp_solver_options, lib, ptr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
L = lib()
check(L.kp_init(0))
cfg = bench.build_problem(name, 0, None, device_apply=True)
svd_r, svd_c = bench.svd_pair(cfg.term, "host")
lam = cfg.lambda_ or 0.01
m = K.build_preconditioner_from_svd(svd_r, svd_c, lam, K.PrecisionFormat.fp16())
solver_name = cfg.solvers[0][0]
solve_fn = L.kp_fpcg if solver_name == "fpcg" else L.kp_pcg
op = cfg.problem.a.handle()
nn = cfg.n * cfg.n


def dalloc(count):
    p = C.c_void_p()
    check(L.kp_device_alloc(count * 8, C.byref(p)))
    return p


d_b, d_x, d_xt = dalloc(nn), dalloc(nn), dalloc(nn)
check(L.kp_memcpy_h2d(d_b, ptr(cfg.problem.b), nn * 8))
check(L.kp_memcpy_h2d(d_xt, ptr(cfg.problem.x_true), nn * 8))


def solve(maxit):
    cap = maxit + 1
    hb = [np.zeros(cap) for _ in range(4)]
    h = kp_history(capacity=cap, relative_error=ptr(hb[0]), residual_norm=ptr(hb[1]),
                   work_units=ptr(hb[2]), residual_cosines=ptr(hb[3]))
    o = kp_solver_options(lambda_=lam, max_iterations=maxit, rel_residual_tol=1e-300,
                          x_true=d_xt.value, device_pointers=1)
    check(L.kp_synchronize())
    check(L.kp_event_record(0))
    check(solve_fn(op, d_b, m.handle(), C.byref(o), d_x, C.byref(h)))
    check(L.kp_event_record(1))
    ms = C.c_float()
    check(L.kp_event_elapsed(0, 1, C.byref(ms)))
    return ms.value * 1e3, h.iterations_used


ks = [1, 2, 4, 8, 16]
res = {}
for k in ks:
    for _ in range(3):
        solve(k)
    ts = [solve(k) for _ in range(15)]
    res[k] = (float(np.median([t for t, _ in ts])), ts[0][1])
for k in ks:
    print(f"{name} maxit {k:3d}: its {res[k][1]:3d}  {res[k][0]:9.1f} us")
x = np.array([res[k][1] for k in ks], float)
y = np.array([res[k][0] for k in ks])
A = np.vstack([x, np.ones_like(x)]).T
slope, icpt = np.linalg.lstsq(A, y, rcond=None)[0]
print(f"{name}: {slope:.1f} us / iteration, {icpt:.1f} us fixed per solve  ({' '.join(sys.argv[2:])})")
