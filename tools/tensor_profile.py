"""Per-kernel-class breakdown of one C5 FPCG solve in each preconditioner mode (dev tool)."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2311_15393_b200 as K
from paper_2311_15393_b200._lib import lib, check
import bench
cfg = bench.build_problem("C5", 0, None, device_apply=True)
sr, sc = bench.svd_pair(cfg.term, "gpu")
H = K.PrecisionFormat.fp16()
L = lib()
opts = K.SolverOptions(lambda_=0.01, max_iterations=30, rel_residual_tol=1e-6, x_true=cfg.problem.x_true)
for accum in ("reference", "tensor"):
    m = K.build_preconditioner_from_svd(sr, sc, 0.01, H, accum=accum)
    K.fpcg(cfg.problem.a, cfg.problem.b, m, opts)
    check(L.kp_profile_reset()); check(L.kp_profile_enable(1))
    t = time.time(); r = K.fpcg(cfg.problem.a, cfg.problem.b, m, opts); dt = time.time() - t
    out = []
    for cls, name in enumerate(["operator", "precond", "vector", "spectral"]):
        tt = C.c_double(); cc = C.c_longlong(); check(L.kp_profile_read(cls, C.byref(tt), C.byref(cc)))
        out.append(f"{name} {tt.value:.1f}ms/{cc.value}")
    check(L.kp_profile_enable(0))
    t = time.time(); r = K.fpcg(cfg.problem.a, cfg.problem.b, m, opts); dt2 = time.time() - t
    print(accum, r.history.iterations_used, f"wall(prof) {dt:.3f}s wall {dt2:.3f}s", out, flush=True)
