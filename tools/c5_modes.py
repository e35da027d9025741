"""C5 solver behaviour in both preconditioner modes + CGLS reference (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import configs
import bench
cfg = bench.build_problem("C5", 0, None, device_apply=True)
sr, sc = bench.svd_pair(cfg.term, "gpu")
H = K.PrecisionFormat.fp16()
opts = K.SolverOptions(lambda_=0.01, max_iterations=100, rel_residual_tol=1e-6, x_true=cfg.problem.x_true)
for name, accum, solver in [("fpcg-exact", "reference", K.fpcg), ("fpcg-tensor", "tensor", K.fpcg),
                            ("pcg-exact", "reference", K.pcg), ("pcg-tensor", "tensor", K.pcg)]:
    m = K.build_preconditioner_from_svd(sr, sc, 0.01, H, accum=accum)
    t = time.time(); r = solver(cfg.problem.a, cfg.problem.b, m, opts); dt = time.time() - t
    h = r.history
    print(name, h.iterations_used, h.converged, repr(h.abort_reason), f"relerr {h.relative_error[-1]:.5f}",
          f"res {h.residual_norm[-1]/h.residual_norm[0]:.3e}", "relerr@k", [round(e, 4) for e in h.relative_error[::5]], f"{dt:.1f}s", flush=True)
m64 = K.build_preconditioner_from_svd(sr, sc, 0.01, K.PrecisionFormat.fp64())
t = time.time(); r = K.pcg(cfg.problem.a, cfg.problem.b, m64, opts); dt = time.time() - t
h = r.history
print("pcg-fp64", h.iterations_used, h.converged, repr(h.abort_reason), f"relerr {h.relative_error[-1]:.5f}", f"{dt:.1f}s", flush=True)
o2 = K.SolverOptions(lambda_=0.01, max_iterations=2000, rel_residual_tol=1e-6, x_true=cfg.problem.x_true)
t = time.time(); r = K.cgls(cfg.problem.a, cfg.problem.b, o2); dt = time.time() - t
h = r.history
print("cgls", h.iterations_used, h.converged, f"relerr {h.relative_error[-1]:.5f}", f"{dt:.1f}s", flush=True)
