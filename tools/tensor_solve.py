"""One short C5 FPCG solve in tensor mode, for ncu launch lists (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_15393_b200 as K
import bench
cfg = bench.build_problem("C5", 0, None, device_apply=True)
sr, sc = bench.svd_pair(cfg.term, "gpu")
m = K.build_preconditioner_from_svd(sr, sc, 0.01, K.PrecisionFormat.fp16(), accum=os.environ.get("ACCUM", "tensor"))
opts = K.SolverOptions(lambda_=0.01, max_iterations=8, rel_residual_tol=1e-6, x_true=cfg.problem.x_true)
for _ in range(2):
    r = K.fpcg(cfg.problem.a, cfg.problem.b, m, opts)
print("done", r.history.iterations_used)
