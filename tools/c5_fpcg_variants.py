"""C5 FPCG (reference-exact fp16) with different setup SVDs (dev tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2311_15393_b200 as K  # noqa: E402

cfg = bench.build_problem("C5", 0, None, device_apply=True)
opts = K.SolverOptions(lambda_=cfg.lambda_, max_iterations=100, rel_residual_tol=cfg.tol,
                       x_true=cfg.problem.x_true)
for how in ("gpu", "host"):
    sr, sc = bench.svd_pair(cfg.term, how)
    m = K.build_preconditioner_from_svd(sr, sc, cfg.lambda_, K.PrecisionFormat.fp16())
    r = K.fpcg(cfg.problem.a, cfg.problem.b, m, opts)
    h = r.history
    print(how, h.iterations_used, h.converged, h.abort_reason, h.relative_error[-1], flush=True)
