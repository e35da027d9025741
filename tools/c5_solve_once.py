"""One C5 FPCG solve (reference-exact fp16) for launch-list profiling."""
import sys
sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200 import configs  # noqa: E402
from paper_2311_15393_b200.kronprec import SolverOptions  # noqa: E402

cfg = configs.build("C5")
m = K.build_preconditioner(cfg.term.row_factor, cfg.term.col_factor, cfg.lambda_, K.PrecisionFormat.fp16())
opts = SolverOptions(lambda_=cfg.lambda_, max_iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 100,
                     rel_residual_tol=cfg.tol, x_true=cfg.problem.x_true)
r = K.fpcg(cfg.problem.a, cfg.problem.b, m, opts)
print("iterations", r.history.iterations_used, r.history.abort_reason, r.history.relative_error[-1])
