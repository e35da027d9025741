"""One C4 image: spectral data, discrepancy lambda, PCG (10 iterations) — for launch lists."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2311_15393_b200 import kronprec as K  # noqa: E402
from paper_2311_15393_b200._lib import check, lib  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard  # noqa: E402

check(lib().kp_init(0))
sh = C4Shard(svd="gpu")
tp = sh.problem(0)
sd = K.make_spectral_data(sh.m0, tp.b)
lam = K.discrepancy(sd, float(np.linalg.norm(tp.noise)), sh.eta).lambda_
m = K.with_lambda(sh.m0, lam)
r = K.pcg(sh.a, tp.b, m, K.SolverOptions(lambda_=lam, max_iterations=10, rel_residual_tol=sh.tol))
print("done", r.history.iterations_used)
