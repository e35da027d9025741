"""Phase breakdown of the per-image C4 pipeline on one GPU."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2311_15393_b200 import kronprec as K  # noqa: E402
from paper_2311_15393_b200._lib import check, lib  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard  # noqa: E402

check(lib().kp_init(0))
sh = C4Shard(svd="gpu")
probs = [sh.problem(i) for i in range(6)]
sh.solve(0, probs[0])
acc = {"spectral": 0.0, "discrepancy": 0.0, "with_lambda": 0.0, "pcg": 0.0}
its = []
for i, tp in enumerate(probs):
    t0 = time.perf_counter()
    sd = K.make_spectral_data(sh.m0, tp.b)
    t1 = time.perf_counter()
    lam = K.discrepancy(sd, float(np.linalg.norm(tp.noise)), sh.eta).lambda_
    t2 = time.perf_counter()
    m = K.with_lambda(sh.m0, lam)
    t3 = time.perf_counter()
    r = K.pcg(sh.a, tp.b, m, K.SolverOptions(lambda_=lam, max_iterations=100,
                                             rel_residual_tol=sh.tol, x_true=tp.x_true))
    t4 = time.perf_counter()
    for k, v in zip(acc, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
        acc[k] += v
    its.append(r.history.iterations_used)
    print(i, f"lam={lam:.4g} it={r.history.iterations_used} rel={r.history.relative_error[-1]:.4f}",
          f"spec={1e3*(t1-t0):.2f} disc={1e3*(t2-t1):.2f} wl={1e3*(t3-t2):.2f} pcg={1e3*(t4-t3):.2f} ms")
print({k: round(1e3 * v / len(probs), 2) for k, v in acc.items()}, "ms/image; mean its", np.mean(its))
