"""Diagnostic: small CGLS / PCG runs on the device against the oracle, printing histories."""
import numpy as np
import paper_2311_15393_b200 as K
from oracle import pyoracle as O
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200.kronprec import KronTerm, KroneckerSum, SolverOptions

for n in (4, 5, 6, 8, 16):
    rng = np.random.default_rng(31)
    a = KroneckerSum([KronTerm(rng.standard_normal((n, n)), rng.standard_normal((n, n)))
                      for _ in range(2)], n)
    b = P.rng_normals(35, n * n)
    ad = sum(np.kron(t.row_factor, t.col_factor) for t in a.terms)
    lam = 0.3 * np.linalg.svd(ad, compute_uv=False)[0]
    o = SolverOptions(lambda_=lam, max_iterations=n * n, rel_residual_tol=1e-10)
    r = K.cgls(a, b, o)
    xo, ho = O.cgls(a, b, o)
    print(n, "gpu", r.history.iterations_used, r.history.converged, np.array(r.history.residual_norm[:6]))
    print(n, "orc", ho.iterations_used, ho.converged, np.array(ho.residual_norm[:6]))
    print("  x diff", np.linalg.norm(r.x - xo) / np.linalg.norm(xo))
