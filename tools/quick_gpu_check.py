"""Quick first-contact GPU parity check against the oracle (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import problems as P
from oracle import pyoracle as O

h = K.PrecisionFormat.fp16(); d = K.PrecisionFormat.fp64()
O.set_threads(8)
for n in [8, 16, 33, 64, 100, 256]:
    psf = P.make_psf("gaussian", 5, sigma=1.5)
    a, _ = P.psf_to_kronsum(psf, n)
    x = np.random.default_rng(n).standard_normal(n * n)
    g = K.kronsum_apply(a, x); o = O.kronsum_apply(a, x)
    gt = K.kronsum_apply_transpose(a, x); ot = O.kronsum_apply_transpose(a, x)
    e1 = np.linalg.norm(g - o) / np.linalg.norm(o); e2 = np.linalg.norm(gt - ot) / np.linalg.norm(ot)
    t = P.nearest_kron(psf, n)
    u_r = P.host_svd(t.row_factor); u_c = P.host_svd(t.col_factor)
    svr = K.kronprec.SvdTriple(*u_r); svc = K.kronprec.SvdTriple(*u_c)
    pg = K.build_preconditioner_from_svd(svr, svc, 0.05, h)
    po = O.build_preconditioner_from_svd(u_r, u_c, 0.05, h)
    r = np.random.default_rng(1).uniform(-1, 1, n * n)
    zg = K.precond_solve(pg, r); zo = O.precond_solve(po, r)
    pg64 = K.build_preconditioner_from_svd(svr, svc, 0.05, d); po64 = O.build_preconditioner_from_svd(u_r, u_c, 0.05, d)
    zg64 = K.precond_solve(pg64, r); zo64 = O.precond_solve(po64, r)
    print(f"n={n:4d} apply {e1:.2e} applyT {e2:.2e} msolve16 bitwise={np.array_equal(zg, zo)} "
          f"(ndiff={np.sum(zg != zo)}) msolve64 {np.linalg.norm(zg64-zo64)/np.linalg.norm(zo64):.2e}", flush=True)

# PCG / FPCG / CGLS small problem
n = 64
psf = P.make_psf("gaussian", 9, sigma=2.0)
img = P.blob_image(n, 7)
tp = P.make_test_problem(img, psf, 0.01, 3)
t = P.nearest_kron(psf, n)
u_r = P.host_svd(t.row_factor); u_c = P.host_svd(t.col_factor)
pg = K.build_preconditioner_from_svd(K.kronprec.SvdTriple(*u_r), K.kronprec.SvdTriple(*u_c), 0.01, h)
po = O.build_preconditioner_from_svd(u_r, u_c, 0.01, h)
opts = K.SolverOptions(lambda_=0.01, max_iterations=50, rel_residual_tol=1e-6, x_true=tp.x_true)
for kind in ["pcg", "fpcg", "cgls"]:
    t0 = time.time()
    rg = getattr(K, kind)(tp.a, tp.b, pg, opts) if kind != "cgls" else K.cgls(tp.a, tp.b, opts)
    t1 = time.time()
    ro = getattr(O, kind)(tp.a, tp.b, po, opts) if kind != "cgls" else O.cgls(tp.a, tp.b, opts)
    xo, ho = ro
    print(kind, "gpu iters", rg.history.iterations_used, "oracle iters", ho.iterations_used,
          "relerr", rg.history.relative_error[-1], ho.relative_error[-1],
          "max hist resid rel diff", max(abs(a - b) / b for a, b in zip(rg.history.residual_norm, ho.residual_norm)),
          "abort", repr(rg.history.abort_reason), f"{t1-t0:.3f}s", flush=True)
