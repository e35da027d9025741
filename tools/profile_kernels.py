"""Exercise the two hot kernels at C5 size for ncu captures (dev tool).

--what op:    2 operator applies (n=4096, r=5 banded factors): gemm_f64_kernel
--what msolve: 2 fp16 reference-exact preconditioner solves: gemm_f16ref_kernel
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200.kronprec import SvdTriple

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="op")
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
n = a.n
psf = P.psf_gauss_motion(41, 4.0, 15, 30.0)
if a.what == "op":
    op, _ = P.psf_to_kronsum(psf, n, max_rank=5)
    x = np.random.default_rng(0).standard_normal(n * n)
    for _ in range(a.reps):
        t = time.time(); y = K.kronsum_apply(op, x); print("apply", time.time() - t, flush=True)
elif a.what == "msolve":
    q = np.linalg.qr(np.random.default_rng(1).standard_normal((n, n)))[0]
    s = np.linspace(1.0, 1e-3, n)
    sv = SvdTriple(np.asfortranarray(q), s, np.asfortranarray(q))
    m = K.build_preconditioner_from_svd(sv, sv, 0.01, K.PrecisionFormat.fp16())
    r = np.random.default_rng(2).standard_normal(n * n)
    for _ in range(a.reps):
        t = time.time(); z = K.precond_solve(m, r); print("msolve", time.time() - t, flush=True)
if a.what == "msolve_tc":
    q = np.linalg.qr(np.random.default_rng(1).standard_normal((n, n)))[0]
    s = np.linspace(1.0, 1e-3, n)
    sv = SvdTriple(np.asfortranarray(q), s, np.asfortranarray(q))
    m = K.build_preconditioner_from_svd(sv, sv, 0.01, K.PrecisionFormat.fp16(), accum="tensor")
    r = np.random.default_rng(2).standard_normal(n * n)
    for _ in range(a.reps):
        t = time.time(); z = K.precond_solve(m, r); print("msolve_tc", time.time() - t, flush=True)
