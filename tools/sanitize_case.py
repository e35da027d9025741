"""Small cases that launch every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck): operator (banded and dense), fp16 M-solve on
both engines at ragged sizes, generic formats, PCG / FPCG / CGLS, batched
solves, GCV / discrepancy, tensor mode, device problem generation."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200 import problems as P  # noqa: E402
from paper_2311_15393_b200.kronprec import SolverOptions, SvdTriple  # noqa: E402

rng = np.random.default_rng(5)
F16 = K.PrecisionFormat.fp16()
for n in (72, 200):
    psf = P.make_psf("gaussian", 9, sigma=2.0)
    tp = P.make_test_problem(P.blob_image(n, 11), psf, 0.01, 3)
    term = P.nearest_kron(psf, n)
    sr, sc = SvdTriple(*P.host_svd(term.row_factor)), SvdTriple(*P.host_svd(term.col_factor))
    r = rng.uniform(-1, 1, n * n)
    zs = []
    for eng in ("cuda", "tensor"):  # gemm_f16ref, gemm_f16x
        K.set_fp16_products(eng)
        m = K.build_preconditioner_from_svd(sr, sc, 0.01, F16)
        zs.append(K.precond_solve(m, r))
    assert np.array_equal(zs[0], zs[1]), "engines differ"
    K.set_fp16_products("auto")
    for fmt in (K.PrecisionFormat.bfloat16(), K.PrecisionFormat.fp64()):
        K.precond_solve(K.build_preconditioner_from_svd(sr, sc, 0.01, fmt), r)
    K.precond_solve(K.build_preconditioner_from_svd(sr, sc, 0.01, F16, accum="tensor"), r)
    y = K.kronsum_apply(tp.a, tp.x_true)
    tp.a.set_mode("dense")
    yd = K.kronsum_apply(tp.a, tp.x_true)
    K.kronsum_apply_transpose(tp.a, tp.x_true)
    tp.a.set_mode("auto")
    assert np.linalg.norm(y - yd) <= 1e-12 * np.linalg.norm(y)
    opts = SolverOptions(lambda_=0.01, max_iterations=12, rel_residual_tol=1e-6, x_true=tp.x_true)
    for eng in ("cuda", "tensor"):
        K.set_fp16_products(eng)
        m = K.build_preconditioner_from_svd(sr, sc, 0.01, F16)
        K.pcg(tp.a, tp.b, m, opts)
        K.fpcg(tp.a, tp.b, m, opts)
        bs = np.stack([tp.b, 0.5 * tp.b, tp.b + 1e-3])
        K.pcg_batch(tp.a, bs, m, [0.01, 0.02, 0.03], opts)
    K.set_fp16_products("auto")
    K.cgls(tp.a, tp.b, opts)
    sd = K.make_spectral_data(m, tp.b, tp.x_true)
    K.gcv_grid(sd, np.logspace(-4, 0, 64))
    K.gcv(sd)
    K.discrepancy(sd, float(np.linalg.norm(tp.noise)), 1.01)
    K.discrepancy_batch(m, bs, [float(np.linalg.norm(tp.noise))] * 3, 1.01)
    K.lambda_opt(sd)
    K.filtered_solution(m, tp.b, 0.01)
    K.round_array(r, F16)
    K.lp_matmul(rng.standard_normal((37, 70)), rng.standard_normal((70, 19)), F16)
    print("case", n, "ok", flush=True)
print("sanitize cases ok")
