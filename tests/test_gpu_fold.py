"""PCG scalar steps folded into the vector kernels (pcg_alpha_scalar into
pcg_update's CTAs, pcg_resid_scalar into its last CTA, pcg_beta_scalar into
pcg_p_update — krylov.cpp:100-138) give bit-identical solves to the separate
scalar kernels (KP_FOLD_SCALARS=0): same iterates, histories, stop / abort,
single and batched, with fewer launches where the folds apply (small n)."""
import os

import numpy as np
import pytest

import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200._lib import lib
from paper_2311_15393_b200.kronprec import SolverOptions

pytestmark = pytest.mark.gpu


def with_fold(on, fn):
    old = os.environ.get("KP_FOLD_SCALARS")
    os.environ["KP_FOLD_SCALARS"] = "1" if on else "0"
    try:
        c0 = lib().kp_launch_count()
        out = fn()
        return out, lib().kp_launch_count() - c0
    finally:
        if old is None:
            del os.environ["KP_FOLD_SCALARS"]
        else:
            os.environ["KP_FOLD_SCALARS"] = old


def same(r1, r2):
    h1, h2 = r1.history, r2.history
    assert h1.iterations_used == h2.iterations_used
    assert h1.converged == h2.converged and h1.abort_reason == h2.abort_reason
    assert h1.msolve_count == h2.msolve_count
    assert h1.residual_norm == h2.residual_norm
    assert h1.relative_error == h2.relative_error
    assert h1.residual_cosines == h2.residual_cosines
    assert np.array_equal(r1.x, r2.x)


def problem(n, seed=11):
    psf = P.make_psf("gaussian", 17, sigma=2.5)
    a, _ = P.psf_to_kronsum(psf, n)
    term = P.nearest_kron(psf, n)
    tp = P.make_test_problem(P.blob_image(n, seed), psf, 0.01, seed + 1, a=a)
    return a, term, tp, psf


@pytest.mark.parametrize("n", [64, 97, 256, 1024])
@pytest.mark.parametrize("solver", ["pcg", "fpcg"])
@pytest.mark.parametrize("fmt", ["fp16", "fp64"])
def test_fold_equals_separate(n, solver, fmt):
    a, term, tp, _ = problem(n)
    lam = 0.02
    m = K.build_preconditioner(term.row_factor, term.col_factor, lam, K.PrecisionFormat.parse(fmt))
    o = SolverOptions(lambda_=lam, max_iterations=30, rel_residual_tol=1e-7, x_true=tp.x_true,
                      track_search_direction_orthogonality=True)
    fn = lambda: getattr(K, solver)(a, tp.b, m, o)  # noqa: E731
    fn()  # lazy set-up launches out of the counts
    r1, c1 = with_fold(True, fn)
    r0, c0 = with_fold(False, fn)
    same(r1, r0)
    if n <= 256:  # every fold applies: 3 fewer launches per iteration
        assert c0 - c1 >= 3 * r1.history.iterations_used


def test_fold_abort_paths():
    """Stops inside the folded steps: the iteration cap / convergence in the
    folded residual step and a positivity abort in the folded rho step (a
    tiny lambda with fp16 products), same as the separate kernels."""
    a, term, tp, _ = problem(96)
    for lam, tol, maxit in [(1e-6, 1e-15, 300), (0.02, 1e-15, 6), (0.5, 1e-3, 100)]:
        m = K.build_preconditioner(term.row_factor, term.col_factor, lam, K.PrecisionFormat.fp16())
        o = SolverOptions(lambda_=lam, max_iterations=maxit, rel_residual_tol=tol, x_true=tp.x_true)
        fn = lambda: K.pcg(a, tp.b, m, o)  # noqa: E731
        same(with_fold(True, fn)[0], with_fold(False, fn)[0])


@pytest.mark.parametrize("solver", ["pcg_batch", "fpcg_batch"])
def test_fold_batch(solver):
    a, term, _, psf = problem(96)
    tps = [P.make_test_problem(P.blob_image(96, 40 + i), psf, [0.001, 0.01, 0.05][i % 3], 50 + i, a=a)
           for i in range(5)]
    m0 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, K.PrecisionFormat.fp16())
    lams = [0.01, 0.03, 0.1, 0.3, 1e-6]
    opts = SolverOptions(max_iterations=40, rel_residual_tol=1e-5)
    bs = np.stack([tp.b for tp in tps])
    xts = np.stack([tp.x_true for tp in tps])
    fn = lambda: getattr(K, solver)(a, bs, m0, lams, opts, x_true=xts)  # noqa: E731
    rf, _ = with_fold(True, fn)
    rs, _ = with_fold(False, fn)
    for x, y in zip(rf, rs):
        same(x, y)
    for i, tp in enumerate(tps):  # and each image equals its single (folded) solve
        o = SolverOptions(lambda_=lams[i], max_iterations=40, rel_residual_tol=1e-5, x_true=tp.x_true)
        single = getattr(K, solver.replace("_batch", ""))(a, tp.b, K.with_lambda(m0, lams[i]), o)
        same(rf[i], single)
