"""Device emulated low-precision BLAS vs the oracle: round_array for any
format (precision.cpp:15-41, 82-95), lp_matmul / lp_matvec / lp_dot /
pairwise_sum (lpblas.cpp:13-70) — bit-identical — plus the reference's own
pins from test_lpblas.cpp, and Kronecker-SVD preconditioners in formats
other than fp16 / fp64 (the generic emulation path)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2311_15393_b200 as K
from oracle import pyoracle as O
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200.kronprec import PrecisionFormat as F
from paper_2311_15393_b200.kronprec import SvdTriple

pytestmark = pytest.mark.gpu

H, BF, S, D = F.fp16(), F.bfloat16(), F.fp32(), F.fp64()
TINY = F.parse("custom:t=5,emax=4,subnormals=1")
TINY_FLUSH = F.parse("custom:t=5,emax=4,subnormals=0")
FORMATS = [H, BF, S, D, TINY, TINY_FLUSH]


def same_bits(a, b):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def edge_values(fmt, rng):
    t, emax = fmt.significand_bits, fmt.max_exponent
    if fmt.covers_double():
        thr, mx = np.inf, np.finfo(np.float64).max
    else:
        thr, mx = fmt.overflow_threshold(), fmt.max_finite()
    emin = fmt.min_exponent()
    vals = [0.0, -0.0, np.inf, -np.inf, thr, -thr, np.nextafter(thr, 0), mx, -mx,
            2.0 ** emin, 2.0 ** (emin - t + 1), 2.0 ** (emin - t), 1.5 * 2.0 ** (emin - t + 1),
            1.0 + 2.0 ** -t, 1.0 + 3 * 2.0 ** -t, 5e-324, -5e-324, 1e300, -1e-300]
    vals += list(rng.standard_normal(200) * 10.0 ** rng.uniform(-6, 6, 200))
    vals += list(np.ldexp(rng.uniform(1, 2, 100), rng.integers(emin - t - 2, emax + 2, 100)))
    return np.array([v for v in vals if np.isfinite(v) or np.isinf(v)])


@pytest.mark.parametrize("fmt", FORMATS, ids=lambda f: f.name)
def test_round_array_matches_oracle(fmt):
    rng = np.random.default_rng(17)
    x = edge_values(fmt, rng)
    assert same_bits(K.round_array(x, fmt), O.round_array(x, fmt))
    assert np.isnan(K.round_value(np.nan, fmt))


@pytest.mark.parametrize("fmt", FORMATS, ids=lambda f: f.name)
@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (3, 5, 7), (7, 17, 4), (33, 65, 9), (5, 128, 3),
                                   (2, 1000, 2), (64, 64, 64)])
def test_lp_matmul_matches_oracle(fmt, m, k, n):
    rng = np.random.default_rng(m * 1000 + k * 10 + n)
    a = rng.uniform(-3, 3, (m, k))
    b = rng.uniform(-3, 3, (k, n))
    assert same_bits(K.lp_matmul(a, b, fmt), O.lp_matmul(a, b, fmt, mode=1))
    # binary16-representable inputs: the f16x2 GEMM path for fp16
    ar, br = O.round_array(a, H), O.round_array(b, H)
    assert same_bits(K.lp_matmul(ar, br, fmt), O.lp_matmul(ar, br, fmt, mode=1))


def test_lp_matmul_f16_path_ragged_large():
    rng = np.random.default_rng(5)
    for m, k, n in [(100, 333, 70), (129, 1, 65), (31, 4097, 3)]:
        a = O.round_array(rng.uniform(-1, 1, (m, k)), H)
        b = O.round_array(rng.uniform(-1, 1, (k, n)), H)
        assert same_bits(K.lp_matmul(a, b, H), O.lp_matmul(a, b, H))


def test_lpblas_pins():  # test_lpblas.cpp:37-63, 102-222
    assert K.pairwise_sum(np.ones(8), H) == 8.0
    assert K.pairwise_sum(np.arange(1, 9.0), H) == 36.0
    assert K.pairwise_sum([2048, 2, 1, 1], H) == 2052.0
    assert K.pairwise_sum([2048, 1, 1, 1], H) == 2050.0
    assert K.pairwise_sum([7.0], H) == 7.0
    with pytest.raises(ValueError):
        K.pairwise_sum(np.zeros(0), H)
    e3 = np.zeros(8)
    e3[2] = 1
    assert K.lp_dot(e3, np.arange(1, 9.0), H) == 3.0
    assert K.lp_dot(np.ones(16), np.ones(16), H) == 16.0
    with pytest.raises(ValueError):
        K.lp_dot(np.ones(3), np.ones(4), H)
    rng = np.random.default_rng(4242)
    for fmt in (H, BF):
        for n in (10, 64, 100, 1000):
            x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
            got = K.lp_dot(x, y, fmt)
            assert got == O.lp_dot(x, y, fmt)
            bound = (np.ceil(np.log2(n)) + 2) * fmt.unit_roundoff() * np.abs(x * y).sum()
            assert abs(got - x @ y) <= bound
    v = rng.uniform(-2, 2, 8)
    assert same_bits(K.lp_matvec(np.eye(8), v, H), O.round_array(v, H))
    b = rng.uniform(-3, 3, (4, 6))
    assert same_bits(K.lp_matmul(np.eye(4), b, H), O.round_array(b, H))
    a = rng.uniform(-3, 3, (3, 5))
    assert same_bits(K.lp_matmul(a, np.eye(5), H), O.round_array(a, H))
    assert np.array_equal(K.lp_matmul([[1, 2], [3, 4]], [[5, 6], [7, 8]], H), [[19, 22], [43, 50]])
    with pytest.raises(ValueError):
        K.lp_matmul([[1, 2], [3, 4]], np.ones((3, 2)), H)
    for k in (4, 17, 32):
        m = rng.uniform(-1, 1, (7, k))
        w = rng.uniform(-1, 1, k)
        assert same_bits(K.lp_matmul(m, w.reshape(-1, 1), H)[:, 0], K.lp_matvec(m, w, H))
        assert same_bits(K.lp_matvec(m, w, H), O.lp_matvec(m, w, H))
    for _ in range(20):
        x = np.floor(rng.uniform(-8, 9, (6, 6)))
        y = np.floor(rng.uniform(-8, 9, (6, 6)))
        assert np.array_equal(K.lp_matmul(x, y, H), x @ y)
    x = rng.uniform(-1, 1, 100)
    assert K.lp_dot(x, x, D) == O.lp_dot(x, x, D)  # unrounded FP64 tree, same order


MID = F.parse("custom:t=9,emax=20,subnormals=0")


@pytest.mark.parametrize("fmt", [BF, S, MID], ids=lambda f: f.name)
def test_generic_format_preconditioner_bitwise(fmt):
    n = 24
    psf = P.make_psf("gaussian", 7, sigma=1.5)
    term = P.nearest_kron(psf, n)
    g = K.build_preconditioner(term.row_factor, term.col_factor, 0.05, fmt)
    o = O.build_preconditioner(term.row_factor, term.col_factor, 0.05, fmt)
    rng = np.random.default_rng(9)
    for _ in range(3):
        r = rng.standard_normal(n * n)
        zg, zo = K.precond_solve(g, r), O.precond_solve(o, r)
        # the FP64 SVDs of the two sides may differ in the last bits; with a
        # shared SVD the solve is bit-identical
        assert np.linalg.norm(zg - zo) <= 1e-2 * np.linalg.norm(zo) + 1e-300
    sr = SvdTriple(*P.host_svd(term.row_factor))
    sc = SvdTriple(*P.host_svd(term.col_factor))
    g = K.build_preconditioner_from_svd(sr, sc, 0.05, fmt)
    o = O.build_preconditioner_from_svd((sr.u, sr.s, sr.v), (sc.u, sc.s, sc.v), 0.05, fmt)
    for _ in range(3):
        r = rng.standard_normal(n * n)
        assert same_bits(K.precond_solve(g, r), O.precond_solve(o, r))


def test_generic_format_pcg_matches_oracle():
    n = 32
    psf = P.make_psf("gaussian", 7, sigma=1.5)
    tp = P.make_test_problem(P.blob_image(n, 77), psf, 0.01, 78)
    term = P.nearest_kron(psf, n)
    sr = SvdTriple(*P.host_svd(term.row_factor))
    sc = SvdTriple(*P.host_svd(term.col_factor))
    g = K.build_preconditioner_from_svd(sr, sc, 0.02, BF)
    o = O.build_preconditioner_from_svd((sr.u, sr.s, sr.v), (sc.u, sc.s, sc.v), 0.02, BF)
    opts = K.SolverOptions(lambda_=0.02, max_iterations=40, rel_residual_tol=1e-6, x_true=tp.x_true)
    for solver in ("pcg", "fpcg"):
        r = getattr(K, solver)(tp.a, tp.b, g, opts)
        xo, ho = getattr(O, solver)(tp.a, tp.b, o, opts)
        h = r.history
        assert h.residual_norm[0] == pytest.approx(ho.residual_norm[0], rel=1e-12)
        assert abs(h.iterations_used - ho.iterations_used) <= 2
        assert h.converged == ho.converged
        assert abs(h.relative_error[-1] - ho.relative_error[-1]) <= 1e-3


def test_round_call_session_matches_reference_budget():
    """RoundCallSession (precision.hpp:55-66): the reference's own budgets -
    test_factor.cpp:302-317 (2 + 4 (1 + 3) calls per fp16 M-solve at n = 8,
    none for fp64) and test_krylov.cpp:259-287 (all rounding happens inside
    the preconditioner solves) - and the oracle's tally for the BLAS calls."""
    n = 8
    t = 0.5 * np.eye(n) + 0.25 * (np.eye(n, k=1) + np.eye(n, k=-1))
    p16 = K.build_preconditioner(t, t, 0.05, H)
    s = K.RoundCallSession()
    K.precond_solve(p16, np.ones(n * n))
    assert s.count() == 2 + 4 * (1 + 3)
    p64 = K.build_preconditioner(t, t, 0.05, D)
    s2 = K.RoundCallSession()
    K.precond_solve(p64, np.ones(n * n))
    assert s2.count() == 0
    a = K.KroneckerSum([K.KronTerm(t, t)], n)
    b = np.sin(0.3 + np.arange(n * n))
    opts = K.SolverOptions(lambda_=0.05, max_iterations=10, rel_residual_tol=1e-12)
    base = K.RoundCallSession()
    K.cgls(a, b, opts)
    assert K.round_call_count(base) == 0
    prec = K.RoundCallSession()
    rp = K.pcg(a, b, p16, opts)
    assert K.round_call_count(prec) == 18 * rp.history.msolve_count
    assert rp.history.msolve_count >= rp.history.iterations_used
    flex = K.RoundCallSession()
    rf = K.fpcg(a, b, p16, opts)
    assert flex.count() == 18 * rf.history.msolve_count
    dbl = K.RoundCallSession()
    K.pcg(a, b, p64, opts)
    assert dbl.count() == 0
    # sessions nest; scalar rounding is not tallied; BLAS calls against the oracle's tally
    outer = K.RoundCallSession()
    K.round_value(0.1, H)
    assert outer.count() == 0
    rng = np.random.default_rng(2)
    x, y = rng.standard_normal((5, 37)), rng.standard_normal((37, 3))
    for fmt in (H, BF, D):
        inner = K.RoundCallSession()
        o0 = O.round_calls()
        K.round_array(x, fmt), O.round_array(x, fmt)
        K.lp_matmul(x, y, fmt), O.lp_matmul(x, y, fmt)
        K.lp_matvec(x, y[:, 0], fmt), O.lp_matvec(x, y[:, 0], fmt)
        K.lp_dot(x[0], y[:, 0], fmt), O.lp_dot(x[0], y[:, 0], fmt)
        K.pairwise_sum(K.round_array(x[0], fmt), fmt), O.pairwise_sum(O.round_array(x[0], fmt), fmt)
        assert inner.count() == O.round_calls() - o0
    assert outer.count() > 0
    b0 = K.RoundCallSession()
    q = K.build_preconditioner(t, t, 0.05, H)
    assert b0.count() == 3
    K.with_lambda(q, 0.1)
    assert b0.count() == 4
