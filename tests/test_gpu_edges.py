"""Edge cases of the solve path on the device vs the oracle: n = 1, zero and
non-finite right-hand sides, one-iteration budgets, iterate / cosine
recording, the banded-detection limits (r = 8 terms, 64 diagonals) and
ragged n around the 64-element padding of the fp16 operands."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2311_15393_b200 as K
from oracle import pyoracle as O
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200.kronprec import KronTerm, KroneckerSum, SolverOptions, SvdTriple

pytestmark = pytest.mark.gpu

H, D = K.PrecisionFormat.fp16(), K.PrecisionFormat.fp64()


def preconds(term, lam, fmt):
    sr = SvdTriple(*P.host_svd(term.row_factor))
    sc = SvdTriple(*P.host_svd(term.col_factor))
    g = K.build_preconditioner_from_svd(sr, sc, lam, fmt)
    o = O.build_preconditioner_from_svd((sr.u, sr.s, sr.v), (sc.u, sc.s, sc.v), lam, fmt)
    return g, o


def same_history(h, ho, rel=1e-10):
    assert h.iterations_used == ho.iterations_used
    assert h.converged == ho.converged
    assert h.abort_reason == ho.abort_reason
    assert h.msolve_count == ho.msolve_count
    assert len(h.residual_norm) == len(ho.residual_norm)
    scale = abs(ho.residual_norm[0]) if ho.residual_norm and np.isfinite(ho.residual_norm[0]) else 1.0
    for a, b in zip(h.residual_norm, ho.residual_norm):
        if np.isfinite(b):  # FP64 re-association: relative, or absolute vs ||r0|| near 0
            assert a == pytest.approx(b, rel=rel, abs=1e-14 * scale)
        else:
            assert not np.isfinite(a)


def banded_toeplitz(w, c, n):  # deblur.cpp:157-165
    t = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            k = i - j + c
            if 0 <= k < len(w):
                t[i, j] = w[k]
    return t


def blur(n, n_p=5, sigma=1.0, seed=3, noise=0.01):
    psf = P.make_psf("gaussian", n_p, sigma=sigma)
    tp = P.make_test_problem(P.blob_image(n, seed + 100), psf, noise, seed)
    return tp, P.nearest_kron(psf, n)


def test_one_by_one_system():
    a = KroneckerSum([KronTerm(np.array([[2.0]]), np.array([[3.0]]))], 1)
    b = np.array([1.5])
    assert K.kronsum_apply(a, b)[0] == 9.0
    assert K.kronsum_apply_transpose(a, b)[0] == 9.0
    for fmt in (H, D):
        g, o = preconds(KronTerm(np.array([[2.0]]), np.array([[3.0]])), 0.5, fmt)
        assert K.precond_solve(g, b)[0] == O.precond_solve(o, b)[0]
        opts = SolverOptions(lambda_=0.5, max_iterations=5, rel_residual_tol=1e-12)
        for solver in ("pcg", "fpcg"):
            r = getattr(K, solver)(a, b, g, opts)
            xo, ho = getattr(O, solver)(a, b, o, opts)
            same_history(r.history, ho)
            assert r.x[0] == pytest.approx(xo[0], rel=1e-14)
    r = K.cgls(a, b, SolverOptions(lambda_=0.5, max_iterations=5, rel_residual_tol=1e-12))
    xo, ho = O.cgls(a, b, SolverOptions(lambda_=0.5, max_iterations=5, rel_residual_tol=1e-12))
    same_history(r.history, ho)
    assert r.x[0] == pytest.approx(6.0 * 1.5 / (36.0 + 0.25), rel=1e-14)  # A = 2 (x) 3 = 6


def test_zero_rhs_converges_immediately():
    tp, term = blur(16)
    g, o = preconds(term, 0.1, H)
    z = np.zeros(16 * 16)
    opts = SolverOptions(lambda_=0.1, max_iterations=10, rel_residual_tol=1e-8)
    for solver in ("pcg", "fpcg"):
        r = getattr(K, solver)(tp.a, z, g, opts)
        _, ho = getattr(O, solver)(tp.a, z, o, opts)
        same_history(r.history, ho)
        assert r.history.converged and r.history.iterations_used == 0
        assert not r.x.any()
    r = K.cgls(tp.a, z, opts)
    _, ho = O.cgls(tp.a, z, opts)
    same_history(r.history, ho)
    assert not r.x.any()


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_non_finite_rhs_aborts_like_the_reference(bad):
    tp, term = blur(16)
    g, o = preconds(term, 0.1, H)
    b = tp.b.copy()
    b[37] = bad
    opts = SolverOptions(lambda_=0.1, max_iterations=10, rel_residual_tol=1e-8)
    for solver in ("pcg", "fpcg"):
        r = getattr(K, solver)(tp.a, b, g, opts)
        _, ho = getattr(O, solver)(tp.a, b, o, opts)
        assert r.history.converged == ho.converged
        assert r.history.abort_reason == ho.abort_reason
        assert r.history.iterations_used == ho.iterations_used
    r = K.cgls(tp.a, b, opts)
    _, ho = O.cgls(tp.a, b, opts)
    assert (r.history.converged, r.history.abort_reason, r.history.iterations_used) == \
           (ho.converged, ho.abort_reason, ho.iterations_used)


def test_single_iteration_budget_and_recording():
    tp, term = blur(24)
    g, o = preconds(term, 0.05, H)
    opts = SolverOptions(lambda_=0.05, max_iterations=1, rel_residual_tol=1e-14, x_true=tp.x_true,
                         record_iterates=True, track_search_direction_orthogonality=True)
    for solver in ("pcg", "fpcg"):
        r = getattr(K, solver)(tp.a, tp.b, g, opts)
        xo, ho = getattr(O, solver)(tp.a, tp.b, o, opts)
        same_history(r.history, ho)
        assert r.history.iterations_used == 1 and len(r.history.residual_norm) == 2
        assert len(r.history.iterates) == len(ho.iterates) == 2
        assert not r.history.iterates[0].any()
        assert np.linalg.norm(r.history.iterates[1] - ho.iterates[1]) <= 1e-12 * np.linalg.norm(ho.iterates[1])
        assert len(r.history.residual_cosines) == len(ho.residual_cosines)
        for a, b in zip(r.history.residual_cosines, ho.residual_cosines):
            assert a == pytest.approx(b, rel=1e-8, abs=1e-12)
    opts8 = SolverOptions(lambda_=0.05, max_iterations=8, rel_residual_tol=1e-14, x_true=tp.x_true,
                          track_search_direction_orthogonality=True)
    r = K.cgls(tp.a, tp.b, opts8)
    xo, ho = O.cgls(tp.a, tp.b, opts8)
    same_history(r.history, ho, rel=1e-9)
    assert len(r.history.residual_cosines) == len(ho.residual_cosines)
    for a, b in zip(r.history.residual_cosines, ho.residual_cosines):
        assert a == pytest.approx(b, rel=1e-6, abs=1e-10)


@pytest.mark.parametrize("n_p,expect_banded", [(63, True), (65, False)])
def test_banded_detection_limit(n_p, expect_banded):
    n = 80
    psf = P.make_psf("gaussian", n_p, sigma=n_p / 6.0)
    a, _ = P.psf_to_kronsum(psf, n, max_rank=1)
    mode, ct, rt = a.mode()
    assert mode.startswith("banded") == expect_banded
    x = np.random.default_rng(1).standard_normal(n * n)
    want = O.kronsum_apply(a, x)
    assert np.linalg.norm(K.kronsum_apply(a, x) - want) <= 1e-13 * np.linalg.norm(want)


@pytest.mark.parametrize("r,expect_banded", [(8, True), (9, False)])
def test_banded_term_limit(r, expect_banded):
    n = 40
    rng = np.random.default_rng(r)
    terms = []
    for _ in range(r):
        cols = [banded_toeplitz(rng.standard_normal(5), 2, n) for _ in range(2)]
        terms.append(KronTerm(cols[0], cols[1]))
    a = KroneckerSum(terms, n)
    assert (a.mode()[0].startswith("banded")) == expect_banded
    x = rng.standard_normal(n * n)
    for f, fo in ((K.kronsum_apply, O.kronsum_apply), (K.kronsum_apply_transpose, O.kronsum_apply_transpose)):
        want = fo(a, x)
        assert np.linalg.norm(f(a, x) - want) <= 1e-13 * np.linalg.norm(want)


@pytest.mark.parametrize("n", [63, 65, 127, 129, 513])
def test_ragged_sizes_fp16_bitwise(n):
    tp, term = blur(n, n_p=7, sigma=1.5)
    g, o = preconds(term, 0.03, H)
    rng = np.random.default_rng(n)
    r = rng.standard_normal(n * n)
    zg, zo = K.precond_solve(g, r), O.precond_solve(o, r)
    assert np.array_equal(zg.view(np.uint64), zo.view(np.uint64))


def test_device_pointer_mode_matches_host_mode():
    """kp_solver_options.device_pointers = 1: b, x_true and x live in device
    memory (the bench's value path); results equal the host-buffer path."""
    import ctypes as C

    from paper_2311_15393_b200._lib import check, kp_history, kp_solver_options, lib, ptr
    tp, term = blur(32)
    g, _ = preconds(term, 0.05, H)
    L = lib()
    nn = 32 * 32
    opts = SolverOptions(lambda_=0.05, max_iterations=12, rel_residual_tol=1e-9, x_true=tp.x_true)

    def dev(a):
        p = C.c_void_p()
        check(L.kp_device_alloc(nn * 8, C.byref(p)))
        if a is not None:
            check(L.kp_memcpy_h2d(p, ptr(np.ascontiguousarray(a)), nn * 8))
        return p

    for kind in ("cgls", "pcg", "fpcg"):
        ref = K.cgls(tp.a, tp.b, opts) if kind == "cgls" else getattr(K, kind)(tp.a, tp.b, g, opts)
        db, dxt, dx = dev(tp.b), dev(tp.x_true), dev(None)
        cap = 13
        bufs = [np.zeros(cap) for _ in range(4)]
        h = kp_history(capacity=cap, relative_error=ptr(bufs[0]), residual_norm=ptr(bufs[1]),
                       work_units=ptr(bufs[2]), residual_cosines=ptr(bufs[3]))
        o = kp_solver_options(lambda_=0.05, max_iterations=12, rel_residual_tol=1e-9,
                              x_true=dxt.value, device_pointers=1)
        if kind == "cgls":
            check(L.kp_cgls(tp.a.handle(), db, C.byref(o), dx, C.byref(h)))
        else:
            f = L.kp_pcg if kind == "pcg" else L.kp_fpcg
            check(f(tp.a.handle(), db, g.handle(), C.byref(o), dx, C.byref(h)))
        x = np.empty(nn)
        check(L.kp_memcpy_d2h(ptr(x), dx, nn * 8))
        assert h.iterations_used == ref.history.iterations_used
        assert np.array_equal(x, ref.x)
        assert np.array_equal(bufs[1][:h.rows], np.array(ref.history.residual_norm))
        assert np.array_equal(bufs[0][:h.rows], np.array(ref.history.relative_error))
        for p in (db, dxt, dx):
            L.kp_device_free(p)


@pytest.mark.parametrize("n,r", [(1546, 2), (700, 5), (905, 3)])
def test_dense_operator_tma_tiles_ragged(n, r):
    """The 128 x 128 DMMA tiles staged by TMA (big-tile grid: n = 1546, or the
    M = r n product at n = 700), ragged in M, N and K: rows, columns and the K
    tail outside the matrix come from the TMA zero fill; odd n (905: rows not
    16-byte aligned) takes the cp.async staging. kron.cpp:62-88 against numpy."""
    rng = np.random.default_rng(17)
    terms = [KronTerm(rng.standard_normal((n, n)), rng.standard_normal((n, n))) for _ in range(r)]
    op = KroneckerSum(terms, n)
    op.set_mode("dense")
    x = rng.standard_normal(n * n)
    X = x.reshape(n, n, order="F")
    ref = sum(t.col_factor @ X @ t.row_factor.T for t in terms).reshape(-1, order="F")
    reft = sum(t.col_factor.T @ X @ t.row_factor for t in terms).reshape(-1, order="F")
    y, yt = K.kronsum_apply(op, x), K.kronsum_apply_transpose(op, x)
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    assert np.linalg.norm(yt - reft) <= 1e-13 * np.linalg.norm(reft)
