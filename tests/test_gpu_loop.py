"""The device-side solve loop (drive(): one CUDA graph whose WHILE
conditional node replays the iteration until the status word leaves
RUNNING) against the host-polled graph replay it replaces by default: same
iterates bit for bit, same histories and stop reasons, for every solver
(krylov.cpp:58-142 pcg / fpcg, :154-208 cgls), preconditioner format and
batched solve — stopping by convergence, by the iteration cap and by an
abort — and the loop actually runs (kp_drive_stats)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200._lib import check, lib
from paper_2311_15393_b200.kronprec import SolverOptions

pytestmark = pytest.mark.gpu


def stats():
    a, b = C.c_longlong(), C.c_longlong()
    check(lib().kp_drive_stats(C.byref(a), C.byref(b)))
    return a.value, b.value


def run(fn, loop: bool):
    old = os.environ.get("KP_GRAPH_LOOP")
    os.environ["KP_GRAPH_LOOP"] = "1" if loop else "0"
    try:
        s0 = stats()
        out = fn()
        s1 = stats()
    finally:
        if old is None:
            del os.environ["KP_GRAPH_LOOP"]
        else:
            os.environ["KP_GRAPH_LOOP"] = old
    return out, (s1[0] - s0[0], s1[1] - s0[1])


def same(r1, r2):
    h1, h2 = r1.history, r2.history
    assert h1.iterations_used == h2.iterations_used
    assert h1.converged == h2.converged and h1.abort_reason == h2.abort_reason
    assert h1.residual_norm == h2.residual_norm
    assert h1.relative_error == h2.relative_error
    assert h1.work_units == h2.work_units
    assert h1.residual_cosines == h2.residual_cosines
    assert np.array_equal(r1.x, r2.x)


@pytest.fixture(scope="module")
def prob():
    n = 96
    psf = P.make_psf("gaussian", 17, sigma=2.5)
    a, _ = P.psf_to_kronsum(psf, n)
    term = P.nearest_kron(psf, n)
    tp = P.make_test_problem(P.blob_image(n, 11), psf, 0.01, 12, a=a)
    return a, term, tp


@pytest.mark.parametrize("solver", ["pcg", "fpcg", "cgls"])
@pytest.mark.parametrize("fmt", ["fp16", "fp64", "bfloat16"])
@pytest.mark.parametrize("stop", ["converged", "maxit"])
def test_loop_equals_polled(prob, solver, fmt, stop):
    a, term, tp = prob
    lam = 0.02
    maxit, tol = (200, 1e-4) if stop == "converged" else (7, 1e-14)
    opts = SolverOptions(lambda_=lam, max_iterations=maxit, rel_residual_tol=tol, x_true=tp.x_true,
                         track_search_direction_orthogonality=True)
    if solver == "cgls":
        if fmt != "fp16":
            pytest.skip("cgls has no preconditioner")
        fn = lambda: K.cgls(a, tp.b, opts)  # noqa: E731
    else:
        m = K.build_preconditioner(term.row_factor, term.col_factor, lam, K.PrecisionFormat.parse(fmt))
        fn = lambda: getattr(K, solver)(a, tp.b, m, opts)  # noqa: E731
    r_loop, st_loop = run(fn, True)
    r_poll, st_poll = run(fn, False)
    assert st_loop == (1, 0), "the solve did not run as a device loop"
    assert st_poll == (0, 1)
    same(r_loop, r_poll)
    if stop == "maxit":  # (an fp64 preconditioner of this separable PSF is exact: it may stop sooner)
        h = r_loop.history
        assert h.iterations_used == maxit or h.converged or h.abort_reason
        assert h.iterations_used <= maxit
    else:
        assert r_loop.history.converged or r_loop.history.abort_reason


def test_loop_abort_and_immediate_stop(prob):
    """An abort inside the loop (tensor-mode products lose positivity on a
    tiny tolerance) and a solve that stops before the first iteration
    (b = 0: converged at iteration 0) both match the polled driver."""
    a, term, tp = prob
    m = K.build_preconditioner(term.row_factor, term.col_factor, 1e-6, K.PrecisionFormat.fp16())
    o = SolverOptions(lambda_=1e-6, max_iterations=300, rel_residual_tol=1e-15, x_true=tp.x_true)
    r1, _ = run(lambda: K.pcg(a, tp.b, m, o), True)
    r2, _ = run(lambda: K.pcg(a, tp.b, m, o), False)
    same(r1, r2)
    o0 = SolverOptions(lambda_=0.02, max_iterations=50, rel_residual_tol=1e-6)
    z = np.zeros_like(tp.b)

    def outcome(loop):
        try:
            return run(lambda: K.pcg(a, z, m, o0), loop)[0]
        except Exception as e:  # the same error either way
            return f"{type(e).__name__}: {e}"
    r1, r2 = outcome(True), outcome(False)
    if isinstance(r1, str) or isinstance(r2, str):
        assert r1 == r2
    else:
        same(r1, r2)
        assert r1.history.iterations_used <= 1


@pytest.mark.parametrize("solver", ["pcg_batch", "fpcg_batch"])
def test_loop_batch_equals_polled(prob, solver):
    a, term, _ = prob
    n = 96
    psf = P.make_psf("gaussian", 17, sigma=2.5)
    tps = [P.make_test_problem(P.blob_image(n, 40 + i), psf, [0.001, 0.01, 0.05][i % 3], 50 + i, a=a)
           for i in range(4)]
    m0 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, K.PrecisionFormat.fp16())
    lams = [0.01, 0.03, 0.1, 0.3]
    opts = SolverOptions(max_iterations=40, rel_residual_tol=1e-5)
    bs = np.stack([tp.b for tp in tps])
    xts = np.stack([tp.x_true for tp in tps])
    fn = lambda: getattr(K, solver)(a, bs, m0, lams, opts, x_true=xts)  # noqa: E731
    rl, st = run(fn, True)
    rp, _ = run(fn, False)
    assert st == (1, 0)
    for x, y in zip(rl, rp):
        same(x, y)
    assert len({r.history.iterations_used for r in rl}) > 1  # images stop at different iterations


def test_loop_counts_working_launches(prob):
    """gpu_launches accounting: a looped solve counts the head kernel plus
    (iteration kernels + the condition kernel) per body run. Solves capped
    at 5 and 9 iterations (no overshoot in the polled driver either: its
    chunks never pass max_iterations) differ by 4 bodies in both modes."""
    a, term, tp = prob
    m = K.build_preconditioner(term.row_factor, term.col_factor, 0.02, K.PrecisionFormat.fp16())
    L = lib()

    def count(maxit, loop):
        o = SolverOptions(lambda_=0.02, max_iterations=maxit, rel_residual_tol=1e-15, x_true=tp.x_true)
        run(lambda: K.pcg(a, tp.b, m, o), loop)  # first use of m: lazy buffer set-up launches
        c0 = L.kp_launch_count()
        r, _ = run(lambda: K.pcg(a, tp.b, m, o), loop)
        assert r.history.iterations_used == maxit
        return L.kp_launch_count() - c0
    d_loop = count(9, True) - count(5, True)
    d_poll = count(9, False) - count(5, False)
    assert d_poll > 0 and d_loop == d_poll + 4
