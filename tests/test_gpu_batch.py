"""Batched PCG / FPCG (kp_pcg_batch): a batch of right-hand sides with one
lambda each, solved in one device state machine (images stacked along the
GEMM N dimension of the M-solve products, grid.z of the banded operator
passes, one DevState per image) must give, image by image, exactly what the
single solve gives (cli.cpp:469-486: with_lambda + pcg per image) — same
iterates bit for bit, same histories, same stop / abort."""
import numpy as np
import pytest

import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200.kronprec import SolverOptions

pytestmark = pytest.mark.gpu
H = K.PrecisionFormat.fp16()


def batch_problem(n, count, sigma=2.5, np_=17):
    psf = P.make_psf("gaussian", np_, sigma=sigma)
    a, _ = P.psf_to_kronsum(psf, n)
    term = P.nearest_kron(psf, n)
    tps = [P.make_test_problem(P.blob_image(n, 4000 + i), psf, [0.001, 0.01, 0.05][i % 3], 5000 + i, a=a)
           for i in range(count)]
    return a, term, tps


@pytest.fixture(params=["auto", "cuda", "tensor"])
def engine(request):
    K.set_fp16_products(request.param)
    yield request.param
    K.set_fp16_products("auto")


@pytest.mark.parametrize("solver", ["pcg", "fpcg"])
@pytest.mark.parametrize("n,count", [(64, 5), (96, 3), (100, 2), (128, 4)])
def test_batch_equals_single_solves(engine, solver, n, count):
    a, term, tps = batch_problem(n, count)
    m0 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, H)
    lams = [0.02 * (1 + i) for i in range(count)]
    opts = SolverOptions(max_iterations=25, rel_residual_tol=1e-6)
    bs = np.stack([tp.b for tp in tps])
    xts = np.stack([tp.x_true for tp in tps])
    res = getattr(K, f"{solver}_batch")(a, bs, m0, lams, opts, x_true=xts)
    for i, tp in enumerate(tps):
        o = SolverOptions(lambda_=lams[i], max_iterations=25, rel_residual_tol=1e-6, x_true=tp.x_true)
        single = getattr(K, solver)(a, tp.b, K.with_lambda(m0, lams[i]), o)
        hb, hs = res[i].history, single.history
        assert hb.iterations_used == hs.iterations_used
        assert hb.converged == hs.converged and hb.abort_reason == hs.abort_reason
        assert hb.msolve_count == hs.msolve_count
        assert hb.residual_norm == hs.residual_norm
        assert hb.relative_error == hs.relative_error
        assert np.array_equal(res[i].x, single.x)


def test_batch_dense_operator_path():
    a, term, tps = batch_problem(64, 3)
    a.set_mode("dense")
    m0 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, H)
    lams = [0.03, 0.01, 0.2]
    opts = SolverOptions(max_iterations=15, rel_residual_tol=1e-6)
    res = K.pcg_batch(a, np.stack([tp.b for tp in tps]), m0, lams, opts,
                      x_true=np.stack([tp.x_true for tp in tps]))
    for i, tp in enumerate(tps):
        o = SolverOptions(lambda_=lams[i], max_iterations=15, rel_residual_tol=1e-6, x_true=tp.x_true)
        single = K.pcg(a, tp.b, K.with_lambda(m0, lams[i]), o)
        assert res[i].history.residual_norm == single.history.residual_norm
        assert np.array_equal(res[i].x, single.x)


def test_batch_mixed_stops():
    """Images that converge, abort and run to the cap in one batch: each one
    freezes at its own stop while the others continue."""
    a, term, tps = batch_problem(64, 3)
    m0 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, H)
    bs = np.stack([tps[0].b, np.zeros_like(tps[1].b), tps[2].b])  # image 1: b = 0 -> converged at once
    lams = [0.5, 0.05, 0.004]
    opts = SolverOptions(max_iterations=40, rel_residual_tol=1e-3)
    res = K.pcg_batch(a, bs, m0, lams, opts)
    for i in range(3):
        o = SolverOptions(lambda_=lams[i], max_iterations=40, rel_residual_tol=1e-3)
        single = K.pcg(a, bs[i], K.with_lambda(m0, lams[i]), o)
        assert res[i].history.iterations_used == single.history.iterations_used
        assert res[i].history.abort_reason == single.history.abort_reason
        assert np.array_equal(res[i].x, single.x)
    assert res[1].history.iterations_used == 0 and res[1].history.converged


def test_batch_validation():
    a, term, tps = batch_problem(32, 2)
    m0 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, H)
    bs = np.stack([tp.b for tp in tps])
    with pytest.raises(ValueError):
        K.pcg_batch(a, bs, m0, [0.1], SolverOptions())
    m64 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, K.PrecisionFormat.fp64())
    with pytest.raises(Exception, match="fp16 preconditioner"):
        K.pcg_batch(a, bs, m64, [0.1, 0.2], SolverOptions())


@pytest.mark.parametrize("n,count", [(128, 4), (96, 3)])
def test_tensor_mode_batch_equals_single_solves(n, count):
    """KP_ACCUM_TENSOR batches: tcgen05 products with the images stacked along
    M (n % 128 == 0) or one image at a time; each image equals the single
    tensor-mode solve bit for bit."""
    a, term, tps = batch_problem(n, count)
    m0 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, H, accum="tensor")
    lams = [0.02 * (1 + i) for i in range(count)]
    opts = SolverOptions(max_iterations=20, rel_residual_tol=1e-6)
    res = K.pcg_batch(a, np.stack([tp.b for tp in tps]), m0, lams, opts,
                      x_true=np.stack([tp.x_true for tp in tps]))
    for i, tp in enumerate(tps):
        o = SolverOptions(lambda_=lams[i], max_iterations=20, rel_residual_tol=1e-6, x_true=tp.x_true)
        single = K.pcg(a, tp.b, K.with_lambda(m0, lams[i]), o)
        assert res[i].history.iterations_used == single.history.iterations_used
        assert res[i].history.residual_norm == single.history.residual_norm
        assert np.array_equal(res[i].x, single.x)


def test_discrepancy_batch_equals_per_image():
    a, term, tps = batch_problem(96, 6)
    m0 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, H)
    noise = [float(np.linalg.norm(tp.noise)) for tp in tps]
    noise[4] *= 1e6  # eta * ||e|| beyond the reachable residual: no root
    lam, st = K.discrepancy_batch(m0, np.stack([tp.b for tp in tps]), noise, 1.01)
    for i, tp in enumerate(tps):
        sd = K.make_spectral_data(m0, tp.b)
        if i == 4:
            with pytest.raises(K.NoRootError):
                K.discrepancy(sd, noise[i], 1.01)
            assert st[i] != 0 and np.isnan(lam[i])
            continue
        assert st[i] == 0
        assert lam[i] == K.discrepancy(sd, noise[i], 1.01).lambda_  # bit-identical
    # the same batch left in device memory (kp_discrepancy_batch_ex, device_pointers = 1)
    import ctypes as C

    from paper_2311_15393_b200._lib import check, lib, ptr
    L = lib()
    bs = np.ascontiguousarray(np.stack([tp.b for tp in tps]))
    d_b = C.c_void_p()
    check(L.kp_device_alloc(bs.nbytes, C.byref(d_b)))
    check(L.kp_memcpy_h2d(d_b, ptr(bs), bs.nbytes))
    nz = np.asarray(noise, dtype=np.float64)
    lam_d, st_d = np.zeros(len(tps)), np.zeros(len(tps), dtype=np.int32)
    check(L.kp_discrepancy_batch_ex(m0.handle(), len(tps), d_b, ptr(nz), 1.01, ptr(lam_d),
                                    st_d.ctypes.data_as(C.c_void_p), 1))
    check(L.kp_device_free(d_b))
    assert np.array_equal(st_d, np.asarray(st)) and np.array_equal(lam_d, np.asarray(lam), equal_nan=True)


def test_device_svd_backend():
    """svd_dense on the device (cuSOLVER): a = u diag(s) v^T, orthonormal
    factors, s nonincreasing and equal to LAPACK's; a preconditioner built
    from the device factors is bit-identical to the oracle's built from the
    same factors."""
    from oracle import pyoracle as O
    from paper_2311_15393_b200.kronprec import SvdTriple
    psf = P.psf_aniso_gaussian(31, [[4.0, 1.0], [1.0, 2.0]])
    term = P.nearest_kron(psf, 256)
    for f in (term.row_factor, term.col_factor):
        u, s, v = K.svd(f, "device")
        uh, sh, vh = K.svd(f, "host")
        assert np.all(np.diff(s) <= 0)
        assert np.allclose(s, sh, rtol=1e-12, atol=1e-14 * sh[0])
        assert np.linalg.norm(u * s @ v.T - f) <= 1e-13 * np.linalg.norm(f)
        assert np.linalg.norm(u.T @ u - np.eye(256)) <= 1e-12
        assert np.linalg.norm(v.T @ v - np.eye(256)) <= 1e-12
    sr = SvdTriple(*K.svd(term.row_factor, "device"))
    sc = SvdTriple(*K.svd(term.col_factor, "device"))
    g = K.build_preconditioner_from_svd(sr, sc, 0.01, H)
    o = O.build_preconditioner_from_svd((sr.u, sr.s, sr.v), (sc.u, sc.s, sc.v), 0.01, H)
    r = np.random.default_rng(3).standard_normal(256 * 256)
    assert np.array_equal(K.precond_solve(g, r), O.precond_solve(o, r))
    # build_preconditioner through the device backend equals the from-SVD build
    K.set_svd_backend("device")
    try:
        gd = K.build_preconditioner(term.row_factor, term.col_factor, 0.01, H)
    finally:
        K.set_svd_backend("host")
    assert np.array_equal(K.precond_solve(gd, r), K.precond_solve(g, r))


def test_zero_x_true_rejected_single_and_batch():
    """krylov.cpp:21-25: an all-zero x_true is invalid_argument("solver:
    x_true must be nonzero") — raised by the library's device-side check for
    single and batched solves (no host pass over x_true)."""
    a, term, tps = batch_problem(64, 3)
    m0 = K.build_preconditioner(term.row_factor, term.col_factor, 1.0, H)
    z = np.zeros_like(tps[0].x_true)
    with pytest.raises(ValueError, match="x_true must be nonzero"):
        K.pcg(a, tps[0].b, K.with_lambda(m0, 0.05),
              SolverOptions(lambda_=0.05, max_iterations=5, rel_residual_tol=1e-6, x_true=z))
    bs = np.stack([tp.b for tp in tps])
    xts = np.stack([tps[0].x_true, z, tps[2].x_true])
    with pytest.raises(ValueError, match="x_true must be nonzero"):
        K.pcg_batch(a, bs, m0, [0.05] * 3, SolverOptions(max_iterations=5, rel_residual_tol=1e-6), x_true=xts)
