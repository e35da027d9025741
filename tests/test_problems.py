"""Host problem generator (restates deblur.cpp) and the BASELINE configs.
CPU only: the operator checks use the CPU oracle."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2311_15393_b200 import configs
from paper_2311_15393_b200 import problems as P


def conv_zero_bc(x, psf):
    """Brute-force zero-boundary 2-D convolution (test_deblur.cpp:18-55)."""
    n = x.shape[0]
    v, c = psf.values, psf.center_row
    out = np.zeros_like(x)
    npk = v.shape[0]
    for k in range(npk):
        for l in range(npk):
            di, dj = k - c, l - psf.center_col
            src = x[max(0, -di):n - max(0, di), max(0, -dj):n - max(0, dj)]
            out[max(0, di):n - max(0, -di), max(0, dj):n - max(0, -dj)] += v[k, l] * src
    return out


@pytest.mark.parametrize("kind", ["gaussian", "defocus", "motion", "shake", "speckle"])
@pytest.mark.parametrize("n", [8, 16])
def test_kronsum_equals_convolution(kind, n):  # acceptance criterion 4
    psf = P.make_psf(kind, 5, sigma=1.3, radius=2.0, length=3, steps=16, blob_count=3, seed=7)
    assert psf.values.min() >= 0 and abs(psf.values.sum() - 1.0) < 1e-14
    a, _ = P.psf_to_kronsum(psf, n, truncation_tol=0.0)
    x = np.random.default_rng(n).standard_normal((n, n))
    want = conv_zero_bc(x, psf)
    got = O.kronsum_apply(a, x.reshape(-1, order="F")).reshape(n, n, order="F")
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())
    # the transpose is correlation = convolution with the flipped kernel
    flipped = P.Psf(psf.values[::-1, ::-1].copy(), 4 - psf.center_row, 4 - psf.center_col)
    gt = O.kronsum_apply_transpose(a, x.reshape(-1, order="F")).reshape(n, n, order="F")
    assert np.abs(gt - conv_zero_bc(x, flipped)).max() <= 1e-12 * max(1.0, np.abs(gt).max())


def test_gaussian_is_rank_one_and_nearest_kron_exact():
    psf = P.make_psf("gaussian", 5, sigma=1.5)
    a, _ = P.psf_to_kronsum(psf, 8)  # default tol 1e-12 drops the roundoff terms
    assert len(a.terms) == 1
    t = P.nearest_kron(psf, 8)
    dense = np.kron(a.terms[0].row_factor, a.terms[0].col_factor)
    approx = np.kron(t.row_factor, t.col_factor)
    assert np.linalg.norm(dense - approx) <= 1e-12 * np.linalg.norm(dense)
    delta = P.make_psf("defocus", 5, radius=0.0)
    t = P.nearest_kron(delta, 8)
    assert np.abs(t.row_factor - np.eye(8)).max() <= 1e-12


def test_nearest_kron_matches_oracle_restatement():
    psf = P.make_psf("speckle", 7, blob_count=5, seed=11)
    t = P.nearest_kron(psf, 12)
    rf, cf = O.nearest_kron(psf, 12)
    assert np.allclose(t.row_factor, rf, rtol=0, atol=1e-14)
    assert np.allclose(t.col_factor, cf, rtol=0, atol=1e-14)


def test_banded_toeplitz_structure():
    psf = P.make_psf("gaussian", 5, sigma=1.0)
    a, _ = P.psf_to_kronsum(psf, 9)
    c = a.terms[0].col_factor
    for i in range(9):
        for j in range(9):
            if abs(i - j) > 2:
                assert c[i, j] == 0.0
            elif i + 1 < 9 and j + 1 < 9:
                assert c[i, j] == c[i + 1, j + 1]


def test_make_test_problem_noise_scaling():  # deblur.cpp:214-227
    psf = P.make_psf("gaussian", 5, sigma=1.5)
    tp = P.make_test_problem(P.default_test_image(16), psf, 0.05, 9)
    assert np.linalg.norm(tp.noise) / np.linalg.norm(tp.b_true) == pytest.approx(0.05, rel=1e-14)
    assert np.array_equal(tp.b, tp.b_true + tp.noise)
    tp2 = P.make_test_problem(P.default_test_image(16), psf, 0.05, 9)
    assert np.array_equal(tp.b, tp2.b)
    tp0 = P.make_test_problem(P.default_test_image(16), psf, 0.0, 9)
    assert np.array_equal(tp0.noise, np.zeros(256))
    with pytest.raises(ValueError):
        P.make_test_problem(P.default_test_image(16), psf, -0.1, 9)


def test_rng_is_deterministic_and_normal():
    a, b = P.rng_normals(42, 200000), P.rng_normals(42, 200000)
    assert np.array_equal(a, b)
    assert abs(a.mean()) < 0.01 and abs(a.std() - 1.0) < 0.01


def test_default_image_and_blobs():
    img = P.default_test_image(20)
    assert set(np.unique(img)) <= {0.1, 0.7, 1.0}
    b = P.blob_image(64, 5)
    assert b.min() >= 0.0 and b.max() <= 1.0 and b.max() > 0.0
    assert np.array_equal(b, P.blob_image(64, 5)) and not np.array_equal(b, P.blob_image(64, 6))


def test_config_shapes_reduced():
    c1 = configs.build("C1", n=64)
    assert len(c1.problem.a.terms) == 1 and c1.lambda_ == 0.01
    c2 = configs.build("C2", n=64)
    assert len(c2.problem.a.terms) == 3 and c2.lambda_ == 0.005
    c5 = configs.build("C5", n=64)
    assert len(c5.problem.a.terms) == 5
    assert c5.problem.psf.values.shape == (41, 41)
    c4 = [configs.build("C4", image=i, n=64).problem.noise_level for i in range(3)]
    assert c4 == [0.001, 0.01, 0.05]
    assert configs.GCV_GRID[0] == 1e-4 and configs.GCV_GRID[-1] == 1.0 and configs.GCV_GRID.size == 64


def test_c_abi_psf_to_kronsum_and_nearest_kron():
    """kp_psf_to_kronsum / kp_nearest_kron (the boundary's operator setup,
    deblur.hpp:69-70, factor.hpp:34-35) are host-only: they run here without a
    GPU and agree with the package wrappers and the oracle."""
    import ctypes as C
    from paper_2311_15393_b200._lib import check, lib, ptr
    from oracle import pyoracle as O
    L = lib()
    psf = P.make_psf("gaussian", 9, sigma=1.5)
    n = 24
    v = np.asfortranarray(psf.values)
    rows = np.zeros((n, n * 9), order="F")
    cols = np.zeros((n, n * 9), order="F")
    r = C.c_int()
    check(L.kp_psf_to_kronsum(ptr(v), 9, psf.center_row, psf.center_col, n, 1e-12, 0, 9, ptr(rows),
                              ptr(cols), C.byref(r)))
    a, _ = P.psf_to_kronsum(psf, n)
    assert r.value == len(a.terms)
    for k, t in enumerate(a.terms):
        assert np.array_equal(rows[:, k * n:(k + 1) * n], t.row_factor)
        assert np.array_equal(cols[:, k * n:(k + 1) * n], t.col_factor)
    for weighting, code in (("uniform", 0), ("toeplitz", 1)):
        rf = np.zeros((n, n), order="F")
        cf = np.zeros((n, n), order="F")
        check(L.kp_nearest_kron(ptr(v), 9, psf.center_row, psf.center_col, n, code, ptr(rf), ptr(cf)))
        t = P.nearest_kron(psf, n, weighting)
        assert np.array_equal(rf, t.row_factor) and np.array_equal(cf, t.col_factor)
        if weighting == "toeplitz":  # the oracle restates the reference default
            orf, ocf = O.nearest_kron(psf, n)
            assert np.allclose(rf, orf, rtol=0, atol=1e-12) and np.allclose(cf, ocf, rtol=0, atol=1e-12)
    # argument errors are KP_ERR_INVALID_ARGUMENT with the reference's message
    assert L.kp_nearest_kron(ptr(v), 9, 4, 4, 5, 1, ptr(rf), ptr(cf)) == 1
    assert b"image smaller than psf" in L.kp_last_error()
