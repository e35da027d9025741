"""Seeded synthetic test problems (host side, not on the hot path).

Restates the reference generator (deblur.cpp: Rng, make_psf, banded_toeplitz,
psf_to_kronsum, make_test_problem, default_test_image) and adds the BASELINE
configs' generators the reference cannot express (blob image, anisotropic
Gaussian, Gaussian*motion PSF, rank cap). Implemented in C++
(csrc/problem.cpp) so the mt19937_64 streams match the reference bit for bit.
Both arms (CUDA path and CPU oracle) consume these arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import f64, lib, ptr
from .kronprec import KronTerm, KroneckerSum

BLUR_KINDS = {"gaussian": 0, "defocus": 1, "motion": 2, "shake": 3, "speckle": 4}


def _chk(status: int) -> None:
    if status == 0:
        return
    msg = lib().kpg_last_error().decode()
    raise ValueError(msg) if status == 1 else RuntimeError(msg)


@dataclass
class Psf:
    values: np.ndarray
    center_row: int
    center_col: int
    kind: str = "gaussian"
    seed: int = 0
    # BlurParams (deblur.hpp): sigma, radius, length, steps, blob_count, blob_sigma
    params: dict = field(default_factory=lambda: {
        "sigma": 2.0, "radius": 3.0, "length": 5, "steps": 64, "blob_count": 10,
        "blob_sigma": 1.0})


def rng_normals(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().kpg_rng_normals(C.c_uint64(seed), C.c_long(count), ptr(out))
    return out


def make_psf(kind: str, n_p: int, sigma: float = 2.0, radius: float = 3.0, length: int = 5,
             steps: int = 64, blob_count: int = 10, blob_sigma: float = 1.0, seed: int = 0) -> Psf:
    """make_psf (deblur.cpp:130-155)."""
    out = np.empty((n_p, n_p), order="F")
    L = lib()
    _chk(L.kpg_make_psf(BLUR_KINDS[kind], n_p, sigma, radius, length, steps, blob_count,
                        blob_sigma, seed, ptr(out)))
    return Psf(out, n_p // 2, n_p // 2, kind, seed,
               {"sigma": sigma, "radius": radius, "length": length, "steps": steps,
                "blob_count": blob_count, "blob_sigma": blob_sigma})


def psf_aniso_gaussian(n_p: int, cov) -> Psf:
    out = np.empty((n_p, n_p), order="F")
    L = lib()
    _chk(L.kpg_psf_aniso_gaussian(n_p, cov[0][0], cov[0][1], cov[1][1], ptr(out)))
    return Psf(out, n_p // 2, n_p // 2, "aniso_gaussian")


def psf_gauss_motion(n_p: int, sigma: float, length: int, angle_deg: float) -> Psf:
    out = np.empty((n_p, n_p), order="F")
    L = lib()
    _chk(L.kpg_psf_gauss_motion(n_p, sigma, length, angle_deg, ptr(out)))
    return Psf(out, n_p // 2, n_p // 2, "gauss_motion")


def default_test_image(n: int) -> np.ndarray:
    out = np.empty((n, n), order="F")
    _chk(lib().kpg_default_test_image(n, ptr(out)))
    return out


def blob_image(n: int, seed: int, blobs: int = 20) -> np.ndarray:
    out = np.empty((n, n), order="F")
    L = lib()
    _chk(L.kpg_blob_image(n, seed, blobs, ptr(out)))
    return out


def psf_to_kronsum(psf: Psf, n: int, truncation_tol: float = 1e-12,
                   max_rank: int = 0) -> tuple[KroneckerSum, np.ndarray]:
    """psf_to_kronsum (deblur.cpp:167-199) + optional rank cap. Returns the
    operator and the (capped) PSF array sum_{k<r} s_k u_k v_k^T."""
    np_ = psf.values.shape[0]
    cap = np_ if max_rank <= 0 else min(max_rank, np_)
    rows = np.empty((n, n * cap), order="F")
    cols = np.empty((n, n * cap), order="F")
    trunc = np.empty((np_, np_), order="F")
    r = C.c_int()
    v = f64(psf.values)
    L = lib()
    _chk(L.kpg_psf_to_kronsum(ptr(v), np_, psf.center_row, psf.center_col, n, truncation_tol,
                              max_rank, cap, ptr(rows), ptr(cols), C.byref(r), ptr(trunc)))
    terms = [KronTerm(np.asfortranarray(rows[:, k * n:(k + 1) * n]),
                      np.asfortranarray(cols[:, k * n:(k + 1) * n])) for k in range(r.value)]
    return KroneckerSum(terms, n), trunc


def nearest_kron(psf: Psf, n: int, weighting: str = "toeplitz") -> KronTerm:
    """nearest_kron (factor.cpp:25-58)."""
    rf = np.empty((n, n), order="F")
    cf = np.empty((n, n), order="F")
    v = f64(psf.values)
    L = lib()
    _chk(L.kpg_nearest_kron(ptr(v), v.shape[0], psf.center_row, psf.center_col, n,
                            1 if weighting == "toeplitz" else 0, ptr(rf), ptr(cf)))
    return KronTerm(rf, cf)


def kronsum_apply_host(k: KroneckerSum, x: np.ndarray) -> np.ndarray:
    """Host FP64 A x (setup only: b_true)."""
    r = len(k.terms)
    n = k.n
    rows = np.empty((n, n * r), order="F")
    cols = np.empty((n, n * r), order="F")
    for i, t in enumerate(k.terms):
        rows[:, i * n:(i + 1) * n] = t.row_factor
        cols[:, i * n:(i + 1) * n] = t.col_factor
    xv = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1, order="F"))
    out = np.empty(n * n)
    _chk(lib().kpg_kronsum_apply_host(n, r, ptr(rows), ptr(cols), ptr(xv), ptr(out)))
    return out


@dataclass
class TestProblem:
    __test__ = False  # not a pytest class
    a: KroneckerSum
    x_true: np.ndarray
    b_true: np.ndarray
    noise: np.ndarray
    b: np.ndarray
    noise_level: float
    seed: int
    psf: Psf
    n: int


def make_test_problem(image: np.ndarray, psf: Psf, noise_level: float, seed: int,
                      a: KroneckerSum | None = None) -> TestProblem:
    """make_test_problem (deblur.cpp:201-229); `a` overrides psf_to_kronsum
    (rank-capped configs)."""
    image = f64(image)
    n = image.shape[0]
    if image.size == 0:
        raise ValueError("make_test_problem: empty image")
    if image.shape != (n, n):
        raise ValueError("make_test_problem: image must be square")
    if a is None:
        a, _ = psf_to_kronsum(psf, n)
    x_true = image.reshape(-1, order="F").copy()
    b_true = kronsum_apply_host(a, x_true)
    noise = np.empty_like(b_true)
    b = np.empty_like(b_true)
    L = lib()
    _chk(L.kpg_add_noise(b_true.size, ptr(b_true), noise_level, seed, ptr(noise), ptr(b)))
    return TestProblem(a, x_true, b_true, noise, b, noise_level, seed, psf, n)


def make_test_problems_device(a: KroneckerSum, image_seeds, noise_seeds, noise_levels, blobs: int = 20,
                              device_out=None):
    """make_test_problem (deblur.cpp:201-229) for a batch of blob images on
    the device (kp_generate_test_problems): returns (x_true, b, noise,
    noise_norms) as batch x n^2 host arrays, or writes x_true / b into the
    caller's device buffers `device_out = (x_ptr, b_ptr)` and returns the
    noise norms only."""
    n = a.n
    batch = len(image_seeds)
    seeds = np.ascontiguousarray(np.asarray(image_seeds, dtype=np.uint64))
    nseeds = np.ascontiguousarray(np.asarray(noise_seeds, dtype=np.uint64))
    lev = np.ascontiguousarray(np.asarray(noise_levels, dtype=np.float64))
    if nseeds.size != batch or lev.size != batch:
        raise ValueError("make_test_problems_device: one noise seed and level per image")
    norms = np.empty(batch)
    from ._lib import check
    L = lib()
    if device_out is not None:
        check(L.kp_generate_test_problems(a.handle(), batch, seeds.ctypes.data, blobs, nseeds.ctypes.data,
                                          ptr(lev), device_out[0], device_out[1], None, ptr(norms), 1))
        return norms
    x, b, e = np.empty((batch, n * n)), np.empty((batch, n * n)), np.empty((batch, n * n))
    check(L.kp_generate_test_problems(a.handle(), batch, seeds.ctypes.data, blobs, nseeds.ctypes.data,
                                      ptr(lev), ptr(x), ptr(b), ptr(e), ptr(norms), 0))
    return x, b, e, norms


def rng_raw_device(seeds, count: int) -> np.ndarray:
    """std::mt19937_64 outputs on the device (count per seed)."""
    from ._lib import check
    s = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
    out = np.empty((s.size, count), dtype=np.uint64)
    check(lib().kp_rng_raw(s.ctypes.data, s.size, count, out.ctypes.data))
    return out


def host_svd(a: np.ndarray):
    """LAPACK dgesdd (same backend the device path uses for its setup)."""
    a = f64(a)
    m, n = a.shape
    u = np.empty((m, m), order="F")
    s = np.empty(min(m, n))
    v = np.empty((n, n), order="F")
    _chk(lib().kpg_svd(ptr(a), m, n, ptr(u), ptr(s), ptr(v)))
    return u, s, v


def set_blas_threads(t: int) -> None:
    lib().kpg_set_blas_threads(int(t))
