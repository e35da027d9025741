"""Bitwise parity of the reference-exact binary16 GEMMs at the tile
configurations the BASELINE configs actually run, and FP64 iterate parity at
n = 4096.

* gemm_f16ref switches to 32 x 64 tiles (BN = 64) once the 32 x 64 grid has
  >= 8 CTAs per SM (n >~ 1600, the C3 / C5 sizes), and gemm_f16x (tcgen05
  rounded products, the default engine from n >= 512) runs everywhere from
  C2 up. Both engines are checked bit for bit — sign of zero included —
  against the oracle (lp_matmul, lpblas.cpp:59-70) and against committed
  oracle digests of precond_solve (factor.cpp:117-132) at n = 1664 and at the
  headline n = 4096 (tests/golden/msolve_n*.json).
* CGLS (FP64 only) at C5: the first five iterates agree with the oracle's to
  1e-10 relative (north star), fingerprinted by their norms and projections
  on four seeded vectors (tests/golden/C5_cgls_iterates.json).
"""
import json
import os
import sys

import numpy as np
import pytest

import paper_2311_15393_b200 as K
from oracle import pyoracle as O
from paper_2311_15393_b200 import configs
from paper_2311_15393_b200.kronprec import SolverOptions, SvdTriple

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from msolve_inputs import digest, msolve_case  # noqa: E402

H = K.PrecisionFormat.fp16()


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return False
    nan = np.isnan(a)
    return (np.array_equal(nan, np.isnan(b)) and np.array_equal(a[~nan], b[~nan])
            and np.array_equal(np.signbit(a[~nan]), np.signbit(b[~nan])))


@pytest.fixture(params=["cuda", "tensor"])
def engine(request):
    K.set_fp16_products(request.param)
    yield request.param
    K.set_fp16_products("auto")


def f16(x):
    return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)


@pytest.mark.parametrize("case", ["normal", "tiny_signed", "zero_cols"])
def test_lp_matmul_bn64_tiles_bitwise(engine, case):
    """2048 x 300 x 1280: 64 x 20 tiles of 32 x 64 = 1280 CTAs >= 8 per SM,
    so gemm_f16ref runs its BN = 64 configuration (the C3 / C5 one)."""
    m, k, n = 2048, 300, 1280
    rng = np.random.default_rng(64)
    a = f16(rng.uniform(-1, 1, (m, k)))
    b = f16(rng.uniform(-1, 1, (k, n)))
    if case == "tiny_signed":  # products underflow: all-zero trees, sign rule decides
        b = f16(b * 1e-7)
    elif case == "zero_cols":
        b[:, ::7] = 0.0
        b[:, 3::7] = -0.0
        a[::5, :] = -0.0
    c = K.lp_matmul(a, b, H)
    co = O.lp_matmul(a, b, H)
    assert same_bits(c, co)


def test_lp_matmul_engine_is_what_the_solve_uses():
    assert K.fp16_products_engine(4096) == "tensor"
    assert K.fp16_products_engine(1024) == "tensor"
    assert K.fp16_products_engine(256) == "cuda"


@pytest.mark.parametrize("n", [1664, 4096])
@pytest.mark.parametrize("regime", ["wide", "low"])
def test_precond_solve_golden_digest(engine, n, regime):
    """precond_solve at the C5 size (and at n = 1664, the first BN = 64
    size) is bit-identical to the oracle's committed result."""
    path = os.path.join(HERE, "golden", f"msolve_n{n}.json")
    if not os.path.exists(path):
        pytest.skip(f"golden msolve_n{n}.json not generated")
    g = json.load(open(path))
    ref = g["cases"][regime]
    sr, sc, lam, r = msolve_case(n, g["seed"], regime)
    m = K.build_preconditioner_from_svd(SvdTriple(*sr), SvdTriple(*sc), lam, H)
    z = K.precond_solve(m, r)
    d = digest(z)
    assert d["zeros"] == ref["digest"]["zeros"]
    assert d["neg_zeros"] == ref["digest"]["neg_zeros"]
    assert d["sha256"] == ref["digest"]["sha256"]


def test_precond_solve_n1664_live_vs_oracle():
    """Same case run through the oracle here (no golden involved)."""
    sr, sc, lam, r = msolve_case(1664, 77, "low")
    m = K.build_preconditioner_from_svd(SvdTriple(*sr), SvdTriple(*sc), lam, H)
    mo = O.build_preconditioner_from_svd(sr, sc, lam, H)
    assert same_bits(K.precond_solve(m, r), O.precond_solve(mo, r))


def test_c5_cgls_first_iterates_1e10():
    """North star: the unpreconditioned CGLS path agrees to 1e-10 per
    iterate. Fingerprints: ||x_k|| and <x_k, w_j> for four seeded w_j; a
    1e-10 relative iterate difference bounds each by 1e-10 ||x_k|| ||w_j||."""
    path = os.path.join(HERE, "golden", "C5_cgls_iterates.json")
    if not os.path.exists(path):
        pytest.skip("golden C5_cgls_iterates.json not generated")
    g = json.load(open(path))
    cfg = configs.build("C5")
    opts = SolverOptions(lambda_=cfg.lambda_, max_iterations=g["iterations"], rel_residual_tol=cfg.tol,
                         x_true=cfg.problem.x_true, record_iterates=True)
    res = K.cgls(cfg.problem.a, cfg.problem.b, opts)
    its = res.history.iterates
    assert len(its) == len(g["iterates"])
    nn = cfg.n * cfg.n
    probes = [np.random.default_rng(s).standard_normal(nn) for s in g["probe_seeds"]]
    for k, (x, ref) in enumerate(zip(its, g["iterates"])):
        nx = float(np.linalg.norm(x))
        if ref["norm"] == 0.0:
            assert nx == 0.0
            continue
        assert abs(nx - ref["norm"]) <= 1e-10 * ref["norm"], k
        for w, wn, pr in zip(probes, g["probe_norms"], ref["proj"]):
            assert abs(float(x @ w) - pr) <= 1e-10 * ref["norm"] * wn, k
    for k in range(len(g["residual_norm"])):
        assert res.history.residual_norm[k] == pytest.approx(g["residual_norm"][k], rel=1e-10)
        assert res.history.relative_error[k] == pytest.approx(g["relative_error"][k], rel=1e-10)


@pytest.mark.parametrize("seed", range(10))
def test_lp_matmul_random_shapes_bitwise(engine, seed):
    """Ragged shapes (M, N not multiples of the tiles, K not a multiple of
    64, K = 1, single rows / columns) and mixed magnitudes incl. signed zeros,
    subnormal products and a few infinities in B (A must stay finite for
    gemm_f16x, see gemm_f16x.cu): both engines against the oracle, bit for
    bit."""
    rng = np.random.default_rng(1000 + seed)
    m, k, n = (int(x) for x in rng.integers(1, 300, 3))
    if seed == 0:
        m, k, n = 1, 1, 1
    elif seed == 1:
        k = 1
    scale_a = 2.0 ** rng.integers(-14, 6, (m, k))
    scale_b = 2.0 ** rng.integers(-14, 6, (k, n))
    a = f16(rng.standard_normal((m, k)) * scale_a)
    b = f16(rng.standard_normal((k, n)) * scale_b)
    a[rng.random((m, k)) < 0.05] = -0.0
    b[rng.random((k, n)) < 0.05] = 0.0
    if seed % 3 == 2:
        b[rng.random((k, n)) < 0.01] = np.inf
    c = K.lp_matmul(a, b, H)
    assert same_bits(c, O.lp_matmul(a, b, H))
