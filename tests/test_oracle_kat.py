"""Pins the CPU oracle (oracle/kp_oracle.cpp) to the reference's own
known-answer tests for the hot path. Each case cites the reference test it
re-expresses (/root/reference/proj/tests/*.cpp). CPU only."""
import math
import struct

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2311_15393_b200 import PrecisionFormat as PF
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200.kronprec import KronTerm, KroneckerSum, SolverOptions

H = PF.fp16()
BF = PF.bfloat16()
S32 = PF.fp32()
D = PF.fp64()


def ref_uniforms(seed, count, lo, hi):
    """std::mt19937_64 stream mapped like the reference tests' uniform()."""
    from paper_2311_15393_b200._lib import lib
    out = np.empty(count)
    lib().kpg_rng_uniforms(seed, count, lo, hi, out.ctypes.data)
    return out


def fp16_bit_oracle(x: float) -> float:
    """Independent integer-only binary64 -> binary16 -> binary64 conversion
    (re-expression of test_precision.cpp:17-63)."""
    bits = struct.unpack("<Q", struct.pack("<d", x))[0]
    neg = bits >> 63
    ebits = (bits >> 52) & 0x7FF
    frac = bits & ((1 << 52) - 1)
    if ebits == 0x7FF or (ebits == 0 and frac == 0):
        return x
    if ebits == 0:
        m, e = frac, -1074
    else:
        m, e = frac | (1 << 52), ebits - 1075
    exp = e + m.bit_length() - 1
    q = exp - 10 if exp >= -14 else -24
    shift = q - e
    if shift <= 0:
        k = m << -shift
    elif shift >= 54:
        k = 0
    else:
        keep, rem, half = m >> shift, m & ((1 << shift) - 1), 1 << (shift - 1)
        k = keep + 1 if (rem > half or (rem == half and (keep & 1))) else keep
    r = math.ldexp(float(k), q)
    if r > 65504.0:
        r = math.inf
    return -r if neg else r


# ---- precision (test_precision.cpp) ----------------------------------------
def test_format_presets():  # :72-103
    assert H.unit_roundoff() == 2.0 ** -11
    assert H.max_finite() == 65504.0 and H.overflow_threshold() == 65520.0
    assert H.min_exponent() == -14 and not H.covers_double()
    assert S32.max_finite() == float(np.finfo(np.float32).max)
    assert D.covers_double()
    c = PF.parse("custom:t=5,emax=3,subnormals=0")
    assert (c.significand_bits, c.max_exponent, c.subnormals_enabled) == (5, 3, False)
    for bad in ("fp12", "custom:t=1,emax=3,subnormals=0"):
        with pytest.raises(ValueError):
            PF.parse(bad)


def test_scalar_pins():  # :105-156
    r = O.round_value
    assert r(1.0, H) == 1.0
    assert r(0.1, H) == 0.0999755859375
    assert r(0.2, H) == 0.199951171875
    assert r(70000.0, H) == math.inf and r(-70000.0, H) == -math.inf
    assert r(65504.0, H) == 65504.0 and r(65519.999, H) == 65504.0 and r(65520.0, H) == math.inf
    assert r(2049.0, H) == 2048.0 and r(2051.0, H) == 2052.0 and r(2053.0, H) == 2052.0
    assert r(0.1, BF) == 0.10009765625 and r(257.0, BF) == 256.0
    assert r(2.0 ** -24, H) == 2.0 ** -24
    assert r(1.5 * 2.0 ** -25, H) == 2.0 ** -24
    assert r(2.0 ** -25, H) == 0.0
    assert math.copysign(1.0, r(-(2.0 ** -25), H)) < 0
    flush = PF.parse("custom:t=11,emax=15,subnormals=0")
    assert r(2.0 ** -14, flush) == 2.0 ** -14
    assert r(0.6 * 2.0 ** -14, flush) == 2.0 ** -14
    assert r(0.4 * 2.0 ** -14, flush) == 0.0
    assert r(2.0 ** -15, flush) == 0.0
    assert math.isnan(r(math.nan, H))
    assert r(math.inf, H) == math.inf and r(-math.inf, H) == -math.inf
    assert math.copysign(1.0, r(-0.0, H)) < 0
    assert r(np.finfo(float).max, D) == np.finfo(float).max
    assert r(0.1, D) == 0.1


def test_round_array_tally():  # :158-204
    s0 = O.round_calls()
    out = O.round_array([0.1, 0.2], H)
    assert list(out) == [0.0999755859375, 0.199951171875]
    O.round_array(np.zeros(0), H)
    assert O.round_calls() - s0 == 2
    s1 = O.round_calls()
    O.round_value(0.1, H)
    assert O.round_calls() == s1


def test_rounding_invariants_seeded():  # :206-245 (sampled)
    rng = np.random.default_rng(12345)
    for fmt in (H, BF):
        mant = rng.uniform(1.0, 2.0, 4000)
        expo = np.floor(rng.uniform(-30.0, 18.0, 4000)).astype(int)
        sign = np.where(rng.integers(0, 2, 4000) == 1, -1.0, 1.0)
        for m, e, s in zip(mant, expo, sign):
            x = s * math.ldexp(m, int(e))
            rr = O.round_value(x, fmt)
            assert O.round_value(rr, fmt) == rr
            assert O.round_value(-x, fmt) == -rr
            mag = abs(x)
            if math.ldexp(1.0, fmt.min_exponent()) <= mag <= fmt.max_finite():
                assert abs(rr - x) <= fmt.unit_roundoff() * mag
    for k in range(2049):
        assert O.round_value(float(k), H) == float(k)


def test_fp16_conformance_vs_bit_oracle():  # :247-281 and acceptance.cpp:89-177
    edges = [0.1, 1 / 3, 65503.999, 65519.99, 65520.0, 65536.0, 1e-5, 2.0 ** -24, 2.0 ** -25,
             math.ldexp(1.0078125, -25), 0.49 * 2.0 ** -24, 0.51 * 2.0 ** -24, 2051.0, 2049.0,
             6e4, -6e4, 0.0, -0.0, math.inf, -math.inf]
    for x in edges:
        a, b = O.round_value(x, H), fp16_bit_oracle(x)
        assert a == b and math.copysign(1, a) == math.copysign(1, b), x
    # the reference's exact seeded sample stream: mt19937_64(987654321), 1e5 draws
    xs = ref_uniforms(987654321, 100000, -6e4, 6e4)
    got = O.round_array(xs, H)
    want = np.array([fp16_bit_oracle(float(x)) for x in xs])
    assert np.array_equal(got, want)
    # and numpy's direct double -> half conversion agrees too
    assert np.array_equal(got, xs.astype(np.float16).astype(np.float64))
    # exact ties
    rng = np.random.default_rng(31337)
    e = np.floor(rng.uniform(-14.0, 15.0, 20000)).astype(int)
    k = rng.uniform(0.0, 1023.0, 20000).astype(np.int64)
    ties = np.array([math.ldexp(float(2 * kk + 1), int(ee) - 11) for kk, ee in zip(k, e)])
    assert np.array_equal(O.round_array(ties, H), [fp16_bit_oracle(t) for t in ties])
    assert np.array_equal(O.round_array(-ties, H), [fp16_bit_oracle(-t) for t in ties])


def test_fp32_matches_hardware():  # :283-295
    rng = np.random.default_rng(55555)
    mant = rng.uniform(1.0, 2.0, 3000)
    expo = np.floor(rng.uniform(-140.0, 128.0, 3000)).astype(int)
    xs = np.array([math.ldexp(m, int(e)) for m, e in zip(mant, expo)])
    with np.errstate(over="ignore"):
        assert np.array_equal(O.round_array(xs, S32), xs.astype(np.float32).astype(np.float64))


# ---- lpblas (test_lpblas.cpp) ------------------------------------------------
def test_pairwise_pins():  # :37-63
    assert O.pairwise_sum(np.ones(8), H) == 8.0
    assert O.pairwise_sum(np.arange(1, 9.0), H) == 36.0
    assert O.pairwise_sum([2048, 2, 1, 1], H) == 2052.0
    assert O.pairwise_sum([2048, 1, 1, 1], H) == 2050.0
    assert O.pairwise_sum([7.0], H) == 7.0
    with pytest.raises(ValueError):
        O.pairwise_sum(np.zeros(0), H)


def test_rounding_call_budgets():  # :65-100
    rng = np.random.default_rng(777)
    for n in (1, 2, 3, 5, 8, 64, 100, 1024):
        z = O.round_array(rng.uniform(-1, 1, n), H)
        stages = 0 if n == 1 else math.ceil(math.log2(n))
        s = O.round_calls()
        O.pairwise_sum(z, H)
        assert O.round_calls() - s == stages
        s = O.round_calls()
        O.lp_dot(z, z, H)
        assert O.round_calls() - s == stages + 1
    s = O.round_calls()
    x = rng.uniform(-1, 1, 100)
    got = O.lp_dot(x, x, D)
    assert O.round_calls() == s and got == pytest.approx(x @ x, rel=1e-14)


def test_lp_dot_values_and_bound():  # :102-133
    e3 = np.zeros(8)
    e3[2] = 1
    assert O.lp_dot(e3, np.arange(1, 9.0), H) == 3.0
    assert O.lp_dot(np.ones(16), np.ones(16), H) == 16.0
    with pytest.raises(ValueError):
        O.lp_dot(np.ones(3), np.ones(4), H)
    rng = np.random.default_rng(4242)
    for fmt in (H, BF):
        for n in (10, 64, 100, 1000):
            for _ in range(10):
                x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
                bound = (math.ceil(math.log2(n)) + 2) * fmt.unit_roundoff() * np.abs(x * y).sum()
                assert abs(O.lp_dot(x, y, fmt) - x @ y) <= bound


def test_lp_matvec_and_matmul():  # :135-222
    rng = np.random.default_rng(999)
    v = rng.uniform(-2, 2, 8)
    assert np.array_equal(O.lp_matvec(np.eye(8), v, H), O.round_array(v, H))
    b = rng.uniform(-3, 3, (4, 6))
    assert np.array_equal(O.lp_matmul(np.eye(4), b, H), O.round_array(b, H))
    a = rng.uniform(-3, 3, (3, 5))
    assert np.array_equal(O.lp_matmul(a, np.eye(5), H), O.round_array(a, H))
    assert np.array_equal(O.lp_matmul([[1, 2], [3, 4]], [[5, 6], [7, 8]], H), [[19, 22], [43, 50]])
    with pytest.raises(ValueError):
        O.lp_matmul([[1, 2], [3, 4]], np.ones((3, 2)), H)
    for k in (4, 17, 32):  # single-column product == lp_matvec, tallies too
        m = rng.uniform(-1, 1, (7, k))
        w = rng.uniform(-1, 1, k)
        s = O.round_calls()
        mv = O.lp_matvec(m, w, H)
        c1 = O.round_calls() - s
        s = O.round_calls()
        mm = O.lp_matmul(m, w.reshape(-1, 1), H)
        assert np.array_equal(mm[:, 0], mv) and O.round_calls() - s == c1
    for _ in range(50):  # exact on small integers
        x = np.floor(rng.uniform(-8, 9, (6, 6)))
        y = np.floor(rng.uniform(-8, 9, (6, 6)))
        assert np.array_equal(O.lp_matmul(x, y, H), x @ y)


@pytest.mark.parametrize("K", [1, 2, 3, 5, 6, 7, 8, 11, 13, 16, 17, 31, 33, 63, 64, 65, 100, 128, 200])
def test_streamed_tree_equals_literal(K):
    """The streamed per-element tree (and its fast F16C path) is bit-identical
    to the literal materialising lpblas.cpp transcription, for every K shape
    of the odd-carry tree, including overflow and subnormal operands."""
    rng = np.random.default_rng(K)
    a = O.round_array(rng.uniform(-4, 4, (9, K)) * 10.0 ** rng.integers(-7, 4, (9, K)), H)
    b = O.round_array(rng.uniform(-4, 4, (K, 5)) * 10.0 ** rng.integers(-7, 4, (K, 5)), H)
    a[0, :] = 300.0  # overflowing products/sums
    lit = O.lp_matmul(a, b, H, mode=1)
    for mode in (0, 2):
        got = O.lp_matmul(a, b, H, mode=mode)
        assert np.array_equal(np.isnan(got), np.isnan(lit))
        m = ~np.isnan(lit)
        assert np.array_equal(got[m], lit[m])
        assert np.array_equal(np.signbit(got[m]), np.signbit(lit[m]))
    # non-fp16 formats use the generic streamed path
    for fmt in (BF, PF.parse("custom:t=6,emax=5,subnormals=0")):
        x = rng.uniform(-2, 2, (4, K))
        y = rng.uniform(-2, 2, (K, 3))
        assert np.array_equal(O.lp_matmul(x, y, fmt, 2), O.lp_matmul(x, y, fmt, 1))
    # fp64: the eight-row tree path (mode 0) == generic streamed == literal;
    # 13 rows exercise a partial group of eight, wide magnitudes the order
    x = rng.uniform(-2, 2, (13, K)) * 10.0 ** rng.integers(-8, 8, (13, K))
    y = rng.uniform(-2, 2, (K, 3)) * 10.0 ** rng.integers(-8, 8, (K, 3))
    lit = O.lp_matmul(x, y, PF.fp64(), 1)
    assert np.array_equal(O.lp_matmul(x, y, PF.fp64(), 0), lit)
    assert np.array_equal(O.lp_matmul(x, y, PF.fp64(), 2), lit)


def test_fast_fp16_path_exhaustive_pairs():
    """binary32 arithmetic + one RNE conversion == correctly rounded binary16
    for products and sums: checked on all products/sums of a dense sample of
    binary16 values (incl. subnormals, ties and overflow)."""
    vals = np.arange(0, 0x7C00, 37, dtype=np.uint16).view(np.float16).astype(np.float64)
    vals = np.concatenate([vals, -vals, [2.0 ** -24, 65504.0, 2048.0, 1.0]])
    a = vals[:400].reshape(-1, 1)
    b = vals[::7][None, :400]
    # products, K = 1
    got = O.lp_matmul(a, b, H, 0)
    want = np.vectorize(fp16_bit_oracle)(a * b)
    assert np.array_equal(got, want)
    # sums of two binary16 values via K = 2 with unit weights
    aa = np.concatenate([a, a[::-1]], axis=1)
    got = O.lp_matmul(aa, np.ones((2, 1)), H, 0)
    assert np.array_equal(got[:, 0], np.vectorize(fp16_bit_oracle)(aa[:, 0] + aa[:, 1]))


# ---- factor (test_factor.cpp) -----------------------------------------------------
def gaussian_term(n, np_=5, sigma=1.5):
    return P.nearest_kron(P.make_psf("gaussian", np_, sigma=sigma), n)


def test_svd_contract():  # :57-95
    u, s, v = O.svd(np.eye(3))
    assert np.array_equal(s, np.ones(3))
    perm = np.array([[0, 2, 0], [0, 0, 1], [3, 0, 0.0]])
    assert np.max(np.abs(O.svd(perm)[1] - [3, 2, 1])) <= 1e-12
    rng = np.random.default_rng(808)
    for _ in range(10):
        a = rng.uniform(-1, 1, (6, 6))
        u, s, v = O.svd(a)
        assert np.abs(u.T @ u - np.eye(6)).max() <= 1e-10
        assert np.all(np.diff(s) <= 0) and s[-1] >= 0
        assert np.abs(u @ np.diag(s) @ v.T - a).max() <= 1e-10 * s[0]
        ev = np.sqrt(np.maximum(np.linalg.eigvalsh(a.T @ a), 0))[::-1]
        assert np.allclose(s, ev, rtol=1e-8)
    with pytest.raises(ValueError):
        O.svd(np.array([[1, 2], [3, np.nan]]))


def test_preconditioner_construction_pins():  # :177-238
    p = O.build_preconditioner(np.eye(4), np.eye(4), 1.0, H)
    assert np.array_equal(p.s_weights, np.full((4, 4), 0.5))
    assert np.array_equal(p.s_lp, np.full((4, 4), 0.5))
    p = O.build_preconditioner(np.diag([2.0, 1.0]), np.eye(2), 0.0, D)
    assert np.array_equal(p.s_weights, [[0.25, 1.0], [0.25, 1.0]])
    with pytest.raises(ValueError):
        O.build_preconditioner(np.diag([1.0, 0.0]), np.eye(2), 0.0, D)
    with pytest.raises(ValueError):
        O.build_preconditioner(np.diag([1.0, 0.0]), np.eye(2), -1.0, D)
    with pytest.raises(ValueError):
        O.build_preconditioner(np.diag([1.0, 0.0]), np.eye(3), 1.0, D)
    t = gaussian_term(8)
    p = O.build_preconditioner(t.row_factor, t.col_factor, 0.05, H)
    _, sr, _ = p.svd_r
    _, sc, _ = p.svd_c
    sw = p.s_weights
    for j in range(8):
        for i in range(8):
            den = (sr[j] * sc[i]) ** 2 + 0.05 ** 2
            assert sw[i, j] == 1.0 / den and 0 < sw[i, j] <= 1 / 0.05 ** 2
    assert np.array_equal(p.vr_lp, O.round_array(p.vr_lp, H))
    assert np.array_equal(p.s_lp, O.round_array(sw, H))
    q = O.with_lambda(p, 0.1)
    assert q.s_weights[0, 0] == 1.0 / ((sr[0] * sc[0]) ** 2 + 0.1 * 0.1)


def apply_m(t, lam, z):
    n = t.row_factor.shape[0]
    k = KroneckerSum([KronTerm(t.row_factor, t.col_factor)], n)
    return O.normal_matvec(k, lam, z)


def test_precond_solve_kats():  # :240-318
    rng = np.random.default_rng(11)
    p = O.build_preconditioner(np.eye(4), np.eye(4), 1.0, H)
    r = rng.uniform(-1, 1, 16)
    assert np.array_equal(O.precond_solve(p, r), 0.5 * O.round_array(r, H))
    t = gaussian_term(8)
    p64 = O.build_preconditioner(t.row_factor, t.col_factor, 0.01, D)
    r = rng.uniform(-1, 1, 64)
    z = O.precond_solve(p64, r)
    assert np.linalg.norm(apply_m(t, 0.01, z) - r) <= 1e-10 * np.linalg.norm(r)
    ah = np.kron(t.row_factor, t.col_factor)
    zs = np.linalg.solve(ah.T @ ah + 1e-4 * np.eye(64), r)
    assert np.linalg.norm(z - zs) <= 1e-10 * np.linalg.norm(zs)
    p16 = O.build_preconditioner(t.row_factor, t.col_factor, 0.05, H)
    z = O.precond_solve(p16, r)
    kappa = p16.s_weights.max() / p16.s_weights.min()
    assert np.linalg.norm(apply_m(t, 0.05, z) - r) / np.linalg.norm(r) <= 50 * 2 ** -11 * kappa
    s = O.round_calls()
    O.precond_solve(p16, np.ones(64))
    assert O.round_calls() - s == 2 + 4 * (1 + 3)  # 18 roundings per M-solve at n = 8
    p64b = O.build_preconditioner(t.row_factor, t.col_factor, 0.05, D)
    s = O.round_calls()
    O.precond_solve(p64b, np.ones(64))
    assert O.round_calls() == s
    with pytest.raises(ValueError):
        O.precond_solve(p16, np.ones(63))
    for n in (8, 16, 32):
        tt = gaussian_term(n)
        probe = O.build_preconditioner(tt.row_factor, tt.col_factor, 1.0, D)
        lam = 0.02 * probe.svd_r[1][0] * probe.svd_c[1][0]
        a16 = O.build_preconditioner(tt.row_factor, tt.col_factor, lam, H)
        a64 = O.build_preconditioner(tt.row_factor, tt.col_factor, lam, D)
        r = rng.uniform(-1, 1, n * n)
        z16, z64 = O.precond_solve(a16, r), O.precond_solve(a64, r)
        assert np.linalg.norm(z16 - z64) / np.linalg.norm(z64) <= 1e3 * 2 ** -11


def test_spectrum_and_projection():  # :320-408
    p = O.build_preconditioner(np.eye(3), np.eye(3), 1.0, D)
    b = np.random.default_rng(2025).uniform(-1, 1, 9)
    s, bh = O.spectral(p, b)
    assert np.array_equal(s, np.ones(9)) and np.array_equal(bh, b)
    p = O.build_preconditioner(np.diag([2.0, 1.0]), np.diag([3.0, 1.0]), 0.5, D)
    assert list(O.spectral(p, np.ones(4))[0]) == [6, 3, 2, 1]
    rng = np.random.default_rng(7)
    ar, ac = rng.uniform(-1, 1, (4, 4)), rng.uniform(-1, 1, (4, 4))
    p = O.build_preconditioner(ar, ac, 0.1, D)
    s, bh = O.spectral(p, np.ones(16))
    assert np.abs(s - np.linalg.svd(np.kron(ar, ac), compute_uv=False)).max() <= 1e-10
    x = rng.uniform(-1, 1, 16)
    ax = np.kron(ar, ac) @ x
    s, bh, xh = O.spectral(p, ax, x)
    assert np.abs(bh - s * xh).max() <= 1e-10
    assert np.linalg.norm(O.spectral(p, x)[1]) == pytest.approx(np.linalg.norm(x), rel=1e-10)


# ---- krylov (test_krylov.cpp) ------------------------------------------------------
def desk(kind, n, noise, seed):  # test_krylov.cpp:41-54
    psf = P.make_psf(kind, 7, sigma=1.2, radius=2.0, seed=seed + 1)
    tp = P.make_test_problem(P.default_test_image(n), psf, noise, seed)
    return tp, P.nearest_kron(psf, n)


def random_sum(n, seeds, scale=None):
    def rm(s):
        return P.rng_normals(s, n * n).reshape(n, n, order="F")
    terms = []
    for i in range(0, len(seeds), 2):
        rf = rm(seeds[i])
        if scale and i // 2 in scale:
            rf = scale[i // 2] * rf
        terms.append(KronTerm(rf, rm(seeds[i + 1])))
    return KroneckerSum(terms, n)


def dense(k):
    return sum(np.kron(t.row_factor, t.col_factor) for t in k.terms)


def test_normal_matvec():  # :91-108
    eye = KroneckerSum([KronTerm(np.eye(4), np.eye(4))], 4)
    p = P.rng_normals(3, 16)
    assert np.linalg.norm(O.normal_matvec(eye, 0.0, p) - p) == 0.0
    a = random_sum(4, [10, 11, 12, 13])
    ad = dense(a)
    for lam in (0.0, 0.7):
        want = ad.T @ (ad @ p) + lam * lam * p
        assert np.linalg.norm(O.normal_matvec(a, lam, p) - want) <= 1e-12 * np.linalg.norm(want)


def test_cgls_kats():  # :110-206
    eye = KroneckerSum([KronTerm(np.eye(4), np.eye(4))], 4)
    b = P.rng_normals(21, 16)
    x, h = O.cgls(eye, b, SolverOptions(lambda_=0.0, x_true=b))
    assert h.converged and h.iterations_used == 1
    assert np.linalg.norm(x - b) <= 1e-14 * np.linalg.norm(b)
    assert h.relative_error[0] == 1.0
    a = random_sum(4, [31, 32, 33, 34], scale={1: 0.4})
    ad = dense(a)
    b = P.rng_normals(35, 16)
    lam = 0.3 * np.linalg.svd(ad, compute_uv=False)[0]
    want = np.linalg.solve(ad.T @ ad + lam * lam * np.eye(16), ad.T @ b)
    x, h = O.cgls(a, b, SolverOptions(lambda_=lam, max_iterations=16, rel_residual_tol=1e-10))
    assert h.converged and np.linalg.norm(x - want) <= 1e-8 * np.linalg.norm(want)
    tp, _ = desk("defocus", 8, 0.05, 11)
    x, h = O.cgls(tp.a, tp.b, SolverOptions(lambda_=0.05, max_iterations=5,
                                            rel_residual_tol=1e-14, x_true=tp.x_true))
    assert not h.converged and h.abort_reason == "" and h.iterations_used == 5
    assert len(h.residual_norm) == 6 and h.work_units == [2.0 * k for k in range(6)]
    with pytest.raises(ValueError):
        O.cgls(eye, np.ones(16), SolverOptions(max_iterations=0))


def test_pcg_kats():  # :208-351
    tp, best = desk("gaussian", 8, 0.01, 41)
    m = O.build_preconditioner(best.row_factor, best.col_factor, 0.05, D)
    x, h = O.pcg(tp.a, tp.b, m, SolverOptions(lambda_=0.05, rel_residual_tol=1e-8))
    assert h.converged and h.iterations_used == 1  # exact inverse
    tp, _ = desk("gaussian", 8, 0.01, 43)
    m = O.build_preconditioner(np.eye(8), np.eye(8), 1.0, D)
    x, h = O.pcg(tp.a, tp.b, m, SolverOptions(lambda_=0.07, max_iterations=12,
                                              rel_residual_tol=1e-13, record_iterates=True))
    want = plain_cg(tp.a, tp.b, 0.07, h.iterations_used)
    for k, xk in enumerate(h.iterates):
        assert np.linalg.norm(xk - want[k]) <= 1e-10 * max(1.0, np.linalg.norm(want[k]))
    tp, best = desk("gaussian", 8, 0.01, 47)
    opts = SolverOptions(lambda_=0.05, max_iterations=10, rel_residual_tol=1e-12)
    m16 = O.build_preconditioner(best.row_factor, best.col_factor, 0.05, H)
    s = O.round_calls()
    x, h = O.pcg(tp.a, tp.b, m16, opts)
    assert O.round_calls() - s == 18 * h.msolve_count and h.msolve_count >= h.iterations_used
    x, h = O.pcg(tp.a, np.full(64, 1e300), m16, SolverOptions(lambda_=0.05))
    assert not h.converged and "non-finite" in h.abort_reason


def _dot(x, y):
    """Left-to-right sum, the oracle's reduction order."""
    acc = 0.0
    for u, v in zip(x.tolist(), y.tolist()):
        acc += u * v
    return acc


def plain_cg(a, b, lam, iters):  # test_krylov.cpp:58-79
    x = np.zeros(b.size)
    r = O.kronsum_apply_transpose(a, b)
    p = r.copy()
    g = _dot(r, r)
    xs = [x.copy()]
    for _ in range(iters):
        if g <= 0:
            break
        q = O.normal_matvec(a, lam, p)
        al = g / _dot(p, q)
        x = x + al * p
        r = r - al * q
        xs.append(x.copy())
        gn = _dot(r, r)
        p = r + (gn / g) * p
        g = gn
    return xs


def test_fpcg_kats():  # :353-407
    tp, best = desk("gaussian", 8, 0.01, 61)
    m = O.build_preconditioner(best.row_factor, best.col_factor, 0.06, D)
    opts = SolverOptions(lambda_=0.06, max_iterations=6, rel_residual_tol=1e-13,
                         record_iterates=True)
    _, hp = O.pcg(tp.a, tp.b, m, opts)
    _, hf = O.fpcg(tp.a, tp.b, m, opts)
    for a, b in zip(hp.iterates, hf.iterates):
        assert np.linalg.norm(a - b) <= 1e-8 * max(1.0, np.linalg.norm(a))
    tp, best = desk("defocus", 16, 0.01, 63)
    m16 = O.build_preconditioner(best.row_factor, best.col_factor, 0.03, H)
    opts = SolverOptions(lambda_=0.03, max_iterations=40, rel_residual_tol=1e-9,
                         x_true=tp.x_true)
    _, hp = O.pcg(tp.a, tp.b, m16, opts)
    _, hf = O.fpcg(tp.a, tp.b, m16, opts)
    from paper_2311_15393_b200.kronprec import plateau_iteration
    assert abs(plateau_iteration(hp) - plateau_iteration(hf)) <= 2


# ---- regparam (test_regparam.cpp) ---------------------------------------------------
def random_spectrum(seed, count):
    """Random spectra like test_regparam.cpp:89-104 (sigma = 10^U(-5,0),
    sorted nonincreasing; b, x standard normal). Property tests only."""
    rng = np.random.default_rng(seed)
    s = np.sort(10.0 ** rng.uniform(-5, 0, count))[::-1].copy()
    return s, rng.standard_normal(count), rng.standard_normal(count)


def gcv_ref(s, b, n, lam):
    d = s * s + lam * lam
    return n * np.sum((b / d) ** 2) / np.sum(1 / d) ** 2


def test_objectives_match_plain_loops():  # :220-260
    s, b, x = random_spectrum(11, 12)
    for lam in (0.1, 1.0, 10.0):
        assert O.gcv_objective(s, b, lam) == pytest.approx(gcv_ref(s, b, 12, lam), rel=1e-12)
        want = np.sum((s * b / (s * s + lam * lam) - x) ** 2)
        assert O.opt_objective(s, b, x, lam) == pytest.approx(want, rel=1e-12)


def test_selectors_vs_grid_scan():  # :262-303
    for seed in range(1, 8):
        s, b, x = random_spectrum(seed * 977, 20)
        lo, hi = max(s.min(), 1e-10 * s.max()), s.max()
        grid = np.exp(np.linspace(np.log(lo), np.log(hi), 10000))
        step = (np.log(hi) - np.log(lo)) / 9999
        c = O.select("gcv", s, b)
        vals = [gcv_ref(s, b, 20, l) for l in grid]
        assert abs(np.log(c["lambda"]) - np.log(grid[int(np.argmin(vals))])) <= 1.01 * step


def test_discrepancy_kats():  # :349-425
    c = O.discrepancy([1.0], [2.0], 1.0, 1.0)
    assert c["lambda"] == pytest.approx(1.0, rel=1e-9)
    with pytest.raises(O.NoRootError, match="too large"):
        O.discrepancy([1.0], [2.0], 3.0, 1.0)
    with pytest.raises(O.NoRootError, match="too small"):
        O.discrepancy([1.0], [2.0], 1e-30, 1.0)
    for seed in range(3, 8):
        s, b, _ = random_spectrum(seed * 131, 16)
        lo, hi = max(s.min(), 1e-10 * s.max()), s.max()
        target = np.exp(0.35 * np.log(lo) + 0.65 * np.log(hi))
        eps = math.sqrt(np.sum((target ** 2 * b / (s * s + target ** 2)) ** 2))
        c = O.discrepancy(s, b, eps, 1.0)
        assert c["lambda"] == pytest.approx(target, rel=1e-6)
    s, b, _ = random_spectrum(21, 10)
    prev = -math.inf
    for lam in np.exp(np.linspace(np.log(1e-8 * s.max()), np.log(10 * s.max()), 64)):
        d = O.discrepancy_gap(s, b, 0.5, lam)
        assert d >= prev - 1e-12 * max(1.0, abs(d))
        prev = d


def test_filtered_solution_is_pcg_limit():
    """filtered_solution (regparam.cpp:329-349) is the exact answer for a
    single-term operator: PCG with the fp64 preconditioner lands on it."""
    tp, best = desk("gaussian", 8, 0.01, 5)
    m = O.build_preconditioner(best.row_factor, best.col_factor, 0.05, D)
    xf = O.filtered_solution(m, tp.b, 0.05)
    x, h = O.pcg(tp.a, tp.b, m, SolverOptions(lambda_=0.05, rel_residual_tol=1e-12))
    assert np.linalg.norm(x - xf) <= 1e-8 * np.linalg.norm(xf)
