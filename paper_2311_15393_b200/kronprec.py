"""Host-side mirror of the reference ``kronprec`` solver API for the hot path.

Same names, argument meaning and error behaviour as the reference C++
headers (/root/reference/proj/include/kronprec/*.hpp), with numpy
column-major arrays in place of Eigen matrices. Every compute call goes
through the C ABI (include/kronprec_b200.h) into the sm_100a kernels.

Exceptions: std::invalid_argument -> ValueError, std::runtime_error ->
RuntimeError, kronprec::NoRootError -> NoRootError.
"""
from __future__ import annotations

import ctypes as C
import math
import re
from dataclasses import dataclass, field

import numpy as np

from ._lib import (KP_ACCUM_REFERENCE, KP_ACCUM_TENSOR, NoRootError, check, f64, kp_format,
                   kp_history, kp_param_choice, kp_solver_options, lib, ptr)

__all__ = [
    "PrecisionFormat", "round_value", "round_array", "RoundCallSession", "round_call_count", "lp_matmul", "lp_matvec", "lp_dot",
    "pairwise_sum", "KronTerm", "KroneckerSum", "vec", "unvec", "kron_apply", "kronsum_apply",
    "kronsum_apply_transpose", "normal_matvec", "KronSvdPreconditioner",
    "build_preconditioner", "build_preconditioner_from_svd", "with_lambda", "precond_solve",
    "SolverOptions", "ConvergenceHistory", "SolveResult", "cgls", "pcg", "fpcg", "pcg_batch", "fpcg_batch", "discrepancy_batch", "svd", "svd_dense", "set_svd_backend", "ApproxSpectrum", "approx_spectrum", "project_b", "project_x",
    "plateau_iteration", "WorkReport", "work_report", "SpectralData", "make_spectral_data",
    "ParamChoice", "gcv_objective", "opt_objective", "wgcv_objective", "discrepancy_gap", "gcv",
    "gcv_grid", "lambda_opt", "wgcv", "discrepancy", "filtered_solution", "NoRootError",
    "MinimizeResult", "minimize_1d", "find_root", "param_method_name", "set_fp16_products",
    "fp16_products_engine",
]


# ---------------------------------------------------------------------------
# precision.hpp:14-37
@dataclass(frozen=True)
class PrecisionFormat:
    significand_bits: int = 53
    max_exponent: int = 1023
    subnormals_enabled: bool = True
    name: str = "fp64"

    @staticmethod
    def fp16() -> "PrecisionFormat":
        return PrecisionFormat(11, 15, True, "fp16")

    @staticmethod
    def bfloat16() -> "PrecisionFormat":
        return PrecisionFormat(8, 127, True, "bfloat16")

    @staticmethod
    def fp32() -> "PrecisionFormat":
        return PrecisionFormat(24, 127, True, "fp32")

    @staticmethod
    def fp64() -> "PrecisionFormat":
        return PrecisionFormat(53, 1023, True, "fp64")

    @staticmethod
    def parse(text: str) -> "PrecisionFormat":  # precision.cpp:50-63
        presets = {"fp16": PrecisionFormat.fp16, "bfloat16": PrecisionFormat.bfloat16,
                   "fp32": PrecisionFormat.fp32, "fp64": PrecisionFormat.fp64}
        if text in presets:
            return presets[text]()
        m = re.fullmatch(r"custom:t=(-?\d+),emax=(-?\d+),subnormals=(-?\d+)", text)
        if m:
            t, e, s = (int(g) for g in m.groups())
            if t >= 2 and e >= 1 and s in (0, 1):
                return PrecisionFormat(t, e, s == 1, text)
        raise ValueError(f"unknown precision format: {text}")

    def unit_roundoff(self) -> float:
        return math.ldexp(1.0, -self.significand_bits)

    def max_finite(self) -> float:
        return math.ldexp(2.0 - math.ldexp(1.0, 1 - self.significand_bits), self.max_exponent)

    def overflow_threshold(self) -> float:
        return math.ldexp(2.0 - math.ldexp(1.0, -self.significand_bits), self.max_exponent)

    def min_exponent(self) -> int:
        return 1 - self.max_exponent

    def covers_double(self) -> bool:
        return self.significand_bits >= 53 and self.max_exponent >= 1023 and self.subnormals_enabled

    def c(self) -> kp_format:
        return kp_format(self.significand_bits, self.max_exponent, int(self.subnormals_enabled))


# ---------------------------------------------------------------------------
# precision.hpp:39-51, lpblas.hpp:9-33 — device emulation, any format
def round_value(x: float, fmt: PrecisionFormat) -> float:
    """round_value (precision.cpp:82-86); not tallied by RoundCallSession."""
    out = C.c_double()
    check(lib().kp_round_value(float(x), fmt.c(), C.byref(out)))
    return out.value


class RoundCallSession:
    """Tally of the vectorised rounding calls made on the current thread since
    construction (precision.hpp:55-66); sessions may nest. The device path
    counts the round_inplace calls the reference makes for the same API call."""

    def __init__(self):
        self._start = _round_calls()

    def count(self) -> int:
        return _round_calls() - self._start


def _round_calls() -> int:
    n = C.c_ulonglong()
    check(lib().kp_round_call_count(C.byref(n)))
    return int(n.value)


def round_call_count(session: RoundCallSession) -> int:  # precision.cpp:117-119
    return session.count()


def round_array(a, fmt: PrecisionFormat) -> np.ndarray:
    """round_array (precision.cpp:82-95), same shape as `a`."""
    arr = np.asarray(a, dtype=np.float64)
    x = np.ascontiguousarray(arr.reshape(-1))
    out = np.empty_like(x)
    check(lib().kp_round_array(ptr(x), x.size, fmt.c(), ptr(out)))
    return out.reshape(arr.shape)


def _lp(a, b, fmt: PrecisionFormat, round_leaves: bool) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError("lp_matmul: shape mismatch")
    m, k = a.shape
    n = b.shape[1]
    af = np.asfortranarray(a)
    bf = np.asfortranarray(b)
    c = np.empty((m, n), dtype=np.float64, order="F")
    check(lib().kp_lp_matmul_ex(m, k, n, ptr(af), ptr(bf), fmt.c(), int(round_leaves), ptr(c)))
    return np.ascontiguousarray(c)


_FP16_PRODUCTS = {"auto": 0, "cuda": 1, "tensor": 2}


def set_fp16_products(engine: str) -> None:
    """Engine of the reference-exact binary16 products (bit-identical either
    way): "cuda" (f16x2 HMUL2 + HADD2), "tensor" (tcgen05 rounded leaves +
    HADD2 trees) or "auto" (tensor from n >= 512). Process-wide."""
    if engine not in _FP16_PRODUCTS:
        raise ValueError(f"unknown fp16 product engine: {engine}")
    check(lib().kp_set_fp16_products(_FP16_PRODUCTS[engine]))


def fp16_products_engine(n: int) -> str:
    """Engine "auto" picks for an n x n preconditioner solve."""
    t = C.c_int()
    check(lib().kp_get_fp16_products(int(n), C.byref(t)))
    return "tensor" if t.value else "cuda"


def lp_matmul(a, b, fmt: PrecisionFormat) -> np.ndarray:
    """Pairwise-tree product with every product and stage sum rounded (lpblas.cpp:59-70)."""
    return _lp(a, b, fmt, True)


def lp_matvec(a, v, fmt: PrecisionFormat) -> np.ndarray:  # lpblas.cpp:48-57
    v = np.asarray(v, dtype=np.float64).reshape(-1)
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != v.size:
        raise ValueError("lp_matvec: shape mismatch")
    if v.size == 0:
        raise ValueError("lp_matvec: empty input")
    return _lp(a, v.reshape(-1, 1), fmt, True)[:, 0]


def lp_dot(x, y, fmt: PrecisionFormat) -> float:  # lpblas.cpp:39-46
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    y = np.asarray(y, dtype=np.float64).reshape(-1)
    if x.size != y.size:
        raise ValueError("lp_dot: length mismatch")
    if x.size == 0:
        raise ValueError("lp_dot: empty input")
    return float(_lp(x.reshape(1, -1), y.reshape(-1, 1), fmt, True)[0, 0])


def pairwise_sum(z, fmt: PrecisionFormat) -> float:  # lpblas.cpp:34-37 (pre-rounded addends)
    z = np.asarray(z, dtype=np.float64).reshape(-1)
    if z.size == 0:
        raise ValueError("pairwise_sum: empty input")
    return float(_lp(z.reshape(1, -1), np.ones((z.size, 1)), fmt, False)[0, 0])


# ---------------------------------------------------------------------------
# kron.hpp:9-35
def vec(y: np.ndarray) -> np.ndarray:
    """Column stacking (kron.cpp:52-55)."""
    return np.asarray(y, dtype=np.float64).reshape(-1, order="F").copy()


def unvec(y: np.ndarray, n: int) -> np.ndarray:
    y = np.asarray(y, dtype=np.float64)
    if y.size != n * n:
        raise ValueError("unvec: length is not n^2")
    return y.reshape(n, n, order="F").copy()


@dataclass
class KronTerm:
    row_factor: np.ndarray
    col_factor: np.ndarray


class KroneckerSum:
    """A = sum_k row_factor_k (x) col_factor_k; device copy created lazily."""

    def __init__(self, terms: list[KronTerm], n: int):
        self.terms = list(terms)
        self.n = int(n)
        self._h = None

    def _check(self) -> None:  # kron.cpp:12-20
        if not self.terms:
            raise ValueError("KroneckerSum: no terms")
        for t in self.terms:
            if np.shape(t.row_factor) != (self.n, self.n) or np.shape(t.col_factor) != (self.n, self.n):
                raise ValueError("KroneckerSum: factor shape mismatch")

    def handle(self) -> int:
        if self._h is None:
            self._check()
            r = len(self.terms)
            rows = np.empty((self.n, self.n * r), order="F")
            cols = np.empty((self.n, self.n * r), order="F")
            for k, t in enumerate(self.terms):
                rows[:, k * self.n:(k + 1) * self.n] = t.row_factor
                cols[:, k * self.n:(k + 1) * self.n] = t.col_factor
            h = C.c_void_p()
            check(lib().kp_operator_create(self.n, r, ptr(rows), ptr(cols), C.byref(h)))
            self._h = h
        return self._h

    _MODES = {"auto": 0, "dense": 1, "banded": 2, "banded_fused": 3}

    def set_mode(self, mode: str) -> None:
        """Operator algorithm: "auto" (banded-Toeplitz kernels when the
        factors have that structure), "dense" (DMMA GEMMs, the product the
        reference computes), "banded", or "banded_fused" (both passes in one
        kernel; 17 / 19 diagonals only)."""
        check(lib().kp_operator_set_mode(self.handle(), KroneckerSum._MODES[mode]))

    def mode(self) -> tuple[str, int, int]:
        m, tc, tr = C.c_int(), C.c_int(), C.c_int()
        check(lib().kp_operator_get_mode(self.handle(), C.byref(m), C.byref(tc), C.byref(tr)))
        return {1: "dense", 2: "banded", 3: "banded_fused"}[m.value], tc.value, tr.value

    def release(self) -> None:
        if self._h is not None:
            lib().kp_operator_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def _vec_arg(a, n: int, who: str) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, order="F"))
    if v.size != n * n:
        raise ValueError(f"{who}: vector length is not n^2")
    return v


def kronsum_apply(k: KroneckerSum, y) -> np.ndarray:  # kron.cpp:73-79
    k._check()
    y = _vec_arg(y, k.n, "kronsum_apply")
    out = np.empty_like(y)
    check(lib().kp_kronsum_apply(k.handle(), ptr(y), ptr(out)))
    return out


def kronsum_apply_transpose(k: KroneckerSum, y) -> np.ndarray:  # kron.cpp:81-88
    k._check()
    y = _vec_arg(y, k.n, "kronsum_apply_transpose")
    out = np.empty_like(y)
    check(lib().kp_kronsum_apply_transpose(k.handle(), ptr(y), ptr(out)))
    return out


def kron_apply(c, d, y) -> np.ndarray:  # kron.cpp:62-71
    """(C (x) D) y = vec(D unvec(y) C^T) on the device operator kernels."""
    c = np.asarray(c, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    n = c.shape[0] if c.ndim == 2 else 0
    if c.shape != (n, n) or d.shape != (n, n) or n == 0:
        raise ValueError("kron_apply: factors must be square and equally sized")
    y = np.asarray(y, dtype=np.float64).reshape(-1)
    if y.size != n * n:
        raise ValueError("kron_apply: vector length is not n^2")
    return kronsum_apply(KroneckerSum([KronTerm(c, d)], n), y)


def normal_matvec(a: KroneckerSum, lambda_: float, p) -> np.ndarray:  # krylov.cpp:146-152
    p = np.ascontiguousarray(np.asarray(p, dtype=np.float64).reshape(-1))
    if p.size != a.n * a.n:
        raise ValueError("normal_matvec: length mismatch")
    out = np.empty_like(p)
    check(lib().kp_normal_matvec(a.handle(), float(lambda_), ptr(p), ptr(out)))
    return out


# ---------------------------------------------------------------------------
# factor.hpp:42-71
@dataclass
class SvdTriple:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray


class KronSvdPreconditioner:
    """Device-resident one-term Kronecker-SVD preconditioner (factor.hpp:42-54).

    ``accum``: "reference" (bit-identical to lp_matmul's per-op rounding) or
    "tensor" (tcgen05 fp16 GEMMs with fp32 accumulation)."""

    _FIELDS = {"s_weights": 0, "s_lp": 1, "vr_lp": 2, "vc_lp": 3}

    def __init__(self, handle, n: int, lambda_: float, fmt: PrecisionFormat, accum: str,
                 a_r=None, a_c=None):
        self._h = handle
        self.n = n
        self.lambda_ = lambda_
        self.fmt = fmt
        self.accum = accum
        self.a_r = a_r
        self.a_c = a_c

    def _export(self, field: int, shape) -> np.ndarray:
        out = np.empty(shape, order="F")
        check(lib().kp_precond_export(self._h, field, ptr(out)))
        return out

    def __getattr__(self, name):
        if name in KronSvdPreconditioner._FIELDS:
            return self._export(KronSvdPreconditioner._FIELDS[name], (self.n, self.n))
        if name in ("svd_r", "svd_c"):
            base = 6 if name == "svd_r" else 8
            s = self._export(4 if name == "svd_r" else 5, (self.n,))
            return SvdTriple(self._export(base, (self.n, self.n)), s,
                             self._export(base + 1, (self.n, self.n)))
        raise AttributeError(name)

    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h is not None:
                lib().kp_precond_destroy(self._h)
                self._h = None
        except Exception:
            pass


def _accum_code(accum: str) -> int:
    if accum == "reference":
        return KP_ACCUM_REFERENCE
    if accum == "tensor":
        return KP_ACCUM_TENSOR
    raise ValueError(f"unknown accumulation mode: {accum}")


def build_preconditioner(a_r, a_c, lambda_: float, fmt: PrecisionFormat,
                         accum: str = "reference") -> KronSvdPreconditioner:
    """factor.cpp:80-104 (host LAPACK SVDs, device-resident rounded factors)."""
    a_r = f64(a_r)
    a_c = f64(a_c)
    n = a_r.shape[0]
    if a_r.shape != (n, n) or a_c.shape != (n, n):
        raise ValueError("build_preconditioner: factors must be square and equally sized")
    h = C.c_void_p()
    check(lib().kp_precond_build(ptr(a_r), ptr(a_c), n, float(lambda_), fmt.c(),
                                 _accum_code(accum), C.byref(h)))
    return KronSvdPreconditioner(h, n, float(lambda_), fmt, accum, a_r, a_c)


def build_preconditioner_from_svd(svd_r: SvdTriple, svd_c: SvdTriple, lambda_: float,
                                  fmt: PrecisionFormat, accum: str = "reference"
                                  ) -> KronSvdPreconditioner:
    n = np.shape(svd_r.s)[0]
    arrs = [f64(x) for x in (svd_r.u, svd_r.s, svd_r.v, svd_c.u, svd_c.s, svd_c.v)]
    h = C.c_void_p()
    check(lib().kp_precond_build_from_svd(n, *[ptr(x) for x in arrs], float(lambda_), fmt.c(),
                                          _accum_code(accum), C.byref(h)))
    return KronSvdPreconditioner(h, n, float(lambda_), fmt, accum)


def with_lambda(p: KronSvdPreconditioner, lambda_: float) -> KronSvdPreconditioner:
    """factor.cpp:106-115: same SVDs, new weights."""
    h = C.c_void_p()
    check(lib().kp_precond_with_lambda(p.handle(), float(lambda_), C.byref(h)))
    return KronSvdPreconditioner(h, p.n, float(lambda_), p.fmt, p.accum, p.a_r, p.a_c)


def precond_solve(p: KronSvdPreconditioner, r) -> np.ndarray:  # factor.cpp:117-132
    r = np.ascontiguousarray(np.asarray(r, dtype=np.float64).reshape(-1))
    if r.size != p.n * p.n:
        raise ValueError("precond_solve: vector length is not n^2")
    z = np.empty_like(r)
    check(lib().kp_precond_solve(p.handle(), ptr(r), ptr(z)))
    return z


# ---------------------------------------------------------------------------
# krylov.hpp:14-47
@dataclass
class SolverOptions:
    lambda_: float = 0.0
    max_iterations: int = 100
    rel_residual_tol: float = 1e-8
    x_true: np.ndarray | None = None
    track_search_direction_orthogonality: bool = False
    record_iterates: bool = False


@dataclass
class ConvergenceHistory:
    relative_error: list = field(default_factory=list)
    residual_norm: list = field(default_factory=list)
    work_units: list = field(default_factory=list)
    residual_cosines: list = field(default_factory=list)
    iterates: list = field(default_factory=list)
    iterations_used: int = 0
    converged: bool = False
    abort_reason: str = ""
    msolve_count: int = 0


@dataclass
class SolveResult:
    x: np.ndarray
    history: ConvergenceHistory


def _solve(kind: str, a: KroneckerSum, b, m: KronSvdPreconditioner | None,
           opts: SolverOptions) -> SolveResult:
    nn = a.n * a.n
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(-1))
    if b.size != nn:
        raise ValueError("solver: right-hand side length mismatch")
    if opts.max_iterations < 1:
        raise ValueError("solver: max_iterations must be at least 1")
    if not opts.rel_residual_tol > 0.0:
        raise ValueError("solver: tolerance must be positive")
    xt = None
    if opts.x_true is not None:
        xt = np.ascontiguousarray(np.asarray(opts.x_true, dtype=np.float64).reshape(-1))
        if xt.size != nn:
            raise ValueError("solver: x_true length mismatch")
        # an all-zero x_true is rejected by the library ("solver: x_true must
        # be nonzero", from the device-side check of the initial step)
    cap = opts.max_iterations + 1
    rel = np.zeros(cap)
    res = np.zeros(cap)
    work = np.zeros(cap)
    cos = np.zeros(cap)
    its = np.zeros((cap, nn)) if opts.record_iterates else None
    h = kp_history(capacity=cap, relative_error=ptr(rel), residual_norm=ptr(res),
                   work_units=ptr(work), residual_cosines=ptr(cos), iterates=ptr(its))
    o = kp_solver_options(lambda_=float(opts.lambda_), max_iterations=int(opts.max_iterations),
                          rel_residual_tol=float(opts.rel_residual_tol), x_true=ptr(xt),
                          track_search_direction_orthogonality=int(
                              opts.track_search_direction_orthogonality),
                          record_iterates=int(opts.record_iterates), device_pointers=0)
    x = np.empty(nn)
    L = lib()
    if kind == "cgls":
        st = L.kp_cgls(a.handle(), ptr(b), C.byref(o), ptr(x), C.byref(h))
    else:
        f = L.kp_pcg if kind == "pcg" else L.kp_fpcg
        st = f(a.handle(), ptr(b), m.handle(), C.byref(o), ptr(x), C.byref(h))
    check(st)
    rows = h.rows
    hist = ConvergenceHistory(
        relative_error=list(rel[:rows]) if xt is not None else [],
        residual_norm=list(res[:rows]), work_units=list(work[:rows]),
        residual_cosines=list(cos[:h.n_cosines]),
        iterates=[its[k].copy() for k in range(rows)] if its is not None else [],
        iterations_used=h.iterations_used, converged=bool(h.converged),
        abort_reason=h.abort_reason.decode(), msolve_count=h.msolve_count)
    return SolveResult(x, hist)


def cgls(a: KroneckerSum, b, opts: SolverOptions) -> SolveResult:  # krylov.cpp:154-208
    return _solve("cgls", a, b, None, opts)


def pcg(a: KroneckerSum, b, m: KronSvdPreconditioner, opts: SolverOptions) -> SolveResult:
    """Fletcher-Reeves PCG (krylov.cpp:58-142, 210-213)."""
    if m.n != a.n:
        raise ValueError("solver: preconditioner size mismatch")
    return _solve("pcg", a, b, m, opts)


def fpcg(a: KroneckerSum, b, m: KronSvdPreconditioner, opts: SolverOptions) -> SolveResult:
    """Polak-Ribiere flexible PCG (krylov.cpp:58-142, 215-218)."""
    if m.n != a.n:
        raise ValueError("solver: preconditioner size mismatch")
    return _solve("fpcg", a, b, m, opts)


def _solve_batch(kind: str, a: KroneckerSum, bs, m: KronSvdPreconditioner, lambdas,
                 opts: SolverOptions, x_true=None, out=None) -> list:
    nn = a.n * a.n
    bs = np.ascontiguousarray(np.asarray(bs, dtype=np.float64).reshape(-1, nn))
    batch = bs.shape[0]
    lam = np.ascontiguousarray(np.asarray(lambdas, dtype=np.float64).reshape(-1))
    if lam.size != batch:
        raise ValueError("pcg_batch: one lambda per right-hand side")
    if m.n != a.n:
        raise ValueError("solver: preconditioner size mismatch")
    if opts.max_iterations < 1:
        raise ValueError("solver: max_iterations must be at least 1")
    xt = None
    if x_true is not None:
        xt = np.ascontiguousarray(np.asarray(x_true, dtype=np.float64).reshape(-1, nn))
        if xt.shape[0] != batch:
            raise ValueError("solver: x_true batch mismatch")
        # all-zero rows are rejected by the library (device-side check; a host
        # pass over the whole batch here cost ~0.1 s per C4 step)
    cap = opts.max_iterations + 1
    bufs = [[np.zeros(cap) for _ in range(4)] for _ in range(batch)]
    hs = (kp_history * batch)()
    for i, (rel, res, work, cos) in enumerate(bufs):
        hs[i] = kp_history(capacity=cap, relative_error=ptr(rel), residual_norm=ptr(res),
                           work_units=ptr(work), residual_cosines=ptr(cos))
    o = kp_solver_options(lambda_=0.0, max_iterations=int(opts.max_iterations),
                          rel_residual_tol=float(opts.rel_residual_tol), x_true=ptr(xt),
                          track_search_direction_orthogonality=int(opts.track_search_direction_orthogonality),
                          record_iterates=0, device_pointers=0)
    if out is None:
        x = np.empty((batch, nn))
    else:  # caller's buffer (e.g. pinned host memory), batch x n^2 float64
        x = out.reshape(batch, nn)
        if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"]:
            raise ValueError("pcg_batch: out must be a contiguous float64 batch x n^2 array")
    f = lib().kp_pcg_batch if kind == "pcg" else lib().kp_fpcg_batch
    check(f(a.handle(), m.handle(), batch, ptr(bs), ptr(lam), C.byref(o), ptr(x), hs))
    results = []
    for i in range(batch):
        h = hs[i]
        rel, res, work, cos = bufs[i]
        rows = h.rows
        results.append(SolveResult(x[i], ConvergenceHistory(
            relative_error=list(rel[:rows]) if xt is not None else [],
            residual_norm=list(res[:rows]), work_units=list(work[:rows]),
            residual_cosines=list(cos[:h.n_cosines]), iterates=[],
            iterations_used=h.iterations_used, converged=bool(h.converged),
            abort_reason=h.abort_reason.decode(), msolve_count=h.msolve_count)))
    return results


def pcg_batch(a: KroneckerSum, bs, m: KronSvdPreconditioner, lambdas, opts: SolverOptions,
              x_true=None, out=None) -> list:
    """PCG for a batch of right-hand sides (rows of `bs`), image i with lambda
    lambdas[i] and the factors of `m` (with_lambda per image, cli.cpp:469-486):
    one batched device solve; result i equals pcg(a, bs[i], with_lambda(m,
    lambdas[i]), opts) with opts.x_true = x_true[i]. Result i's x is row i of
    `out` (or of a new batch x n^2 array)."""
    return _solve_batch("pcg", a, bs, m, lambdas, opts, x_true, out)


def fpcg_batch(a: KroneckerSum, bs, m: KronSvdPreconditioner, lambdas, opts: SolverOptions,
               x_true=None, out=None) -> list:
    return _solve_batch("fpcg", a, bs, m, lambdas, opts, x_true, out)


_SVD_BACKENDS = {"host": 0, "device": 1}


def svd(a, backend: str = "host"):
    """svd_dense (factor.cpp:14-23): (u, s, v) with a = u diag(s) v^T, s
    nonincreasing. backend "host": LAPACK dgesdd; "device": cuSOLVER FP64 on
    the B200."""
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    n = a.shape[0]
    if a.ndim != 2 or a.shape != (n, n) or n == 0:
        raise ValueError("svd_dense: square, non-empty matrix expected")
    u, v, sv = np.empty((n, n), order="F"), np.empty((n, n), order="F"), np.empty(n)
    check(lib().kp_svd(ptr(a), n, _SVD_BACKENDS[backend], ptr(u), ptr(sv), ptr(v)))
    return u, sv, v


def svd_dense(a, backend: str = "host") -> SvdTriple:  # factor.cpp:14-23
    return SvdTriple(*svd(a, backend))


def set_svd_backend(backend: str) -> None:
    """Backend of build_preconditioner's factor SVDs (process-wide)."""
    check(lib().kp_set_svd_backend(_SVD_BACKENDS[backend]))


def discrepancy_batch(m: KronSvdPreconditioner, bs, noise_norms, eta: float):
    """discrepancy(make_spectral_data(m, b_i), noise_norms[i], eta) for every
    row b_i of `bs` in one batched device search (regparam.cpp:288-327).
    Returns (lambdas, status): status 0 ok, KP_ERR_NO_ROOT / KP_ERR_RUNTIME
    per image (lambda NaN); lambdas equal discrepancy()'s bit for bit."""
    nn = m.n * m.n
    bs = np.ascontiguousarray(np.asarray(bs, dtype=np.float64).reshape(-1, nn))
    batch = bs.shape[0]
    nz = np.ascontiguousarray(np.asarray(noise_norms, dtype=np.float64).reshape(-1))
    if nz.size != batch:
        raise ValueError("discrepancy_batch: one noise norm per right-hand side")
    lam = np.empty(batch)
    st = np.empty(batch, dtype=np.int32)
    check(lib().kp_discrepancy_batch(m.handle(), batch, ptr(bs), ptr(nz), float(eta), ptr(lam),
                                     st.ctypes.data_as(C.c_void_p)))
    return lam, st


def plateau_iteration(h: ConvergenceHistory, tol: float = 0.01) -> int:  # krylov.cpp:220-231
    if not h.relative_error:
        raise ValueError("plateau_iteration: run has no relative-error track")
    if not tol >= 0.0:
        raise ValueError("plateau_iteration: negative tolerance")
    best = min(h.relative_error)
    for k, e in enumerate(h.relative_error):
        if e <= (1.0 + tol) * best:
            return k
    return len(h.relative_error) - 1


@dataclass
class WorkReport:
    m_precond: int = 0
    m_baseline: int = 0
    threshold: float = 0.0
    preconditioning_pays: bool = False
    plateau_tolerance: float = 0.01


def work_report(h_precond, h_baseline, plateau_tol: float = 0.01) -> WorkReport:
    w = WorkReport(plateau_tolerance=plateau_tol)  # krylov.cpp:233-243
    w.m_precond = plateau_iteration(h_precond, plateau_tol)
    w.m_baseline = plateau_iteration(h_baseline, plateau_tol)
    w.threshold = (8.0 * w.m_baseline) / 9.0
    w.preconditioning_pays = float(w.m_precond) < w.threshold
    return w


# ---------------------------------------------------------------------------
# regparam.hpp:19-90
@dataclass
class ParamChoice:
    lambda_: float = 0.0
    method: str = "gcv"
    omega: float = 0.0
    eta: float = 0.0
    noise_norm: float = 0.0
    objective_value: float = 0.0
    bracket_lo: float = 0.0
    bracket_hi: float = 0.0
    flat_objective: bool = False
    grid_index: int = -1


_METHODS = {0: "opt", 1: "gcv", 2: "wgcv", 3: "discrepancy", 4: "gcv_grid"}


def _choice(c: kp_param_choice) -> ParamChoice:
    return ParamChoice(c.lambda_, _METHODS.get(c.method, "?"), c.omega, c.eta, c.noise_norm,
                       c.objective_value, c.bracket_lo, c.bracket_hi, bool(c.flat_objective),
                       c.grid_index)


class SpectralData:
    """Device-resident sigma_hat = s_r(j) s_c(i) and b_hat = vec(U_c^T B U_r)."""

    def __init__(self, handle, n: int, has_x: bool = False):
        self._h = handle
        self.n = n * n
        self._side = n
        self._has_x = has_x

    def handle(self):
        return self._h

    def exported(self) -> tuple[np.ndarray, np.ndarray]:
        """(sigma_hat, b_hat) sorted like approx_spectrum / project_b."""
        s = np.empty(self.n)
        b = np.empty(self.n)
        check(lib().kp_spectral_export(self._h, ptr(s), ptr(b)))
        return s, b

    @property
    def sigma_hat(self) -> np.ndarray:
        return self.exported()[0]

    @property
    def x_hat(self) -> np.ndarray | None:
        """Coordinates of x_true (same order as exported()), or None."""
        if not self._has_x:
            return None
        x = np.empty(self.n)
        check(lib().kp_spectral_export_xhat(self._h, ptr(x)))
        return x

    @property
    def b_hat(self) -> np.ndarray:
        return self.exported()[1]

    def __del__(self):
        try:
            if self._h is not None:
                lib().kp_spectral_destroy(self._h)
                self._h = None
        except Exception:
            pass


@dataclass
class ApproxSpectrum:  # factor.hpp:76-79
    sigma: np.ndarray
    perm: np.ndarray


def approx_spectrum(p: KronSvdPreconditioner) -> ApproxSpectrum:
    """factor.cpp:134-153: sigma(k) = s_r(j) s_c(i) sorted nonincreasing by a
    stable sort of the column-major index j n + i (index bookkeeping on the
    host, as the device export's ordering)."""
    products = np.outer(np.asarray(p.svd_r.s), np.asarray(p.svd_c.s)).reshape(-1)  # [j*n + i]
    perm = np.argsort(-products, kind="stable")
    return ApproxSpectrum(products[perm], perm)


def project_b(p: KronSvdPreconditioner, b) -> np.ndarray:  # factor.cpp:179-182
    """vec(U_c^T B U_r) reordered like approx_spectrum (device DMMA projections)."""
    return make_spectral_data(p, b).b_hat


def project_x(p: KronSvdPreconditioner, x) -> np.ndarray:  # factor.cpp:184-187
    """vec(V_c^T X V_r) reordered like approx_spectrum."""
    return make_spectral_data(p, x, x).x_hat


def make_spectral_data(p: KronSvdPreconditioner, b, x_true=None) -> SpectralData:
    """regparam.cpp:119-134 (x_true: the overload with x coordinates)."""
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(-1))
    if b.size != p.n * p.n:
        raise ValueError("project: vector length is not n^2")
    h = C.c_void_p()
    if x_true is None:
        check(lib().kp_spectral_create(p.handle(), ptr(b), C.byref(h)))
        return SpectralData(h, p.n)
    x = np.ascontiguousarray(np.asarray(x_true, dtype=np.float64).reshape(-1))
    if x.size != p.n * p.n:
        raise ValueError("project: vector length is not n^2")
    check(lib().kp_spectral_create_x(p.handle(), ptr(b), ptr(x), C.byref(h)))
    return SpectralData(h, p.n, True)


def _probe(f, x: float, who: str) -> float:  # regparam.cpp:37-43
    v = float(f(x))
    if math.isnan(v):
        raise RuntimeError(f"{who}: objective is NaN")
    return v


@dataclass
class MinimizeResult:  # regparam.hpp:55-58
    x: float = 0.0
    fx: float = 0.0


def minimize_1d(f, lo: float, hi: float, tol: float) -> MinimizeResult:
    """Golden-section search (regparam.cpp:150-181); host arithmetic, same
    IEEE double operations as the reference."""
    if not lo < hi:
        raise ValueError("minimize_1d: requires lo < hi")
    if not tol > 0.0:
        raise ValueError("minimize_1d: tol must be positive")
    invphi = 0.6180339887498949
    a, b = lo, hi
    c = b - invphi * (b - a)
    d = a + invphi * (b - a)
    fc, fd = _probe(f, c, "minimize_1d"), _probe(f, d, "minimize_1d")
    it = 0
    while it < 300 and b - a > tol * (1.0 + min(abs(a), abs(b))):
        if fc < fd:
            b, d, fd = d, c, fc
            c = b - invphi * (b - a)
            if c <= a or c >= d:
                break
            fc = _probe(f, c, "minimize_1d")
        else:
            a, c, fc = c, d, fd
            d = a + invphi * (b - a)
            if d <= c or d >= b:
                break
            fd = _probe(f, d, "minimize_1d")
        it += 1
    return MinimizeResult(c, fc) if fc < fd else MinimizeResult(d, fd)


def find_root(f, lo: float, hi: float, tol: float) -> float:
    """Bisection (regparam.cpp:184-214)."""
    if not lo < hi:
        raise ValueError("find_root: requires lo < hi")
    if not tol > 0.0:
        raise ValueError("find_root: tol must be positive")
    flo, fhi = _probe(f, lo, "find_root"), _probe(f, hi, "find_root")
    if not (math.isfinite(flo) and math.isfinite(fhi)):
        raise RuntimeError("find_root: endpoint value not finite")
    if flo == 0.0:
        return lo
    if fhi == 0.0:
        return hi
    if (flo > 0.0) == (fhi > 0.0):
        raise ValueError("find_root: no sign change over [lo, hi]")
    a, b = lo, hi
    while b - a > tol * (1.0 + 0.5 * (abs(a) + abs(b))):
        m = a + 0.5 * (b - a)
        if m <= a or m >= b:
            break
        fm = _probe(f, m, "find_root")
        if not math.isfinite(fm):
            raise RuntimeError("find_root: function value not finite")
        if fm == 0.0:
            return m
        if (fm > 0.0) == (flo > 0.0):
            a, flo = m, fm
        else:
            b = m
    return a + 0.5 * (b - a)


def param_method_name(method: str) -> str:  # regparam.cpp:136-148
    names = {"opt": "opt", "gcv": "gcv", "wgcv": "wgcv", "discrepancy": "discrepancy",
             "gcv_grid": "gcv_grid"}
    if method not in names:
        raise ValueError("unknown parameter method")
    return names[method]


def gcv_objective(sd: SpectralData, lambda_: float) -> float:  # regparam.cpp:224-229
    v = C.c_double()
    check(lib().kp_gcv_objective(sd.handle(), float(lambda_), C.byref(v)))
    return v.value


def opt_objective(sd: SpectralData, lambda_: float) -> float:  # regparam.cpp:216-222
    v = C.c_double()
    check(lib().kp_opt_objective(sd.handle(), float(lambda_), C.byref(v)))
    return v.value


def wgcv_objective(sd: SpectralData, omega: float, lambda_: float) -> float:  # :231-240
    v = C.c_double()
    check(lib().kp_wgcv_objective(sd.handle(), float(omega), float(lambda_), C.byref(v)))
    return v.value


def lambda_opt(sd: SpectralData) -> ParamChoice:  # regparam.cpp:248-252
    c = kp_param_choice()
    check(lib().kp_lambda_opt(sd.handle(), C.byref(c)))
    return _choice(c)


def wgcv(sd: SpectralData, omega: float) -> ParamChoice:  # regparam.cpp:260-286
    c = kp_param_choice()
    check(lib().kp_wgcv(sd.handle(), float(omega), C.byref(c)))
    return _choice(c)


def filtered_solution(p: KronSvdPreconditioner, b, lambda_: float) -> np.ndarray:
    """Direct Tikhonov solution for the Kronecker approximation (regparam.cpp:329-349)."""
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(-1))
    if b.size != p.n * p.n:
        raise ValueError("filtered_solution: vector length is not n^2")
    x = np.empty_like(b)
    check(lib().kp_filtered_solution(p.handle(), ptr(b), float(lambda_), ptr(x)))
    return x


def discrepancy_gap(sd: SpectralData, epsilon: float, lambda_: float) -> float:  # :242-246
    v = C.c_double()
    check(lib().kp_discrepancy_gap(sd.handle(), float(epsilon), float(lambda_), C.byref(v)))
    return v.value


def gcv(sd: SpectralData) -> ParamChoice:  # regparam.cpp:254-258
    c = kp_param_choice()
    check(lib().kp_gcv(sd.handle(), C.byref(c)))
    return _choice(c)


def gcv_grid(sd: SpectralData, lambdas) -> tuple[ParamChoice, np.ndarray]:
    """North-star GCV: one batched reduction over an explicit lambda grid;
    returns the first argmin (grid_index) and the objective values."""
    lam = np.ascontiguousarray(np.asarray(lambdas, dtype=np.float64))
    vals = np.empty_like(lam)
    c = kp_param_choice()
    check(lib().kp_gcv_grid(sd.handle(), ptr(lam), lam.size, ptr(vals), C.byref(c)))
    return _choice(c), vals


def discrepancy(sd: SpectralData, noise_norm: float, eta: float) -> ParamChoice:  # :288-327
    c = kp_param_choice()
    check(lib().kp_discrepancy(sd.handle(), float(noise_norm), float(eta), C.byref(c)))
    return _choice(c)
