"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/_build/libkp_oracle.so, the C++ restatement of the
reference kronprec hot path (see kp_oracle.cpp). Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs
may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from paper_2311_15393_b200._lib import kp_format, kp_history, kp_param_choice, kp_solver_options

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libkp_oracle.so")
_lib = None


class NoRootError(RuntimeError):
    pass


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            import subprocess
            import sys
            subprocess.run(["make", "-C", _HERE, f"PY={sys.executable}"], check=True,
                           capture_output=True)
        L = C.CDLL(LIB_PATH)
        P, D, I, Lg = C.c_void_p, C.c_double, C.c_int, C.c_long
        F = kp_format
        sig = {
            "kpo_last_error": ([], C.c_char_p), "kpo_set_threads": ([I], None),
            "kpo_get_threads": ([], I), "kpo_round_calls": ([], C.c_ulonglong),
            "kpo_round_value": ([D, F], D), "kpo_round_array": ([P, Lg, F], None),
            "kpo_pairwise_sum": ([P, Lg, F, P], I), "kpo_lp_dot": ([P, P, Lg, F, P], I),
            "kpo_lp_matvec": ([P, Lg, Lg, P, F, P], I),
            "kpo_lp_matmul": ([P, Lg, Lg, P, Lg, F, P, I], I),
            "kpo_kronsum_apply": ([I, I, P, P, P, P, I], I),
            "kpo_normal_matvec": ([I, I, P, P, D, P, P], I),
            "kpo_svd": ([P, I, I, P, P, P], I),
            "kpo_nearest_kron": ([P, I, I, I, I, P, P], I),
            "kpo_precond_build": ([P, P, I, D, F, C.POINTER(P)], I),
            "kpo_precond_from_svd": ([I, P, P, P, P, P, P, D, F, C.POINTER(P)], I),
            "kpo_precond_with_lambda": ([P, D, C.POINTER(P)], I),
            "kpo_precond_destroy": ([P], None), "kpo_precond_export": ([P, I, P], I),
            "kpo_precond_solve": ([P, P, P, I], I), "kpo_spectral": ([P, P, P, P, P, P], I),
            "kpo_cgls": ([I, I, P, P, P, C.POINTER(kp_solver_options), P, C.POINTER(kp_history)], I),
            "kpo_pcg": ([I, I, P, P, P, P, C.POINTER(kp_solver_options), I, P,
                         C.POINTER(kp_history)], I),
            "kpo_gcv_objective": ([P, P, Lg, D, C.POINTER(D)], I),
            "kpo_opt_objective": ([P, P, P, Lg, D, C.POINTER(D)], I),
            "kpo_wgcv_objective": ([P, P, Lg, D, D, C.POINTER(D)], I),
            "kpo_discrepancy_gap": ([P, P, Lg, D, D, C.POINTER(D)], I),
            "kpo_select": ([I, P, P, P, Lg, D, C.POINTER(kp_param_choice)], I),
            "kpo_discrepancy": ([P, P, Lg, D, D, C.POINTER(kp_param_choice)], I),
            "kpo_gcv_grid": ([P, P, Lg, P, I, P, C.POINTER(kp_param_choice)], I),
            "kpo_filtered_solution": ([P, P, D, P], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(st: int) -> None:
    if st == 0:
        return
    msg = lib().kpo_last_error().decode()
    if st == 1:
        raise ValueError(msg)
    if st == 3:
        raise NoRootError(msg)
    raise RuntimeError(msg)


def _p(a):
    return None if a is None else a.ctypes.data


def _fmt(f) -> kp_format:
    return kp_format(f.significand_bits, f.max_exponent, int(f.subnormals_enabled))


def _v(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, order="F"))


def _m(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def set_threads(t: int) -> None:
    lib().kpo_set_threads(int(t))


def round_calls() -> int:
    return int(lib().kpo_round_calls())


# ---- precision / lpblas ------------------------------------------------------
def round_value(x: float, fmt) -> float:
    return lib().kpo_round_value(float(x), _fmt(fmt))


def round_array(a, fmt) -> np.ndarray:
    out = np.array(a, dtype=np.float64, order="F", copy=True)
    lib().kpo_round_array(_p(out), out.size, _fmt(fmt))
    return out


def pairwise_sum(z, fmt) -> float:
    z = _v(z)
    out = C.c_double()
    _check(lib().kpo_pairwise_sum(_p(z), z.size, _fmt(fmt), C.byref(out)))
    return out.value


def lp_dot(x, y, fmt) -> float:
    x, y = _v(x), _v(y)
    if x.size != y.size:
        raise ValueError("lp_dot: length mismatch")
    out = C.c_double()
    _check(lib().kpo_lp_dot(_p(x), _p(y), x.size, _fmt(fmt), C.byref(out)))
    return out.value


def lp_matvec(a, v, fmt) -> np.ndarray:
    a, v = _m(a), _v(v)
    if a.shape[1] != v.size:
        raise ValueError("lp_matvec: shape mismatch")
    out = np.empty(a.shape[0])
    _check(lib().kpo_lp_matvec(_p(a), a.shape[0], a.shape[1], _p(v), _fmt(fmt), _p(out)))
    return out


def lp_matmul(a, b, fmt, mode: int = 0) -> np.ndarray:
    """mode 0: streamed (fast fp16 path when applicable), 1: literal
    materialising transcription, 2: streamed generic."""
    a, b = _m(a), _m(b)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if b.ndim == 1:
        b = b.reshape(-1, 1, order="F")
    if a.shape[1] != b.shape[0]:
        raise ValueError("lp_matmul: shape mismatch")
    out = np.empty((a.shape[0], b.shape[1]), order="F")
    _check(lib().kpo_lp_matmul(_p(a), a.shape[0], a.shape[1], _p(b), b.shape[1], _fmt(fmt),
                               _p(out), mode))
    return out


# ---- kron --------------------------------------------------------------------
def _stack(k):
    n, r = k.n, len(k.terms)
    rows = np.empty((n, n * r), order="F")
    cols = np.empty((n, n * r), order="F")
    for i, t in enumerate(k.terms):
        rows[:, i * n:(i + 1) * n] = t.row_factor
        cols[:, i * n:(i + 1) * n] = t.col_factor
    return n, r, rows, cols


def kronsum_apply(k, y) -> np.ndarray:
    n, r, rows, cols = _stack(k)
    y = _v(y)
    out = np.empty(n * n)
    _check(lib().kpo_kronsum_apply(n, r, _p(rows), _p(cols), _p(y), _p(out), 0))
    return out


def kronsum_apply_transpose(k, y) -> np.ndarray:
    n, r, rows, cols = _stack(k)
    y = _v(y)
    out = np.empty(n * n)
    _check(lib().kpo_kronsum_apply(n, r, _p(rows), _p(cols), _p(y), _p(out), 1))
    return out


def normal_matvec(k, lam, p) -> np.ndarray:
    n, r, rows, cols = _stack(k)
    p = _v(p)
    out = np.empty(n * n)
    _check(lib().kpo_normal_matvec(n, r, _p(rows), _p(cols), float(lam), _p(p), _p(out)))
    return out


# ---- factor --------------------------------------------------------------------
class Precond:
    FIELDS = {"s_weights": 0, "s_lp": 1, "vr_lp": 2, "vc_lp": 3}

    def __init__(self, h, n, lam, fmt):
        self._h, self.n, self.lambda_, self.fmt = h, n, lam, fmt

    def export(self, field: int, shape) -> np.ndarray:
        out = np.empty(shape, order="F")
        _check(lib().kpo_precond_export(self._h, field, _p(out)))
        return out

    def __getattr__(self, name):
        if name in Precond.FIELDS:
            return self.export(Precond.FIELDS[name], (self.n, self.n))
        if name in ("svd_r", "svd_c"):
            base = 6 if name == "svd_r" else 8
            return (self.export(base, (self.n, self.n)),
                    self.export(4 if name == "svd_r" else 5, (self.n,)),
                    self.export(base + 1, (self.n, self.n)))
        raise AttributeError(name)

    def __del__(self):
        try:
            lib().kpo_precond_destroy(self._h)
        except Exception:
            pass


def build_preconditioner(a_r, a_c, lam, fmt) -> Precond:
    a_r, a_c = _m(a_r), _m(a_c)
    n = a_r.shape[0]
    if a_r.shape != (n, n) or a_c.shape != (n, n):
        raise ValueError("build_preconditioner: factors must be square and equally sized")
    h = C.c_void_p()
    _check(lib().kpo_precond_build(_p(a_r), _p(a_c), n, float(lam), _fmt(fmt), C.byref(h)))
    return Precond(h, n, float(lam), fmt)


def build_preconditioner_from_svd(svd_r, svd_c, lam, fmt) -> Precond:
    ur, sr, vr = (_m(x) for x in svd_r)
    uc, sc, vc = (_m(x) for x in svd_c)
    n = sr.size
    h = C.c_void_p()
    _check(lib().kpo_precond_from_svd(n, _p(ur), _p(sr), _p(vr), _p(uc), _p(sc), _p(vc),
                                      float(lam), _fmt(fmt), C.byref(h)))
    return Precond(h, n, float(lam), fmt)


def with_lambda(p: Precond, lam) -> Precond:
    h = C.c_void_p()
    _check(lib().kpo_precond_with_lambda(p._h, float(lam), C.byref(h)))
    return Precond(h, p.n, float(lam), p.fmt)


def precond_solve(p: Precond, r, mode: int = 0) -> np.ndarray:
    r = _v(r)
    if r.size != p.n * p.n:
        raise ValueError("precond_solve: vector length is not n^2")
    z = np.empty_like(r)
    _check(lib().kpo_precond_solve(p._h, _p(r), _p(z), mode))
    return z


def svd(a):
    a = _m(a)
    m, n = a.shape
    u, s, v = np.empty((m, m), order="F"), np.empty(min(m, n)), np.empty((n, n), order="F")
    _check(lib().kpo_svd(_p(a), m, n, _p(u), _p(s), _p(v)))
    return u, s, v


def nearest_kron(psf, n):
    v = _m(psf.values)
    rf, cf = np.empty((n, n), order="F"), np.empty((n, n), order="F")
    _check(lib().kpo_nearest_kron(_p(v), v.shape[0], psf.center_row, psf.center_col, n,
                                  _p(rf), _p(cf)))
    return rf, cf


def spectral(p: Precond, b, x_true=None):
    """(sigma_hat, b_hat[, x_hat]) sorted as approx_spectrum / project_b."""
    b = _v(b)
    nn = p.n * p.n
    s, bh = np.empty(nn), np.empty(nn)
    xh = np.empty(nn) if x_true is not None else None
    xt = _v(x_true) if x_true is not None else None
    _check(lib().kpo_spectral(p._h, _p(b), _p(xt), _p(s), _p(bh), _p(xh)))
    return (s, bh, xh) if x_true is not None else (s, bh)


def filtered_solution(p: Precond, b, lam) -> np.ndarray:
    b = _v(b)
    x = np.empty_like(b)
    _check(lib().kpo_filtered_solution(p._h, _p(b), float(lam), _p(x)))
    return x


# ---- krylov ----------------------------------------------------------------------
@dataclass
class History:
    relative_error: list = field(default_factory=list)
    residual_norm: list = field(default_factory=list)
    work_units: list = field(default_factory=list)
    residual_cosines: list = field(default_factory=list)
    iterates: list = field(default_factory=list)
    iterations_used: int = 0
    converged: bool = False
    abort_reason: str = ""
    msolve_count: int = 0


def _solve(kind, k, b, m, opts):
    n, r, rows, cols = _stack(k)
    nn = n * n
    b = _v(b)
    xt = _v(opts.x_true) if opts.x_true is not None else None
    cap = opts.max_iterations + 1
    rel, res, work, cos = np.zeros(cap), np.zeros(cap), np.zeros(cap), np.zeros(cap)
    its = np.zeros((cap, nn)) if opts.record_iterates else None
    h = kp_history(capacity=cap, relative_error=_p(rel), residual_norm=_p(res),
                   work_units=_p(work), residual_cosines=_p(cos), iterates=_p(its))
    o = kp_solver_options(lambda_=float(opts.lambda_), max_iterations=int(opts.max_iterations),
                          rel_residual_tol=float(opts.rel_residual_tol), x_true=_p(xt),
                          track_search_direction_orthogonality=int(
                              opts.track_search_direction_orthogonality),
                          record_iterates=int(opts.record_iterates), device_pointers=0)
    x = np.empty(nn)
    if kind == "cgls":
        st = lib().kpo_cgls(n, r, _p(rows), _p(cols), _p(b), C.byref(o), _p(x), C.byref(h))
    else:
        st = lib().kpo_pcg(n, r, _p(rows), _p(cols), _p(b), m._h, C.byref(o),
                           1 if kind == "fpcg" else 0, _p(x), C.byref(h))
    _check(st)
    rows_ = h.rows
    hist = History(list(rel[:rows_]) if xt is not None else [], list(res[:rows_]),
                   list(work[:rows_]), list(cos[:h.n_cosines]),
                   [its[q].copy() for q in range(rows_)] if its is not None else [],
                   h.iterations_used, bool(h.converged), h.abort_reason.decode(), h.msolve_count)
    return x, hist


def cgls(k, b, opts):
    return _solve("cgls", k, b, None, opts)


def pcg(k, b, m, opts):
    return _solve("pcg", k, b, m, opts)


def fpcg(k, b, m, opts):
    return _solve("fpcg", k, b, m, opts)


# ---- regparam --------------------------------------------------------------------
def _obj(fn, *args):
    out = C.c_double()
    _check(fn(*args, C.byref(out)))
    return out.value


def gcv_objective(s, b, lam):
    s, b = _v(s), _v(b)
    return _obj(lib().kpo_gcv_objective, _p(s), _p(b), s.size, float(lam))


def opt_objective(s, b, x, lam):
    s, b, x = _v(s), _v(b), _v(x)
    return _obj(lib().kpo_opt_objective, _p(s), _p(b), _p(x), s.size, float(lam))


def wgcv_objective(s, b, omega, lam):
    s, b = _v(s), _v(b)
    return _obj(lib().kpo_wgcv_objective, _p(s), _p(b), s.size, float(omega), float(lam))


def discrepancy_gap(s, b, eps, lam):
    s, b = _v(s), _v(b)
    return _obj(lib().kpo_discrepancy_gap, _p(s), _p(b), s.size, float(eps), float(lam))


def _choice(c):
    return {"lambda": c.lambda_, "method": c.method, "omega": c.omega, "eta": c.eta,
            "noise_norm": c.noise_norm, "objective_value": c.objective_value,
            "bracket_lo": c.bracket_lo, "bracket_hi": c.bracket_hi,
            "flat_objective": bool(c.flat_objective), "grid_index": c.grid_index}


def select(method: str, s, b, x=None, omega: float = 1.0):
    code = {"opt": 0, "gcv": 1, "wgcv": 2}[method]
    s, b = _v(s), _v(b)
    x = _v(x) if x is not None else None
    c = kp_param_choice()
    _check(lib().kpo_select(code, _p(s), _p(b), _p(x), s.size, float(omega), C.byref(c)))
    return _choice(c)


def discrepancy(s, b, noise_norm, eta):
    s, b = _v(s), _v(b)
    c = kp_param_choice()
    _check(lib().kpo_discrepancy(_p(s), _p(b), s.size, float(noise_norm), float(eta),
                                 C.byref(c)))
    return _choice(c)


def gcv_grid(s, b, lambdas):
    s, b, lam = _v(s), _v(b), _v(lambdas)
    vals = np.empty_like(lam)
    c = kp_param_choice()
    _check(lib().kpo_gcv_grid(_p(s), _p(b), s.size, _p(lam), lam.size, _p(vals), C.byref(c)))
    return _choice(c), vals
