"""Seeded inputs of the large-size preconditioner-solve goldens (test
infrastructure, shared by tests/golden/gen_goldens.py and the -m gpu tests).

The singular-vector factors are drawn directly as binary16-representable
values (numpy PCG64, platform independent), so build_preconditioner's
rounding of V (factor.cpp:100-104) is the identity and the goldens do not
depend on any LAPACK's last bits. The residual spans 1e-9 .. 1 in magnitude
per column block, so the products reach the binary16 subnormal range and
underflow to signed zeros (the regime where the C5 FPCG run stagnates,
DESIGN.md §4), and a few columns are exactly zero (all-zero output trees,
whose sign the device resolves separately)."""
from __future__ import annotations

import hashlib

import numpy as np


def msolve_case(n: int, seed: int, regime: str = "wide"):
    """(svd_r, svd_c, lam, r) as plain arrays: ((u, s, v), (u, s, v), lam, r).

    regime "wide": column magnitudes 1e-9 .. 1; "low": 1e-10 .. 1e-5, where
    most products underflow and many output trees are all-zero (their sign
    comes from the product sign rule)."""
    rng = np.random.default_rng(seed)

    def factor():
        v = (rng.standard_normal((n, n)) / np.sqrt(n)).astype(np.float16).astype(np.float64)
        s = np.sort(rng.uniform(1e-3, 1.0, n))[::-1].copy()
        return np.asfortranarray(v), s, np.asfortranarray(v)

    u_r, s_r, v_r = factor()
    u_c, s_c, v_c = factor()
    lam = 0.01
    r = rng.standard_normal((n, n))
    lo, hi = (-9.0, 0.0) if regime == "wide" else (-10.0, -5.0)
    scale = 10.0 ** rng.uniform(lo, hi, n)  # per-column magnitude
    r *= scale[None, :]
    r[:, rng.integers(0, n, 3)] = 0.0
    r[rng.integers(0, n, 5), :] *= -0.0  # signed-zero rows mixed in
    return (u_r, s_r, v_r), (u_c, s_c, v_c), lam, r.reshape(-1, order="F")


def digest(z: np.ndarray) -> dict:
    """Bitwise fingerprint of a solve result (sign of zero included)."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    bits = z.view(np.uint64)
    return {"sha256": hashlib.sha256(z.tobytes()).hexdigest(),
            "norm": float(np.linalg.norm(z)),
            "zeros": int(np.count_nonzero(z == 0.0)),
            "neg_zeros": int(np.count_nonzero(bits == np.uint64(1 << 63))),
            "nonfinite": int(np.count_nonzero(~np.isfinite(z))),
            "head": [float(v) for v in z[:4]]}
