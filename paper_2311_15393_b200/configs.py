"""The five BASELINE.json configurations as seeded synthetic problems.

Pinned choices (the reference API cannot express these, so both
arms consume the arrays built here):
  x_true   blob_image(n, seed=1000+cfg) — 20 Gaussian blobs, clipped [0,1]
  noise    make_test_problem noise with seed 2000+cfg (C4: 4000+i / 5000+i)
  C1       Gaussian sigma=3 on 19x19 (2*ceil(3 sigma)+1), rank 1
  C2/C3    anisotropic Gaussian, cov [[4,1],[1,2]] on 31x31, psf_to_kronsum
           capped at rank 3; nearest_kron of the rank-3 PSF array
  C4       Gaussian sigma=2.5 on 17x17, rank 1, noise cycling 0.1/1/5 %
  C5       Gaussian sigma=4 convolved with a 15-sample segment at 30 degrees
           on 41x41, rank-5 cap; nearest_kron of the rank-5 array
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import problems as P
from .kronprec import KronTerm, KroneckerSum

GCV_GRID = 10.0 ** (-4.0 + 4.0 * np.arange(64) / 63.0)  # C3: 64 log-spaced in [1e-4, 1]


@dataclass
class Config:
    name: str
    n: int
    problem: P.TestProblem
    term: KronTerm  # nearest Kronecker product (preconditioner factors)
    lambda_: float | None  # None: chosen by gcv_grid / discrepancy
    solvers: list = field(default_factory=list)  # (solver, fmt, maxit)
    tol: float = 1e-6
    select: str = "fixed"  # fixed | gcv_grid | discrepancy
    eta: float = 1.01


def _psf(name: str) -> tuple[P.Psf, int]:
    if name == "C1":
        return P.make_psf("gaussian", 19, sigma=3.0), 0
    if name in ("C2", "C3"):
        return P.psf_aniso_gaussian(31, [[4.0, 1.0], [1.0, 2.0]]), 3
    if name == "C4":
        return P.make_psf("gaussian", 17, sigma=2.5), 0
    if name == "C5":
        return P.psf_gauss_motion(41, 4.0, 15, 30.0), 5
    raise ValueError(f"unknown config {name}")


def build(name: str, image: int = 0, n: int | None = None) -> Config:
    """Build config `name` (n overridable for scaled-down tests)."""
    sizes = {"C1": 256, "C2": 1024, "C3": 2048, "C4": 1024, "C5": 4096}
    n = n or sizes[name]
    psf, cap = _psf(name)
    a, trunc = P.psf_to_kronsum(psf, n, max_rank=cap)
    psf_for_m = P.Psf(trunc, psf.center_row, psf.center_col, psf.kind) if cap else psf
    term = P.nearest_kron(psf_for_m, n)
    cfg_id = int(name[1])
    if name == "C4":
        xs, ns = 4000 + image, 5000 + image
        noise = [0.001, 0.01, 0.05][image % 3]
    else:
        xs, ns = 1000 + cfg_id + 100 * image, 2000 + cfg_id + 100 * image  # image>0: replicas
        noise = {"C1": 0.01, "C2": 0.01, "C3": 0.005, "C5": 0.01}[name]
    tp = P.make_test_problem(P.blob_image(n, xs), psf, noise, ns, a=a)
    if name == "C1":
        return Config(name, n, tp, term, 0.01, [("pcg", "fp16", 100), ("cgls", None, 2000)])
    if name == "C2":
        return Config(name, n, tp, term, 0.005, [("fpcg", "fp16", 100)])
    if name == "C3":
        return Config(name, n, tp, term, None, [("pcg", "fp16", 100)], select="gcv_grid")
    if name == "C4":
        return Config(name, n, tp, term, None, [("pcg", "fp16", 100)], select="discrepancy")
    return Config(name, n, tp, term, 0.01,
                  [("fpcg", "fp16", 100), ("pcg", "fp64", 100), ("cgls", None, 2000)])
