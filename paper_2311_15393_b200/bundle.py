"""Problem bundles in the reference's on-disk format (deblur.cpp:277-359,
schema "kronprec.problem/1"): a directory with meta.json plus raw
little-endian float64 files psf.f64 (n_p x n_p, column-major), xtrue.f64,
btrue.f64 and b.f64 (vec order). Bundles written here load in the reference
(`load_problem`) and vice versa, so problems and goldens can move between
the two implementations.

The BASELINE configs need two things the reference format cannot name: PSF
kinds it does not have (the anisotropic Gaussian, Gaussian * motion) and the
rank cap of psf_to_kronsum. They are written as extra keys
(``kp_b200_kind``, ``kp_b200_rank_cap``) that the reference ignores; its
``kind`` field then carries the nearest reference kind.
"""
from __future__ import annotations

import json
import os

import numpy as np

from . import problems as P

SCHEMA = "kronprec.problem/1"
REFERENCE_KINDS = ("gaussian", "defocus", "motion", "shake", "speckle")
FILES = ("psf.f64", "xtrue.f64", "btrue.f64", "b.f64")


def _write_f64(path: str, a: np.ndarray) -> None:
    np.ascontiguousarray(a, dtype="<f8").tofile(path)


def _read_f64(path: str, count: int) -> np.ndarray:
    v = np.fromfile(path, dtype="<f8")
    if v.size != count:
        raise RuntimeError(f"short read from {path}")
    return v.astype(np.float64)


def save_problem(tp: P.TestProblem, directory: str, rank_cap: int = 0) -> None:
    """save_problem (deblur.cpp:277-310)."""
    os.makedirs(directory, exist_ok=True)
    psf = tp.psf
    n_p = int(psf.values.shape[0])
    nn = tp.n * tp.n
    kind = psf.kind if psf.kind in REFERENCE_KINDS else "gaussian"
    params = dict(psf.params)
    meta = {
        "schema": SCHEMA,
        "kind": kind,
        "n": int(tp.n),
        "psf_size": n_p,
        "center_row": int(psf.center_row),
        "center_col": int(psf.center_col),
        "seed": int(tp.seed),
        "psf_seed": int(psf.seed),
        "noise_level": float(tp.noise_level),
        "params": {"sigma": float(params["sigma"]), "radius": float(params["radius"]),
                   "length": int(params["length"]), "steps": int(params["steps"]),
                   "blob_count": int(params["blob_count"]),
                   "blob_sigma": float(params["blob_sigma"])},
        "bytes": {"psf.f64": n_p * n_p * 8, "xtrue.f64": nn * 8, "btrue.f64": nn * 8,
                  "b.f64": nn * 8},
    }
    if kind != psf.kind:
        meta["kp_b200_kind"] = psf.kind
    if rank_cap:
        meta["kp_b200_rank_cap"] = int(rank_cap)
    with open(os.path.join(directory, "meta.json"), "w") as f:
        f.write(json.dumps(meta, indent=2) + "\n")
    _write_f64(os.path.join(directory, "psf.f64"), np.asfortranarray(psf.values).reshape(-1, order="F"))
    _write_f64(os.path.join(directory, "xtrue.f64"), tp.x_true)
    _write_f64(os.path.join(directory, "btrue.f64"), tp.b_true)
    _write_f64(os.path.join(directory, "b.f64"), tp.b)


def load_problem(directory: str) -> P.TestProblem:
    """load_problem (deblur.cpp:312-359): the operator is rebuilt from the PSF
    with psf_to_kronsum (rank-capped when the bundle says so)."""
    path = os.path.join(directory, "meta.json")
    if not os.path.exists(path):
        raise RuntimeError(f"missing bundle meta.json in {directory}")
    with open(path) as f:
        meta = json.load(f)
    n = int(meta["n"])
    n_p = int(meta["psf_size"])
    for name in FILES:
        fp = os.path.join(directory, name)
        if not os.path.exists(fp) or os.path.getsize(fp) != int(meta["bytes"][name]):
            raise RuntimeError(f"bundle file {name} is missing or has the wrong size")
    kind = meta.get("kp_b200_kind", meta["kind"])
    if meta["kind"] not in REFERENCE_KINDS:
        raise ValueError(f"unknown blur kind: {meta['kind']}")
    pj = meta["params"]
    params = {"sigma": float(pj["sigma"]), "radius": float(pj["radius"]), "length": int(pj["length"]),
              "steps": int(pj["steps"]), "blob_count": int(pj["blob_count"]),
              "blob_sigma": float(pj["blob_sigma"])}
    values = _read_f64(os.path.join(directory, "psf.f64"), n_p * n_p).reshape(n_p, n_p, order="F")
    psf = P.Psf(np.asfortranarray(values), int(meta["center_row"]), int(meta["center_col"]), kind,
                int(meta["psf_seed"]), params)
    nn = n * n
    x_true = _read_f64(os.path.join(directory, "xtrue.f64"), nn)
    b_true = _read_f64(os.path.join(directory, "btrue.f64"), nn)
    b = _read_f64(os.path.join(directory, "b.f64"), nn)
    a, _ = P.psf_to_kronsum(psf, n, max_rank=int(meta.get("kp_b200_rank_cap", 0)))
    return P.TestProblem(a, x_true, b_true, b - b_true, b, float(meta["noise_level"]),
                         int(meta["seed"]), psf, n)
