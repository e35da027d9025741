"""Problem bundles in the reference format (deblur.cpp:277-359): round trip,
the exact meta.json key set and file sizes the reference's load_problem
checks, and the rank-capped BASELINE PSFs (host only, no GPU)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2311_15393_b200 import bundle as B
from paper_2311_15393_b200 import problems as P

REF_KEYS = {"schema", "kind", "n", "psf_size", "center_row", "center_col", "seed", "psf_seed",
            "noise_level", "params", "bytes"}


def test_round_trip_reference_kind(tmp_path):
    psf = P.make_psf("defocus", 7, radius=2.0, seed=5)
    tp = P.make_test_problem(P.default_test_image(24), psf, 0.02, 11)
    d = str(tmp_path / "b1")
    B.save_problem(tp, d)
    meta = json.load(open(os.path.join(d, "meta.json")))
    assert set(meta) == REF_KEYS and meta["schema"] == "kronprec.problem/1"
    assert set(meta["params"]) == {"sigma", "radius", "length", "steps", "blob_count", "blob_sigma"}
    for name in B.FILES:
        assert os.path.getsize(os.path.join(d, name)) == meta["bytes"][name]
    q = B.load_problem(d)
    assert q.n == tp.n and q.seed == tp.seed and q.noise_level == tp.noise_level
    for f in ("x_true", "b_true", "b"):
        assert np.array_equal(getattr(q, f), getattr(tp, f))
    # the reference reloads noise as b - b_true (deblur.cpp:357), not the draws
    assert np.array_equal(q.noise, tp.b - tp.b_true)
    assert np.allclose(q.noise, tp.noise, rtol=0, atol=1e-15)
    assert np.array_equal(q.psf.values, tp.psf.values)
    assert (q.psf.kind, q.psf.seed, q.psf.params) == (tp.psf.kind, tp.psf.seed, tp.psf.params)
    assert len(q.a.terms) == len(tp.a.terms)
    for s, t in zip(q.a.terms, tp.a.terms):
        assert np.array_equal(s.row_factor, t.row_factor) and np.array_equal(s.col_factor, t.col_factor)


def test_rank_capped_baseline_psf(tmp_path):
    psf = P.psf_aniso_gaussian(31, [[4.0, 1.0], [1.0, 2.0]])
    a, _ = P.psf_to_kronsum(psf, 48, max_rank=3)
    tp = P.make_test_problem(P.blob_image(48, 1002), psf, 0.01, 2002, a=a)
    d = str(tmp_path / "c2")
    B.save_problem(tp, d, rank_cap=3)
    meta = json.load(open(os.path.join(d, "meta.json")))
    assert meta["kind"] == "gaussian" and meta["kp_b200_kind"] == "aniso_gaussian"
    assert REF_KEYS <= set(meta)
    q = B.load_problem(d)
    assert len(q.a.terms) == 3
    for s, t in zip(q.a.terms, a.terms):
        assert np.array_equal(s.row_factor, t.row_factor) and np.array_equal(s.col_factor, t.col_factor)
    assert np.array_equal(q.b, tp.b)


def test_corrupt_bundles_are_rejected(tmp_path):
    tp = P.make_test_problem(P.default_test_image(8), P.make_psf("gaussian", 3), 0.01, 1)
    d = str(tmp_path / "bad")
    B.save_problem(tp, d)
    with open(os.path.join(d, "b.f64"), "ab") as f:
        f.write(b"\0" * 8)
    with pytest.raises(RuntimeError, match="wrong size"):
        B.load_problem(d)
    os.remove(os.path.join(d, "meta.json"))
    with pytest.raises(RuntimeError, match="missing bundle meta.json"):
        B.load_problem(d)
