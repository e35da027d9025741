"""minimize_1d / find_root (regparam.cpp:150-214) — the reference's public
host search helpers, with its own pins (test_regparam.cpp:130-172). Host
code, no GPU."""
from __future__ import annotations

import math

import pytest

from paper_2311_15393_b200 import kronprec as K


def test_minimize_1d_pins():
    r = K.minimize_1d(lambda x: (x - 2.0) * (x - 2.0), 0.0, 5.0, 1e-10)
    assert abs(r.x - 2.0) <= 1e-7 and r.fx <= 1e-13
    r = K.minimize_1d(math.cos, 0.0, 2.0 * math.acos(-1.0), 1e-10)
    assert abs(r.x - math.pi) <= 1e-6 and abs(r.fx + 1.0) <= 1e-12
    r = K.minimize_1d(lambda x: math.inf if x < 1.0 else (x - 2.0) ** 2, 0.0, 5.0, 1e-10)
    assert abs(r.x - 2.0) <= 1e-6


def test_find_root_pins():
    assert abs(K.find_root(lambda t: t - 3.0, 0.0, 10.0, 1e-12) - 3.0) <= 1e-9
    assert K.find_root(lambda t: t, 0.0, 1.0, 1e-12) == 0.0


def test_search_errors():
    with pytest.raises(ValueError):
        K.minimize_1d(lambda x: 0.0, 1.0, 1.0, 1e-8)
    with pytest.raises(RuntimeError):
        K.minimize_1d(lambda x: math.nan, 0.0, 1.0, 1e-8)
    with pytest.raises(ValueError):
        K.find_root(lambda x: 1.0, 0.0, 1.0, 1e-8)
    with pytest.raises(ValueError):
        K.find_root(lambda x: 0.5, 2.0, 1.0, 1e-8)
    with pytest.raises(ValueError):
        K.param_method_name("nope")
