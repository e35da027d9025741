"""Quick gemm_f16x check for kernel variants: bitwise against the committed
n=1664 / n=4096 oracle digests (tests/golden/msolve_n*.json) and per-launch
time of the n=4096 M-solve products (profile events, 3 M-solves)."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200 import _lib  # noqa: E402
from paper_2311_15393_b200.kronprec import SvdTriple  # noqa: E402
from msolve_inputs import digest, msolve_case  # noqa: E402

F16 = K.PrecisionFormat.fp16()
K.set_fp16_products("tensor")
ok = True
for n in (1664, 4096):
    g = json.load(open(f"tests/golden/msolve_n{n}.json"))
    for regime in ("wide", "low"):
        sr, sc, lam, r = msolve_case(n, g["seed"], regime)
        m = K.build_preconditioner_from_svd(SvdTriple(*sr), SvdTriple(*sc), lam, F16)
        for rep in range(2):
            same = digest(K.precond_solve(m, r))["sha256"] == g["cases"][regime]["digest"]["sha256"]
            ok &= same
        print(f"n={n} {regime}: bitwise {same}", flush=True)
L = _lib.lib()
K.precond_solve(m, r)
L.kp_profile_reset()
L.kp_profile_enable(1)
for _ in range(3):
    K.precond_solve(m, r)
t, c = C.c_double(), C.c_longlong()
L.kp_profile_read(1, C.byref(t), C.byref(c))
L.kp_profile_enable(0)
print(f"{os.environ.get('VARIANT', '')}: n=4096 f16x {t.value / c.value:.3f} ms per GEMM ({c.value} launches) "
      f"{'OK' if ok else 'MISMATCH'}", flush=True)
