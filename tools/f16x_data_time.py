"""gemm_f16x time per product vs the data: random residuals, residuals whose
products all underflow (every output an all-zero tree, zero-sign path), and
residuals at the C4 stagnation scale (n = 1024 x 64 images would be the same
shape per image; here one n = 4096 M-solve)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200 import _lib  # noqa: E402
from paper_2311_15393_b200.kronprec import SvdTriple  # noqa: E402

n = 4096
rng = np.random.default_rng(1)
v = (rng.standard_normal((n, n)) / 64).astype(np.float16).astype(np.float64)
trip = SvdTriple(v, np.linspace(1, 1e-3, n), v)
m = K.build_preconditioner_from_svd(trip, trip, 0.01, K.PrecisionFormat.fp16())
K.set_fp16_products("tensor")
L = _lib.lib()
base = rng.standard_normal(n * n)
for label, scale in (("random (scale 1)", 1.0), ("scale 1e-6 (subnormal r16)", 1e-6),
                     ("scale 1e-7 (mostly underflowing leaves)", 1e-7), ("scale 1e-12 (all zero)", 1e-12)):
    r = base * scale
    K.precond_solve(m, r)
    L.kp_profile_reset()
    L.kp_profile_enable(1)
    for _ in range(2):
        z = K.precond_solve(m, r)
    t, c = C.c_double(), C.c_longlong()
    L.kp_profile_read(1, C.byref(t), C.byref(c))
    ta, ca = C.c_double(), C.c_longlong()
    L.kp_profile_read(4, C.byref(ta), C.byref(ca))
    L.kp_profile_enable(0)
    print(f"{label:42s} {t.value / c.value:.3f} ms per product, aux {ta.value / max(1, ca.value):.3f} ms/launch, "
          f"zeros in z {np.count_nonzero(z == 0)}", flush=True)
