"""Per-launch device time of the operator kernels at C5 size (dev tool)."""
import os, sys, ctypes as C, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200._lib import lib, check
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
psf = P.psf_gauss_motion(41, 4.0, 15, 30.0)
op, _ = P.psf_to_kronsum(psf, n, max_rank=5)
x = np.random.default_rng(0).standard_normal(n * n)
L = lib()
for mode in ("banded",):
    op.set_mode(mode)
    y = K.kronsum_apply(op, x); yt = K.kronsum_apply_transpose(op, x)
    check(L.kp_profile_reset()); check(L.kp_profile_enable(1))
    for _ in range(3):
        K.kronsum_apply(op, x); K.kronsum_apply_transpose(op, x)
    t = C.c_double(); c = C.c_longlong(); check(L.kp_profile_read(0, C.byref(t), C.byref(c)))
    check(L.kp_profile_enable(0))
    flops = 2 * 5 * 82 * n * n  # per apply, unpadded taps
    print("RESULT", mode, n, f"{t.value / c.value:.4f} ms/pass", f"{flops / (2 * t.value / c.value / 1e3) / 1e12:.2f} TF/s",
          hashlib.md5(y.tobytes()).hexdigest()[:12], hashlib.md5(yt.tobytes()).hexdigest()[:12], flush=True)
