"""Sweep the DMMA GEMM variants (KP_F64_CFG) at C5 size (dev tool)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, time, hashlib
sys.path.insert(0, %r)
import numpy as np
import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200._lib import lib, check
import ctypes as C
n = 4096
psf = P.psf_gauss_motion(41, 4.0, 15, 30.0)
op, _ = P.psf_to_kronsum(psf, n, max_rank=5)
x = np.random.default_rng(0).standard_normal(n * n)
y = K.kronsum_apply(op, x)
L = lib(); check(L.kp_profile_enable(1)); check(L.kp_profile_reset())
for _ in range(3): y = K.kronsum_apply(op, x)
t = C.c_double(); c = C.c_longlong(); check(L.kp_profile_read(0, C.byref(t), C.byref(c)))
print("RESULT", os.environ.get("KP_F64_CFG", "0"), t.value / c.value, 2 * 5 * n**3 / (t.value / c.value / 1e3) / 1e12, hashlib.md5(y.tobytes()).hexdigest())
''' % ROOT
for cfg in ["0", "1", "2", "3", "4"]:
    env = dict(os.environ, KP_F64_CFG=cfg)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print([l for l in r.stdout.splitlines() if l.startswith("RESULT")] or r.stderr[-500:], flush=True)
