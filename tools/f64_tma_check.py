"""gemm_f64 staging check: dense operator at a ragged size against numpy, then the
time and digest of the C5-size dense operator apply with TMA and with cp.async
staging (KP_F64_TMA=0) - the two must agree bit for bit (same smem layout, same
MMA order)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, hashlib
sys.path.insert(0, %r)
import numpy as np
import ctypes as C
import paper_2311_15393_b200 as K
from paper_2311_15393_b200 import problems as P
from paper_2311_15393_b200._lib import lib, check
rng = np.random.default_rng(3)
n = 1546   # 13 x 13 big tiles, ragged in M, N and K
terms = [K.KronTerm(rng.standard_normal((n, n)), rng.standard_normal((n, n))) for _ in range(2)]
op = K.KroneckerSum(terms, n)
op.set_mode("dense")
x = rng.standard_normal(n * n)
y = K.kronsum_apply(op, x)
yt = K.kronsum_apply_transpose(op, x)
X = x.reshape(n, n, order="F")
ref = sum(t.col_factor @ X @ t.row_factor.T for t in terms).reshape(-1, order="F")
reft = sum(t.col_factor.T @ X @ t.row_factor for t in terms).reshape(-1, order="F")
e1 = np.linalg.norm(y - ref) / np.linalg.norm(ref); e2 = np.linalg.norm(yt - reft) / np.linalg.norm(reft)
n = 4096
psf = P.psf_gauss_motion(41, 4.0, 15, 30.0)
op, _ = P.psf_to_kronsum(psf, n, max_rank=5)
op.set_mode("dense")
x = rng.standard_normal(n * n)
y = K.kronsum_apply(op, x)
L = lib(); check(L.kp_profile_enable(1)); check(L.kp_profile_reset())
for _ in range(3): y = K.kronsum_apply(op, x)
t = C.c_double(); c = C.c_longlong(); check(L.kp_profile_read(0, C.byref(t), C.byref(c)))
ms = t.value / c.value
print("RESULT tma=%%s ragged rel err %%.2e %%.2e | n=4096 r=5: %%.3f ms per GEMM, %%.2f TF/s, digest %%s" %% (
    os.environ.get("KP_F64_TMA", "1"), e1, e2, ms, 2 * 5 * n**3 / (ms / 1e3) / 1e12, hashlib.md5(y.tobytes()).hexdigest()))
''' % ROOT
for tma in ["1", "0"]:
    env = dict(os.environ, KP_F64_TMA=tma)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    print([l for l in r.stdout.splitlines() if l.startswith("RESULT")] or r.stderr[-1500:], flush=True)
