"""GPU check of the tcgen05 rounded-leaf GEMM (gemm_f16x) against gemm_f16ref
and the oracle: bitwise (incl. the sign of zeros) on lp_matmul and
precond_solve, plus per-launch timing of both engines."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200 import _lib  # noqa: E402
from paper_2311_15393_b200.kronprec import SvdTriple  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

F16 = K.PrecisionFormat.fp16()
rng = np.random.default_rng(7)


def f16(x):
    return x.astype(np.float16).astype(np.float64)


def bits_equal(a, b):
    """Bitwise equality (signed zeros included); any NaN equals any NaN."""
    a, b = np.asarray(a), np.asarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    return np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64))


def both(fn):
    K.set_fp16_products("cuda")
    r1 = fn()
    K.set_fp16_products("tensor")
    r2 = fn()
    K.set_fp16_products("auto")
    return r1, r2


ok = True
cases = [(1, 1, 1), (7, 5, 3), (128, 64, 32), (130, 65, 33), (300, 200, 100), (513, 300, 257),
         (1000, 129, 77), (2048, 300, 1280), (256, 4096, 256)]
for (m, k, n) in cases:
    for dist in ("normal", "wide", "zeros", "tinyneg"):
        if dist == "normal":
            a, b = f16(rng.standard_normal((m, k))), f16(rng.standard_normal((k, n)))
        elif dist == "wide":
            a = f16(rng.standard_normal((m, k)) * np.exp2(rng.integers(-20, 10, (m, k))))
            b = f16(rng.standard_normal((k, n)) * np.exp2(rng.integers(-20, 10, (k, n))))
        elif dist == "zeros":
            a = f16(rng.standard_normal((m, k)) * (rng.random((m, k)) < 0.5))
            b = f16(rng.standard_normal((k, n)) * (rng.random((k, n)) < 0.3))
            a[a == 0] = np.where(rng.random(np.count_nonzero(a == 0)) < 0.5, -0.0, 0.0)
        else:  # all products underflow: outputs +-0, signs matter
            a = -np.abs(f16(rng.random((m, k)) * 1e-4))
            b = f16(rng.random((k, n)) * 1e-4)
            if m > 3:
                a[3, :] = np.abs(a[3, :])  # a row with same signs -> +0
        c1, c2 = both(lambda: K.lp_matmul(a, b, F16))
        same = bits_equal(c1, c2)
        orc = O.lp_matmul(a, b, F16) if m * n * k <= 3e8 else None
        so = bits_equal(c2, orc) if orc is not None else None
        nz = int(np.count_nonzero(c2 == 0))
        print(f"lp_matmul {m}x{k}x{n} {dist:8s}: tensor==cuda {same}  tensor==oracle {so}  zeros {nz}", flush=True)
        ok &= same and (so is not False)

for n in (256, 512, 1024, 1664):
    ur, _ = np.linalg.qr(rng.standard_normal((n, n)))
    uc, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sr = np.sort(rng.random(n))[::-1] + 1e-3
    sc = np.sort(rng.random(n))[::-1] + 1e-3
    trip_r, trip_c = SvdTriple(ur, sr, ur.copy()), SvdTriple(uc, sc, uc.copy())
    m = K.build_preconditioner_from_svd(trip_r, trip_c, 0.01, F16)
    for scale in (1.0, 1e-6, 0.0):
        r = rng.standard_normal(n * n) * scale
        z1, z2 = both(lambda: K.precond_solve(m, r))
        print(f"precond_solve n={n} scale={scale}: tensor==cuda {bits_equal(z1, z2)} zeros {int(np.count_nonzero(z2 == 0))}",
              flush=True)
        ok &= bits_equal(z1, z2)

# timing at n = 4096 (one M-solve = 4 GEMMs)
n = 4096
v = f16(rng.standard_normal((n, n)) / 64)
trip = SvdTriple(v, np.linspace(1, 1e-3, n), v)
m = K.build_preconditioner_from_svd(trip, trip, 0.01, F16)
r = rng.standard_normal(n * n)
L = _lib.lib()
for eng in ("cuda", "tensor"):
    K.set_fp16_products(eng)
    K.precond_solve(m, r)
    L.kp_profile_reset()
    L.kp_profile_enable(1)
    for _ in range(3):
        z = K.precond_solve(m, r)
    import ctypes as C
    t, c = C.c_double(), C.c_longlong()
    L.kp_profile_read(1, C.byref(t), C.byref(c))
    L.kp_profile_enable(0)
    per = t.value / c.value
    print(f"n=4096 {eng}: {c.value} precond launches, {per:.3f} ms avg  (GEMM-equivalent {t.value / 12:.3f} ms per GEMM)")
K.set_fp16_products("auto")
print("ALL OK" if ok else "MISMATCH")
