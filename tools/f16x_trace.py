"""Timeline of gemm_f16x's TMEM round trip (profiling build: KP_NVCC_EXTRA=-DKP_F16X_TRACE=1).

Reads the clock64 stamps CTA 0 leaves for its second tile (issuer thread,
epilogue warps 4 and 12) and prints the median phase lengths in cycles."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200 import _lib  # noqa: E402
from paper_2311_15393_b200.kronprec import SvdTriple  # noqa: E402

n = 4096
rng = np.random.default_rng(1)
v = rng.standard_normal((n, n)).astype(np.float16).astype(np.float64) / 64
trip = SvdTriple(v, np.linspace(1, 1e-3, n), v)
m = K.build_preconditioner_from_svd(trip, trip, 0.01, K.PrecisionFormat.fp16())
r = rng.standard_normal(n * n)
K.set_fp16_products("tensor")
for _ in range(2):
    K.precond_solve(m, r)
L = _lib.lib()
buf = (C.c_longlong * 16384)()
rc = L.kp_debug_f16x_trace(buf, 16384)
assert rc == 0, rc
t = np.array(buf[:], dtype=np.int64)
import os
NBUF = int(os.environ.get("NBUF", "2"))
iss = t[:1024 * NBUF].reshape(64, 4, NBUF, 4)  # kt, kk, h, stamp
epi = t[4096:8192].reshape(2, 64, 4, 8)        # warp(4|12), kt, kk, stamp
stg = t[8192:8448].reshape(64, 4)
sl = slice(8, 56)


def med(x):
    x = np.asarray(x).ravel()
    return f"med {np.median(x):7.0f}  p10 {np.percentile(x, 10):7.0f}  p90 {np.percentile(x, 90):7.0f}"


print("tile span (cycles):", iss[63, 3, NBUF - 1, 2] - iss[0, 0, 0, 0], " per kk:", (iss[63, 3, NBUF - 1, 2] - iss[0, 0, 0, 0]) / 256)
for h in range(NBUF):
    print(f"issuer buf{h}: tempty wait      ", med(iss[sl, :, h, 1] - iss[sl, :, h, 0]))
    print(f"issuer buf{h}: fence+mma+commit ", med(iss[sl, :, h, 2] - iss[sl, :, h, 1]))
    seq = iss[sl, :, h, 1].ravel()
    print(f"issuer buf{h}: period            ", med(np.diff(seq)))
print("issuer: wait A stage   ", med(stg[sl, 1] - stg[sl, 0]))
print("issuer: wait B expanded", med(stg[sl, 2] - stg[sl, 1]))
for w, h in ((0, 0), (1, NBUF // 2)):
    e = epi[w, sl]
    print(f"epi warp{4 + 8 * w} (buf{h}): tfull wait        ", med(e[:, :, 1] - e[:, :, 0]))
    print(f"epi warp{4 + 8 * w} (buf{h}): ld + wait::ld     ", med(e[:, :, 2] - e[:, :, 1]))
    print(f"epi warp{4 + 8 * w} (buf{h}): fence+arrive      ", med(e[:, :, 3] - e[:, :, 2]))
    print(f"epi warp{4 + 8 * w} (buf{h}): adds              ", med(e[:, :, 4] - e[:, :, 3]))
    print(f"epi warp{4 + 8 * w} (buf{h}): commit issued -> tfull seen ", med(e[:, :, 1] - iss[sl, :, h, 2]))
    nxt = iss[sl, :, h, 1].ravel()[1:]
    arr = e[:, :, 3].ravel()[:-1]
    print(f"epi warp{4 + 8 * w} (buf{h}): arrive -> issuer sees tempty", med(nxt - arr))
    print(f"epi warp{4 + 8 * w} (buf{h}): tfull seen -> arrive        ", med(e[:, :, 3] - e[:, :, 1]))
np.save("gpurun_out/f16x_trace.npy", t)
