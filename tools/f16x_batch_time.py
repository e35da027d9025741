"""Per-launch time of the batched M-solve products (kp_pcg_batch, 64 x n=1024)
on random data vs the C4 batch's own (stagnating) data, to separate the
shape (K = 1024 per tile) from the data (underflowing products, zero-output
fix-ups)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200._lib import lib  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard  # noqa: E402

L = lib()
sh = C4Shard()
ids = list(range(64))
probs = {i: sh.problem(i) for i in ids}
bs, xts, nz = sh.stack(ids, probs)
lams = sh.select_lambdas_arrays(bs, nz)


def timed(b, x, its, label):
    opts = K.SolverOptions(max_iterations=its, rel_residual_tol=1e-30)
    K.pcg_batch(sh.a, b, sh.m0, lams, opts, x_true=x)
    L.kp_profile_reset()
    L.kp_profile_enable(1)
    res = K.pcg_batch(sh.a, b, sh.m0, lams, opts, x_true=x)
    L.kp_profile_enable(0)
    t, c = C.c_double(), C.c_longlong()
    L.kp_profile_read(1, C.byref(t), C.byref(c))
    ta, ca = C.c_double(), C.c_longlong()
    L.kp_profile_read(4, C.byref(ta), C.byref(ca))
    launches = 4 * max(r.history.msolve_count for r in res)  # the capped last iteration skips its M-solve
    print(f"{label}: {its} iterations, precond {t.value:.1f} ms / {launches} GEMM launches = "
          f"{t.value / launches:.3f} ms per product; aux {ta.value:.1f} ms", flush=True)


for its in (3, 10, 30, 100):
    timed(bs, xts, its, f"C4 data, {its} iterations")
rng = np.random.default_rng(0)
rb = rng.standard_normal(bs.shape)
for its in (3, 30):
    timed(rb, xts, its, f"random rhs, {its} iterations")
