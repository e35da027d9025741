"""Where the time of one batched C4 pass goes (host phases + kernel classes)."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200._lib import lib  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard  # noqa: E402

sh = C4Shard()
ids = list(range(64))
probs = {i: sh.problem(i) for i in ids}
bs, xts, nz = sh.stack(ids, probs)
lv = [probs[i].noise_level for i in ids]
out = np.empty_like(bs)
sh.solve_arrays(ids[:4], np.ascontiguousarray(bs[:4]), np.ascontiguousarray(xts[:4]), nz[:4], lv[:4])
L = lib()
for rep in range(2):
    L.kp_synchronize()
    t0 = time.time()
    lams = sh.select_lambdas_arrays(bs, nz)
    t1 = time.time()
    L.kp_profile_reset()
    L.kp_profile_enable(1 if rep else 0)
    res = sh.solve_arrays(ids, bs, xts, nz, lv, lams, out=out)
    L.kp_synchronize()
    t2 = time.time()
    L.kp_profile_enable(0)
    print(f"pass {rep} ({'profiled' if rep else 'graph'}): lambdas {t1 - t0:.3f} s, batched pcg {t2 - t1:.3f} s, "
          f"iterations {max(r.iterations for r in res)}")
for cls, name in enumerate(["operator", "precond", "vector", "spectral", "precond_aux"]):
    t, c = C.c_double(), C.c_longlong()
    L.kp_profile_read(cls, C.byref(t), C.byref(c))
    print(f"  {name:12s} {t.value:9.1f} ms  {c.value:6d} launches  {t.value / max(1, c.value):.4f} ms/launch")
