"""Device time of the batched lambda sweeps at C4 size (dev tool): one
objective value vs 63 in one launch, and one discrepancy solve."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2311_15393_b200 import kronprec as K  # noqa: E402
from paper_2311_15393_b200._lib import check, lib  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard  # noqa: E402

check(lib().kp_init(0))
sh = C4Shard(svd="gpu")
tp = sh.problem(0)
sd = K.make_spectral_data(sh.m0, tp.b)
nn = float(np.linalg.norm(tp.noise))
lams = np.logspace(-4, 0, 63)
for _ in range(3):
    K.gcv_grid(sd, lams)
    K.discrepancy(sd, nn, 1.01)
    K.discrepancy_gap(sd, nn, 0.01)
for name, fn in (("gap x1", lambda: K.discrepancy_gap(sd, nn, 0.01)),
                 ("gcv_grid x63", lambda: K.gcv_grid(sd, lams)),
                 ("gcv_grid x16", lambda: K.gcv_grid(sd, lams[:16])),
                 ("discrepancy", lambda: K.discrepancy(sd, nn, 1.01))):
    t = time.perf_counter()
    for _ in range(20):
        fn()
    print(f"{name:14s} {(time.perf_counter() - t) / 20 * 1e3:.3f} ms (host wall)")
