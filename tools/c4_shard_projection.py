"""C4 strong-scaling projection from ONE GPU: for N = 1, 2, 4, 8 ranks, time each
rank's shard of the 64 images (its one batched solve, host buffers in and out,
exactly what bench.py --gpus N runs on that rank) one shard at a time on this
GPU. The ranks of the real job share nothing on the data path (NCCL only gathers
the per-image results), so the job time is the slowest shard's time:
projected solves/s = 64 / max over ranks of t_shard. This is a projection, not
a multi-GPU measurement (the pool gives one GPU per call)."""
import ctypes as C
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2311_15393_b200._lib import check, lib  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard, shard  # noqa: E402

L = lib()
check(L.kp_init(0))
images = 64
sh = C4Shard(n=1024, svd="host", device=0)
probs = {i: sh.problem(i) for i in range(images)}
pinned = []


def palloc(shape):
    p = C.c_void_p()
    check(L.kp_host_alloc(int(np.prod(shape)) * 8, C.byref(p)))
    pinned.append(p)
    return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=shape)


def timed(mine, reps=2):
    bs, xts, nzs = sh.stack(mine, probs, palloc)
    xout = palloc(bs.shape)
    levels = [probs[i].noise_level for i in mine]
    sh.solve_arrays(mine, bs, xts, nzs, levels, out=xout)  # warm-up
    best = None
    for _ in range(reps):
        check(L.kp_synchronize())
        check(L.kp_event_record(0))
        res = sh.solve_arrays(mine, bs, xts, nzs, levels, out=xout)
        check(L.kp_event_record(1))
        ms = C.c_float()
        check(L.kp_event_elapsed(0, 1, C.byref(ms)))
        best = ms.value / 1e3 if best is None else min(best, ms.value / 1e3)
    return best, res


rows, base = [], None
for N in (1, 2, 4, 8):
    ts = []
    for r in range(N):
        t, res = timed(list(shard(images, N, r)))
        ts.append(t)
    val = images / max(ts)
    base = base or val
    rows.append({"ranks": N, "images_per_rank": images // N, "shard_s": [round(t, 4) for t in ts],
                 "projected_solves_per_s": round(val, 2), "projected_efficiency": round(val / (N * base), 3)})
    print(json.dumps(rows[-1]), flush=True)
