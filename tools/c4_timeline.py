"""GPU timeline (CUPTI via torch.profiler) of one C4 step as bench.py runs it
(pinned host buffers, one kp_discrepancy_batch + one kp_pcg_batch): device
busy / idle, host->device / device->host copies, and the idle gaps (host
work the device waits for), with the kernels around them.

KP_GRAPH_LOOP=0 is set: CUPTI does not see kernels inside conditional
(device-loop) graph bodies."""
import ctypes as C
import os
import sys
from collections import defaultdict

os.environ.setdefault("KP_GRAPH_LOOP", "0")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2311_15393_b200._lib import check, lib  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard  # noqa: E402

L = lib()
check(L.kp_init(0))
torch.cuda.set_device(0)
sh = C4Shard(svd="gpu")
ids = list(range(64))
probs = {i: sh.problem(i) for i in ids}


def palloc(shape):
    p = C.c_void_p()
    check(L.kp_host_alloc(int(np.prod(shape)) * 8, C.byref(p)))
    return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=shape)


bs, xts, nz = sh.stack(ids, probs, palloc)
xout = palloc(bs.shape)
lv = [probs[i].noise_level for i in ids]
for _ in range(2):
    sh.solve_arrays(ids, bs, xts, nz, lv, out=xout)
check(L.kp_synchronize())
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    import time
    t0 = time.time()
    lams = sh.select_lambdas_arrays(bs, nz)
    check(L.kp_synchronize())
    t1 = time.time()
    sh.solve_arrays(ids, bs, xts, nz, lv, lams, out=xout)
    check(L.kp_synchronize())
    t2 = time.time()
print(f"host wall: lambdas {1e3 * (t1 - t0):.1f} ms, pcg_batch {1e3 * (t2 - t1):.1f} ms")
evs = prof.events()
gpu = sorted([e for e in evs if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
span = gpu[-1].time_range.end - gpu[0].time_range.start
busy = sum(e.time_range.end - e.time_range.start for e in gpu)
print(f"GPU span {span / 1e3:.1f} ms, busy {busy / 1e3:.1f} ms, idle {(span - busy) / 1e3:.1f} ms")
agg = defaultdict(lambda: [0, 0.0])
for e in gpu:
    a = agg[e.name[:60]]
    a[0] += 1
    a[1] += e.time_range.end - e.time_range.start
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {k:60s} n={c:5d} tot={t / 1e3:8.2f} ms mean={t / c:9.1f} us")
print("idle gaps > 100 us:")
prev = gpu[0]
tot_gap = 0.0
for e in gpu[1:]:
    g = e.time_range.start - prev.time_range.end
    if g > 100:
        tot_gap += g
        print(f"  {g / 1e3:7.2f} ms after {prev.name[:45]:45s} before {e.name[:45]}")
    prev = e
print(f"sum of gaps > 100 us: {tot_gap / 1e3:.1f} ms")
api = defaultdict(lambda: [0, 0.0])
for e in evs:
    if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda"):
        a = api[e.name]
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
for k, (c, t) in sorted(api.items(), key=lambda kv: -kv[1][1])[:10]:
    print(f"  host {k:36s} n={c:5d} tot={t / 1e3:8.2f} ms")
