"""GPU timeline of whole solves (CUPTI through torch.profiler): every kernel
and runtime call of a few device-resident solves, so the per-solve fixed cost
(setup kernels, graph capture / update, status polls, history copies) can be
separated from the iterations.

    python tools/solve_timeline.py C1 [solves]
"""
import ctypes as C
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200._lib import check, kp_history, kp_solver_options, lib, ptr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
nsolve = int(sys.argv[2]) if len(sys.argv) > 2 else 3
# CUPTI does not see kernels inside conditional (device-loop) graph bodies
import os  # noqa: E402
os.environ.setdefault("KP_GRAPH_LOOP", "0")
L = lib()
check(L.kp_init(0))
torch.cuda.set_device(0)
cfg = bench.build_problem(name, 0, None, device_apply=True)
svd_r, svd_c = bench.svd_pair(cfg.term, "host")
fmt = K.PrecisionFormat.fp16()
m = K.build_preconditioner_from_svd(svd_r, svd_c, cfg.lambda_ or 0.01, fmt)
solver_name, _, maxit = cfg.solvers[0]
solve_fn = L.kp_fpcg if solver_name == "fpcg" else L.kp_pcg
op = cfg.problem.a.handle()
nn = cfg.n * cfg.n


def dalloc(count):
    p = C.c_void_p()
    check(L.kp_device_alloc(count * 8, C.byref(p)))
    return p


d_b, d_x, d_xt = dalloc(nn), dalloc(nn), dalloc(nn)
check(L.kp_memcpy_h2d(d_b, ptr(cfg.problem.b), nn * 8))
check(L.kp_memcpy_h2d(d_xt, ptr(cfg.problem.x_true), nn * 8))
cap = maxit + 1
hb = [np.zeros(cap) for _ in range(4)]


def solve():
    h = kp_history(capacity=cap, relative_error=ptr(hb[0]), residual_norm=ptr(hb[1]),
                   work_units=ptr(hb[2]), residual_cosines=ptr(hb[3]))
    o = kp_solver_options(lambda_=cfg.lambda_ or 0.01, max_iterations=maxit, rel_residual_tol=cfg.tol,
                          x_true=d_xt.value, device_pointers=1)
    check(solve_fn(op, d_b, m.handle(), C.byref(o), d_x, C.byref(h)))
    return h.iterations_used


for _ in range(5):
    its = solve()
check(L.kp_synchronize())
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(nsolve):
        solve()
    check(L.kp_synchronize())
evs = [e for e in prof.events()]
kern = sorted([e for e in evs if e.device_type == torch.autograd.DeviceType.CUDA],
              key=lambda e: e.time_range.start)
cpu = sorted([e for e in evs if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda")],
             key=lambda e: e.time_range.start)
print(f"{name}: {its} iterations per solve, {len(kern)} GPU records, {len(cpu)} runtime calls")
t0 = kern[0].time_range.start
busy = sum(e.time_range.end - e.time_range.start for e in kern)
span = kern[-1].time_range.end - t0
print(f"GPU span {span:.1f} us for {nsolve} solves ({span / nsolve:.1f} us/solve), busy {busy:.1f} us "
      f"({busy / span:.2%}), idle {span - busy:.1f} us")
agg = defaultdict(lambda: [0, 0.0])
for e in kern:
    a = agg[e.name[:70]]
    a[0] += 1
    a[1] += e.time_range.end - e.time_range.start
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:70s} n={c:4d} mean={t / c:7.2f} us tot={t / nsolve:8.1f} us/solve")
api = defaultdict(lambda: [0, 0.0])
for e in cpu:
    a = api[e.name]
    a[0] += 1
    a[1] += e.time_range.end - e.time_range.start
print("runtime calls (host):")
for k, (c, t) in sorted(api.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:40s} n={c:4d} mean={t / c:7.2f} us tot={t / nsolve:8.1f} us/solve")
print("last solve, GPU timeline (start offset, duration, gap before):")
per = len(kern) // nsolve
last = kern[-per:]
prev_end = last[0].time_range.start
s0 = prev_end
for e in last:
    st, en = e.time_range.start, e.time_range.end
    print(f"  {st - s0:8.1f} {en - st:7.2f} gap {st - prev_end:6.2f}  {e.name[:60]}")
    prev_end = en
