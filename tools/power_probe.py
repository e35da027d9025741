"""Is the batched-product slowdown over a long C4 solve power / clock driven?
Times 3-iteration batched solves right after idle and right after ~1.5 s of
continuous load, and samples NVML SM clock, power and throttle reasons."""
import ctypes as C
import sys
import threading
import time

import numpy as np
import pynvml

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200._lib import lib  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def poll():
    while not stop.wait(0.005):
        samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))


L = lib()
sh = C4Shard()
ids = list(range(64))
probs = {i: sh.problem(i) for i in ids}
bs, xts, nz = sh.stack(ids, probs)
lams = sh.select_lambdas_arrays(bs, nz)


def run(its, label):
    opts = K.SolverOptions(max_iterations=its, rel_residual_tol=1e-30)
    L.kp_profile_reset()
    L.kp_profile_enable(1)
    t0 = time.time()
    K.pcg_batch(sh.a, bs, sh.m0, lams, opts, x_true=xts)
    t1 = time.time()
    L.kp_profile_enable(0)
    t, c = C.c_double(), C.c_longlong()
    L.kp_profile_read(1, C.byref(t), C.byref(c))
    win = [s for s in samples if t0 <= s[0] <= t1]
    clk = np.median([s[1] for s in win]) if win else float("nan")
    pw = max([s[2] for s in win]) if win else float("nan")
    reasons = sorted({s[3] for s in win})
    print(f"{label}: {t.value / (4 * (its + 1)):.3f} ms/product (wall {t1 - t0:.3f} s), SM clock median {clk} MHz, "
          f"power max {pw:.0f} W, reasons {[hex(r) for r in reasons]}", flush=True)


threading.Thread(target=poll, daemon=True).start()
run(3, "warm-up")
time.sleep(3)
run(3, "after 3 s idle, 3 iterations")
run(100, "100 iterations")
run(3, "right after, 3 iterations")
time.sleep(3)
run(3, "after 3 s idle, 3 iterations")
stop.set()
