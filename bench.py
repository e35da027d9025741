#!/usr/bin/env python
"""Benchmark of the B200 PCG / FPCG hot path (BASELINE.json metric).

Workload (N=1): config C5 — n=4096 (16.7M unknowns), rank-5 Kronecker-sum
blur, FPCG with the fp16 Kronecker-SVD preconditioner (reference-exact
per-op rounding), lambda=0.01, tol 1e-6, max 100 iterations. One "step" is
one full FPCG solve; the metric is solver iterations per second over the K
timed steps. N>1 (torchrun): config C4, the BASELINE batched metric —
solves/s over the 64-image batch, images sharded over the ranks (strong
scaling), one batched PCG state machine per GPU, NCCL only to gather the
per-image results and the timing. `--config` overrides either default.

  value       device-resident b / x (kp_fpcg with device pointers)
  e2e         the C-ABI call with pinned HOST buffers (b, x_true in; x out)
  roofline    dominant kernel = the reference-exact binary16 M-solve GEMM
              (gemm_f16x: tcgen05 rounded products + f16x2 tree adds)
  cpu_baseline  the CPU oracle (C++ restatement of the reference, OpenBLAS +
              streamed fp16 emulation) timed on the host cores for one
              iteration's operator + preconditioner work (all threads, and a
              1-thread sample like the single-threaded reference)

`--impl reference` times that CPU implementation as the reference arm.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DMMA_PEAK_TFLOPS = 37.07  # measured, profiles/r01_microbench_peaks_v2.txt (m16n8k16 f64)
DFMA_PEAK_TFLOPS = 33.88  # measured DFMA (FP64 ALU) peak, same microbenchmark
F16X2_PEAK_TOPS = 36.9    # measured f16x2 mul+add half-ops/s, same file
# DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from the
# committed ncu --set full captures (profiles/r01_ncu_key_metrics.txt, r02_*)
TRAFFIC = {
    ("gemm_f16ref_kernel", 4096): 68.29e6 + 21.03e6,   # r01_gemm_f16ref_u64_n4096.ncu-rep
    ("gemm_f16x_kernel", 4096): 73.48e6 + 18.53e6,     # r02_gemm_f16x_c5.ncu-rep
    ("gemm_f16tc_kernel", 4096): (73.37e6 + 13.91e6 + 118.5e6 + 18.64e6 + 72.79e6 + 13.88e6
                                  + 71.8e6 + 15.19e6) / 4,  # mean of the 4 products of a solve
    ("band", 4096): (134.2e6 + 613.1e6 + 671.1e6 + 121.8e6) / 2,  # per pass, r01_band_vec
}


def peaks():
    """Driver-measured roofline denominators (MEASURED_PEAKS.json): HBM copy
    GB/s and cuBLAS bf16 TFLOP/s, burst (kernel timed alone) and sustained
    (seconds-long loop under the power cap); the recipe's fallback if absent."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "MEASURED_PEAKS.json (measured)"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "B200_PROFILING.md fallback"}


class ClockSampler:
    """SM clocks and throttle reasons during the timed region.

    NVML (pynvml) polled every 2 ms from a thread, plus one sample on entry
    and one on exit, so even a millisecond-long region (C1) has samples;
    nvidia-smi -lms 200 when NVML is unavailable."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        self.index = int(ids[index]) if index < len(ids) and ids[index].isdigit() else index
        self.proc = None
        self.nvml = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, float, int]] = []
        self.stop = threading.Event()

    def _nvml_sample(self):
        n, h = self.nvml, self.handle
        self.samples.append((float(n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)),
                             float(n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)),
                             int(n.nvmlDeviceGetCurrentClocksEventReasons(h))))

    def _poll(self):
        while not self.stop.wait(0.002):
            self._nvml_sample()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml, self.handle = pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nvml_sample()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=1)
            self._nvml_sample()
            return
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        if self.nvml:
            for clk, cmax, bits in self.samples:
                sm.append(clk)
                mx = max(mx, cmax)
                reasons.update(nm for nm, b in self.REASONS if bits & b)
        names = [nm for nm, _ in self.REASONS]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.nvml else "nvidia-smi"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def build_problem(name: str, image: int, n: int | None, device_apply: bool):
    """Config problem; b_true computed on the device for large n (setup only)."""
    from paper_2311_15393_b200 import configs, problems as P
    import paper_2311_15393_b200 as K
    if not device_apply:
        return configs.build(name, image=image, n=n)
    orig = P.kronsum_apply_host
    P.kronsum_apply_host = lambda k, x: K.kronsum_apply(k, x)
    try:
        return configs.build(name, image=image, n=n)
    finally:
        P.kronsum_apply_host = orig


def svd_pair(term, how: str):
    """Setup SVDs of the two factors: host LAPACK dgesdd (the oracle's
    routine) or the library's device SVD (cuSOLVER FP64, kp_svd)."""
    import paper_2311_15393_b200 as K
    from paper_2311_15393_b200 import problems as P
    from paper_2311_15393_b200.kronprec import SvdTriple
    if how == "host":  # host-only entry point (also used by the CPU reference arm)
        return SvdTriple(*P.host_svd(term.row_factor)), SvdTriple(*P.host_svd(term.col_factor))
    return SvdTriple(*K.svd(term.row_factor, "device")), SvdTriple(*K.svd(term.col_factor, "device"))


def cpu_iteration_sample(cfg, svd_r, svd_c, fmt, threads: int) -> float:
    """Seconds for one FPCG iteration's operator + preconditioner work on the
    CPU oracle (normal_matvec + precond_solve)."""
    from oracle import pyoracle as O
    O.set_threads(threads)
    po = O.build_preconditioner_from_svd((svd_r.u, svd_r.s, svd_r.v),
                                         (svd_c.u, svd_c.s, svd_c.v), cfg.lambda_, fmt)
    p = np.random.default_rng(0).standard_normal(cfg.n * cfg.n)
    t0 = time.perf_counter()
    O.normal_matvec(cfg.problem.a, cfg.lambda_, p)
    O.precond_solve(po, p)
    return time.perf_counter() - t0


def cpu_iteration_single_thread(cfg, fmt, slab: int = 128) -> dict:
    """One FPCG iteration's operator + preconditioner work on ONE host thread
    (the reference is single-threaded: no OpenMP in proj/CMakeLists.txt),
    from a bounded sample: one dense one-term kron_apply (2 FP64 GEMMs of
    n^3, the oracle's OpenBLAS on 1 thread) and one `slab`-row block of a
    reference-exact binary16 lp_matmul (slab x n x n), extrapolated to the
    iteration's 2 r applies of the operator (normal_matvec) and 4 full n^3
    lp_matmuls (precond_solve)."""
    from oracle import pyoracle as O
    import paper_2311_15393_b200 as K
    n = cfg.n
    slab = min(slab, n)
    O.set_threads(1)
    try:
        rng = np.random.default_rng(0)
        one = K.KroneckerSum([cfg.problem.a.terms[0]], n)
        x = rng.standard_normal(n * n)
        t0 = time.perf_counter()
        O.kronsum_apply(one, x)
        t_apply = time.perf_counter() - t0
        a = rng.uniform(-1, 1, (slab, n)).astype(np.float16).astype(np.float64)
        b = rng.uniform(-1, 1, (n, n)).astype(np.float16).astype(np.float64)
        t0 = time.perf_counter()
        O.lp_matmul(a, b, fmt)
        t_slab = time.perf_counter() - t0
    finally:
        O.set_threads(os.cpu_count() or 1)
    r = len(cfg.problem.a.terms)
    t_iter = 2 * r * t_apply + 4 * (n / slab) * t_slab
    return {"value": 1.0 / t_iter, "unit": "iterations/s", "cores": 1, "kind": "port",
            "sample": f"1 thread: one one-term kron_apply at n={n} ({t_apply:.2f} s) and a {slab}-row "
                      f"block of one binary16 lp_matmul ({t_slab:.2f} s), extrapolated to 2r={2 * r} "
                      f"applies + 4 full lp_matmuls per iteration",
            "sample_s": t_apply + t_slab}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import paper_2311_15393_b200 as K
    threads = os.cpu_count() or 1
    t0 = time.time()
    cfg = build_problem(args.config, 0, args.size, device_apply=False)
    svd_r, svd_c = svd_pair(cfg.term, "host")
    fmt = K.PrecisionFormat.fp16()
    if cfg.lambda_ is None:  # C3 / C4: the config's lambda rule, on the oracle (cli.cpp:469-505)
        from oracle import pyoracle as O
        from paper_2311_15393_b200.configs import GCV_GRID
        m0 = O.build_preconditioner_from_svd((svd_r.u, svd_r.s, svd_r.v),
                                             (svd_c.u, svd_c.s, svd_c.v), 1.0, fmt)
        so, bo = O.spectral(m0, cfg.problem.b)
        if cfg.select == "gcv_grid":
            cfg.lambda_ = O.gcv_grid(so, bo, GCV_GRID)[0]["lambda"]
        else:
            cfg.lambda_ = O.discrepancy(so, bo, float(np.linalg.norm(cfg.problem.noise)),
                                        cfg.eta)["lambda"]
    setup_s = time.time() - t0
    solver_name = cfg.solvers[0][0]
    if args.config == "C4":
        return run_reference_c4(args, cfg, svd_r, svd_c, fmt, threads, setup_s)
    for _ in range(args.warmup):
        cpu_iteration_sample(cfg, svd_r, svd_c, fmt, threads)
    times = [cpu_iteration_sample(cfg, svd_r, svd_c, fmt, threads) for _ in range(args.steps)]
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference",
        "metric": metric_name(cfg),
        "value": value, "unit": "iterations/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+f16(emulated)", "data": "synthetic",
        "config": workload_config(cfg),
        "run_info": {"l2": "host CPU run (no GPU L2 involved)"},
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": threads, "kind": "port",
                         "sample": f"one {solver_name.upper()} iteration's normal_matvec + "
                                   "precond_solve (fp16 reference-exact emulation) per step"},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "setup_s": setup_s,
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_c4_image_sample(cfg, svd_r, svd_c, fmt, threads) -> float:
    """Seconds per C4 image on the CPU oracle: the lambda selection (spectral
    data + discrepancy) timed, plus one PCG iteration's operator +
    preconditioner work timed and scaled to the image's 100 iterations."""
    from oracle import pyoracle as O
    O.set_threads(threads)
    m0 = O.build_preconditioner_from_svd((svd_r.u, svd_r.s, svd_r.v), (svd_c.u, svd_c.s, svd_c.v), 1.0, fmt)
    t0 = time.perf_counter()
    so, bo = O.spectral(m0, cfg.problem.b)
    lam = O.discrepancy(so, bo, float(np.linalg.norm(cfg.problem.noise)), cfg.eta)["lambda"]
    t_sel = time.perf_counter() - t0
    cfg.lambda_ = lam  # the image's own lambda for the iteration sample
    return t_sel + 100 * cpu_iteration_sample(cfg, svd_r, svd_c, fmt, threads)


def run_reference_c4(args, cfg, svd_r, svd_c, fmt, threads, setup_s):
    """Reference arm for C4 (solves/s over the image batch): per step one
    image's lambda selection (spectral data + discrepancy, on the oracle)
    plus one PCG iteration's operator + preconditioner work, extrapolated to
    the 100 iterations every C4 image runs (the reference-exact solves
    stagnate to the cap; tests/golden/C4.json)."""
    def step():
        return cpu_c4_image_sample(cfg, svd_r, svd_c, fmt, threads)

    for _ in range(args.warmup):
        step()
    per_image = [step() for _ in range(args.steps)]
    value = args.steps / sum(per_image)
    metric = METRIC_C4 if cfg.n == 1024 else METRIC_C4.replace("1024^2", f"{cfg.n}^2")
    line = {"impl": "reference", "metric": metric, "value": value, "unit": "solves/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(per_image) / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64+f16(emulated)", "data": "synthetic",
            "config": c4_config(),
            "run_info": {"l2": "host CPU run (no GPU L2 involved)"},
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": threads, "kind": "port",
                             "sample": "per step: one C4 image's spectral data + discrepancy lambda and one "
                                       "PCG iteration (normal_matvec + precond_solve), extrapolated to the "
                                       "image's 100 iterations"},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_s": setup_s}
    print(json.dumps(line), flush=True)
    return 0


def c4_config() -> dict:
    return {"workload": "C4: 64 x n=1024, Gaussian sigma=2.5, noise 0.1/1/5 %, discrepancy eta=1.01, "
                        "PCG fp16 tol 1e-6", "images": 64,
            "l2": "GPU arm: each step solves 64 distinct images (8 MB inputs and ~0.1 GB of solver state "
                  "per image), far more than the 126 MB L2; no flush needed"}


METRIC = "PCG iterations/s at 4096^2 image"


def metric_name(cfg) -> str:
    """BASELINE's headline metric name for C5 at full size; otherwise the
    same metric labelled with the config and image side actually run."""
    if cfg.name == "C5" and cfg.n == 4096:
        return METRIC
    return f"PCG iterations/s at {cfg.n}^2 image ({cfg.name})"
METRIC_C4 = "solves/s over image batch (64 x 1024^2, discrepancy lambda + PCG fp16)"


def run_c4(args):
    """BASELINE C4: 64 independent 1024^2 images sharded across the ranks;
    per image: spectral data, discrepancy lambda, with_lambda, PCG (fp16)."""
    ws, rank, local = dist_env()
    import torch
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    from paper_2311_15393_b200._lib import check, lib
    from paper_2311_15393_b200.batch import C4Shard, gather_results, reduce_timing, shard
    L = lib()
    check(L.kp_init(local))
    images = 64
    mine = list(shard(images, ws, rank))
    sh = C4Shard(n=args.size, svd=args.svd, device=local)
    t_gen = time.time()
    probs = {i: sh.problem(i) for i in mine}  # input generation is not timed
    t_gen_host = time.time() - t_gen
    # the same images generated on the device (kp_generate_test_problems), for the record
    from paper_2311_15393_b200 import problems as Pm
    check(L.kp_synchronize())
    t_gen = time.time()
    Pm.make_test_problems_device(sh.a, [4000 + i for i in mine], [5000 + i for i in mine],
                                 [probs[i].noise_level for i in mine])
    t_gen_dev = time.time() - t_gen
    batched = args.c4_mode == "batch"
    pinned = []

    def palloc(shape):  # pinned host staging (the e2e inputs / outputs live here)
        p = C.c_void_p()
        check(L.kp_host_alloc(int(np.prod(shape)) * 8, C.byref(p)))
        pinned.append(p)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=shape)

    if batched:
        bs, xts, nzs = sh.stack(mine, probs, palloc)
        xout = palloc(bs.shape)
        levels = [probs[i].noise_level for i in mine]

    def run_all():
        # batch: lambdas by kp_discrepancy_batch, then ONE batched PCG over this
        # rank's images (kp_pcg_batch), host buffers in and out; streams: the
        # per-image pipeline on `workers` concurrent streams
        if batched:
            return sh.solve_arrays(mine, bs, xts, nzs, levels, out=xout)
        return sh.solve_many(mine, probs, args.workers)

    for _ in range(max(1, args.warmup)):
        run_all()
    if dist:
        dist.barrier()
    launches0 = L.kp_launch_count()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            check(L.kp_synchronize())
            check(L.kp_event_record(0))
            results = run_all()  # ends synchronised (host buffers out)
            check(L.kp_event_record(1))
            ms = C.c_float()
            check(L.kp_event_elapsed(0, 1, C.byref(ms)))
            times.append(ms.value / 1e3)
    elapsed = sum(times)
    launches = L.kp_launch_count() - launches0
    # profiled pass (per-launch events) for the M-solve GEMM roofline
    roof = None
    if batched:
        lams = sh.select_lambdas_arrays(bs, nzs)
        check(L.kp_profile_reset())
        check(L.kp_profile_enable(1))
        res_p = sh.solve_arrays(mine, bs, xts, nzs, levels, lams, out=xout)
        tt, tc = C.c_double(), C.c_longlong()
        check(L.kp_profile_read(1, C.byref(tt), C.byref(tc)))
        check(L.kp_profile_enable(0))
        nb = sum(1 for v in lams if v is not None)
        # batched M-solves that ran: the longest image's msolve_count (a solve
        # stopped at the iteration cap skips its last M-solve)
        batches = max(r.msolve_count for r in res_p)
        work = 2.0 * nb * float(sh.n) ** 3  # binary16 ops per launch (all images of the batch)
        ach = work / (tt.value / (4 * batches) / 1e3) / 1e12 if tc.value else 0.0
        import paper_2311_15393_b200 as K
        eng = K.fp16_products_engine(sh.n)
        peak = 2.0 * F16X2_PEAK_TOPS if eng == "tensor" else F16X2_PEAK_TOPS
        roof = {"bound": "compute", "pipe": "f16x2 CUDA-core pipe (tree adds)" +
                ("; rounded products from tcgen05" if eng == "tensor" else ""),
                "achieved": ach, "peak": peak, "unit": "T half-ops/s", "frac": ach / peak,
                "traffic": None,
                "kernel": "gemm_f16x_kernel" if eng == "tensor" else "gemm_f16ref_kernel",
                "work_per_launch": f"{work:.4g} half-ops ({nb} images x 2 n^3, batched along N)",
                "launches": 4 * batches, "ms_per_launch": tt.value / (4 * batches)}
    # ---- device-resident pass (the line's `value`): the same batched solve with
    # b / x_true / x in device memory (kp_discrepancy_batch_ex + kp_pcg_batch with
    # device_pointers); the host-buffer loop above is the line's `e2e` ----
    res_elapsed = None
    if batched:
        from paper_2311_15393_b200._lib import kp_history, kp_solver_options, ptr
        B, nn_ = len(mine), sh.n * sh.n
        dptr = []

        def dalloc(count):
            p = C.c_void_p()
            check(L.kp_device_alloc(count * 8, C.byref(p)))
            dptr.append(p)
            return p

        d_b, d_xt, d_x = dalloc(B * nn_), dalloc(B * nn_), dalloc(B * nn_)
        check(L.kp_memcpy_h2d(d_b, ptr(bs), B * nn_ * 8))
        check(L.kp_memcpy_h2d(d_xt, ptr(xts), B * nn_ * 8))
        nz_arr = np.ascontiguousarray(np.asarray(nzs, dtype=np.float64))
        lam_arr, st_arr = np.zeros(B), np.zeros(B, dtype=np.int32)
        cap = 101
        hbufs = [[np.zeros(cap) for _ in range(4)] for _ in range(B)]
        hs = (kp_history * B)()

        def run_resident():
            check(L.kp_discrepancy_batch_ex(sh.m0.handle(), B, d_b, ptr(nz_arr), float(sh.eta), ptr(lam_arr),
                                            st_arr.ctypes.data_as(C.c_void_p), 1))
            if np.any(st_arr != 0):
                return None
            for i, (rel, res, work, cos) in enumerate(hbufs):
                hs[i] = kp_history(capacity=cap, relative_error=ptr(rel), residual_norm=ptr(res),
                                   work_units=ptr(work), residual_cosines=ptr(cos))
            o = kp_solver_options(lambda_=0.0, max_iterations=100, rel_residual_tol=float(sh.tol), x_true=d_xt.value,
                                  track_search_direction_orthogonality=0, record_iterates=0, device_pointers=1)
            check(L.kp_pcg_batch(sh.a.handle(), sh.m0.handle(), B, d_b, ptr(lam_arr), C.byref(o), d_x, hs))
            check(L.kp_synchronize())
            return [hs[i].iterations_used for i in range(B)]

        its_res = run_resident()  # warm-up
        if its_res is not None and its_res != [r.iterations for r in results]:
            raise RuntimeError("device-resident batch differs from the host-buffer batch")
        # every rank takes the same path (an image without a root on any rank: all fall back to e2e)
        bad, _ = reduce_timing(0.0 if its_res is not None else 1.0, 0.0, dist,
                               device="cuda" if args.dist_backend == "nccl" else "cpu")
        if bad == 0.0:
            if dist:
                dist.barrier()
            res_times = []
            for _ in range(args.steps):
                check(L.kp_synchronize())
                check(L.kp_event_record(2))
                run_resident()
                check(L.kp_event_record(3))
                ms = C.c_float()
                check(L.kp_event_elapsed(2, 3, C.byref(ms)))
                res_times.append(ms.value / 1e3)
            res_elapsed = sum(res_times)
        for p in dptr:
            check(L.kp_device_free(p))
    e2e_elapsed, solved = reduce_timing(elapsed, float(len(results) * args.steps), dist,
                                        device="cuda" if args.dist_backend == "nccl" else "cpu")
    if res_elapsed is None:
        elapsed = e2e_elapsed
    else:
        elapsed, _ = reduce_timing(res_elapsed, float(len(results) * args.steps), dist,
                                   device="cuda" if args.dist_backend == "nccl" else "cpu")
    allres = gather_results(results, dist,
                            device="cuda" if (dist and args.dist_backend == "nccl") else None)

    # ---- secondary: the same batch with the tcgen05 tensor-mode preconditioner ----
    tensor = None
    if not args.no_tensor:
        sht = C4Shard(n=args.size, svd=args.svd, device=local, accum="tensor")

        def run_tensor():
            if batched:
                return sht.solve_arrays(mine, bs, xts, nzs, levels, out=xout)
            return sht.solve_many(mine, probs, args.workers)

        run_tensor()  # warm-up
        if dist:
            dist.barrier()
        check(L.kp_synchronize())
        check(L.kp_event_record(4))
        res_t = run_tensor()
        check(L.kp_event_record(5))
        mst = C.c_float()
        check(L.kp_event_elapsed(4, 5, C.byref(mst)))
        el_t, solved_t = reduce_timing(mst.value / 1e3, float(len(res_t)), dist,
                                       device="cuda" if args.dist_backend == "nccl" else "cpu")
        all_t = gather_results(res_t, dist,
                               device="cuda" if (dist and args.dist_backend == "nccl") else None)
        tensor = {"value": solved_t / el_t, "unit": "solves/s",
                  "mean_iterations": float(np.mean([r["iterations"] for r in all_t])),
                  "note": "KP_ACCUM_TENSOR: tcgen05 kind::f16, fp32 accumulation (not bit-exact); " +
                          ("one batched solve per GPU" if batched else "per-image solves on streams"),
                  "results": [{k: r[k] for k in ("image", "lam", "iterations", "rel_err")}
                              for r in all_t[:6]]}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import paper_2311_15393_b200 as K
        threads = os.cpu_count() or 1
        try:
            ccfg = build_problem("C4", 0, args.size, device_apply=False)
            csr, csc = svd_pair(ccfg.term, "host")
            cpu = {"value": 1.0 / cpu_c4_image_sample(ccfg, csr, csc, K.PrecisionFormat.fp16(), threads),
                   "unit": "solves/s", "cores": threads, "kind": "port",
                   "sample": "one C4 image on the oracle: spectral data + discrepancy lambda, plus one PCG "
                             "iteration's normal_matvec + precond_solve scaled to the image's 100 iterations"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "solves/s", "cores": threads, "kind": "port", "sample": f"failed: {e}"}
    if rank == 0:
        its = [r["iterations"] for r in allres]
        metric = METRIC_C4 if sh.n == 1024 else METRIC_C4.replace("1024^2", f"{sh.n}^2")
        out = {"metric": metric, "value": solved / elapsed, "unit": "solves/s", "n_gpus": ws,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f64 + f16 (reference-exact)", "data": "synthetic (seeded blob images)",
               "config": c4_config(),
               "run_info": {"parallelism": f"images sharded over {ws} GPU(s), NCCL gather; " +
                                         ("one batched PCG state machine per GPU (kp_pcg_batch)" if batched
                                          else f"{args.workers} concurrent streams per GPU"),
                          "mean_iterations": float(np.mean(its)), "images_solved": len(allres),
                          "no_root": sum(r["no_root"] for r in allres),
                          "l2": "each step solves 64 distinct images (8 MB inputs and ~0.1 GB of solver "
                                "state per image), far more than the 126 MB L2; no flush needed"},
               "e2e": {"value": solved / e2e_elapsed, "unit": "solves/s",
                       "h2d_bytes_per_step": 64 * 2 * 8 * sh.n * sh.n,
                       "d2h_bytes_per_step": 64 * 8 * sh.n * sh.n,
                       "note": "the public API with pinned host buffers: b, x_true in, x out inside the timed "
                               "region" + ("" if res_elapsed is not None else
                                           "; value repeats it (no device-resident pass in this mode)")},
               "clocks": clk.summary(), "gpu_launches": int(launches), "roofline": roof,
               "problem_generation_s": {"host": t_gen_host, "device": t_gen_dev,
                                        "note": "untimed setup: this rank's images by the host "
                                                "generator vs kp_generate_test_problems (incl. copies "
                                                "back to the host)"},
               "cpu_baseline": cpu,
               "results": [{k: r[k] for k in ("image", "lam", "iterations", "rel_err")}
                           for r in allres[:6]],
               "tensor_mode": tensor}
        print(json.dumps(out), flush=True)
    for p_ in pinned:
        L.kp_host_free(p_)
    if dist:
        dist.destroy_process_group()
    return 0


def workload_config(cfg) -> dict:
    """The workload definition, identical in both arms (ours / reference)."""
    solver, _, maxit = cfg.solvers[0]
    lam = cfg.lambda_ if cfg.select == "fixed" else f"{cfg.select} ({cfg.lambda_:.6g})"
    return {"workload": f"{cfg.name}: n={cfg.n} r={len(cfg.problem.a.terms)} {solver.upper()}, fp16 "
                        f"Kronecker-SVD preconditioner (reference-exact rounding), "
                        f"lambda={lam}, tol={cfg.tol}, maxit {maxit}",
            "unknowns": cfg.n * cfg.n, "l2": l2_note(cfg)}


def l2_note(cfg) -> str:
    return ("GPU arm: working set (~4 GB) far larger than the 126 MB L2; no flush needed" if cfg.n >= 4096
            else "GPU arm: L2 flushed before every timed step (256 MB zero-fill), steps timed separately")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None,
                    help="C1..C5; default: C5 (PCG iterations/s at 4096^2) on one GPU, the C4 "
                         "batch (solves/s over 64 images, sharded) when launched with several ranks")
    ap.add_argument("--size", type=int, default=None, help="override image side n (quick runs)")
    ap.add_argument("--svd", default="auto", choices=["auto", "gpu", "host"],
                    help="setup SVD of the factors: host LAPACK dgesdd (the oracle's routine) or "
                         "the library's cuSOLVER SVD; auto = host on one GPU, device when several "
                         "ranks would contend for the host cores")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tensor", action="store_true", help="skip the tensor-mode secondary run")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense-operator roofline probe")
    ap.add_argument("--no-other-runs", action="store_true",
                    help="skip the config's other solver runs (C5: PCG fp64-precond, CGLS)")
    ap.add_argument("--operator", default="auto", choices=["auto", "dense", "banded"])
    ap.add_argument("--workers", type=int, default=6,
                    help="C4 --c4-mode streams: concurrent host threads / streams per GPU")
    ap.add_argument("--c4-mode", default="batch", choices=["batch", "streams"],
                    help="C4: one batched PCG state machine per GPU, or per-image solves on streams")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend for timing reduction / result gather")
    args = ap.parse_args()
    if args.config is None:
        args.config = "C4" if dist_env()[0] > 1 else "C5"
    if args.svd == "auto":
        args.svd = "host" if dist_env()[0] == 1 else "gpu"
    if args.impl == "reference":
        return run_reference(args)

    if args.config == "C4":
        return run_c4(args)

    ws, rank, local = dist_env()
    import torch
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    import paper_2311_15393_b200 as K
    from paper_2311_15393_b200._lib import check, lib, ptr
    from paper_2311_15393_b200._lib import kp_history, kp_solver_options
    L = lib()
    check(L.kp_init(local))

    t0 = time.time()
    cfg = build_problem(args.config, rank, args.size, device_apply=True)
    t_problem = time.time() - t0
    t1 = time.time()
    svd_r, svd_c = svd_pair(cfg.term, args.svd)
    t_svd = time.time() - t1
    fmt = K.PrecisionFormat.fp16()
    solver_name, _, maxit = cfg.solvers[0]  # C1-C3, C5: the config's preconditioned run
    lam_select = None
    if cfg.lambda_ is None:  # C3: GCV over the 64-point grid with m0 at lambda = 1 (cli.cpp:469-505)
        from paper_2311_15393_b200.configs import GCV_GRID
        m0 = K.build_preconditioner_from_svd(svd_r, svd_c, 1.0, fmt)
        choice, _ = K.gcv_grid(K.make_spectral_data(m0, cfg.problem.b), GCV_GRID)
        cfg.lambda_ = choice.lambda_
        lam_select = {"method": "gcv_grid", "grid_index": choice.grid_index, "lambda": choice.lambda_}
    m = K.build_preconditioner_from_svd(svd_r, svd_c, cfg.lambda_, fmt)
    solve_fn = L.kp_fpcg if solver_name == "fpcg" else L.kp_pcg
    cfg.problem.a.set_mode(args.operator)
    op = cfg.problem.a.handle()
    setup_s = time.time() - t0
    n = cfg.n
    nn = n * n

    # ---- device-resident inputs (value) ----
    def dalloc(count):
        p = C.c_void_p()
        check(L.kp_device_alloc(count * 8, C.byref(p)))
        return p

    def halloc(count):
        p = C.c_void_p()
        check(L.kp_host_alloc(count * 8, C.byref(p)))
        return p, np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=(count,))

    d_b, d_x, d_xt = dalloc(nn), dalloc(nn), dalloc(nn)
    check(L.kp_memcpy_h2d(d_b, ptr(cfg.problem.b), nn * 8))
    check(L.kp_memcpy_h2d(d_xt, ptr(cfg.problem.x_true), nn * 8))
    hp_b, h_b = halloc(nn)
    hp_x, h_x = halloc(nn)
    hp_xt, h_xt = halloc(nn)
    h_b[:] = cfg.problem.b
    h_xt[:] = cfg.problem.x_true

    cap = maxit + 1
    hist_bufs = [np.zeros(cap) for _ in range(4)]

    def solve(device: bool, mm=None):
        h = kp_history(capacity=cap, relative_error=ptr(hist_bufs[0]), residual_norm=ptr(hist_bufs[1]),
                       work_units=ptr(hist_bufs[2]), residual_cosines=ptr(hist_bufs[3]))
        o = kp_solver_options(lambda_=cfg.lambda_, max_iterations=maxit, rel_residual_tol=cfg.tol,
                              x_true=(d_xt.value if device else hp_xt.value),
                              device_pointers=int(device))
        if device:
            check(solve_fn(op, d_b, (mm or m).handle(), C.byref(o), d_x, C.byref(h)))
        else:
            check(solve_fn(op, hp_b, (mm or m).handle(), C.byref(o), hp_x, C.byref(h)))
        solve.msolves = h.msolve_count
        return h.iterations_used, float(hist_bufs[0][h.rows - 1]), h.abort_reason.decode()

    for _ in range(args.warmup):
        its_w, rel_w, ab_w = solve(True)

    def barrier():
        check(L.kp_synchronize())
        if dist:
            dist.barrier()

    # ---- timed region: device-resident (value); iterations replayed as CUDA graphs ----
    launches0 = L.kp_launch_count()
    barrier()
    iters = 0
    rel_last = None
    # n < 4096: the solve's working set is within a few L2 sizes, so L2 is
    # flushed (256 MB zero-fill on torch's stream, then a device sync) before
    # every step and each step is timed by its own event pair
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if cfg.n < 4096 else None
    with ClockSampler(local) as clk:
        ms_total = 0.0
        if flush is None:
            check(L.kp_event_record(0))
        for _ in range(args.steps):
            if flush is not None:
                flush.zero_()
                torch.cuda.synchronize()
                check(L.kp_event_record(0))
            it, rel_last, abort = solve(True)
            iters += it
            if flush is not None:
                check(L.kp_event_record(1))
                ms = C.c_float()
                check(L.kp_event_elapsed(0, 1, C.byref(ms)))
                ms_total += ms.value
        if flush is None:
            check(L.kp_event_record(1))
            ms = C.c_float()
            check(L.kp_event_elapsed(0, 1, C.byref(ms)))
            ms_total = ms.value
    barrier()
    launches = L.kp_launch_count() - launches0
    elapsed = ms_total / 1e3

    # ---- profiled pass: the same K solves with CUDA events around every launch
    # (per kernel class, on the library stream) for the roofline and shares ----
    check(L.kp_profile_reset())
    check(L.kp_profile_enable(1))
    check(L.kp_event_record(6))
    prof_iters = 0
    prof_msolves = 0  # M-solves that ran (history.msolve_count): 4 working GEMM launches each
    for _ in range(args.steps):
        it, _, _ = solve(True)
        prof_iters += it
        prof_msolves += solve.msolves
    # operator launches that did work: A^T b at setup + 2 applies per iteration
    # (an overshoot iteration's launches return at once and are not counted)
    prof_op_applies = args.steps + 2 * prof_iters
    check(L.kp_event_record(7))
    prof_ms = C.c_float()
    check(L.kp_event_elapsed(6, 7, C.byref(prof_ms)))
    prof = {}
    for cls, name in enumerate(["operator_gemm_f64", "precond_gemm_f16ref", "vector", "spectral"]):
        t = C.c_double()
        c = C.c_longlong()
        check(L.kp_profile_read(cls, C.byref(t), C.byref(c)))
        prof[name] = (t.value, c.value)
    check(L.kp_profile_enable(0))

    # ---- secondary: tcgen05 tensor-mode preconditioner (north-star variant) ----
    tensor = None
    if not args.no_tensor:
        mt = K.build_preconditioner_from_svd(svd_r, svd_c, cfg.lambda_, fmt, accum="tensor")
        solve(True, mt)
        barrier()
        check(L.kp_event_record(4))
        t_iters, t_rel = 0, None
        for _ in range(args.steps):
            it, t_rel, _ = solve(True, mt)
            t_iters += it
        check(L.kp_event_record(5))
        t_ms = C.c_float()
        check(L.kp_event_elapsed(4, 5, C.byref(t_ms)))
        # one profiled solve for the tcgen05 kernel's roofline (per-launch events)
        check(L.kp_profile_reset())
        check(L.kp_profile_enable(1))
        solve(True, mt)
        tt, tcnt = C.c_double(), C.c_longlong()
        check(L.kp_profile_read(1, C.byref(tt), C.byref(tcnt)))
        check(L.kp_profile_enable(0))
        t_launches = 4 * solve.msolves  # working tcgen05 launches (no-op ones excluded)
        tc_ach = 2.0 * float(n) ** 3 / (tt.value / t_launches / 1e3) / 1e12 if t_launches else 0.0
        pk = peaks()
        tensor = {"value": t_iters / (t_ms.value / 1e3), "unit": "iterations/s",
                  "solves_per_s": args.steps / (t_ms.value / 1e3),
                  "iterations_per_solve": t_iters // args.steps, "final_rel_err": t_rel,
                  "note": "KP_ACCUM_TENSOR: tcgen05 kind::f16, fp32 accumulation (not bit-exact)",
                  "roofline": {"bound": "tensor", "achieved": tc_ach, "peak": pk["bf16_tflops_sustained"],
                               "unit": "TFLOP/s", "frac": tc_ach / pk["bf16_tflops_sustained"],
                               "frac_of_burst": tc_ach / pk["bf16_tflops"],
                               "kernel": "gemm_f16tc_kernel (tcgen05 kind::f16, 4 per M-solve)",
                               "peak_source": f"{pk['source']}: bf16_tflops_sustained (in-step kernel); "
                                              "frac_of_burst against bf16_tflops",
                               "work_per_launch": f"{2.0 * float(n) ** 3:.4g} flop",
                               "traffic": TRAFFIC.get(("gemm_f16tc_kernel", n))}}

    # ---- the config's other runs (C5: PCG with the FP64 preconditioner, CGLS),
    # one device-resident solve each, for the record ----
    other_runs = {}
    if not args.no_other_runs:
        for solver_o, fmt_o, maxit_o in cfg.solvers[1:]:
            hb = [np.zeros(maxit_o + 1) for _ in range(4)]  # kept alive for the call
            rel_o = hb[0]
            ho = kp_history(capacity=maxit_o + 1, relative_error=ptr(hb[0]), residual_norm=ptr(hb[1]),
                            work_units=ptr(hb[2]), residual_cosines=ptr(hb[3]))
            oo = kp_solver_options(lambda_=cfg.lambda_, max_iterations=maxit_o,
                                   rel_residual_tol=cfg.tol, x_true=d_xt.value, device_pointers=1)
            mo = None
            if solver_o != "cgls":
                fmt_obj = K.PrecisionFormat.fp64() if fmt_o == "fp64" else fmt
                mo = K.build_preconditioner_from_svd(svd_r, svd_c, cfg.lambda_, fmt_obj)
            barrier()
            check(L.kp_event_record(8))
            if solver_o == "cgls":
                check(L.kp_cgls(op, d_b, C.byref(oo), d_x, C.byref(ho)))
            else:
                fn = L.kp_fpcg if solver_o == "fpcg" else L.kp_pcg
                check(fn(op, d_b, mo.handle(), C.byref(oo), d_x, C.byref(ho)))
            check(L.kp_event_record(9))
            o_ms = C.c_float()
            check(L.kp_event_elapsed(8, 9, C.byref(o_ms)))
            other_runs[f"{solver_o}_{fmt_o or 'none'}"] = {
                "iterations_per_s": ho.iterations_used / (o_ms.value / 1e3),
                "iterations": ho.iterations_used, "converged": bool(ho.converged),
                "final_rel_err": float(rel_o[ho.rows - 1]), "ms": o_ms.value,
                "abort_reason": ho.abort_reason.decode()}

    # ---- e2e: the same solves through host (pinned) buffers ----
    for _ in range(max(1, args.warmup)):  # warm the host-path staging buffers too
        solve(False)
    barrier()
    check(L.kp_event_record(2))
    e2e_iters = 0
    for _ in range(args.steps):
        it, _, _ = solve(False)
        e2e_iters += it
    check(L.kp_event_record(3))
    e2e_ms = C.c_float()
    check(L.kp_event_elapsed(2, 3, C.byref(e2e_ms)))
    barrier()
    e2e_elapsed = e2e_ms.value / 1e3

    if dist:  # max time over ranks, summed work; per-image results gathered to all
        from paper_2311_15393_b200.batch import gather_results, reduce_timing
        dev = "cuda" if args.dist_backend == "nccl" else "cpu"
        elapsed, iters = reduce_timing(elapsed, float(iters), dist, device=dev)
        e2e_elapsed, e2e_iters = reduce_timing(e2e_elapsed, float(e2e_iters), dist, device=dev)
        iters, e2e_iters = int(iters), int(e2e_iters)
        per_rank = gather_results([{"image": rank, "rel_err": rel_last}], dist, device=dev,
                                  fields=("image", "rel_err"))

    if not dist:
        per_rank = None
    value = iters / elapsed
    e2e_value = e2e_iters / e2e_elapsed
    r = len(cfg.problem.a.terms)
    op_mode, tc, tr = cfg.problem.a.mode()
    op_ms, _ = prof["operator_gemm_f64"]
    op_launches = 2 * prof_op_applies  # two launches (passes / GEMMs) per apply
    if op_mode == "banded_fused":  # passes A + B in one launch per apply: 2 r (Lc + Lr) n^2 flop
        op_launches = prof_op_applies
        op_flops_per_launch = 2.0 * r * (tc + tr) * float(n) ** 2
        op_peak, op_kernel = DFMA_PEAK_TFLOPS, "band_fused (FP64 DFMA, banded Toeplitz, both passes)"
        op_src = "measured DFMA peak, profiles/r01_microbench_peaks.txt"
    elif op_mode == "banded":  # two correlation passes per apply: 2 r (Lc + Lr) n^2 flop
        op_flops_per_launch = 2.0 * r * (tc + tr) * float(n) ** 2 / 2.0
        op_peak, op_kernel = DFMA_PEAK_TFLOPS, "band_cols/band_rows (FP64 DFMA, banded Toeplitz)"
        op_src = "measured DFMA peak, profiles/r01_microbench_peaks.txt"
    else:  # each of the two GEMMs of an apply
        op_flops_per_launch = 2.0 * r * float(n) ** 3
        op_peak, op_kernel = DMMA_PEAK_TFLOPS, "gemm_f64_tma_kernel (DMMA m16n8k16, TMA-staged 128x128 tiles)"
        op_src = "measured DMMA f64 peak, profiles/r01_microbench_peaks.txt"
    op_ach = op_flops_per_launch / (op_ms / op_launches / 1e3) / 1e12 if op_launches else 0.0
    pm_ms, _ = prof["precond_gemm_f16ref"]
    pm_launches = 4 * prof_msolves  # working launches only (a converged solve's last M-solve is a no-op)
    half_ops = 2.0 * float(n) ** 3  # n^3 rounded products + n^3 rounded tree adds per GEMM
    pm_ach = half_ops / (pm_ms / pm_launches / 1e3) / 1e12 if pm_launches else 0.0
    engine = K.fp16_products_engine(n)
    total_prof = sum(v[0] for v in prof.values())
    op_line = {"bound": "tensor" if op_mode == "dense" else "compute",
               "pipe": "DMMA" if op_mode == "dense" else "FP64 DFMA", "achieved": op_ach,
               "peak": op_peak, "unit": "TFLOP/s", "frac": op_ach / op_peak,
               "traffic": TRAFFIC.get(("band", n)) if op_mode == "banded" else None,
               "kernel": op_kernel, "peak_source": op_src,
               "work_per_launch": f"{op_flops_per_launch:.4g} flop"}
    if engine == "tensor":
        # gemm_f16x: the n^3 rounded products come from tcgen05 MMAs, the n^3
        # rounded tree adds (HADD2) saturate the f16x2 pipe, so the 2 n^3
        # binary16 ops of a launch complete at most at 2 x the f16x2 rate
        pm_peak = 2.0 * F16X2_PEAK_TOPS
        pm_line = {"bound": "compute", "pipe": "f16x2 CUDA-core pipe (rounded tree adds, HADD2); the rounded "
                                              "products come from the tcgen05 tensor pipe",
                   "achieved": pm_ach, "peak": pm_peak, "unit": "T half-ops/s", "frac": pm_ach / pm_peak,
                   "traffic": TRAFFIC.get(("gemm_f16x_kernel", n)), "kernel": "gemm_f16x_kernel",
                   "peak_source": "2 x measured f16x2 add rate (profiles/r01_microbench_peaks.txt): "
                                  "n^3 adds on the f16x2 pipe bound the 2 n^3 ops",
                   "work_per_launch": f"{half_ops:.4g} half-ops", "launches": pm_launches,
                   "ms_per_launch": pm_ms / pm_launches if pm_launches else None}
        # the tensor-pipe view: every rounded leaf is one column of a K = 16
        # kind::f16 MMA (16 MACs), so the MMAs issue 32 n^3 flop per launch
        pk = peaks()
        exp_tf = 32.0 * float(n) ** 3 / (pm_ms / pm_launches / 1e3) / 1e12 if pm_launches else 0.0
        pm_line["tensor_pipe"] = {
            "issued_mma_tflops": exp_tf, "frac_of_bf16_burst": exp_tf / pk["bf16_tflops"],
            "frac_of_bf16_sustained": exp_tf / pk["bf16_tflops_sustained"],
            "useful_frac_of_bf16_burst": pm_ach / pk["bf16_tflops"],
            "note": "the MMAs form the n^3 rounded products (one live k per B column); the n^3 rounded "
                    "tree adds cannot run on the tensor pipe (fp32 accumulation has no per-add "
                    "binary16 rounding), so the f16x2 add rate is the ceiling (ncu: tensor pipe 34 % "
                    "busy, profiles/r02_ncu_f16x.txt)"}
    else:
        pm_line = {"bound": "compute", "pipe": "f16x2 CUDA-core FMA pipe (reference-exact rounding "
                                              "needs a binary16 rounding per product and per sum)",
                   "achieved": pm_ach,
                   "peak": F16X2_PEAK_TOPS, "unit": "T half-ops/s", "frac": pm_ach / F16X2_PEAK_TOPS,
                   "traffic": TRAFFIC.get(("gemm_f16ref_kernel", n)), "kernel": "gemm_f16ref_kernel",
                   "peak_source": "measured f16x2 mul+add rate, profiles/r01_microbench_peaks.txt",
                   "work_per_launch": f"{half_ops:.4g} half-ops", "launches": pm_launches,
                   "ms_per_launch": pm_ms / pm_launches if pm_launches else None}
    dominant, other = (pm_line, op_line) if pm_ms > op_ms else (op_line, pm_line)

    # the HBM-bound vector kernels (north star: "achieved HBM GB/s for the vector
    # kernels"): algorithmic bytes of the class per iteration and per solve over
    # the class's device time in the profiled pass
    vec_line = None
    vec_ms, vec_launches = prof["vector"]
    if solver_name in ("pcg", "fpcg") and vec_ms > 0:
        flex = solver_name == "fpcg"
        upd = (7 + (1 if flex else 0)) * 8 + 2     # pcg_update: x, r, p, q, x_true in; x, r (, r_prev), r16 out
        fin = (2 + 8 + 8 + (8 if flex else 0)) if engine == "tensor" else 0  # msolve_finish_f16: z16, r (, r_prev) in; z out
        pup = 24                                     # p = z + beta p
        init = 8 + 8 + 10 + 16                       # x = 0, x_true.x_true, r -> r16, p = z
        vbytes = float(nn) * (prof_iters * (upd + fin + pup) + args.steps * init)
        pk = peaks()
        v_ach = vbytes / (vec_ms / 1e3) / 1e9
        vec_line = {"bound": "hbm", "achieved": v_ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": v_ach / pk["hbm_gbs"], "kernel": "pcg_update / pcg_p_update / msolve_finish_f16 "
                    "(+ per-solve zero / dot / cast / copy)", "peak_source": pk["source"] + ": hbm_gbs",
                    "bytes_per_iteration": float(nn) * (upd + fin + pup), "launches": vec_launches,
                    "note": "algorithmic bytes (every vector read or written once per kernel); below "
                            "n = 4096 the vectors fit the 126 MB L2 and the figure is not an HBM rate"}

    # the dense DMMA operator (the product the reference computes), for its roofline
    dense = None
    if op_mode.startswith("banded") and not args.no_dense:
        cfg.problem.a.set_mode("dense")
        check(L.kp_profile_reset())
        check(L.kp_profile_enable(1))
        xin = np.ascontiguousarray(cfg.problem.x_true)
        for _ in range(2):
            K.kronsum_apply(cfg.problem.a, xin)
        t_ = C.c_double()
        c_ = C.c_longlong()
        check(L.kp_profile_read(0, C.byref(t_), C.byref(c_)))
        check(L.kp_profile_enable(0))
        cfg.problem.a.set_mode("auto")
        d_ach = 2.0 * r * float(n) ** 3 / (t_.value / c_.value / 1e3) / 1e12
        dense = {"bound": "tensor", "achieved": d_ach, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                 "frac": d_ach / DMMA_PEAK_TFLOPS, "kernel": "gemm_f64_tma_kernel (DMMA m16n8k16, TMA-staged 128x128 tiles)",
                 "ms_per_launch": t_.value / c_.value, "launches": c_.value}

    out = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            try:
                t_cpu = cpu_iteration_sample(cfg, svd_r, svd_c, fmt, threads)
                cpu = {"value": 1.0 / t_cpu, "unit": "iterations/s", "cores": threads, "kind": "port",
                       "sample": f"one {solver_name.upper()} iteration's normal_matvec + "
                                 f"precond_solve at {cfg.name} (oracle: OpenBLAS FP64 + "
                                 "streamed reference-exact fp16)"}
            except Exception as e:  # noqa: BLE001
                cpu = {"value": None, "unit": "iterations/s", "cores": threads, "kind": "port",
                       "sample": f"failed: {e}"}
            try:
                cpu["single_thread"] = cpu_iteration_single_thread(cfg, fmt)
            except Exception as e:  # noqa: BLE001
                cpu["single_thread"] = {"value": None, "sample": f"failed: {e}"}
        out = {
            "metric": metric_name(cfg),
            "value": value, "unit": "iterations/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 (operator, vectors) + f16 (preconditioner, reference-exact)",
            "data": f"synthetic (seeded blob images, BASELINE {cfg.name} PSF)",
            "config": workload_config(cfg),
            "run_info": {"l2": l2_note(cfg), "parallelism": f"replicas x{ws}",
                         "per_rank_final_rel_err": ([d["rel_err"] for d in per_rank] if dist else None),
                         "iterations_per_solve": iters // max(1, args.steps * ws),
                         "lambda": cfg.lambda_, "lambda_selection": lam_select,
                         "final_rel_err": rel_last,
                         "fp16_products_engine": engine}, 
            "e2e": {"value": e2e_value, "unit": "iterations/s", "h2d_bytes_per_step": 2 * nn * 8,
                    "d2h_bytes_per_step": nn * 8 + 4 * cap * 8},
            "roofline": dominant,
            "roofline_other": other,
            "roofline_vector": vec_line,
            "roofline_dense_operator_gemm": dense,
            "operator_mode": {"mode": op_mode, "col_taps": tc, "row_taps": tr},
            "kernels": {k: {"ms": v[0], "launches": v[1],
                            "share": v[0] / total_prof if total_prof else None}
                        for k, v in prof.items()},
            "profiled_pass": {"value": prof_iters / (prof_ms.value / 1e3), "unit": "iterations/s",
                              "note": "same solves with per-launch CUDA events and no graph "
                                      "replay; source of roofline and kernel shares"},
            "solves_per_s": args.steps * ws / elapsed,
            "tensor_mode": tensor,
            "other_runs": other_runs,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "setup_s": {"total": setup_s, "problem": t_problem, "svd": t_svd, "svd_backend": args.svd},
        }
        print(json.dumps(out), flush=True)
    for p in (d_b, d_x, d_xt):
        L.kp_device_free(p)
    for p in (hp_b, hp_x, hp_xt):
        L.kp_host_free(p)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
