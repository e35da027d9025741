"""Batches of independent solves sharded across GPUs (BASELINE config C4).

A single solve does not shard; batches of independent images
do. Each rank takes a contiguous block of image indices, runs the full
reference pipeline per image on its own GPU — spectral data, discrepancy-
principle lambda (regparam.cpp:288-327, eta = 1.01), with_lambda, PCG with the
fp16 preconditioner — and the per-image results are gathered with one
collective (NCCL on GPUs, gloo in the CPU tests). No data-path collective.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass


def shard(num_items: int, world: int, rank: int) -> range:
    """Contiguous, balanced block of item indices for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard: bad world/rank")
    base, extra = divmod(num_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass
class ImageResult:
    image: int
    noise_level: float
    lam: float
    iterations: int
    converged: bool
    rel_err: float
    abort_reason: str = ""
    no_root: bool = False
    msolve_count: int = 0  # M-solves that ran (history.msolve_count)


RESULT_FIELDS = ("image", "noise_level", "lam", "iterations", "converged", "rel_err", "no_root")
_INT_FIELDS = {"image", "iterations"}
_BOOL_FIELDS = {"converged", "no_root"}


def gather_results(local: list, dist=None, device=None, fields=RESULT_FIELDS) -> list:
    """All ranks' results, sorted by image. The numeric fields travel as one
    float64 tensor per rank (dist.all_gather: ncclAllGather on the NCCL
    backend, `device` = "cuda"); abort-reason strings, when any rank has one,
    follow in a small object gather."""
    items = [asdict(r) if isinstance(r, ImageResult) else dict(r) for r in local]
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return sorted(items, key=lambda d: d["image"])
    import torch
    world = dist.get_world_size()
    cnt = torch.tensor([len(items)], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt)
    counts = [int(c.item()) for c in counts]
    rows = max(1, max(counts))
    buf = torch.full((rows, len(fields)), float("nan"), dtype=torch.float64)
    for i, d in enumerate(items):
        buf[i] = torch.tensor([float(d[f]) for f in fields], dtype=torch.float64)
    buf = buf.to(device) if device else buf
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    has_reason = torch.tensor([int(any(d.get("abort_reason") for d in items))], device=device)
    dist.all_reduce(has_reason, op=dist.ReduceOp.MAX)
    reasons = {}
    if has_reason.item():
        objs = [None] * world
        dist.all_gather_object(objs, {d["image"]: d["abort_reason"] for d in items
                                      if d.get("abort_reason")})
        for o in objs:
            reasons.update(o)
    out = []
    for r, b in enumerate(bufs):
        for row in b[:counts[r]].cpu().tolist():
            d = {}
            for f, v in zip(fields, row):
                d[f] = int(v) if f in _INT_FIELDS else bool(v) if f in _BOOL_FIELDS else v
            if "image" in d and "abort_reason" in ImageResult.__dataclass_fields__ and \
                    fields is RESULT_FIELDS:
                d["abort_reason"] = reasons.get(d["image"], "")
            out.append(d)
    return sorted(out, key=lambda d: d["image"])


def reduce_timing(elapsed_s: float, units: float, dist=None, device=None) -> tuple[float, float]:
    """(max elapsed over ranks, sum of units over ranks) — the whole-job
    throughput is units / elapsed."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return elapsed_s, units
    import torch
    t = torch.tensor([elapsed_s], dtype=torch.float64, device=device)
    u = torch.tensor([units], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


class C4Shard:
    """Shared operator / preconditioner factors for the C4 batch on one GPU
    (all 64 images share the PSF, hence A and the Kronecker factors).

    accum="tensor" builds the tcgen05 tensor-mode preconditioner (not
    bit-exact; the bench's secondary C4 run). solve_many() runs `workers`
    host threads; each has its own library
    context (stream) and its own operator handle, so independent images
    overlap on the device (the kernels of one image at n = 1024 do not fill
    the 148 SMs on their own)."""

    def __init__(self, n: int | None = None, svd: str = "host", device: int = 0,
                 accum: str = "reference"):
        import numpy as np

        from . import configs
        from . import kronprec as K
        from . import problems as P
        from .kronprec import SvdTriple

        self.K, self.P, self.np = K, P, np
        self.device = device
        base = configs.build("C4", image=0, n=n)
        self.n = base.n
        self.a = base.problem.a
        self.psf = base.problem.psf
        self.eta = base.eta
        self.tol = base.tol
        if svd == "gpu":  # the library's device SVD (cuSOLVER, svd_dev.cu)
            pair = [SvdTriple(*K.svd(f, "device")) for f in (base.term.row_factor, base.term.col_factor)]
            self.m0 = K.build_preconditioner_from_svd(pair[0], pair[1], 1.0, K.PrecisionFormat.fp16(),
                                                      accum=accum)
        else:
            self.m0 = K.build_preconditioner(base.term.row_factor, base.term.col_factor, 1.0,
                                             K.PrecisionFormat.fp16(), accum=accum)

    def problem(self, image: int):
        P, np = self.P, self.np
        noise = [0.001, 0.01, 0.05][image % 3]
        return P.make_test_problem(P.blob_image(self.n, 4000 + image), self.psf, noise, 5000 + image,
                                   a=self.a)

    def solve_many(self, images, probs: dict, workers: int = 1) -> list:
        """Solve `images` (problems in `probs`) on `workers` concurrent streams."""
        import threading

        from ._lib import check, lib
        images = list(images)
        workers = max(1, min(workers, len(images)))
        if workers == 1:
            return [self.solve(i, probs[i]) for i in images]
        out, errors = {}, []

        def run(w):
            try:
                check(lib().kp_init(self.device))  # this thread's context and stream
                a = self.K.KroneckerSum(list(self.a.terms), self.a.n)  # own operator handle
                for i in images[w::workers]:
                    out[i] = self.solve(i, probs[i], a=a)
            except Exception as e:  # noqa: BLE001
                errors.append(e)

        threads = [threading.Thread(target=run, args=(w,)) for w in range(workers)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return [out[i] for i in images]

    def stack(self, images, probs: dict, alloc=None):
        """(b, x_true) of `images` as two contiguous batch x n^2 arrays and the
        noise norms; `alloc(shape)` provides the arrays (e.g. pinned host
        memory), numpy by default."""
        np = self.np
        images = list(images)
        nn = self.n * self.n
        alloc = alloc or (lambda shape: np.empty(shape))
        bs, xts = alloc((len(images), nn)), alloc((len(images), nn))
        for q, i in enumerate(images):
            bs[q] = probs[i].b
            xts[q] = probs[i].x_true
        return bs, xts, [float(np.linalg.norm(probs[i].noise)) for i in images]

    def select_lambdas_arrays(self, bs, noise_norms) -> list:
        """Discrepancy-principle lambda per row of bs (regparam.cpp:288-327),
        all images' bisections advancing together (kp_discrepancy_batch; equal
        to discrepancy() per image); None when the bracket has no root."""
        lam, st = self.K.discrepancy_batch(self.m0, bs, noise_norms, self.eta)
        return [float(v) if c == 0 else None for v, c in zip(lam, st)]

    def select_lambdas(self, images, probs: dict) -> dict:
        images = list(images)
        bs, _, nz = self.stack(images, probs)
        return dict(zip(images, self.select_lambdas_arrays(bs, nz)))

    def solve_arrays(self, images, bs, xts, noise_norms, noise_levels, lams=None, out=None) -> list:
        """The images' PCG solves (rows of bs / xts) as ONE batched device
        solve (kp_pcg_batch: images stacked along the M-solve GEMMs' N
        dimension, one DevState per image); lambdas by the discrepancy
        principle unless given. Image by image the result equals solve()."""
        K, np = self.K, self.np
        images = list(images)
        lams = lams if lams is not None else self.select_lambdas_arrays(bs, noise_norms)
        ok = [q for q in range(len(images)) if lams[q] is not None]
        res = {}
        if ok:
            opts = K.SolverOptions(max_iterations=100, rel_residual_tol=self.tol)
            full = len(ok) == len(images)
            sub = (lambda a: a) if full else (lambda a: np.ascontiguousarray(a[ok]))
            rr = K.pcg_batch(self.a, sub(bs), self.m0, [lams[q] for q in ok], opts, x_true=sub(xts),
                             out=out if full else None)
            res = dict(zip(ok, rr))
        outl = []
        for q, i in enumerate(images):
            if q not in res:
                outl.append(ImageResult(i, noise_levels[q], float("nan"), 0, False, float("nan"), "", True))
                continue
            h = res[q].history
            outl.append(ImageResult(i, noise_levels[q], lams[q], h.iterations_used, h.converged,
                                    h.relative_error[-1], h.abort_reason, msolve_count=h.msolve_count))
        return outl

    def solve_batch(self, images, probs: dict, lams: dict | None = None) -> list:
        images = list(images)
        bs, xts, nz = self.stack(images, probs)
        return self.solve_arrays(images, bs, xts, nz, [probs[i].noise_level for i in images],
                                 None if lams is None else [lams[i] for i in images])

    def solve(self, image: int, tp=None, a=None) -> ImageResult:
        K, np = self.K, self.np
        tp = tp or self.problem(image)
        a = a if a is not None else self.a
        sd = K.make_spectral_data(self.m0, tp.b)
        try:
            lam = K.discrepancy(sd, float(np.linalg.norm(tp.noise)), self.eta).lambda_
        except K.NoRootError:
            return ImageResult(image, tp.noise_level, float("nan"), 0, False, float("nan"),
                               "", True)
        m = K.with_lambda(self.m0, lam)
        r = K.pcg(a, tp.b, m, K.SolverOptions(lambda_=lam, max_iterations=100,
                                                   rel_residual_tol=self.tol, x_true=tp.x_true))
        h = r.history
        return ImageResult(image, tp.noise_level, lam, h.iterations_used, h.converged,
                           h.relative_error[-1], h.abort_reason)
