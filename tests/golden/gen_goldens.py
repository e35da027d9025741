"""Generate the config goldens with the CPU oracle (test infrastructure).

The reference cannot be built here (Eigen absent), so the goldens for the
BASELINE configs come from the oracle restatement, run on the
same seeded inputs the device tests build (paper_2311_15393_b200.configs).
Full sizes where the oracle finishes in minutes; C5 (n=4096) as a prefix of
iterations. Output: tests/golden/<config>.json (histories, iteration counts,
lambda choices, solution checksums). Usage:

    python tests/golden/gen_goldens.py C1 C2 C3 C4 C5 [C5fpcg] [--threads 8]

C4 covers all 64 images of the batch and resumes from the images already in
C4.json (it checkpoints after every image).

C5fpcg writes C5_fpcg_full.json: the headline FPCG run to its end;
C5cgls writes C5_cgls_full.json: the CGLS run to convergence;
C5pcg64 writes C5_pcg64_full.json: PCG with the FP64 preconditioner.
C5cglsiter writes C5_cgls_iterates.json: the first 5 CGLS iterates at n=4096
  as norms + projections on 4 seeded vectors (the iterates themselves are
  134 MB each).
M4096 / M1664 write msolve_n<n>.json: bitwise digests of precond_solve on the
  seeded binary16-exact factors of tests/golden/msolve_inputs.py.
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import pyoracle as O  # noqa: E402
from paper_2311_15393_b200 import configs  # noqa: E402
from paper_2311_15393_b200 import PrecisionFormat as PF  # noqa: E402
from paper_2311_15393_b200.kronprec import SolverOptions  # noqa: E402

FMT = {"fp16": PF.fp16(), "fp64": PF.fp64()}


def hist_dict(x, h):
    return {"iterations_used": h.iterations_used, "converged": h.converged,
            "abort_reason": h.abort_reason, "msolve_count": h.msolve_count,
            "residual_norm": h.residual_norm, "relative_error": h.relative_error,
            "x_sum": float(np.sum(x)), "x_norm": float(np.linalg.norm(x))}


def run_solver(cfg, solver, fmt, maxit, lam, m0):
    opts = SolverOptions(lambda_=lam, max_iterations=maxit, rel_residual_tol=cfg.tol,
                         x_true=cfg.problem.x_true)
    t0 = time.time()
    if solver == "cgls":
        x, h = O.cgls(cfg.problem.a, cfg.problem.b, opts)
    else:
        m = O.with_lambda(m0[fmt], lam)
        x, h = getattr(O, solver)(cfg.problem.a, cfg.problem.b, m, opts)
    d = hist_dict(x, h)
    d.update(solver=solver, fmt=fmt, max_iterations=maxit, seconds=time.time() - t0)
    return d


def gen(name: str, prefix: int | None = None, images=(0,), only=None, tag=None, resume=False):
    out = {"config": name, "generator": "oracle/kp_oracle.cpp via tests/golden/gen_goldens.py",
           "images": []}
    path = os.path.join(HERE, f"{tag or name}.json")
    done = {}
    if resume and os.path.exists(path):  # keep images already generated
        with open(path) as f:
            done = {rec["image"]: rec for rec in json.load(f)["images"]}
    for img in images:
        if img in done:
            out["images"].append(done[img])
            continue
        cfg = configs.build(name, image=img)
        m0 = {}
        fmts = {f for _, f, _ in cfg.solvers if f}
        for f in fmts:  # build_preconditioner at lambda = 1 (cli.cpp:192-198)
            m0[f] = O.build_preconditioner(cfg.term.row_factor, cfg.term.col_factor, 1.0, FMT[f])
        rec = {"image": img, "n": cfg.n, "rank": len(cfg.problem.a.terms),
               "noise_level": cfg.problem.noise_level,
               "noise_norm": float(np.linalg.norm(cfg.problem.noise)),
               "b_norm": float(np.linalg.norm(cfg.problem.b)), "select": cfg.select}
        lam = cfg.lambda_
        if cfg.select != "fixed":
            s, bh = O.spectral(m0["fp16"], cfg.problem.b)
            if cfg.select == "gcv_grid":
                c, vals = O.gcv_grid(s, bh, configs.GCV_GRID)
                rec["gcv_index"] = c["grid_index"]
                rec["gcv_values"] = list(map(float, vals))
            else:
                c = O.discrepancy(s, bh, float(np.linalg.norm(cfg.problem.noise)), cfg.eta)
            lam = c["lambda"]
        rec["lambda"] = lam
        rec["runs"] = []
        for solver, fmt, maxit in cfg.solvers:
            if only and solver != only:
                continue
            mi = min(maxit, prefix) if prefix else maxit
            rec["runs"].append(run_solver(cfg, solver, fmt, mi, lam, m0))
            print(name, img, solver, fmt, rec["runs"][-1]["iterations_used"],
                  f"{rec['runs'][-1]['seconds']:.1f}s", flush=True)
        out["images"].append(rec)
        if resume:  # checkpoint after every image (the 64-image C4 run takes hours)
            with open(path, "w") as f:
                json.dump(out, f, indent=1)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, flush=True)


def projection_vectors(nn: int, count: int = 4):
    """Seeded probe vectors for iterate fingerprints (shared with the tests)."""
    return [np.random.default_rng(9000 + j).standard_normal(nn) for j in range(count)]


def gen_cgls_iterates(iters: int = 5):
    cfg = configs.build("C5")
    opts = SolverOptions(lambda_=cfg.lambda_, max_iterations=iters, rel_residual_tol=cfg.tol,
                         x_true=cfg.problem.x_true, record_iterates=True)
    t0 = time.time()
    _, h = O.cgls(cfg.problem.a, cfg.problem.b, opts)
    w = projection_vectors(cfg.n * cfg.n)
    rows = [{"norm": float(np.linalg.norm(x)), "proj": [float(x @ v) for v in w]} for x in h.iterates]
    out = {"config": "C5", "solver": "cgls", "iterations": iters, "lambda": cfg.lambda_,
           "probe_seeds": [9000 + j for j in range(len(w))], "probe_norms": [float(np.linalg.norm(v)) for v in w],
           "iterates": rows, "residual_norm": h.residual_norm, "relative_error": h.relative_error,
           "seconds": time.time() - t0,
           "generator": "oracle/kp_oracle.cpp via tests/golden/gen_goldens.py C5cglsiter"}
    path = os.path.join(HERE, "C5_cgls_iterates.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, f"{out['seconds']:.1f}s", flush=True)


def gen_msolve(n: int, seed: int = 4242):
    sys.path.insert(0, HERE)
    from msolve_inputs import digest, msolve_case
    out = {"n": n, "seed": seed, "cases": {},
           "generator": f"oracle/kp_oracle.cpp via tests/golden/gen_goldens.py M{n}"}
    for regime in ("wide", "low"):
        sr, sc, lam, r = msolve_case(n, seed, regime)
        t0 = time.time()
        m = O.build_preconditioner_from_svd(sr, sc, lam, FMT["fp16"])
        z = O.precond_solve(m, r)
        out["cases"][regime] = {"lambda": lam, "digest": digest(z), "seconds": time.time() - t0}
        print(n, regime, out["cases"][regime], flush=True)
    path = os.path.join(HERE, f"msolve_n{n}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, flush=True)


if __name__ == "__main__":
    threads = 8
    args = [a for a in sys.argv[1:]]
    if "--threads" in args:
        i = args.index("--threads")
        threads = int(args[i + 1])
        del args[i:i + 2]
    O.set_threads(threads)
    for name in args:
        if name == "C4":  # all 64 images of the batch (resumable; ~110 s per image on 8 threads)
            gen("C4", images=tuple(range(64)), resume=True)
        elif name == "C5":
            gen("C5", prefix=3)
        elif name == "C5fpcg":  # the headline run in full (about 45 min on 8 threads)
            gen("C5", only="fpcg", tag="C5_fpcg_full")
        elif name == "C5cgls":  # CGLS to convergence (about 45 min on 8 threads)
            gen("C5", only="cgls", tag="C5_cgls_full")
        elif name == "C5cglsiter":
            gen_cgls_iterates()
        elif name.startswith("M") and name[1:].isdigit():
            gen_msolve(int(name[1:]))
        elif name == "C5pcg64":  # PCG with the FP64 preconditioner to convergence
            gen("C5", only="pcg", tag="C5_pcg64_full")
        else:
            gen(name)
