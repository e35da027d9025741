"""Reference-compatible experiment verbs over the B200 solve path
(proj/src/cli.cpp:532-780, proj/include/kronprec/cli.hpp).

    python -m paper_2311_15393_b200 {generate,decompose,solve,compare,sweep}
        [--config FILE] [--blur ..] [--n ..] [--noise ..] ... [--include-fpcg]

Same config keys, defaults, validation messages, output files and schemas as
the reference CLI (kronprec.summary/1, kronprec.convergence/1,
kronprec.work_report/1, kronprec.comparison/1, kronprec.sweep/1,
kronprec.decompose/1, the kronprec.problem/1 bundle of `generate`) and the
same exit codes (2 config error, 3 io error, 4 other). The problem setup
(PSF, test image, noise) is the host code of problems.py; every solve,
preconditioner solve and lambda search runs on the device through the C ABI.
`decompose` (the Table-1 Frobenius report, kron.cpp:90-139) is host numpy:
it is a report, not part of the solve path.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from dataclasses import dataclass, field

import numpy as np

from . import kronprec as K
from . import problems as P


class ConfigError(Exception):
    pass


class IoError(Exception):
    pass


@dataclass
class ExperimentConfig:  # cli.hpp:34-62
    blur: str = "gaussian"
    n: int = 32
    noise: float = 0.01
    seed: int = 1
    psf_size: int = 9
    psf_seed: int = 0
    psf_sigma: float = 2.0
    psf_radius: float = 3.0
    psf_length: int = 5
    psf_steps: int = 64
    psf_blob_count: int = 10
    psf_blob_sigma: float = 1.0
    fmt: str = "fp16"
    solver: str = "pcg"
    param: str = "opt"
    omega: float = 1.0
    eta: float = 1.0
    lambda_: float = 0.0
    precond_lambda: float | None = None
    maxit: int = 50
    tol: float = 1e-8
    out: str = "out"
    include_fpcg: bool = False
    sweep_key: str = ""
    sweep_values: list = field(default_factory=list)


def _bad(key, value, want):
    raise ConfigError(f'config key {key}: cannot parse "{value}" as {want}')


def _double(key, value):  # cli.cpp:40-48
    t = value.strip()
    try:
        v = float(t)
    except ValueError:
        _bad(key, value, "a number")
    if not math.isfinite(v):
        _bad(key, value, "a finite number")
    return v


def _int(key, value):
    t = value.strip()
    try:
        v = int(t, 10)
    except ValueError:
        _bad(key, value, "an integer")
    if not -2**31 <= v < 2**31:
        _bad(key, value, "an integer in range")
    return v


def _u64(key, value):
    t = value.strip()
    if not t or t.startswith("-"):
        _bad(key, value, "a nonnegative integer")
    try:
        return int(t, 10)
    except ValueError:
        _bad(key, value, "a nonnegative integer")


def _bool(key, value):
    t = value.strip()
    if t in ("1", "true"):
        return True
    if t in ("0", "false"):
        return False
    _bad(key, value, "a boolean (0/1/true/false)")


def _split(key, value):
    items = [s.strip() for s in value.split(",")]
    if len(items) == 1 and not items[0]:
        return []
    if any(not s for s in items):
        raise ConfigError(f'config key {key}: empty item in "{value}"')
    return items


_KEYS = {  # cli.cpp:282-317 apply_key
    "blur": ("blur", str.strip), "n": ("n", _int), "noise": ("noise", _double), "seed": ("seed", _u64),
    "psf_size": ("psf_size", _int), "psf_seed": ("psf_seed", _u64), "psf_sigma": ("psf_sigma", _double),
    "psf_radius": ("psf_radius", _double), "psf_length": ("psf_length", _int),
    "psf_steps": ("psf_steps", _int), "psf_blob_count": ("psf_blob_count", _int),
    "psf_blob_sigma": ("psf_blob_sigma", _double), "fmt": ("fmt", str.strip),
    "solver": ("solver", str.strip), "param": ("param", str.strip), "omega": ("omega", _double),
    "eta": ("eta", _double), "lambda": ("lambda_", _double), "precond_lambda": ("precond_lambda", _double),
    "maxit": ("maxit", _int), "tol": ("tol", _double), "out": ("out", str.strip),
    "include_fpcg": ("include_fpcg", _bool), "sweep_key": ("sweep_key", str.strip),
    "sweep_values": ("sweep_values", _split),
}


def apply_key(cfg: ExperimentConfig, key: str, value: str) -> None:
    if key not in _KEYS:
        raise ConfigError(f"unknown config key: {key}")
    attr, conv = _KEYS[key]
    setattr(cfg, attr, conv(key, value) if conv not in (str.strip,) else value.strip())


def load_config_file(cfg: ExperimentConfig, path: str) -> None:  # cli.cpp:325-343
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise IoError(f"cannot read config file {path}")
    for lineno, line in enumerate(lines, 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"{path}:{lineno}: expected key=value")
        key, value = line.split("=", 1)
        if not key.strip():
            raise ConfigError(f"{path}:{lineno}: empty key")
        apply_key(cfg, key.strip(), value)


_BLURS = ("gaussian", "defocus", "motion", "shake", "speckle")


def validate(cfg: ExperimentConfig) -> None:  # cli.cpp:345-375
    if cfg.blur not in _BLURS:
        raise ConfigError(f"config key blur: unknown blur kind: {cfg.blur}")
    try:
        K.PrecisionFormat.parse(cfg.fmt)
    except ValueError as e:
        raise ConfigError(f"config key fmt: {e}")
    if cfg.solver not in ("cgls", "pcg", "fpcg"):
        raise ConfigError(f"config key solver: unknown solver {cfg.solver}")
    if cfg.param not in ("opt", "gcv", "wgcv", "discrepancy", "fixed"):
        raise ConfigError(f"config key param: unknown method {cfg.param}")
    if cfg.n < 2:
        raise ConfigError("config key n: need n >= 2")
    if cfg.psf_size < 1 or cfg.psf_size % 2 == 0:
        raise ConfigError("config key psf_size: need a positive odd size")
    if cfg.psf_size > cfg.n:
        raise ConfigError("config key psf_size: PSF larger than the image")
    if cfg.noise < 0.0:
        raise ConfigError("config key noise: must be >= 0")
    if cfg.omega <= 0.0:
        raise ConfigError("config key omega: must be > 0")
    if cfg.eta <= 0.0:
        raise ConfigError("config key eta: must be > 0")
    if cfg.lambda_ < 0.0:
        raise ConfigError("config key lambda: must be >= 0")
    if cfg.precond_lambda is not None and cfg.precond_lambda < 0.0:
        raise ConfigError("config key precond_lambda: must be >= 0")
    if cfg.maxit < 1:
        raise ConfigError("config key maxit: must be >= 1")
    if cfg.tol <= 0.0:
        raise ConfigError("config key tol: must be > 0")
    if not cfg.out:
        raise ConfigError("config key out: must not be empty")


def config_json(cfg: ExperimentConfig) -> dict:  # cli.cpp:409-437
    return {"blur": cfg.blur, "n": cfg.n, "noise": cfg.noise, "seed": cfg.seed, "psf_size": cfg.psf_size,
            "psf_seed": cfg.psf_seed, "psf_sigma": cfg.psf_sigma, "psf_radius": cfg.psf_radius,
            "psf_length": cfg.psf_length, "psf_steps": cfg.psf_steps, "psf_blob_count": cfg.psf_blob_count,
            "psf_blob_sigma": cfg.psf_blob_sigma, "fmt": cfg.fmt, "solver": cfg.solver, "param": cfg.param,
            "omega": cfg.omega, "eta": cfg.eta, "lambda": cfg.lambda_, "precond_lambda": cfg.precond_lambda,
            "maxit": cfg.maxit, "tol": cfg.tol, "out": cfg.out, "include_fpcg": cfg.include_fpcg,
            "sweep_key": cfg.sweep_key, "sweep_values": list(cfg.sweep_values)}


def _psf(cfg):
    try:
        return P.make_psf(cfg.blur, cfg.psf_size, sigma=cfg.psf_sigma, radius=cfg.psf_radius,
                          length=cfg.psf_length, steps=cfg.psf_steps, blob_count=cfg.psf_blob_count,
                          blob_sigma=cfg.psf_blob_sigma, seed=cfg.psf_seed)
    except ValueError as e:
        raise ConfigError(str(e))


def build_problem(cfg: ExperimentConfig) -> P.TestProblem:  # cli.cpp:398-407
    psf = _psf(cfg)
    try:
        return P.make_test_problem(P.default_test_image(cfg.n), psf, cfg.noise, cfg.seed)
    except ValueError as e:
        raise ConfigError(str(e))


@dataclass
class Selection:  # cli.hpp:96-108
    method: str = ""
    lambda_: float = 0.0
    objective_value: float = 0.0
    bracket_lo: float = 0.0
    bracket_hi: float = 0.0
    flat_objective: bool = False
    omega: float = 0.0
    eta: float = 0.0
    noise_norm: float = 0.0
    no_root: bool = False
    diagnostic: str = ""


def _num(v) -> str:  # "%.17g"
    return "%d" % v if isinstance(v, (int, np.integer)) and not isinstance(v, bool) else "%.17g" % v


def _csv(path, header, rows):  # RFC 4180 with CRLF (cli.cpp:110-140)
    def q(cell):
        return '"' + cell.replace('"', '""') + '"' if any(c in cell for c in ',"\r\n') else cell
    try:
        with open(path, "w", newline="") as f:
            for r in [header] + rows:
                f.write(",".join(q(c) for c in r) + "\r\n")
    except OSError:
        raise IoError(f"cannot write {path}")


def _write_json(path, j):
    try:
        with open(path, "w") as f:
            f.write(json.dumps(j, indent=2) + "\n")
    except OSError:
        raise IoError(f"cannot write {path}")


def save_pgm(image: np.ndarray, path: str) -> None:  # deblur.cpp:361-371
    img = np.clip(np.asarray(image, dtype=np.float64), 0.0, 1.0)
    px = np.floor(img * 255.0 + 0.5).astype(np.uint8)  # lround of nonnegative values
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{img.shape[1]} {img.shape[0]}\n255\n".encode())
            f.write(px.tobytes(order="C"))
    except OSError:
        raise IoError(f"cannot write {path}")


def selection_json(sel: Selection) -> dict:  # cli.cpp:149-169
    j = {"method": sel.method, "no_root": sel.no_root}
    if sel.no_root:
        j["diagnostic"] = sel.diagnostic
        return j
    j["lambda"] = sel.lambda_
    if sel.method == "fixed":
        return j
    j.update(objective_value=sel.objective_value, bracket_lo=sel.bracket_lo, bracket_hi=sel.bracket_hi,
             flat_objective=sel.flat_objective)
    if sel.method == "wgcv":
        j["omega"] = sel.omega
    if sel.method == "discrepancy":
        j["eta"] = sel.eta
        j["noise_norm"] = sel.noise_norm
    return j


def solver_json(name: str, r: K.SolveResult, plateau: int) -> dict:  # cli.cpp:171-183
    h = r.history
    return {"name": name, "iterations": h.iterations_used, "converged": h.converged,
            "abort_reason": h.abort_reason, "final_relative_error": h.relative_error[-1],
            "final_residual_norm": h.residual_norm[-1], "plateau_iteration": plateau,
            "msolve_count": h.msolve_count, "work_units_total": h.work_units[-1]}


class Prepared:  # cli.cpp:186-198
    def __init__(self, cfg: ExperimentConfig):
        self.tp = build_problem(cfg)
        self.term = P.nearest_kron(self.tp.psf, cfg.n)
        self.m0 = K.build_preconditioner(self.term.row_factor, self.term.col_factor, 1.0,
                                         K.PrecisionFormat.parse(cfg.fmt))


def select_lambda(cfg: ExperimentConfig, m0, tp) -> Selection:  # cli.cpp:200-233
    sel = Selection(method=cfg.param)
    if cfg.param == "fixed":
        sel.lambda_ = cfg.lambda_
        return sel
    try:
        if cfg.param == "opt":
            pc = K.lambda_opt(K.make_spectral_data(m0, tp.b, tp.x_true))
        elif cfg.param == "gcv":
            pc = K.gcv(K.make_spectral_data(m0, tp.b))
        elif cfg.param == "wgcv":
            pc = K.wgcv(K.make_spectral_data(m0, tp.b), cfg.omega)
        else:
            pc = K.discrepancy(K.make_spectral_data(m0, tp.b), float(np.linalg.norm(tp.noise)), cfg.eta)
        sel.lambda_ = pc.lambda_
        sel.objective_value, sel.bracket_lo, sel.bracket_hi = pc.objective_value, pc.bracket_lo, pc.bracket_hi
        sel.flat_objective, sel.omega, sel.eta, sel.noise_norm = (pc.flat_objective, pc.omega, pc.eta,
                                                                  pc.noise_norm)
    except K.NoRootError as e:
        sel.no_root = True
        sel.diagnostic = str(e)
    return sel


def _opts(cfg, lam, tp):  # cli.cpp:235-243
    return K.SolverOptions(lambda_=lam, max_iterations=cfg.maxit, rel_residual_tol=cfg.tol, x_true=tp.x_true)


def precond_for(cfg, p: Prepared, chosen: float):  # cli.cpp:245-254
    ml = cfg.precond_lambda if cfg.precond_lambda is not None else chosen
    if ml == 0.0 and p.m0.svd_r.s.min() * p.m0.svd_c.s.min() == 0.0:
        raise ConfigError("preconditioner lambda is 0 but the approximate operator is singular; set lambda "
                          "or precond_lambda > 0")
    return K.with_lambda(p.m0, ml)


def run_single(cfg: ExperimentConfig) -> dict:  # cli.cpp:469-486
    validate(cfg)
    p = Prepared(cfg)
    oc = {"selection": select_lambda(cfg, p.m0, p.tp), "solved": False}
    if oc["selection"].no_root:
        return oc
    opts = _opts(cfg, oc["selection"].lambda_, p.tp)
    if cfg.solver == "cgls":
        r = K.cgls(p.tp.a, p.tp.b, opts)
    else:
        m = precond_for(cfg, p, oc["selection"].lambda_)
        r = (K.fpcg if cfg.solver == "fpcg" else K.pcg)(p.tp.a, p.tp.b, m, opts)
    oc.update(solved=True, result=r, final_relative_error=r.history.relative_error[-1],
              plateau=K.plateau_iteration(r.history))
    return oc


def write_solve_outputs(cfg: ExperimentConfig, oc: dict) -> None:  # cli.cpp:263-283
    os.makedirs(cfg.out, exist_ok=True)
    summary = {"schema": "kronprec.summary/1", "config": config_json(cfg),
               "selection": selection_json(oc["selection"])}
    if oc["solved"]:
        summary["solver"] = solver_json(cfg.solver, oc["result"], oc["plateau"])
        h = oc["result"].history
        _csv(os.path.join(cfg.out, "convergence.csv"),
             ["schema", "iteration", "relative_error", "residual_norm", "cumulative_work_units"],
             [["kronprec.convergence/1", _num(k), _num(h.relative_error[k]), _num(h.residual_norm[k]),
               _num(h.work_units[k])] for k in range(len(h.residual_norm))])
        save_pgm(K.unvec(oc["result"].x, cfg.n), os.path.join(cfg.out, "reconstruction.pgm"))
    _write_json(os.path.join(cfg.out, "summary.json"), summary)


def _fro2(a_terms, b_terms) -> float:
    """<sum_k R_k (x) C_k, sum_l S_l (x) D_l>_F = sum tr(R^T S) tr(C^T D)."""
    return float(sum(np.sum(r * s) * np.sum(c * d) for r, c in a_terms for s, d in b_terms))


def decompose_row(cfg: ExperimentConfig) -> dict:  # cli.cpp:505-530 (kron.cpp:90-139 distances)
    validate(cfg)
    psf = _psf(cfg)
    a, _ = P.psf_to_kronsum(psf, cfg.n)
    term = P.nearest_kron(psf, cfg.n)
    fmt = K.PrecisionFormat.parse(cfg.fmt)
    at = [(t.row_factor, t.col_factor) for t in a.terms]
    one = [(term.row_factor, term.col_factor)]
    rnd = [(K.round_array(term.row_factor, fmt), K.round_array(term.col_factor, fmt))]
    norm2 = _fro2(at, at)

    def dist(b):
        return math.sqrt(max(0.0, norm2 + _fro2(b, b) - 2.0 * _fro2(at, b)))
    norm = math.sqrt(norm2)
    return {"terms": len(a.terms), "rel_error": dist(one) / norm, "rel_error_rounded": dist(rnd) / norm}


def cmd_generate(cfg):  # cli.cpp:532-546
    from .bundle import save_problem
    validate(cfg)
    tp = build_problem(cfg)
    try:
        save_problem(tp, cfg.out)
    except OSError as e:
        raise IoError(str(e))
    save_pgm(K.unvec(tp.x_true, cfg.n), os.path.join(cfg.out, "xtrue.pgm"))
    save_pgm(K.unvec(tp.b_true, cfg.n), os.path.join(cfg.out, "btrue.pgm"))
    save_pgm(K.unvec(tp.b, cfg.n), os.path.join(cfg.out, "b.pgm"))
    print(f"wrote problem bundle to {cfg.out}")


def cmd_decompose(cfg):  # cli.cpp:548-561
    row = decompose_row(cfg)
    os.makedirs(cfg.out, exist_ok=True)
    _write_json(os.path.join(cfg.out, "decompose.json"),
                {"schema": "kronprec.decompose/1", "config": config_json(cfg), **row})
    print(f"blur={cfg.blur} n={cfg.n} terms={row['terms']} rel_error={_num(row['rel_error'])} "
          f"rel_error_rounded={_num(row['rel_error_rounded'])}")


def cmd_solve(cfg):  # cli.cpp:563-576
    oc = run_single(cfg)
    write_solve_outputs(cfg, oc)
    if oc["solved"]:
        print(f"solver={cfg.solver} lambda={_num(oc['selection'].lambda_)} "
              f"iterations={oc['result'].history.iterations_used} "
              f"final_relative_error={_num(oc['final_relative_error'])}")
    else:
        print(f"parameter search failed: {oc['selection'].diagnostic}")


def cmd_compare(cfg):  # cli.cpp:578-646 (run_compare :488-503)
    validate(cfg)
    p = Prepared(cfg)
    sel = select_lambda(cfg, p.m0, p.tp)
    os.makedirs(cfg.out, exist_ok=True)
    j = {"schema": "kronprec.work_report/1", "config": config_json(cfg), "selection": selection_json(sel)}
    header = ["schema", "iteration", "cgls_relative_error", "cgls_residual_norm", "cgls_work_units",
              "pcg_relative_error", "pcg_residual_norm", "pcg_work_units"]
    if cfg.include_fpcg:
        header += ["fpcg_relative_error", "fpcg_residual_norm", "fpcg_work_units"]
    rows = []
    if not sel.no_root:
        opts = _opts(cfg, sel.lambda_, p.tp)
        m = precond_for(cfg, p, sel.lambda_)
        base = K.cgls(p.tp.a, p.tp.b, opts)
        pre = K.pcg(p.tp.a, p.tp.b, m, opts)
        flex = K.fpcg(p.tp.a, p.tp.b, m, opts) if cfg.include_fpcg else None
        rep = K.work_report(pre.history, base.history)
        j["baseline"] = solver_json("cgls", base, rep.m_baseline)
        j["precond"] = solver_json("pcg", pre, rep.m_precond)
        if flex is not None:
            j["flexible"] = solver_json("fpcg", flex, K.plateau_iteration(flex.history))
        j.update(m_baseline=rep.m_baseline, m_precond=rep.m_precond, threshold=rep.threshold,
                 preconditioning_pays=rep.preconditioning_pays, plateau_tolerance=rep.plateau_tolerance)
        runs = [base.history, pre.history] + ([flex.history] if flex is not None else [])
        for k in range(max(len(h.residual_norm) for h in runs)):
            row = ["kronprec.comparison/1", _num(k)]
            for h in runs:
                row += ([_num(h.relative_error[k]), _num(h.residual_norm[k]), _num(h.work_units[k])]
                        if k < len(h.residual_norm) else ["", "", ""])
            rows.append(row)
        print(f"m_baseline={rep.m_baseline} m_precond={rep.m_precond} "
              f"preconditioning_pays={'true' if rep.preconditioning_pays else 'false'}")
    else:
        print(f"parameter search failed: {sel.diagnostic}")
    _csv(os.path.join(cfg.out, "comparison.csv"), header, rows)
    _write_json(os.path.join(cfg.out, "work_report.json"), j)


def cmd_sweep(cfg):  # cli.cpp:648-688
    validate(cfg)
    if not cfg.sweep_key:
        raise ConfigError("sweep needs sweep_key")
    if cfg.sweep_key in ("out", "sweep_key", "sweep_values"):
        raise ConfigError(f"config key sweep_key: cannot sweep {cfg.sweep_key}")
    if not cfg.sweep_values:
        raise ConfigError("sweep needs a nonempty sweep_values list")
    os.makedirs(cfg.out, exist_ok=True)
    rows = []
    for i, value in enumerate(cfg.sweep_values):
        sub = ExperimentConfig(**{k: (list(v) if isinstance(v, list) else v) for k, v in vars(cfg).items()})
        sub.sweep_key, sub.sweep_values = "", []
        sub.out = os.path.join(cfg.out, f"run_{i}")
        status, oc = "ok", None
        try:
            apply_key(sub, cfg.sweep_key, value)
            oc = run_single(sub)
            write_solve_outputs(sub, oc)
            if not oc["solved"]:
                status = oc["selection"].diagnostic
            elif oc["result"].history.abort_reason:
                status = oc["result"].history.abort_reason
        except Exception as e:  # noqa: BLE001  (the reference records any failure per run)
            status = str(e)
        if oc is not None and oc["solved"]:
            rows.append(["kronprec.sweep/1", value, _num(oc["selection"].lambda_),
                         _num(oc["final_relative_error"]), _num(oc["plateau"]), status])
        else:
            rows.append(["kronprec.sweep/1", value, "", "", "", status])
    _csv(os.path.join(cfg.out, "sweep.csv"),
         ["schema", "value", "lambda", "final_relative_error", "plateau_iteration", "status"], rows)
    print(f"swept {cfg.sweep_key} over {len(cfg.sweep_values)} values into {cfg.out}")


_FLAGS = [("--blur", "blur"), ("--n", "n"), ("--noise", "noise"), ("--seed", "seed"), ("--fmt", "fmt"),
          ("--solver", "solver"), ("--param", "param"), ("--omega", "omega"), ("--eta", "eta"),
          ("--lambda", "lambda"), ("--maxit", "maxit"), ("--tol", "tol"),
          ("--precond-lambda", "precond_lambda"), ("--out", "out"), ("--psf-size", "psf_size"),
          ("--psf-seed", "psf_seed"), ("--psf-sigma", "psf_sigma"), ("--psf-radius", "psf_radius"),
          ("--psf-length", "psf_length"), ("--psf-steps", "psf_steps"), ("--psf-blob-count", "psf_blob_count"),
          ("--psf-blob-sigma", "psf_blob_sigma"), ("--sweep-key", "sweep_key"),
          ("--sweep-values", "sweep_values")]
_VERBS = {"generate": cmd_generate, "decompose": cmd_decompose, "solve": cmd_solve, "compare": cmd_compare,
          "sweep": cmd_sweep}


def main(argv=None) -> int:  # cli.cpp:724-780 dispatch
    ap = argparse.ArgumentParser(prog="kronprec-b200",
                                 description="Kronecker-SVD preconditioned image deblurring experiments (B200)")
    sub = ap.add_subparsers(dest="verb", required=True)
    for verb in _VERBS:
        sp = sub.add_parser(verb)
        sp.add_argument("--config")
        for flag, key in _FLAGS:
            sp.add_argument(flag, dest="k_" + key)
        sp.add_argument("--include-fpcg", action="store_true")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        cfg = ExperimentConfig()
        if args.config:
            load_config_file(cfg, args.config)
        for _, key in _FLAGS:
            v = getattr(args, "k_" + key)
            if v is not None:
                apply_key(cfg, key, v)
        if args.include_fpcg:
            cfg.include_fpcg = True
        _VERBS[args.verb](cfg)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except IoError as e:
        print(f"io error: {e}", file=sys.stderr)
        return 3
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 4
    return 0
