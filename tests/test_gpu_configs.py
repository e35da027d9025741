"""BASELINE configurations on the device vs the oracle.

C1 (n=256) runs the oracle at test time; C2-C5 compare against the committed
oracle goldens (tests/golden/*.json, made by tests/golden/gen_goldens.py;
C5 as a 3-iteration prefix). Bounds from the north star: reference-exact
preconditioned runs within +-2 iterations and 1e-3 final relative error of
the reference, identical GCV grid index, FP64 histories 1e-10 over a prefix."""
import json
import os

import numpy as np
import pytest

import paper_2311_15393_b200 as K
from oracle import pyoracle as O
from paper_2311_15393_b200 import configs
from paper_2311_15393_b200.kronprec import SolverOptions, SvdTriple
from paper_2311_15393_b200 import problems as P

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
FMT = {"fp16": K.PrecisionFormat.fp16(), "fp64": K.PrecisionFormat.fp64()}


def golden(name):
    path = os.path.join(HERE, "golden", f"{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"golden {name}.json not generated (tests/golden/gen_goldens.py)")
    with open(path) as f:
        return json.load(f)


def device_runs(cfg, lam, solvers, accum="reference", prefix=None):
    m0 = {}
    out = []
    for solver, fmt, maxit in solvers:
        opts = SolverOptions(lambda_=lam, max_iterations=min(maxit, prefix or maxit),
                             rel_residual_tol=cfg.tol, x_true=cfg.problem.x_true)
        if solver == "cgls":
            r = K.cgls(cfg.problem.a, cfg.problem.b, opts)
        else:
            if fmt not in m0:
                m0[fmt] = K.build_preconditioner(cfg.term.row_factor, cfg.term.col_factor, 1.0,
                                                 FMT[fmt], accum=accum if fmt == "fp16" else "reference")
            m = K.with_lambda(m0[fmt], lam)
            r = getattr(K, solver)(cfg.problem.a, cfg.problem.b, m, opts)
        out.append(r)
    return out


def check_against(run, ref, prefix_rows=3, final=True):
    """North-star bounds. Row 0 (A^T b, ||x_true||) is FP64-only: 1e-10.
    Later rows of fp16-preconditioned runs depend on the last bits of the
    host LAPACK SVD (CPU model / thread count differ between the golden
    machine and the GPU box), which flip rare fp16 roundings of V, so for
    them only the north-star end bounds apply (the M-solve itself is checked
    bit for bit with a shared SVD); FP64-only runs (CGLS, fp64 format) keep
    1e-8 per row."""
    h = run.history
    assert abs(h.iterations_used - ref["iterations_used"]) <= 2
    assert h.converged == ref["converged"]
    if final:
        assert abs(h.relative_error[-1] - ref["relative_error"][-1]) <= 1e-3
    fp16 = ref.get("fmt") == "fp16"
    rows = 1 if fp16 else prefix_rows
    for k in range(min(rows, len(h.residual_norm), len(ref["residual_norm"]))):
        tol = 1e-10 if k == 0 else 1e-8
        assert h.residual_norm[k] == pytest.approx(ref["residual_norm"][k], rel=tol)
        assert h.relative_error[k] == pytest.approx(ref["relative_error"][k], rel=tol)


def test_c1_vs_oracle_now():
    cfg = configs.build("C1")
    g = golden("C1")["images"][0]
    runs = device_runs(cfg, cfg.lambda_, cfg.solvers)
    for run, ref in zip(runs, g["runs"]):
        check_against(run, ref)
    # and against an oracle run made here with the same SVD (bit-exact M)
    sr = SvdTriple(*P.host_svd(cfg.term.row_factor))
    sc = SvdTriple(*P.host_svd(cfg.term.col_factor))
    mg = K.build_preconditioner_from_svd(sr, sc, cfg.lambda_, FMT["fp16"])
    mo = O.build_preconditioner_from_svd((sr.u, sr.s, sr.v), (sc.u, sc.s, sc.v), cfg.lambda_, FMT["fp16"])
    opts = SolverOptions(lambda_=cfg.lambda_, max_iterations=100, rel_residual_tol=cfg.tol,
                         x_true=cfg.problem.x_true)
    rg = K.pcg(cfg.problem.a, cfg.problem.b, mg, opts)
    _, ho = O.pcg(cfg.problem.a, cfg.problem.b, mo, opts)
    assert rg.history.iterations_used == ho.iterations_used
    assert abs(rg.history.relative_error[-1] - ho.relative_error[-1]) <= 1e-6


def test_c2_fpcg_vs_golden():
    cfg = configs.build("C2")
    g = golden("C2")["images"][0]
    (run,) = device_runs(cfg, cfg.lambda_, cfg.solvers)
    ref = g["runs"][0]
    check_against(run, ref, prefix_rows=5)
    assert run.history.abort_reason.split(" at ")[0] == ref["abort_reason"].split(" at ")[0]
    # the M-solve at n=1024 is bit-identical to the reference emulation
    sr = SvdTriple(*P.host_svd(cfg.term.row_factor))
    sc = SvdTriple(*P.host_svd(cfg.term.col_factor))
    mg = K.build_preconditioner_from_svd(sr, sc, cfg.lambda_, FMT["fp16"])
    mo = O.build_preconditioner_from_svd((sr.u, sr.s, sr.v), (sc.u, sc.s, sc.v), cfg.lambda_,
                                         FMT["fp16"])
    r = K.kronsum_apply_transpose(cfg.problem.a, cfg.problem.b)
    assert np.array_equal(K.precond_solve(mg, r), O.precond_solve(mo, r))


def test_c3_gcv_index_and_pcg():
    g = golden("C3")["images"][0]
    cfg = configs.build("C3")
    m0 = K.build_preconditioner(cfg.term.row_factor, cfg.term.col_factor, 1.0, FMT["fp16"])
    sd = K.make_spectral_data(m0, cfg.problem.b)
    c, vals = K.gcv_grid(sd, configs.GCV_GRID)
    assert c.grid_index == g["gcv_index"]
    assert np.allclose(vals, g["gcv_values"], rtol=1e-10)
    (run,) = device_runs(cfg, c.lambda_, cfg.solvers)
    check_against(run, g["runs"][0])


def test_c4_discrepancy_and_batched_pcg_vs_golden():
    """C4: every image of the golden (all 64 of the batch once generated):
    discrepancy lambda (1e-9) and the batched PCG solve (kp_pcg_batch) within
    the north-star bounds of the oracle's per-image run."""
    from paper_2311_15393_b200.batch import C4Shard
    g = golden("C4")
    sh = C4Shard()
    ids = [rec["image"] for rec in g["images"]]
    probs = {i: sh.problem(i) for i in ids}
    results = sh.solve_batch(ids, probs)
    for rec, res in zip(g["images"], results):
        assert res.image == rec["image"]
        assert res.lam == pytest.approx(rec["lambda"], rel=1e-9)
        ref = rec["runs"][0]
        assert abs(res.iterations - ref["iterations_used"]) <= 2
        assert res.converged == ref["converged"]
        assert abs(res.rel_err - ref["relative_error"][-1]) <= 1e-3


def test_c4_batched_equals_per_image_solves():
    """Two C4 images at full size: the batched solve equals the per-image
    pipeline (solve()) exactly."""
    from paper_2311_15393_b200.batch import C4Shard
    sh = C4Shard()
    probs = {i: sh.problem(i) for i in (1, 2)}
    batched = sh.solve_batch([1, 2], probs)
    for i, rb in zip((1, 2), batched):
        rs = sh.solve(i, probs[i])
        assert (rb.lam, rb.iterations, rb.converged, rb.rel_err) == (rs.lam, rs.iterations, rs.converged, rs.rel_err)


def test_c5_prefix_vs_golden():
    g = golden("C5")["images"][0]
    cfg = configs.build("C5")
    runs = device_runs(cfg, cfg.lambda_, cfg.solvers, prefix=3)
    for run, ref in zip(runs, g["runs"]):
        assert run.history.iterations_used == ref["iterations_used"]
        check_against(run, ref, prefix_rows=len(ref["residual_norm"]), final=False)


def test_c5_operator_full_size_properties():
    """Size-independent checks at BASELINE size (n = 4096, r = 5): the banded
    operator equals the dense DMMA product, is linear, and A^T is its adjoint."""
    psf, cap = configs._psf("C5")
    a, _ = P.psf_to_kronsum(psf, 4096, max_rank=cap)
    assert a.mode()[0].startswith("banded")
    rng = np.random.default_rng(55)
    x, y = rng.standard_normal(4096 * 4096), rng.standard_normal(4096 * 4096)
    ax = K.kronsum_apply(a, x)
    aty = K.kronsum_apply_transpose(a, y)
    assert abs(ax @ y - x @ aty) <= 1e-12 * np.linalg.norm(ax) * np.linalg.norm(y)
    axy = K.kronsum_apply(a, 2.0 * x - 3.0 * y)
    assert np.linalg.norm(axy - (2.0 * ax - 3.0 * K.kronsum_apply(a, y))) <= 1e-13 * np.linalg.norm(axy)
    a.set_mode("dense")
    dx = K.kronsum_apply(a, x)
    a.set_mode("auto")
    assert np.linalg.norm(ax - dx) <= 1e-13 * np.linalg.norm(dx)


def test_setup_svd_backend_invariance():
    """The factor SVDs may come from host LAPACK or the library's cuSOLVER SVD (kp_svd);
    their vectors differ in sign and last bits. M, the GCV sums and the
    discrepancy lambda are invariant (SURVEY §7 'setup cost')."""
    cfg = configs.build("C1")
    term = cfg.term
    host = [SvdTriple(*P.host_svd(f)) for f in (term.row_factor, term.col_factor)]
    dev = [SvdTriple(*K.svd(f, "device")) for f in (term.row_factor, term.col_factor)]  # cuSOLVER
    r = np.random.default_rng(8).standard_normal(cfg.n * cfg.n)
    for fmt, tol in ((K.PrecisionFormat.fp64(), 1e-10), (K.PrecisionFormat.fp16(), 2e-3)):
        mh = K.build_preconditioner_from_svd(host[0], host[1], 0.01, fmt)
        md = K.build_preconditioner_from_svd(dev[0], dev[1], 0.01, fmt)
        zh, zd = K.precond_solve(mh, r), K.precond_solve(md, r)
        assert np.linalg.norm(zh - zd) <= tol * np.linalg.norm(zh)
    m0h = K.build_preconditioner_from_svd(host[0], host[1], 1.0, K.PrecisionFormat.fp16())
    m0d = K.build_preconditioner_from_svd(dev[0], dev[1], 1.0, K.PrecisionFormat.fp16())
    sh, sd = K.make_spectral_data(m0h, cfg.problem.b), K.make_spectral_data(m0d, cfg.problem.b)
    ch, vh_ = K.gcv_grid(sh, configs.GCV_GRID)
    cd, vd = K.gcv_grid(sd, configs.GCV_GRID)
    assert ch.grid_index == cd.grid_index
    assert np.allclose(vh_, vd, rtol=1e-10)
    nn = float(np.linalg.norm(cfg.problem.noise))
    assert K.discrepancy(sh, nn, 1.01).lambda_ == pytest.approx(K.discrepancy(sd, nn, 1.01).lambda_,
                                                                 rel=1e-9)


def test_c5_fpcg_full_solve_vs_golden():
    """The headline run end to end at BASELINE size: C5 FPCG with the fp16
    reference-exact preconditioner, against the oracle's complete run
    (tests/golden/C5_fpcg_full.json: iterations, stop / abort reason,
    final relative error)."""
    path = os.path.join(os.path.dirname(__file__), "golden", "C5_fpcg_full.json")
    if not os.path.exists(path):
        pytest.skip("C5_fpcg_full.json not generated")
    ref = json.load(open(path))["images"][0]["runs"][0]
    cfg = configs.build("C5")
    # the library's LAPACK setup SVD (the oracle's routine); cuSOLVER factors
    # move the stagnation-point abort by a few iterations
    m = K.build_preconditioner(cfg.term.row_factor, cfg.term.col_factor, cfg.lambda_,
                               FMT["fp16"])
    opts = SolverOptions(lambda_=cfg.lambda_, max_iterations=100, rel_residual_tol=cfg.tol,
                         x_true=cfg.problem.x_true)
    run = K.fpcg(cfg.problem.a, cfg.problem.b, m, opts)
    check_against(run, ref, prefix_rows=1)
    assert run.history.abort_reason.split(" at ")[0] == ref["abort_reason"].split(" at ")[0]


def test_c5_cgls_full_solve_vs_golden():
    """C5's CGLS run to convergence at BASELINE size (FP64 only) against the
    oracle's complete run: iteration count, convergence, final error, and the
    residual / error history over a 20-row prefix at 1e-8 (later rows drift
    with FP64 re-association)."""
    path = os.path.join(os.path.dirname(__file__), "golden", "C5_cgls_full.json")
    if not os.path.exists(path):
        pytest.skip("C5_cgls_full.json not generated")
    ref = json.load(open(path))["images"][0]["runs"][0]
    cfg = configs.build("C5")
    (run,) = device_runs(cfg, cfg.lambda_, [("cgls", None, 2000)])
    check_against(run, ref, prefix_rows=20)


def test_c5_pcg_fp64_full_solve_vs_golden():
    """C5's third run: PCG with the FP64 Kronecker-SVD preconditioner to
    convergence, against the oracle's complete run
    (tests/golden/C5_pcg64_full.json): iteration count, convergence, final
    relative error, residual / error history over a 20-row prefix at 1e-8."""
    path = os.path.join(os.path.dirname(__file__), "golden", "C5_pcg64_full.json")
    if not os.path.exists(path):
        pytest.skip("C5_pcg64_full.json not generated")
    ref = json.load(open(path))["images"][0]["runs"][0]
    assert ref["solver"] == "pcg" and ref["fmt"] == "fp64"
    cfg = configs.build("C5")
    (run,) = device_runs(cfg, cfg.lambda_, [("pcg", "fp64", 100)])
    check_against(run, ref, prefix_rows=20)


@pytest.mark.parametrize("name", ["C1", "C2", "C5"])
def test_tensor_mode_at_config_scale(name):
    """The tcgen05 tensor-mode preconditioner (fp32 accumulation, one binary16
    rounding per product matrix; KP_ACCUM_TENSOR) at BASELINE sizes, against
    the reference-exact run (goldens from the oracle).

    C1: the reference converges; tensor mode must land within 1e-3 of its
    final relative error and need no more than 2 extra iterations.
    C2 / C5: the reference's per-product rounding underflows once the
    residual reaches ~1e-6 and it stagnates until the positivity abort
    (DESIGN.md §4). Tensor mode does not stagnate there, so the north star's
    +-2-iteration bound cannot hold by construction; asserted instead: tensor
    mode reaches a final relative error no worse than the reference's, and
    never reports the reference's abort."""
    cfg = configs.build(name)
    g = golden({"C5": "C5_fpcg_full"}.get(name, name))["images"][0]["runs"][0]
    (run,) = device_runs(cfg, cfg.lambda_, cfg.solvers[:1], accum="tensor")
    h = run.history
    if name == "C1":
        assert g["converged"] and h.converged
        assert abs(h.relative_error[-1] - g["relative_error"][-1]) <= 1e-3
        assert h.iterations_used <= g["iterations_used"] + 2
    else:
        assert not g["converged"] and "lost positivity" in g["abort_reason"]
        assert "lost positivity" not in h.abort_reason
        assert h.relative_error[-1] <= g["relative_error"][-1] + 1e-3
