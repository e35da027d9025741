"""Sweep reference-exact fp16 GEMM variants (KP_F16REF_CFG) (dev tool)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, hashlib
sys.path.insert(0, %r)
import numpy as np, ctypes as C
import paper_2311_15393_b200 as K
from paper_2311_15393_b200.kronprec import SvdTriple
from paper_2311_15393_b200._lib import lib, check
for n in (1024, 4096):
    q = np.linalg.qr(np.random.default_rng(1).standard_normal((n, n)))[0] if n <= 1024 else None
    if q is None:
        import torch
        q = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1)))[0].cpu().numpy()
    sv = SvdTriple(np.asfortranarray(q), np.linspace(1.0, 1e-3, n), np.asfortranarray(q))
    m = K.build_preconditioner_from_svd(sv, sv, 0.01, K.PrecisionFormat.fp16())
    r = np.random.default_rng(2).standard_normal(n * n)
    z = K.precond_solve(m, r)
    L = lib(); check(L.kp_profile_enable(1)); check(L.kp_profile_reset())
    for _ in range(3): z = K.precond_solve(m, r)
    t = C.c_double(); c = C.c_longlong(); check(L.kp_profile_read(1, C.byref(t), C.byref(c)))
    check(L.kp_profile_enable(0))
    ms = t.value / c.value
    print("RESULT", os.environ.get("KP_F16REF_CFG", "0"), n, f"{ms:.4f} ms/GEMM", f"{2*n**3/(ms/1e3)/1e12:.2f} Tops", hashlib.md5(z.tobytes()).hexdigest(), flush=True)
''' % ROOT
for cfg in sys.argv[1:] or ["0", "1", "5", "6"]:
    env = dict(os.environ, KP_F16REF_CFG=cfg)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    print([l for l in r.stdout.splitlines() if l.startswith("RESULT")] or r.stderr[-800:], flush=True)
