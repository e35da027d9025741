"""Per-launch device time of gemm_f16x vs gemm_f16ref at n=4096 (one M-solve each)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200.kronprec import SvdTriple  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(1)
v = rng.standard_normal((n, n)).astype(np.float16).astype(np.float64) / 64
trip = SvdTriple(v, np.linspace(1, 1e-3, n), v)
m = K.build_preconditioner_from_svd(trip, trip, 0.01, K.PrecisionFormat.fp16())
r = rng.standard_normal(n * n)
for eng in sys.argv[2:] or ["cuda", "tensor"]:
    K.set_fp16_products(eng)
    for _ in range(2):
        K.precond_solve(m, r)
