"""A few dense-mode operator applies at C5 size (ncu capture target for gemm_f64_tma_kernel)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200 import problems as P  # noqa: E402

n = 4096
psf = P.psf_gauss_motion(41, 4.0, 15, 30.0)
op, _ = P.psf_to_kronsum(psf, n, max_rank=5)
op.set_mode("dense")
x = np.random.default_rng(0).standard_normal(n * n)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    y = K.kronsum_apply(op, x)
print("ok", float(np.linalg.norm(y)))
