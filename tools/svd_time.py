"""Setup SVD timing at the C5 size: host LAPACK vs cuSOLVER (gesvd / gesvdj
via KP_SVD_ALGO) on the C5 nearest-Kronecker factors, plus the C5 FPCG
iteration count with the device factors."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200 import configs  # noqa: E402

cfg = configs.build("C5")
f = cfg.term.row_factor
K.svd(f[:256, :256].copy(), "device")  # warm cuSOLVER
for backend in sys.argv[1:] or ["device", "host"]:
    t0 = time.time()
    u, s, v = K.svd(f, backend)
    dt = time.time() - t0
    err = np.linalg.norm((u * s) @ v.T - f) / np.linalg.norm(f)
    print(f"{backend} ({os.environ.get('KP_SVD_ALGO', 'gesvd')}): {dt:.2f} s, reconstruction {err:.2e}", flush=True)
