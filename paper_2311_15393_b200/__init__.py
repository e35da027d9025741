"""B200-native PCG / FPCG / CGLS hot path of arXiv 2311.15393 (kronprec).

Drop-in for the reference's solver path: Kronecker-sum operator, half-
precision Kronecker-SVD preconditioner, Krylov solvers and lambda selection,
computed by hand-written sm_100a kernels behind the C ABI in
include/kronprec_b200.h. See DESIGN.md.
"""
from .kronprec import *  # noqa: F401,F403
from .kronprec import __all__ as _k_all
from . import problems  # noqa: F401

__all__ = list(_k_all) + ["problems"]
