import numpy as np, sys
sys.path.insert(0, '.')
import paper_2311_15393_b200 as K
from oracle import pyoracle as O
from paper_2311_15393_b200.kronprec import KronTerm, KroneckerSum, SolverOptions
a = KroneckerSum([KronTerm(np.array([[2.0]]), np.array([[3.0]]))], 1)
b = np.array([1.5])
o = SolverOptions(lambda_=0.5, max_iterations=5, rel_residual_tol=1e-12)
r = K.cgls(a, b, o); xo, ho = O.cgls(a, b, o)
print(r.x, xo, r.history.residual_norm, ho.residual_norm, r.history.iterations_used, ho.iterations_used, r.history.converged, ho.converged)
