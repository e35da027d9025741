"""One batched C4 PCG solve (64 x 1024^2, 100 iterations) for ncu captures."""
import sys

sys.path.insert(0, ".")
import paper_2311_15393_b200 as K  # noqa: E402
from paper_2311_15393_b200.batch import C4Shard  # noqa: E402

sh = C4Shard()
ids = list(range(64))
probs = {i: sh.problem(i) for i in ids}
bs, xts, nz = sh.stack(ids, probs)
lams = sh.select_lambdas_arrays(bs, nz)
its = int(sys.argv[1]) if len(sys.argv) > 1 else 100
res = K.pcg_batch(sh.a, bs, sh.m0, lams, K.SolverOptions(max_iterations=its, rel_residual_tol=1e-30), x_true=xts)
print("done", max(r.history.iterations_used for r in res))
