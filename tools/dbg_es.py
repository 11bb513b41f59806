"""Debug: fast vs direct (sampled targets) for cfg1 at several sizes."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1905_08375_b200 import nonloc as N, configs
for lg in [int(x) for x in sys.argv[1:]] or [18, 20, 22]:
    n = 1 << lg
    w = configs.cfg1(n)
    op = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
    fast = op.apply(w.u)
    tg = np.unique(np.concatenate([np.arange(0, 50), np.arange(n - 50, n),
                                   np.random.default_rng(0).integers(0, n, 400)])).astype(np.int64)
    d = op.plan.apply_direct_at(w.u, tg)
    err = np.abs(fast[tg] - d) / np.max(np.abs(d))
    bad = tg[err > 1e-10]
    print(lg, op.info.exp_terms, "maxerr %.3e" % err.max(), "bad", len(bad), bad[:10], flush=True)
