"""Debug: fast vs direct (sampled) for cfg1 family with clip / collar."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1905_08375_b200 import nonloc as N, configs
for lg in [16]:
    for ext in (0, 1):
        n = 1 << lg
        w = configs.cfg1(n, exterior=ext)
        op = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
        fast = op.apply(w.u)
        tg = np.arange(0, n, 7).astype(np.int64)
        d = op.plan.apply_direct_at(w.u, tg)
        err = np.abs(fast[tg] - d) / np.max(np.abs(d))
        bad = tg[err > 1e-10]
        print(lg, ext, op.info.exp_terms, "maxerr %.3e" % err.max(), "bad", len(bad), bad[:5], bad[-5:], flush=True)
        ones = op.apply(np.ones(n))
        print("  ones max", np.max(np.abs(ones)), "at", np.argmax(np.abs(ones)))
