import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1905_08375_b200 import nonloc as N, configs
n = int(sys.argv[1]); order = sys.argv[2]
ops = []
for ext in [int(c) for c in order]:
    w = configs.cfg1(n, exterior=ext)
    op = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
    e = np.zeros(n); e[n // 2] = 1.0
    g = op.apply(e)
    print(n, "ext", ext, "impulse center", g[n // 2], "L?", op.info.exp_terms, flush=True)
    ops.append(op)
