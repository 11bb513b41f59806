import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1905_08375_b200 import nonloc as N, configs
n = 1 << 16
w0 = configs.cfg1(n, exterior=0)
w1 = configs.cfg1(n, exterior=1)
op0 = N.NonlocalOperator(w0.dim, w0.n, **w0.op_kwargs())
op1 = N.NonlocalOperator(w1.dim, w1.n, **w1.op_kwargs())
print("infos", op0.info.n_in, op0.info.halo_lo, op1.info.n_in, op1.info.halo_lo, op0.info.fast_method, op1.info.fast_method, flush=True)
f0 = op0.apply(w0.u); f1 = op1.apply(w1.u)
i = np.arange(2000, 2010)
print("ratio (f1-f0)/u", (f1[i] - f0[i]) / w0.u[i])
# linearity test: apply to delta function at center
e = np.zeros(n); e[n // 2] = 1.0
g0 = op0.apply(e); g1 = op1.apply(e)
print("impulse diff max", np.max(np.abs(g0 - g1)), "g0 center", g0[n//2-2:n//2+3], "g1 center", g1[n//2-2:n//2+3])
k = np.nonzero(np.abs(g0 - g1) > 1e-9 * np.max(np.abs(g0)))[0]
print("impulse diff at", k[:10], k[-10:], k.size)
