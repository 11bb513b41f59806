import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1905_08375_b200 import nonloc as N, configs
n = 1 << 16
w0 = configs.cfg1(n, exterior=0)
w1 = configs.cfg1(n, exterior=1)
op0 = N.NonlocalOperator(w0.dim, w0.n, **w0.op_kwargs())
op1 = N.NonlocalOperator(w1.dim, w1.n, **w1.op_kwargs())
print("infos", op0.info.n_in, op0.info.n_out, op0.info.halo_lo, op1.info.n_in, op1.info.n_out, op1.info.halo_lo, op0.info.exp_terms, op1.info.exp_terms)
f0 = op0.apply(w0.u); f1 = op1.apply(w1.u)
mid = slice(2000, n - 2000)
print("clip vs collar interior max diff", np.max(np.abs(f0[mid] - f1[mid])) / np.max(np.abs(f0)))
print("u equal", np.array_equal(w0.u, w1.u), "kappa equal", np.array_equal(w0.kappa, w1.kappa))
d0 = op0.plan.apply_direct_at(w0.u, np.arange(2000, 2010))
d1 = op1.plan.apply_direct_at(w1.u, np.arange(2000, 2010))
print(f0[2000:2003], d0[:3]); print(f1[2000:2003], d1[:3])
o1 = op1.apply(np.ones(n))
print("collar apply(1): interior max", np.max(np.abs(o1[mid])), "edge", o1[:3], o1[-3:])
i = np.argmax(np.abs(o1[mid])) + 2000
print("at", i, o1[i-2:i+3])
nz = np.nonzero(np.abs(o1) > 1e-6 * np.max(np.abs(o1)))[0]
print("nonzero count", nz.size, nz[:10], nz[-10:])
