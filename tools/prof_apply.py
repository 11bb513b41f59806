"""Small driver for ncu: build a workload at reduced size and run its fast apply."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1905_08375_b200 import nonloc as N, configs
name = sys.argv[1]
n = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = configs.WORKLOADS[name](n)
op = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
for _ in range(reps):
    op.apply(w.u)
print("ok", name, n, op.info.fast_method)
