"""ncu driver for the direct-sum kernel (direct.cu): the BASELINE operator's
literal form (apply_full_dense + eval_omega, operators.cpp:236-260) through
nlg_apply_direct on a cfg-family workload at reduced size. Prints the pair
count (the reference's pair_count) for the FLOP/s arithmetic.

  python tools/prof_direct.py cfg2 1024
"""
import sys
import time
sys.path.insert(0, ".")
from paper_1905_08375_b200 import nonloc as N, configs
name, n = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = configs.WORKLOADS[name](n)
op = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
for _ in range(reps):
    t0 = time.perf_counter()
    out, pairs = op.plan.apply_direct(w.u)
    el = time.perf_counter() - t0
print(f"ok {name} n={n} pairs={pairs} wall={el:.4f}s pairs/s={pairs / el:.4g}")
