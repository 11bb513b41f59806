"""Small driver for ncu: build a workload (optionally at reduced size) and run
its fast apply on device buffers (nlg_apply_fast_dev: one launch per kernel of
the whole apply, not the host entry's chunked copy pipeline).

  python tools/prof_apply.py cfg4 768 [reps]
"""
import sys
sys.path.insert(0, ".")
import torch
from paper_1905_08375_b200 import nonloc as N, configs
name = sys.argv[1]
n = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = configs.WORKLOADS[name](n)
op = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
plan = op.plan
u = torch.from_numpy(w.u).cuda()
out = torch.empty(plan.components * plan.n_out, dtype=torch.float64, device="cuda")
for _ in range(reps):
    plan.apply_fast_dev(u.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", name, n, op.info.fast_method)
