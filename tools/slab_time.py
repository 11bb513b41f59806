"""Device time of one rank's slab apply for the headline cfg1 at N = 1, 2, 4, 8
(the middle rank: two halos), on this one GPU. Predicts the compute part of the
strong scaling (the NCCL halo exchange is not included)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1905_08375_b200 import nonloc as N, configs
from paper_1905_08375_b200.slabs import Slab

w = configs.cfg1()
dmax = float(w.delta.max())
halo = N.halo_rows(dim=1, n=w.n, family=4, delta_max=dmax)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
base = None
for world in (1, 2, 4, 8):
    r = world // 2
    sl = Slab(w.n, 1, halo if world > 1 else 0, r, world)
    kw = w.op_kwargs()
    for key in ("delta", "coeff", "kappa"):
        kw[key] = sl.input_slice(kw[key])
    op = N.NonlocalOperator(1, w.n, row_begin=sl.row_begin, row_end=sl.row_end,
                            reach=dmax if world > 1 else 0.0, **kw)
    u = torch.from_numpy(sl.input_slice(w.u)).to(dev)
    out = torch.empty(op.plan.n_out, dtype=torch.float64, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    with torch.cuda.stream(stream):
        for _ in range(5):
            op.plan.apply_fast_dev(u.data_ptr(), out.data_ptr(), stream.cuda_stream)
        for a, b in ev:
            flush.fill_(1.0)
            a.record(stream)
            op.plan.apply_fast_dev(u.data_ptr(), out.data_ptr(), stream.cuda_stream)
            b.record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / len(ev)
    base = base or ms
    print(f"N={world}: rank {r} n_in={op.plan.n_in} n_out={op.plan.n_out} fft_len={op.info.fft_len} "
          f"{ms:.4f} ms/apply  compute-only efficiency {base / (world * ms):.2f}")
