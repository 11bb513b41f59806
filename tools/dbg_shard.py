import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import oracle as O
from paper_1905_08375_b200 import nonloc as N, configs
from paper_1905_08375_b200.slabs import Slab
w = configs.cfg1(1 << 16)
kw = w.op_kwargs()
full = N.NonlocalOperator(1, w.n, **kw)
ref = full.apply(w.u)
dref,_ = full.apply_direct(w.u)
print("full fast vs direct", O.rel_inf(ref, dref), "M", full.info.exp_terms)
dmax = float(w.delta.max())
halo = N.halo_rows(dim=1, n=w.n, family=4, delta_max=dmax)
for r in range(3):
    sl = Slab(w.n, 1, halo, r, 3)
    k2 = dict(kw)
    for key in ("delta","coeff","kappa"):
        k2[key] = sl.input_slice(k2[key])
    op = N.NonlocalOperator(1, w.n, row_begin=sl.row_begin, row_end=sl.row_end, reach=dmax, **k2)
    ui = sl.input_slice(w.u)
    f = op.apply(ui); d,_ = op.apply_direct(ui)
    seg = slice(sl.row_begin, sl.row_end)
    err = np.abs(f - dref[seg]); errd = np.abs(d - dref[seg])
    print(r, "method", op.info.fast_method, "M", op.info.exp_terms, "halo", op.info.halo_lo, op.info.halo_hi,
          "fast rel", O.rel_inf(f, dref[seg]), "direct rel", O.rel_inf(d, dref[seg]), "worst idx", int(np.argmax(err)), "of", len(f))
    bad = np.where(err > 1e-8*np.abs(dref).max())[0]
    if len(bad): print("   bad range", bad.min(), bad.max(), len(bad))
