"""Randomised parity sweep of the column-lane stencils (GPU): fast apply vs the
GPU direct sum (itself pinned to the CPU oracle by the test suite) over random
grids, horizon ranges, weightings, exteriors and slab cuts.

  python tools/fuzz_cy.py [cases] [seed]
"""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1905_08375_b200 import nonloc as N

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rg = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
worst = 0.0
for c in range(cases):
    dim = int(rg.choice([2, 2, 3]))
    n = int(rg.integers(10, 72) * 2) if dim == 2 else int(rg.integers(6, 26) * 2)
    hi = float(rg.uniform(1.5, 12.0 if dim == 2 else 8.0))
    lo = float(rg.uniform(0.5, hi))
    peri = dim == 2 and rg.random() < 0.3
    kw = (not peri) and rg.random() < 0.7
    ext = int(rg.integers(0, 2))
    h = 1.0 / n
    idx = np.indices((n,) * dim).reshape(dim, -1)
    kvec = rg.integers(1, 4, dim)
    phase = sum(int(kvec[a]) * idx[a] for a in range(dim)) * (2.0 * np.pi / n) + rg.uniform(0, 6.28)
    delta = h * (0.5 * (lo + hi) + 0.5 * (hi - lo) * np.sin(phase))
    if rg.random() < 0.15:          # piecewise jump (cfg3 style)
        delta = np.where(idx[0] < n // 2, h * lo, h * hi) + 0.0 * delta
    Nn = n ** dim
    coeff = 1.0 + rg.random(Nn)
    kappa = np.exp(0.4 * rg.standard_normal(Nn)) if kw else None
    u = rg.standard_normal((2 if peri else 1) * Nn)
    kwargs = dict(delta=delta, coeff=coeff, exterior=ext)
    if peri:
        kwargs["kernel"] = "peridynamic"
    else:
        kwargs.update(alpha=dim + float(rg.uniform(0.2, 1.8)), kappa=kappa)
    op = N.NonlocalOperator(dim, n, **kwargs)
    fast = op.apply(u)
    direct, _ = op.apply_direct(u)
    err = float(np.max(np.abs(fast - direct)) / np.max(np.abs(direct)))
    worst = max(worst, err)
    tag = f"case {c}: dim {dim} n {n} delta/h [{lo:.2f}, {hi:.2f}] peri {peri} kappa {kw} ext {ext} rel {err:.2e}"
    if not err <= 1e-10:
        print("FAIL", tag)
        sys.exit(1)
    # a slab cut of the same operator (scalar only)
    if not peri and rg.random() < 0.5:
        dmax = float(delta.max())
        halo = N.halo_rows(dim=dim, n=n, family=4, delta_max=dmax)
        rb = int(rg.integers(0, n - 2))
        re = int(rg.integers(rb + 1, n + 1))
        ib, ie = max(0, rb - halo), min(n, re + halo)
        st = n ** (dim - 1)
        sl = slice(ib * st, ie * st)
        ops = N.NonlocalOperator(dim, n, alpha=kwargs["alpha"], delta=delta[sl], coeff=coeff[sl],
                                 kappa=None if kappa is None else kappa[sl], exterior=ext,
                                 row_begin=rb, row_end=re, reach=dmax)
        part = ops.apply(u[sl].copy())
        e2 = float(np.max(np.abs(part - fast[rb * st:re * st])) / np.max(np.abs(fast)))
        if not e2 <= 1e-12:
            print("FAIL slab", tag, rb, re, e2)
            sys.exit(1)
    print(tag)
print("fuzz ok", cases, "cases, worst rel", worst)
