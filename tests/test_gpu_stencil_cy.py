"""Column-lane stencil kernels (stencil_cy_kernel / stencil_cyp_kernel: per-node
horizons in 2-D / 3-D, sources staged by TMA): fast apply vs the restated CPU
oracle (operators.cpp:236-260 with eval_omega, kernel.cpp:275-287) and vs the
GPU direct sum, over the cases the blocking is sensitive to — odd and even
reach (the box halo is rounded to even columns), grids that are not a multiple
of the 32-column tile, odd n (no tensor map: the row-lane fallback), horizons
narrower than a cell, a constant array that puts every target on a tie band,
and slab plans. The row-lane sweep (NLG_ST_CY=0) must agree to rounding."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
FAST_TOL = 1e-10


@pytest.fixture(scope="module")
def N():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1905_08375_b200 import nonloc
    return nonloc


def _fields(dim, n, lo, hi, seed):
    rg = np.random.default_rng(seed)
    N_ = n ** dim
    h = 1.0 / n
    idx = np.indices((n,) * dim).reshape(dim, -1)
    phase = sum((a + 1) * idx[a] for a in range(dim)) * (2.0 * np.pi / n)
    delta = h * (0.5 * (lo + hi) + 0.5 * (hi - lo) * np.sin(phase + 0.3))
    u = rg.standard_normal(N_)
    kappa = np.exp(0.3 * rg.standard_normal(N_))
    coeff = 1.0 + 0.5 * rg.random(N_)
    return delta, u, kappa, coeff


# (dim, n, lowest, highest horizon in cells, kappa weighting)
SCALAR = [(2, 96, 2.0, 5.5, True), (2, 100, 3.0, 7.9, True), (2, 100, 3.0, 7.9, False), (2, 72, 4.0, 12.0, True),
          (2, 101, 2.0, 6.3, True), (2, 64, 0.4, 3.2, True), (3, 40, 2.0, 4.9, True), (3, 36, 3.0, 5.5, True),
          (3, 34, 2.0, 4.2, False), (3, 48, 4.0, 8.0, True),
          (2, 16, 2.0, 6.0, True), (3, 12, 2.0, 5.0, True)]   # boxes wider than the grid


@pytest.mark.parametrize("dim,n,lo,hi,kw", SCALAR)
@pytest.mark.parametrize("exterior", [0, 1])
def test_cy_scalar_vs_oracle_and_direct(N, orc, dim, n, lo, hi, kw, exterior):
    delta, u, kappa, coeff = _fields(dim, n, lo, hi, 11)
    alpha = dim + 0.7
    op = N.NonlocalOperator(dim, n, alpha=alpha, delta=delta, coeff=coeff, kappa=kappa if kw else None,
                            exterior=exterior)
    assert op.info.fast_method == 3
    fast = op.apply(u)
    direct, _ = op.apply_direct(u)
    assert orc.rel_inf(fast, direct) <= FAST_TOL
    tg = np.unique(np.concatenate([np.random.default_rng(1).integers(0, n ** dim, 400),
                                   np.arange(0, min(n ** dim, 3 * n)), np.arange(n ** dim - n, n ** dim)]))
    ref, _ = orc.apply(dim, n, u, targets=tg, family=orc.FRACTIONAL, alpha=alpha, delta=delta, coeff=coeff,
                       kappa=kappa if kw else None, exterior=exterior)
    assert orc.rel_inf(fast[tg], ref) <= FAST_TOL


@pytest.mark.parametrize("n,lo,hi", [(96, 3.0, 8.0), (100, 2.0, 4.9), (72, 2.5, 6.5)])
def test_cy_peridynamic_vs_oracle_and_direct(N, orc, n, lo, hi):
    delta, _, _, coeff = _fields(2, n, lo, hi, 12)
    u = np.random.default_rng(13).standard_normal(2 * n * n)
    op = N.NonlocalOperator(2, n, kernel="peridynamic", delta=delta, coeff=coeff)
    fast = op.apply(u)
    direct, _ = op.apply_direct(u)
    assert orc.rel_inf(fast, direct) <= FAST_TOL
    tg = np.unique(np.random.default_rng(2).integers(0, n * n, 400))
    ref, _ = orc.apply(2, n, u, targets=tg, family=orc.PERIDYNAMIC, delta=delta, coeff=coeff, peri=True)
    assert orc.rel_inf(fast.reshape(2, -1)[:, tg].reshape(-1), ref) <= FAST_TOL


def test_cy_every_target_on_a_tie_band(N, orc):
    """A horizon ARRAY equal to 5h everywhere: |d|^2 = 25 sits on every target's
    tie band, so the band pass (reference float predicate, from global memory)
    decides 12 offsets per target in 2-D."""
    n = 64
    h = 1.0 / n
    _, u, kappa, coeff = _fields(2, n, 3.0, 5.0, 14)
    delta = np.full(n * n, 5.0 * h)
    op = N.NonlocalOperator(2, n, alpha=2.6, delta=delta, coeff=coeff, kappa=kappa)
    fast = op.apply(u)
    direct, pairs = op.apply_direct(u)
    ref, rp = orc.apply(2, n, u, family=orc.FRACTIONAL, alpha=2.6, delta=delta, coeff=coeff, kappa=kappa)
    assert pairs == rp
    assert orc.rel_inf(fast, ref) <= FAST_TOL


@pytest.mark.parametrize("dim,n,lo,hi", [(2, 96, 3.0, 7.9), (3, 40, 2.0, 4.9)])
def test_cy_matches_row_lane_sweep(N, dim, n, lo, hi):
    delta, u, kappa, coeff = _fields(dim, n, lo, hi, 15)
    kw = dict(alpha=dim + 0.5, delta=delta, coeff=coeff, kappa=kappa)
    a = N.NonlocalOperator(dim, n, **kw).apply(u)
    os.environ["NLG_ST_CY"] = "0"
    try:
        b = N.NonlocalOperator(dim, n, **kw).apply(u)
    finally:
        del os.environ["NLG_ST_CY"]
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


@pytest.mark.parametrize("dim,n,lo,hi", [(2, 128, 3.0, 7.9), (3, 40, 2.0, 4.9)])
def test_cy_slab_plans_reassemble(N, dim, n, lo, hi):
    """Slab plans (input rows = owned rows + halo, tensor-map coordinates
    relative to the slab) reassemble to the whole-grid apply."""
    from paper_1905_08375_b200 import nonloc as NL
    delta, u, kappa, coeff = _fields(dim, n, lo, hi, 16)
    alpha = dim + 0.5
    whole = N.NonlocalOperator(dim, n, alpha=alpha, delta=delta, coeff=coeff, kappa=kappa).apply(u)
    dmax = float(delta.max())
    halo = NL.halo_rows(dim=dim, n=n, family=4, delta_max=dmax)
    cuts = [0, n // 3, n // 3 + 9, n]
    st = n ** (dim - 1)
    parts = []
    for rb, re in zip(cuts[:-1], cuts[1:]):
        ib, ie = max(0, rb - halo), min(n, re + halo)
        sl = slice(ib * st, ie * st)
        op = N.NonlocalOperator(dim, n, alpha=alpha, delta=delta[sl], coeff=coeff[sl], kappa=kappa[sl],
                                row_begin=rb, row_end=re, reach=dmax)
        parts.append(op.apply(u[sl].copy()))
    got = np.concatenate(parts)
    assert np.max(np.abs(got - whole)) <= 1e-12 * np.max(np.abs(whole))
