"""The chunked host pipeline of nlg_apply_fast (plan.cu apply_fast_pipelined:
row chunks of u H2D on one copy stream, the apply of every output row range
whose window is resident, D2H of finished rows on a second copy stream) and
the split-phase device apply used for the multi-GPU halo overlap
(nlg_apply_fast_dev_begin / _end). Each piece runs the same per-element
arithmetic as the single-shot device apply, so the results must be identical
to the last bit; the pipeline is also checked against the GPU direct
quadrature (exact pair sets) on sampled targets within the north-star 1e-10."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1905_08375_b200 import nonloc
    return nonloc


def _dev_apply(op, u, split=False):
    import torch
    plan = op.plan
    ud = torch.from_numpy(u).cuda()
    od = torch.empty(plan.n_out, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    if split:
        plan.apply_fast_dev_begin(ud.data_ptr(), od.data_ptr(), s)
        plan.apply_fast_dev_end(ud.data_ptr(), od.data_ptr(), s)
    else:
        plan.apply_fast_dev(ud.data_ptr(), od.data_ptr(), s)
    torch.cuda.synchronize()
    return od.cpu().numpy()


def _box_op(N, n, dh=6.0, s=0.25, **kw):
    from paper_1905_08375_b200 import nonloc as NL
    rng = np.random.default_rng(2)
    d0 = dh / n
    return N.NonlocalOperator(3, n, alpha=3 + 2 * s, delta0=d0, coeff0=float(NL.fractional_cdelta(3, s, d0)),
                              kappa=rng.lognormal(0.0, 0.5, n ** 3), **kw)


@pytest.mark.parametrize("n", [162, 192])
def test_pipeline_box_fft_bitwise(N, n):
    """3-D constant horizon (box FFT + tie pass), >= 4 Mi nodes: the pipelined
    host apply equals the device apply bit for bit."""
    op = _box_op(N, n)
    assert op.info.fast_method == 3 and op.info.fft_len > 0
    u = np.random.default_rng(1).standard_normal(n ** 3)
    host = op.apply(u)
    dev = _dev_apply(op, u)
    assert np.array_equal(host, dev)
    tg = np.random.default_rng(3).choice(n ** 3, 512, replace=False)
    tg = np.concatenate([tg, [0, n ** 3 - 1, (n // 2) * n * n]])
    ref = op.apply_direct_at(u, tg)
    assert np.max(np.abs(host[tg] - ref)) <= 1e-10 * np.max(np.abs(ref))


def test_pipeline_stencil_2d_bitwise(N):
    """2-D variable horizon (offset-table stencil, cfg2 family) at 2048^2."""
    from paper_1905_08375_b200 import configs
    w = configs.cfg2(2048)
    op = N.NonlocalOperator(2, 2048, **w.op_kwargs())
    host = op.apply(w.u)
    dev = _dev_apply(op, w.u)
    assert np.array_equal(host, dev)


def test_pipeline_peridynamic_2d_bitwise(N):
    """2-D peridynamics (cfg3 family, two component planes) at 2048^2: the row
    chunks of both planes travel and are computed per output row range."""
    import torch
    from paper_1905_08375_b200 import configs
    w = configs.cfg3(2048)
    op = N.NonlocalOperator(2, 2048, **w.op_kwargs())
    host = op.apply(w.u)
    plan = op.plan
    ud = torch.from_numpy(w.u).cuda()
    od = torch.empty(2 * plan.n_out, dtype=torch.float64, device="cuda")
    plan.apply_fast_dev(ud.data_ptr(), od.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(host, od.cpu().numpy())
    tg = np.random.default_rng(3).choice(2048 ** 2, 512, replace=False)
    ref = op.apply_direct_at(w.u, tg)
    assert np.max(np.abs(host.reshape(2, -1)[:, tg].reshape(-1) - ref)) <= 1e-10 * np.max(np.abs(ref))


def test_pipeline_stencil_3d_variable_bitwise(N):
    """3-D variable horizon (cfg4-B family) at 168^3."""
    from paper_1905_08375_b200 import configs
    w = configs.cfg4(168, variable=True)
    op = N.NonlocalOperator(3, 168, **w.op_kwargs())
    assert op.info.fft_len == 0
    host = op.apply(w.u)
    dev = _dev_apply(op, w.u)
    assert np.array_equal(host, dev)


def test_pipeline_off_matches(N, monkeypatch):
    op = _box_op(N, 162)
    u = np.random.default_rng(5).standard_normal(162 ** 3)
    a = op.apply(u)
    monkeypatch.setenv("NLG_NO_PIPELINE", "1")
    b = op.apply(u)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("rows", [(0, 40), (40, 90), (90, 128)])
def test_split_phase_box_slab(N, rows):
    """begin + end on a sharded box-FFT slab plan equals the one-call device apply."""
    from paper_1905_08375_b200 import nonloc as NL
    n, dh = 128, 6.0
    d0 = dh / n
    rng = np.random.default_rng(2)
    kappa = rng.lognormal(0.0, 0.5, n ** 3)
    halo = NL.halo_rows(dim=3, n=n, family=4, delta_max=d0)
    rb, re = rows
    ib, ie = max(0, rb - halo), min(n, re + halo)
    sl = slice(ib * n * n, ie * n * n)
    op = N.NonlocalOperator(3, n, alpha=3.5, delta0=d0, coeff0=float(NL.fractional_cdelta(3, 0.25, d0)),
                            kappa=kappa[sl], row_begin=rb, row_end=re, reach=d0)
    u = np.random.default_rng(1).standard_normal(n ** 3)[sl].copy()
    a = _dev_apply(op, u)
    b = _dev_apply(op, u, split=True)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("dim,n,rows", [(2, 512, (128, 320)), (2, 512, (0, 200)), (3, 96, (30, 70)), (3, 96, (60, 96))])
def test_split_phase_stencil_slab(N, dim, n, rows):
    """begin (interior output rows) + end (edge rows) on a sharded stencil slab
    (variable horizon: cfg2 / cfg4-B families) equals the one-call device apply."""
    from paper_1905_08375_b200 import configs, nonloc as NL
    w = configs.cfg2(n) if dim == 2 else configs.cfg4(n, variable=True)
    dmax = float(w.delta.max())
    halo = NL.halo_rows(dim=dim, n=n, family=4, delta_max=dmax)
    rb, re = rows
    st = n ** (dim - 1)
    ib, ie = max(0, rb - halo), min(n, re + halo)
    sl = slice(ib * st, ie * st)
    kw = w.op_kwargs()
    for key in ("delta", "coeff", "kappa"):
        kw[key] = kw[key][sl] if kw[key] is not None else None
    op = N.NonlocalOperator(dim, n, row_begin=rb, row_end=re, reach=dmax, **kw)
    assert op.info.fast_method == 3 and op.info.fft_len == 0
    u = w.u[sl].copy()
    a = _dev_apply(op, u)
    b = _dev_apply(op, u, split=True)
    assert np.array_equal(a, b)


def test_split_phase_peridynamic_slab(N):
    """begin + end on a sharded 2-D peridynamic slab (two component planes,
    strided by the slab's n_in / n_out) equals the one-call device apply."""
    import torch
    from paper_1905_08375_b200 import configs, nonloc as NL
    n, (rb, re) = 512, (128, 330)
    w = configs.cfg3(n)
    dmax = float(w.delta.max())
    halo = NL.halo_rows(dim=2, n=n, family=5, delta_max=dmax)
    ib, ie = max(0, rb - halo), min(n, re + halo)
    sl = slice(ib * n, ie * n)
    kw = w.op_kwargs()
    for key in ("delta", "coeff"):
        kw[key] = kw[key][sl] if kw[key] is not None else None
    op = N.NonlocalOperator(2, n, row_begin=rb, row_end=re, reach=dmax, **kw)
    u = np.concatenate([w.u[:n * n][sl], w.u[n * n:][sl]])
    plan = op.plan
    ud = torch.from_numpy(u).cuda()
    s = torch.cuda.current_stream().cuda_stream
    outs = []
    for split in (False, True):
        od = torch.zeros(2 * plan.n_out, dtype=torch.float64, device="cuda")
        if split:
            plan.apply_fast_dev_begin(ud.data_ptr(), od.data_ptr(), s)
            plan.apply_fast_dev_end(ud.data_ptr(), od.data_ptr(), s)
        else:
            plan.apply_fast_dev(ud.data_ptr(), od.data_ptr(), s)
        torch.cuda.synchronize()
        outs.append(od.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    whole = N.NonlocalOperator(2, n, **w.op_kwargs()).apply(w.u).reshape(2, n, n)[:, rb:re].reshape(-1)
    assert np.max(np.abs(outs[0] - whole)) <= 1e-12 * np.max(np.abs(whole))


@pytest.mark.parametrize("case", ["box", "stencil3d"])
def test_pipeline_sharded_slab_bitwise(N, case):
    """The host pipeline on a sharded slab plan (input rows = owned rows +
    halos, the per-rank e2e path of bench.py --gpus N) equals its device apply."""
    from paper_1905_08375_b200 import configs, nonloc as NL
    n = 192
    w = configs.cfg4(n) if case == "box" else configs.cfg4(n, variable=True)
    dmax = float(w.delta.max()) if w.delta is not None else w.delta0
    halo = NL.halo_rows(dim=3, n=n, family=4, delta_max=dmax)
    rb, re = 70, 190
    st = n * n
    ib, ie = rb - halo, min(n, re + halo)
    sl = slice(ib * st, ie * st)
    kw = w.op_kwargs()
    for key in ("delta", "coeff", "kappa"):
        kw[key] = kw[key][sl] if kw[key] is not None else None
    op = N.NonlocalOperator(3, n, row_begin=rb, row_end=re, reach=dmax, **kw)
    assert (op.info.fft_len > 0) == (case == "box")
    assert op.plan.n_out >= 1 << 22   # the pipelined host path
    u = w.u[sl].copy()
    assert np.array_equal(op.apply(u), _dev_apply(op, u))
