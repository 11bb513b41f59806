"""Multi-GPU plans inside the C-ABI (nlg_group_*, csrc/group.cu): axis-0
slabs, one sharded plan per device, halo rows exchanged device to device
(NCCL point-to-point when the devices are distinct, peer copies when one GPU
stands in for several slabs), overlapped with the halo-independent part of
each slab's apply. The reassembled output must equal the single-plan apply:
the slab plans evaluate the same sums (sharded vs unsharded
<= 1e-12)."""
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


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def _group_vs_single(N, w, devices):
    A = N.A
    fam = A.PERIDYNAMIC if w.kernel == "peridynamic" else A.FRACTIONAL
    kw = dict(dim=w.dim, n=w.n, family=fam, alpha=w.alpha, exterior=w.exterior, delta=w.delta, delta0=w.delta0,
              coeff=w.coeff, coeff0=w.coeff0, kappa=w.kappa)
    g = N.Group(devices, **kw)
    out = g.apply(w.u)
    single = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs()).apply(w.u)
    return g, out, single


@pytest.mark.parametrize("ndev", [1, 3])
def test_group_box_fft(N, ndev):
    from paper_1905_08375_b200 import configs
    w = configs.cfg4(64)
    g, out, single = _group_vs_single(N, w, [0] * ndev)
    assert g.ndev == ndev and not g.nccl
    assert list(g.row_begin) == sorted(g.row_begin) and g.row_end[-1] == 64
    assert _rel(out, single) <= 1e-12


def test_group_stencil_2d(N):
    from paper_1905_08375_b200 import configs
    w = configs.cfg2(256)
    _, out, single = _group_vs_single(N, w, [0, 0, 0, 0])
    assert _rel(out, single) <= 1e-12


def test_group_stencil_3d_variable(N):
    from paper_1905_08375_b200 import configs
    w = configs.cfg4(64, variable=True)
    _, out, single = _group_vs_single(N, w, [0, 0])
    assert _rel(out, single) <= 1e-12


def test_group_peridynamics(N):
    from paper_1905_08375_b200 import configs
    w = configs.cfg3(128)
    _, out, single = _group_vs_single(N, w, [0, 0, 0])
    assert _rel(out, single) <= 1e-12


def test_group_expsum_1d(N):
    from paper_1905_08375_b200 import configs
    w = configs.cfg1(1 << 16)
    _, out, single = _group_vs_single(N, w, [0, 0, 0])
    assert _rel(out, single) <= 1e-11


def test_group_dev_pointers(N):
    """nlg_group_apply_fast_dev: only the owned rows are filled by the caller."""
    import torch
    from paper_1905_08375_b200 import configs
    w = configs.cfg4(48)
    A = N.A
    g = N.Group([0, 0], dim=3, n=48, family=A.FRACTIONAL, alpha=w.alpha, delta0=w.delta0, coeff0=w.coeff0,
                kappa=w.kappa)
    st = 48 * 48
    us, outs = [], []
    for k in range(2):
        u = torch.full((int(g.n_in[k]),), float("nan"), dtype=torch.float64, device="cuda")
        us.append(u)
        outs.append(torch.empty((int(g.row_end[k]) - int(g.row_begin[k])) * st, dtype=torch.float64, device="cuda"))
    # owned rows at offset halo_lo rows of each input buffer
    halo_lo = [0, int(g.n_in[1]) // st - (int(g.row_end[1]) - int(g.row_begin[1]))]
    for k in range(2):
        rb, re = int(g.row_begin[k]), int(g.row_end[k])
        us[k][halo_lo[k] * st:(halo_lo[k] + re - rb) * st] = torch.from_numpy(w.u[rb * st:re * st]).cuda()
    g.apply_dev([u.data_ptr() for u in us], [o.data_ptr() for o in outs])
    out = torch.cat(outs).cpu().numpy()
    single = N.NonlocalOperator(3, 48, **w.op_kwargs()).apply(w.u)
    assert _rel(out, single) <= 1e-12


def test_group_nccl_single_device(N, monkeypatch):
    """NLG_GROUP_NCCL=1 builds an NCCL communicator even for one device (the
    dlopen / ncclCommInitAll / async-error path on a one-GPU box)."""
    from paper_1905_08375_b200 import configs
    monkeypatch.setenv("NLG_GROUP_NCCL", "1")
    w = configs.cfg4(40)
    g, out, single = _group_vs_single(N, w, [0])
    assert g.nccl
    assert _rel(out, single) <= 1e-12


def test_group_nccl_two_devices(N):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_1905_08375_b200 import configs
    w = configs.cfg4(64)
    g, out, single = _group_vs_single(N, w, [0, 1])
    assert g.nccl
    assert _rel(out, single) <= 1e-12


def test_group_rejects_thin_slabs(N):
    from paper_1905_08375_b200 import configs
    w = configs.cfg4(32)
    with pytest.raises(ValueError):
        _group_vs_single(N, w, [0] * 8)   # 4-plane slabs, 8-plane halo
