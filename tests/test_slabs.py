"""Slab sharding along axis 0.

CPU (not gpu): world_size-2 gloo processes exchange u halos through
paper_1905_08375_b200.slabs and each rank evaluates its rows with the oracle
from ONLY its input slab; the result must equal the whole-grid oracle.
GPU: sharded plans (row_begin/row_end) for every fast method, run one after
another on one device, reassemble to the unsharded result."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _worker(rank, world, port, dim, n, delta, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import oracle as O
    from paper_1905_08375_b200.slabs import Slab
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N = n ** dim
    stride = n ** (dim - 1)
    u = O.random_vector(N, 5)
    halo = int(np.floor(delta * n)) + 2
    sl = Slab(n, stride, halo, rank, world)
    u_in = torch.zeros(sl.n_in, dtype=torch.float64)
    own = sl.output_slice()
    u_in[sl.halo_lo * stride: sl.halo_lo * stride + sl.n_out] = torch.from_numpy(u[own])
    sl.exchange(u_in)
    # rebuild a full-grid array that is zero outside this rank's input slab
    v = np.zeros(N)
    v[sl.in_begin * stride: sl.in_end * stride] = u_in.numpy()
    tg = np.arange(own.start, own.stop)
    got, _ = O.apply(dim, n, v, targets=tg, family=O.FRACTIONAL, alpha=1.5, delta0=delta)
    ref, _ = O.apply(dim, n, u, targets=tg, family=O.FRACTIONAL, alpha=1.5, delta0=delta)
    q.put((rank, O.rel_inf(got, ref), bool(np.array_equal(u_in.numpy(), u[sl.in_begin * stride: sl.in_end * stride]))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dim,n,delta", [(1, 512, 0.05), (2, 32, 0.2)])
def test_gloo_halo_exchange_world2(dim, n, delta):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + dim * 7 + n % 97
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dim, n, delta, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, err, exact in res:
        assert exact, f"rank {rank}: halo rows differ"
        assert err == 0.0, f"rank {rank}: rel {err}"


class _OraclePlan:
    """Stands in for a sharded plan in bench.py's N > 1 step: begin() sees u_in
    before the exchange (records that its halo rows are still unset), end()
    evaluates the slab's output rows with the oracle from u_in alone."""

    def __init__(self, O, sl, dim, n, delta, u_in):
        self.O, self.sl, self.dim, self.n, self.delta, self.u_in = O, sl, dim, n, delta, u_in
        self.begin_saw = None

    def apply_fast_dev_begin(self, u_ptr, out_ptr, stream):
        self.begin_saw = self.u_in.clone()

    def apply_fast_dev_end(self, u_ptr, out_ptr, stream):
        sl, N = self.sl, self.n ** self.dim
        v = np.zeros(N)
        v[sl.in_begin * sl.stride: sl.in_end * sl.stride] = self.u_in.numpy()
        own = sl.output_slice()
        self.out, _ = self.O.apply(self.dim, self.n, v, targets=np.arange(own.start, own.stop),
                                   family=self.O.FRACTIONAL, alpha=1.5, delta0=self.delta)


def _bench_seq_worker(rank, world, port, dim, n, delta, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import oracle as O
    from paper_1905_08375_b200.slabs import Slab, slab_apply
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, stride = n ** dim, n ** (dim - 1)
    u = O.random_vector(N, 6)
    sl = Slab(n, stride, int(np.floor(delta * n)) + 2, rank, world)
    u_in = torch.full((sl.n_in,), float("nan"), dtype=torch.float64)   # halos unset until the exchange
    u_in[sl.halo_lo * stride: sl.halo_lo * stride + sl.n_out] = torch.from_numpy(u[sl.output_slice()])
    plan = _OraclePlan(O, sl, dim, n, delta, u_in)
    slab_apply(sl, plan, u_in, u_in, 0)
    own = sl.output_slice()
    ref, _ = O.apply(dim, n, u, targets=np.arange(own.start, own.stop), family=O.FRACTIONAL, alpha=1.5,
                     delta0=delta)
    halos_unset_at_begin = bool(torch.isnan(plan.begin_saw).any()) if sl.n_in > sl.n_out else True
    q.put((rank, O.rel_inf(plan.out, ref), halos_unset_at_begin))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dim,n,delta", [(1, 512, 0.05), (3, 16, 0.25)])
def test_gloo_bench_slab_sequence_world2(dim, n, delta):
    """bench.py's N > 1 step (slabs.slab_apply: begin -> exchange -> end) with
    the oracle standing in for the plan reproduces the whole-grid oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29650 + dim * 11 + n % 89
    procs = [ctx.Process(target=_bench_seq_worker, args=(r, 2, port, dim, n, delta, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, err, unset in res:
        assert err == 0.0, f"rank {rank}: rel {err}"
        assert unset, f"rank {rank}: begin() already saw halo values"


def test_bench_multi_gpu_fails_loudly_without_gpus():
    """--gpus 2 on a box without two GPUs must not silently run one rank."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "--gpus 2" in (r.stderr + r.stdout)


def test_slab_rows_partition():
    from paper_1905_08375_b200.slabs import slab_rows
    for n in (7, 64, 4096, 768):
        for w in (1, 2, 3, 4, 8):
            rows = [slab_rows(n, w, r) for r in range(w)]
            assert rows[0][0] == 0 and rows[-1][1] == n
            assert all(rows[i][1] == rows[i + 1][0] for i in range(w - 1))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cfg1_small", "trunc2d", "frac2d", "peri2d"])
def test_sharded_plans_match_unsharded(case, orc):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1905_08375_b200 import nonloc as N, configs
    from paper_1905_08375_b200.slabs import Slab
    if case == "cfg1_small":
        w = configs.cfg1(1 << 16)
        kw = w.op_kwargs()
        dim, n, u, comps = 1, w.n, w.u, 1
    elif case == "trunc2d":
        dim, n, comps = 2, 64, 1
        u = orc.random_vector(n * n, 3)
        kw = None
    elif case == "frac2d":
        dim, n, comps = 2, 64, 1
        rng = np.random.default_rng(2)
        u = rng.standard_normal(n * n)
        kw = dict(kernel="fractional", alpha=3.0, delta=(4 + 8 * rng.random(n * n)) / n,
                  coeff=1 + rng.random(n * n), kappa=np.exp(0.5 * rng.standard_normal(n * n)))
    else:
        dim, n, comps = 2, 64, 2
        rng = np.random.default_rng(3)
        u = rng.standard_normal(2 * n * n)
        kw = dict(kernel="peridynamic", delta=(3 + 5 * rng.random(n * n)) / n, coeff=1 + 9 * (rng.random(n * n) < .3))
    N_ = n ** dim
    stride = n ** (dim - 1)
    if kw is None:
        full = N.Plan(dim=dim, n=n, family=0, route=0, poly=np.array([1.0]), rule=0, form=0, delta0=0.2)
        ref = full.apply_fast(u)
    else:
        ref = N.NonlocalOperator(dim, n, **kw).apply(u)
    world = 3
    parts = []
    for r in range(world):
        if kw is None:
            halo = N.halo_rows(dim=dim, n=n, family=0, delta_max=0.2, route=0, rule=0, form=0)
        else:
            dmax = float(np.max(kw["delta"])) if kw.get("delta") is not None else kw["delta0"]
            halo = N.halo_rows(dim=dim, n=n, family=4 if kw["kernel"] == "fractional" else 5, delta_max=dmax)
        sl = Slab(n, stride, halo, r, world)
        if kw is None:
            p = N.Plan(dim=dim, n=n, family=0, route=0, poly=np.array([1.0]), rule=0, form=0, delta0=0.2,
                       row_begin=sl.row_begin, row_end=sl.row_end)
        else:
            k2 = dict(kw)
            for key in ("delta", "coeff", "kappa"):
                if k2.get(key) is not None:
                    k2[key] = sl.input_slice(k2[key])
            p = N.NonlocalOperator(dim, n, row_begin=sl.row_begin, row_end=sl.row_end, reach=dmax, **k2).plan
        assert p.info.halo_lo == sl.halo_lo and p.info.halo_hi == sl.halo_hi
        if comps == 1:
            ui = sl.input_slice(u)
        else:
            ui = np.concatenate([sl.input_slice(u[c * N_:(c + 1) * N_]) for c in range(comps)])
        parts.append(p.apply_fast(ui).reshape(comps, -1))
    got = np.concatenate(parts, axis=1).reshape(-1)
    # each shard fits its own far-tail exponential sum from its own horizons
    # (1-D FFT mode), so the 1-D case agrees to the fit level, not bit-near
    assert orc.rel_inf(got, ref) <= (1e-11 if case == "cfg1_small" else 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
def test_cfg1_full_size_slabs_as_in_bench(world, orc):
    """The exact slab plans bench.py --gpus N builds for the headline cfg1
    (2^22 nodes, 62916-cell halos), applied one after the other on this GPU,
    reassemble to the single-plan output; each slab's FFT length comes from its
    own input rows."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1905_08375_b200 import nonloc as N, configs
    from paper_1905_08375_b200.slabs import Slab
    w = configs.cfg1()
    ref = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs()).apply(w.u)
    dmax = float(w.delta.max())
    halo = N.halo_rows(dim=1, n=w.n, family=4, delta_max=dmax)
    parts = []
    for r in range(world):
        sl = Slab(w.n, 1, halo, r, world)
        kw = w.op_kwargs()
        for key in ("delta", "coeff", "kappa"):
            kw[key] = sl.input_slice(kw[key])
        op = N.NonlocalOperator(1, w.n, row_begin=sl.row_begin, row_end=sl.row_end, reach=dmax, **kw)
        assert op.info.fast_method == 2 and op.info.fft_len > 0
        parts.append(op.apply(sl.input_slice(w.u)))
    got = np.concatenate(parts)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))

def _two_plane_worker(rank, world, port, n, halo, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_1905_08375_b200.slabs import Slab, slab_apply
    dist.init_process_group("gloo", rank=rank, world_size=world)
    stride = n
    u = np.random.default_rng(8).standard_normal(2 * n * n)
    sl = Slab(n, stride, halo, rank, world)
    own = sl.output_slice()
    u_in = torch.full((2 * sl.n_in,), float("nan"), dtype=torch.float64)
    for c in range(2):
        o = c * sl.n_in + sl.halo_lo * stride
        u_in[o:o + sl.n_out] = torch.from_numpy(u[c * n * n:(c + 1) * n * n][own])

    class P:
        components = 2

        def apply_fast_dev_begin(self, *a):
            pass

        def apply_fast_dev_end(self, *a):
            pass

    slab_apply(sl, P(), u_in, u_in, 0)
    want = np.concatenate([u[c * n * n:(c + 1) * n * n][sl.in_begin * stride: sl.in_end * stride] for c in range(2)])
    q.put((rank, bool(np.array_equal(u_in.numpy(), want))))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_component_halo_exchange_world2():
    """slab_apply on a two-component field (peridynamics, SoA planes): every
    plane's halo rows arrive from the neighbour's owned rows of the same plane."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_plane_worker, args=(r, 2, 29811, 48, 9, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, exact in res:
        assert exact, f"rank {rank}: halo rows of a component plane differ"
