"""The reference's own fast route (TruncatedOperator, operators.cpp:102-167) on
the GPU scan kernels (csrc/spans.cu):
  * K = 0, any d: single-pass row prefix sums with decoupled look-back
    (scan_lookback) + exact Leaf spans;
  * 1-D K = 1..3: centred moment scans (moment_scan / moment_eval), the
    re-based Steps 2 + 3 (tree.cpp:115-161, operators.cpp:139-164).
Checked against the restated dense Leaf oracle (apply_truncated_dense,
operators.cpp:169-204) and the GPU direct quadrature at sizes where the oracle
is slow: K = 0 <= 1e-12 (test_operators.cpp:64,85), K >= 1 <= 1e-10
(nonloc_main.cpp:85)."""
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


def _dense(dim, n, K, hk, d0, u):
    import oracle as O
    out, _ = O.apply(dim, n, u, family=O.TRUNCATED, route=O.ROUTE_TRUNCATED, poly=O.match_polynomial(K),
                     rule=O.LEAF, form=O.MASS, delta=O.bump_horizon(dim, n, d0) if hk else None, delta0=d0)
    return out


def _op(N, dim, n, K, hk, d0):
    spec = N.KernelSpec(dim, N.RadialProfile.truncated_polynomial(K), N.HorizonField(N.HorizonKind(hk), d0))
    return N.TruncatedOperator(spec, N.Grid.make(dim, n))


@pytest.mark.parametrize("K", [1, 2, 3])
@pytest.mark.parametrize("n,hk,d0", [(4096, 0, 0.01), (4096, 0, 0.02), (2048, 1, 0.25), (8192, 1, 0.005),
                                     (1024, 0, 0.003)])
def test_moment_scans_vs_dense_leaf(N, K, n, hk, d0):
    """1-D K >= 1 fast apply (method 4) vs the dense Leaf oracle, incl. delta = 0.01
    (where the reference's raw-moment fast path loses digits for K >= 2) and
    horizons narrower than a 16-node segment."""
    u = np.random.default_rng(40 + K).standard_normal(n)
    op = _op(N, 1, n, K, hk, d0)
    assert op.fast_method() == 4
    out = op.apply(u)
    assert _rel(out, _dense(1, n, K, hk, d0, u)) <= 1e-10


@pytest.mark.parametrize("K", [0, 3])
def test_scans_large_vs_direct(N, K):
    """2^20 nodes, bump horizon delta0 = 0.005 (5-10k cells, hundreds of
    look-back tiles / moment segments per span) vs the GPU direct Leaf sum on
    sampled targets, both ends included."""
    n, d0 = 1 << 20, 0.005
    u = np.random.default_rng(7).standard_normal(n)
    op = _op(N, 1, n, K, 1, d0)
    out = op.apply(u)
    tg = np.concatenate([[0, 1, n // 2, n - 2, n - 1], np.random.default_rng(8).choice(n, 256, replace=False)])
    ref = op._plan.apply_direct_at(u, tg)
    tol = 1e-12 if K == 0 else 1e-10
    assert np.max(np.abs(out[tg] - ref)) <= tol * np.max(np.abs(out))


def test_lookback_repeat_bitwise(N):
    """The look-back flags carry the apply's epoch: repeated applies (no reset
    between them) give identical results, and a different u gives its own."""
    n = 1 << 18
    op = _op(N, 1, n, 0, 1, 0.01)
    u1 = np.random.default_rng(1).standard_normal(n)
    u2 = np.random.default_rng(2).standard_normal(n)
    a = op.apply(u1)
    b = op.apply(u2)
    c = op.apply(u1)
    d = op.apply(u2)
    assert np.array_equal(a, c) and np.array_equal(b, d)
    assert _rel(a, _dense(1, n, 0, 1, 0.01, u1)) <= 1e-12


@pytest.mark.parametrize("dim,n,d0", [(2, 256, 8.0 / 256), (2, 2048, 4.0 / 2048), (3, 32, 6.0 / 32)])
def test_lookback_rows_2d_3d(N, dim, n, d0):
    """K = 0 in 2-D / 3-D: one look-back chain per grid row (several tiles per
    row at n = 2048)."""
    u = np.random.default_rng(3).standard_normal(n ** dim)
    op = _op(N, dim, n, 0, 0, d0)
    out = op.apply(u)
    if n ** dim <= 1 << 17:
        assert _rel(out, _dense(dim, n, 0, 0, d0, u)) <= 1e-12
    tg = np.random.default_rng(4).choice(n ** dim, 256, replace=False)
    ref = op._plan.apply_direct_at(u, tg)
    assert np.max(np.abs(out[tg] - ref)) <= 1e-12 * np.max(np.abs(out))


def test_moment_scans_sharded(N):
    """Slab plans (row ranges + halos) of the moment scans reassemble to the
    whole-grid apply."""
    from paper_1905_08375_b200 import nonloc as NL
    n, K, d0 = 4096, 2, 0.01
    u = np.random.default_rng(9).standard_normal(n)
    whole = _op(N, 1, n, K, 0, d0).apply(u)
    poly = NL.match_polynomial(K)
    halo = NL.halo_rows(dim=1, n=n, family=NL.A.TRUNCATED, delta_max=d0, route=NL.A.ROUTE_TRUNCATED,
                        rule=NL.A.LEAF, form=NL.A.MASS, poly=poly)
    parts = []
    for rb, re in [(0, 1000), (1000, 3001), (3001, 4096)]:
        ib, ie = max(0, rb - halo), min(n, re + halo)
        p = NL.Plan(dim=1, n=n, family=NL.A.TRUNCATED, route=NL.A.ROUTE_TRUNCATED, poly=poly, rule=NL.A.LEAF,
                    form=NL.A.MASS, delta0=d0, reach=d0, row_begin=rb, row_end=re)
        assert p.info.fast_method == 4
        parts.append(p.apply_fast(u[ib:ie]))
    assert _rel(np.concatenate(parts), whole) <= 1e-12
