"""The reference's own pinned behaviours of the dense truncated oracle, mirrored
on the GPU routes (each test cites the reference case it restates), plus the
peridynamic known-answer tests SURVEY §8(c) derives for cfg3 (there is no
reference peridynamics): a symmetric discrete operator and exact row
translation invariance for constant c and delta."""
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


def _truncated(N, dim, K, kind, d0):
    return N.KernelSpec(dim, N.RadialProfile.truncated_polynomial(K), N.HorizonField(kind, d0))


def test_point_rule_mass_defect(N):
    """test_operators.cpp:107-115: constant u, Point rule, K=0, 1-D n=512,
    delta=1/4 -> |out(mid)| <= 2h/delta^3 (h #included - 2 delta is O(h))."""
    g = N.Grid.make(1, 512)
    spec = _truncated(N, 1, 0, N.HorizonKind.Constant, 0.25)
    out = N.apply_truncated_dense(spec, g, N.InclusionRule.Point, np.ones(g.total))
    bound = 2.0 * g.h / 0.25 ** 3 + 1e-12
    assert abs(out[g.total // 2]) <= bound


def test_leaf_point_gap_shrinks_with_h(N, orc):
    """test_operators.cpp:116-133: Leaf and Point rules differ (K=1, delta=1/4)
    and halving h shrinks the gap."""
    prev = None
    for n in (512, 1024):
        g = N.Grid.make(1, n)
        spec = _truncated(N, 1, 1, N.HorizonKind.Constant, 0.25)
        u = orc.random_vector(g.total, 3)
        leaf = N.apply_truncated_dense(spec, g, N.InclusionRule.Leaf, u)
        point = N.apply_truncated_dense(spec, g, N.InclusionRule.Point, u)
        diff = np.max(np.abs(leaf - point))
        assert diff > 0.0
        if prev is not None:
            assert diff < prev
        prev = diff


def test_dense_rows_translation_invariant(N):
    """test_operators.cpp:214-234: rows of the assembled Leaf/Mass matrix
    (1-D n=128, K=1, delta=1/8) whose stencils clear the boundary hold the same
    multiset of nonzeros, compared EXACTLY."""
    g = N.Grid.make(1, 128)
    spec = _truncated(N, 1, 1, N.HorizonKind.Constant, 0.125)
    a = N.assemble_dense_matrix(spec, g, N.InclusionRule.Leaf, N.ApplyForm.Mass).reshape(g.total, g.total)
    lo, hi = 32, 96
    base = np.sort(a[lo][a[lo] != 0.0])
    for i in range(lo + 1, hi):
        row = np.sort(a[i][a[i] != 0.0])
        assert row.size == base.size
        assert np.array_equal(row, base)


def test_fast_truncated_rows_translation_invariant(N):
    """The same invariance through the fast route (TruncatedOperator, K=0): the
    response to a unit impulse shifted by s is the shifted response, on nodes
    whose windows clear the boundary (span sums of a single nonzero)."""
    n = 256
    g = N.Grid.make(1, n)
    op = N.TruncatedOperator(_truncated(N, 1, 0, N.HorizonKind.Constant, 0.0625), g)
    W = int(0.0625 * n) + 2
    resp = []
    for j in (100, 101, 117, 140):
        e = np.zeros(n)
        e[j] = 1.0
        resp.append((j, op.apply(e)))
    j0, r0 = resp[0]
    for j, r in resp[1:]:
        s = j - j0
        win = slice(j0 - W, j0 + W + 1)
        win_s = slice(j0 - W + s, j0 + W + 1 + s)
        assert np.max(np.abs(r[win_s] - r0[win])) <= 1e-15 * np.max(np.abs(r0))


def _peri(N, n, dh=4.5, c=2.0):
    h = 1.0 / n
    return N.NonlocalOperator(2, n, kernel="peridynamic", delta0=dh * h, coeff0=c)


@pytest.mark.parametrize("route", ["direct", "fast"])
def test_peridynamics_symmetric_operator(N, route):
    """SURVEY §8(c) derived KAT: for constant c and delta the discrete
    peridynamic operator is symmetric, <A u, v> = <u, A v>, and its explicit
    matrix (columns = responses to unit impulses, 2-D n=12, both components)
    equals its transpose."""
    n = 12
    op = _peri(N, n)
    apply = (lambda x: op.apply_direct(x)[0]) if route == "direct" else op.apply
    M = 2 * n * n
    A = np.empty((M, M))
    for j in range(M):
        e = np.zeros(M)
        e[j] = 1.0
        A[:, j] = apply(e)
    assert np.max(np.abs(A - A.T)) <= 1e-13 * np.max(np.abs(A))
    rng = np.random.default_rng(7)
    u, v = rng.standard_normal(M), rng.standard_normal(M)
    lhs, rhs = np.dot(apply(u), v), np.dot(u, apply(v))
    assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + abs(rhs))


@pytest.mark.parametrize("route", ["direct", "fast"])
def test_peridynamics_row_translation_invariance(N, route):
    """SURVEY §8(c) derived KAT: for constant c and delta, interior rows of the
    peridynamic operator are shifts of each other. The response to a unit
    impulse (each component) moved by (sy, sx) is the moved response; the
    direct route reproduces it bit for bit."""
    n = 64   # power of two: node coordinates and offsets are exact dyadics
    op = _peri(N, n)
    apply = (lambda x: op.apply_direct(x)[0]) if route == "direct" else op.apply
    tol = 0.0 if route == "direct" else 1e-14
    R = 7
    for comp in (0, 1):
        def resp(y, x):
            e = np.zeros(2 * n * n)
            e[comp * n * n + y * n + x] = 1.0
            return apply(e).reshape(2, n, n)
        y0, x0 = 20, 20
        r0 = resp(y0, x0)
        sc = np.max(np.abs(r0))
        for sy, sx in ((0, 1), (3, -2), (-5, 4)):
            r = resp(y0 + sy, x0 + sx)
            a = r0[:, y0 - R:y0 + R + 1, x0 - R:x0 + R + 1]
            b = r[:, y0 + sy - R:y0 + sy + R + 1, x0 + sx - R:x0 + sx + R + 1]
            assert np.max(np.abs(a - b)) <= tol * sc
