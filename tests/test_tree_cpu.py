"""Step-1 tree API (§8(f) row 3; reference include/nonloc/tree.hpp,
src/tree.cpp, tests/test_tree.cpp): panel lists, recursion counts and moments
against the compiled reference (tests/golden/tree_api.npz), plus the
reference's own properties (cover equivalence, disjointness, no listed
ancestor, slopes). Host code in libnlgpu; no GPU needed."""
import numpy as np
import pytest

from conftest import golden


@pytest.fixture(scope="module")
def N():
    from paper_1905_08375_b200 import build
    build.build()
    from paper_1905_08375_b200 import nonloc
    return nonloc


def test_decompositions_match_reference(N):
    g = golden("tree_api")
    for k in range(int(g["ndecomp"])):
        dim, n = int(g[f"d{k}_dim"]), int(g[f"d{k}_n"])
        d = N.decompose_region(N.build_tree(N.Grid.make(dim, n)), g[f"d{k}_c"], float(g[f"d{k}_r"]))
        assert d.recur_calls == int(g[f"d{k}_recur"])
        assert [p.level for p in d.panels] == list(g[f"d{k}_levels"])       # same order
        assert [p.index for p in d.panels] == list(g[f"d{k}_indices"])


def test_count_recur_calls_matches_reference(N):
    g = golden("tree_api")
    for dim, n in ((1, 256), (2, 32), (3, 8)):
        t = N.build_tree(N.Grid.make(dim, n))
        assert N.count_recur_calls(t, g[f"radii{dim}"]) == int(g[f"recur{dim}"])


def test_moments_match_reference(N):
    g = golden("tree_api")
    for dim, n, K in ((1, 16, 0), (1, 16, 3), (2, 8, 0), (3, 4, 0)):
        adds = []
        m = N.accumulate_moments(N.build_tree(N.Grid.make(dim, n)), g[f"mom{dim}_{K}_u"], K, adds)
        assert np.array_equal(np.concatenate(m.levels), g[f"mom{dim}_{K}"])   # bit-identical
        assert adds[0] == int(g[f"mom{dim}_{K}_adds"])
    with pytest.raises(ValueError):                      # test_tree.cpp:208-212
        N.accumulate_moments(N.build_tree(N.Grid.make(2, 4)), np.zeros(16), 1)


def brute(grid, c, r):
    """leaf-rule node set of the ball (cube_intersects_ball on leaf boxes)"""
    out = set()
    for i in range(grid.total):
        x = N_node_k(grid, i)
        d2 = 0.0
        for j in range(grid.dim):
            lo, hi = x[j] * grid.h, (x[j] + 1) * grid.h
            if lo > c[j]:
                d2 += (lo - c[j]) ** 2
            elif hi < c[j]:
                d2 += (hi - c[j]) ** 2
        if d2 < r * r:
            out.add(i)
    return out


def N_node_k(grid, i):
    k, rest = [0, 0, 0], i
    for j in range(grid.dim - 1, -1, -1):
        k[j] = rest % grid.n
        rest //= grid.n
    return k


def covered(tree, d):
    nodes = []
    g = tree.grid
    for p in d.panels:
        span = 1 << (tree.depth - p.level)
        per = 1 << p.level
        k, rest = [0, 0, 0], p.index
        for j in range(g.dim - 1, -1, -1):
            k[j] = rest % per
            rest //= per
        ranges = [range(k[j] * span, (k[j] + 1) * span) for j in range(g.dim)]
        import itertools
        for idx in itertools.product(*ranges):
            f = 0
            for j in range(g.dim):
                f = f * g.n + idx[j]
            nodes.append(f)
    return nodes


def test_cover_equivalence_and_disjointness(N):         # test_tree.cpp:91-133
    rng = np.random.default_rng(5)
    for dim, n in ((1, 32), (2, 16), (3, 8)):
        grid = N.Grid.make(dim, n)
        t = N.build_tree(grid)
        for _ in range(20):
            c = rng.random(dim)
            r = 0.05 + 0.6 * rng.random()
            d = N.decompose_region(t, c, r)
            nodes = covered(t, d)
            assert len(nodes) == len(set(nodes))              # disjoint
            assert set(nodes) == brute(grid, c, r)            # exactly the leaf-rule set
            listed = {(p.level, p.index) for p in d.panels}
            for p in d.panels:                                 # no listed ancestor
                q = p
                while q.level > 0:
                    q = t.parent(q)
                    assert (q.level, q.index) not in listed


def test_recur_count_slopes(N):                          # test_tree.cpp:214-249
    t = N.build_tree(N.Grid.make(1, 64))
    assert N.count_recur_calls(t, np.full(64, 2.0)) == 64
    xs, ys = [], []
    for n in (256, 512, 1024, 2048, 4096):
        t = N.build_tree(N.Grid.make(1, n))
        xs.append(n)
        ys.append(N.count_recur_calls(t, np.full(n, 0.05)))
    slope = np.polyfit(np.log(xs), np.log(ys), 1)[0]
    assert 1.0 <= slope <= 1.2
    xs, ys = [], []
    for n in (16, 32, 64, 128):
        t = N.build_tree(N.Grid.make(2, n))
        xs.append(n * n)
        ys.append(N.count_recur_calls(t, np.full(n * n, 0.1)))
    slope = np.polyfit(np.log(xs), np.log(ys), 1)[0]
    assert 1.35 <= slope <= 1.65


@pytest.mark.parametrize("name", ["trunc_2d_n64_k0", "trunc_1d_n2048_k3_bump", "trunc_3d_n8_k0",
                                  "trunc_1d_n512_k2_bump", "trunc_2d_n128_k0_bump"])
def test_reference_counters_from_the_tree(N, name):
    """recur_calls / step2_ops / step3_ops of the reference's TruncatedOperator
    (one apply) from the host tree instruments."""
    g = golden(name)
    dim, n, K, hk, d0 = int(g["dim"]), int(g["n"]), int(g["K"]), int(g["horizon_kind"]), float(g["delta0"])
    grid = N.Grid.make(dim, n)
    spec = N.KernelSpec(dim, N.RadialProfile.truncated_polynomial(K), N.HorizonField(N.HorizonKind(hk), d0))
    r = spec.horizon.nodes(grid)
    r = np.full(grid.total, d0) if r is None else r
    rc, panels = N.count_tree(grid, r)
    nm = 2 * K + 1 if dim == 1 else 1
    step2 = sum((1 << (dim * l)) * (1 << dim) * nm for l in range(grid.levels()))
    assert [rc, step2, panels * nm] == [int(v) for v in g["counters"]]
