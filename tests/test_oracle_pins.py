"""Pin the restated CPU oracle (oracle/nonloc_oracle.c) before trusting it.

(a) against the committed golden vectors produced by the COMPILED REFERENCE
    (tests/golden/make_golden.py) — runs everywhere;
(b) against the compiled reference live (oracle/_ref) on fresh random cases —
    runs where the reference was built (this container).
Tolerances: inclusion sets and pair counts exact; values 1e-14 relative (the
restatement follows the reference's operation order, so most cases are 0).
"""
import numpy as np
import pytest

from conftest import golden

TOL = 1e-14


def test_random_vector_matches_reference_bench_cpp(orc):
    # bench.cpp:10-16 — the seeds the reference tests use (test_operators.cpp:60,71,81)
    for name, seed in (("trunc_2d_n64_k0", 42), ("trunc_1d_n2048_k3_bump", 43), ("trunc_3d_n8_k0", 44)):
        g = golden(name)
        assert np.array_equal(orc.random_vector(len(g["u"]), seed), g["u"])


def test_matching_polynomials(orc):
    g = golden("kernel_algebra")
    for K in range(5):
        assert np.array_equal(orc.match_polynomial(K), g[f"p{K}"])
    # test_kernel.cpp:95-101 — K=3 is 35/16, -35/16, 21/16, -5/16
    assert list(orc.match_polynomial(3)) == [35 / 16, -35 / 16, 21 / 16, -5 / 16]


@pytest.mark.parametrize("name", ["trunc_2d_n64_k0", "trunc_1d_n2048_k3_bump", "trunc_3d_n8_k0",
                                  "trunc_1d_n512_k2_bump", "trunc_1d_n4096_k0_d002",
                                  "trunc_1d_n4096_k3_d002", "trunc_2d_n128_k0_bump"])
def test_truncated_dense_golden(orc, name):
    g = golden(name)
    dim, n, K, hk, d0 = int(g["dim"]), int(g["n"]), int(g["K"]), int(g["horizon_kind"]), float(g["delta0"])
    delta = orc.bump_horizon(dim, n, d0) if hk else None
    poly = orc.match_polynomial(K)
    for rule, form, key, pk in ((orc.LEAF, orc.MASS, "dense_leaf", "leaf_pairs"),
                                (orc.POINT, orc.MASS, "dense_point", "point_pairs"),
                                (orc.POINT, orc.DIFFERENCE, "dense_point_diff", None)):
        out, pairs = orc.apply(dim, n, g["u"], family=orc.TRUNCATED, route=orc.ROUTE_TRUNCATED,
                               poly=poly, rule=rule, form=form, delta=delta, delta0=d0)
        assert orc.rel_inf(out, g[key]) <= TOL
        if pk:
            assert pairs == int(g[pk])
    # the reference's own pin: fast == dense Leaf (test_operators.cpp:64,75,85)
    tol = 1e-12 if K == 0 else 1e-10
    if name != "trunc_1d_n4096_k3_d002":  # raw-moment conditioning, SURVEY §0.5
        assert orc.rel_inf(g["fast"], g["dense_leaf"]) <= tol


def test_smooth_full_split_golden(orc):
    g = golden("split_1d_n256")
    ka = golden("kernel_algebra")
    u = g["u"]
    out, pairs = orc.apply(1, 256, u, family=orc.KAPPA, route=orc.ROUTE_SMOOTH,
                           poly=ka["split_poly2"], tail=ka["split_tail2"], order=2, delta0=0.25)
    assert orc.rel_inf(out, g["smooth_k2"]) <= TOL and pairs == int(g["smooth_pairs"])
    full, fp = orc.apply(1, 256, u, family=orc.INVERSE_S, route=orc.ROUTE_FULL, delta0=0.25, reach=0.25)
    assert orc.rel_inf(full, g["full"]) <= TOL and fp == int(g["full_pairs"])
    # test_operators.cpp:170-177 — smooth + truncated(Point, Difference) == full to 1e-12
    tr, _ = orc.apply(1, 256, u, family=orc.TRUNCATED, route=orc.ROUTE_TRUNCATED,
                      poly=ka["split_poly2"], rule=orc.POINT, form=orc.DIFFERENCE, delta0=0.25)
    assert orc.rel_inf(out + tr, g["full"]) <= 1e-12
    assert orc.rel_inf(out + tr, g["split_k2_pointdiff"]) <= TOL


@pytest.mark.parametrize("dim,n", [(1, 256), (2, 16)])
def test_full_families_golden(orc, dim, n):
    g = golden("full_families")
    ka = golden("kernel_algebra")
    u = g[f"u{dim}"]
    delta = orc.bump_horizon(dim, n, 0.25)
    fams = {0: orc.INVERSE_S, 1: orc.CONICAL, 2: orc.KAPPA, 3: orc.TRUNCATED}
    for fam, f in fams.items():
        poly = orc.match_polynomial(2) if fam == 3 else ka["split_poly2"]
        for div in (0, 1):
            out, pairs = orc.apply(dim, n, u, family=f, route=orc.ROUTE_FULL, poly=poly,
                                   tail=ka["split_tail2"], order=2, delta=delta, delta0=0.25,
                                   reach=0.5, divergence=bool(div))
            assert orc.rel_inf(out, g[f"full{dim}_f{fam}_div{div}"]) <= TOL
            assert pairs == int(g[f"pairs{dim}_f{fam}_div{div}"])


@pytest.mark.parametrize("tag,dim,n", [("1d", 1, 2048), ("2d", 2, 64), ("3d", 3, 16)])
def test_fractional_kappa_variable_delta_golden(orc, tag, dim, n):
    g = golden("fractional_general")
    kw, p1 = orc.apply(dim, n, g[f"{tag}_u"], family=orc.FRACTIONAL, alpha=float(g[f"{tag}_alpha"]),
                       delta=g[f"{tag}_delta"], coeff=g[f"{tag}_cx"], kappa=g[f"{tag}_kappa"])
    assert orc.rel_inf(kw, g[f"{tag}_kw"]) <= 1e-13 and p1 == int(g[f"{tag}_kw_pairs"])
    pl, p0 = orc.apply(dim, n, g[f"{tag}_u"], family=orc.FRACTIONAL, alpha=float(g[f"{tag}_alpha"]),
                       delta=g[f"{tag}_delta"])
    assert orc.rel_inf(pl, g[f"{tag}_plain"]) <= 1e-13 and p0 == int(g[f"{tag}_plain_pairs"])


def test_cfg0_clip_golden_and_collar_identity(orc):
    g = golden("fractional_general")
    n = 4096
    cd = float(g["cfg0_cdelta"])
    clip, pc = orc.apply(1, n, g["cfg0_u"], family=orc.FRACTIONAL, alpha=1.5, delta0=0.02, coeff0=cd)
    assert orc.rel_inf(clip, g["cfg0_out_clip"]) <= 1e-13 and pc == int(g["cfg0_pairs"])
    # collar = clip - u_i h^d sum_{y outside, in rule} omega(x_i, y)
    col, _ = orc.apply(1, n, g["cfg0_u"], family=orc.FRACTIONAL, alpha=1.5, delta0=0.02, coeff0=cd,
                       exterior=orc.COLLAR)
    ones_col, _ = orc.apply(1, n, np.ones(n), family=orc.FRACTIONAL, alpha=1.5, delta0=0.02,
                            coeff0=cd, exterior=orc.COLLAR)
    # for u = 1 the clip operator vanishes, so collar(1) = -h sum_ext omega
    assert orc.rel_inf(col, clip + g["cfg0_u"] * ones_col) <= 1e-12
    assert np.all(ones_col[100:-100] == 0.0) and ones_col[0] < 0


@pytest.fixture(scope="module")
def ref(orc):
    if not orc.ref_available():
        try:
            orc.build(ref=True)
        except Exception:
            pass
    if not orc.ref_available():
        pytest.skip("compiled reference (oracle/_ref) not available")
    return orc


def test_live_reference_random_cases(ref):
    rng = np.random.default_rng(7)
    O = ref
    for dim, n in ((1, 128), (2, 16), (3, 8)):
        for trial in range(3):
            d0 = float(0.05 + 0.4 * rng.random())
            hk = int(rng.integers(0, 2))
            K = int(rng.integers(0, 4)) if dim == 1 else 0
            u = O.random_vector(n ** dim, int(rng.integers(1 << 30)))
            delta = O.bump_horizon(dim, n, d0) if hk else None
            for rule in (O.LEAF, O.POINT):
                for form in (O.MASS, O.DIFFERENCE):
                    a, pa = O.ref_truncated_dense(dim, n, K, hk, d0, u, rule, form)
                    b, pb = O.apply(dim, n, u, family=O.TRUNCATED, route=O.ROUTE_TRUNCATED,
                                    poly=O.match_polynomial(K), rule=rule, form=form,
                                    delta=delta, delta0=d0)
                    assert O.rel_inf(b, a) <= TOL and pa == pb


def test_inclusion_predicates_exact(orc):
    """Leaf / Point membership vs brute-force integer reasoning on dyadic grids
    (the survey's 553,793-case probe, SURVEY §7 hard part 1, in miniature)."""
    import ctypes as C
    rng = np.random.default_rng(3)
    lib = orc.orc()
    for _ in range(3000):
        dim = int(rng.integers(1, 4))
        n = int(2 ** rng.integers(3, 23)) if dim == 1 else int(2 ** rng.integers(3, 12))
        h = 1.0 / n
        kx = rng.integers(0, n, size=3).astype(np.int64)
        # delta on half-integer ties half the time
        m = float(rng.integers(1, 20))
        delta = (m + (0.5 if rng.random() < 0.5 else rng.random())) * h
        dk = rng.integers(-22, 23, size=3)
        ky = (kx + dk).astype(np.int64)
        pk = kx.ctypes.data_as(C.POINTER(C.c_int64))
        py = ky.ctypes.data_as(C.POINTER(C.c_int64))
        leaf = lib.orc_leaf_in(dim, n, pk, py, delta)
        point = lib.orc_point_in(dim, n, pk, py, delta)
        # integer forms: Leaf  sum ((2|dk|-1)_+)^2 h^2/4 < fl(delta^2)
        #                Point sqrt(sum dk^2) h < delta
        s = sum(max(2 * abs(int(dk[j])) - 1, 0) ** 2 for j in range(dim))
        assert leaf == int(s * h * h / 4 < delta * delta)
        r2 = sum(int(dk[j]) ** 2 for j in range(dim))
        assert point == int(np.sqrt(r2 * h * h) < delta)
