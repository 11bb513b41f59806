"""Krylov consumer on the GPU (§8(f) row 1): dense assembly and transpose
apply of the direct operators, and the device-resident CG / CGNR
(nlg_solve_dirichlet) against the compiled reference's solve path
(tests/golden/solve_dirichlet.npz, assemble_dense.npz; reference
tests/test_solve.cpp:47-170, tools/nonloc_main.cpp:189-222)."""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1905_08375_b200 import nonloc
    return nonloc


def rel_inf(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def spec_t(N, K, kind, d0, dim=1):
    return N.KernelSpec(dim, N.RadialProfile.truncated_polynomial(K), N.HorizonField(kind, d0))


ASM = [("k1_const_leaf_mass", 1, 128, "t", 1, 0, "leaf", "mass", False),
       ("k0_bump_leaf_mass", 1, 128, "t", 0, 1, "leaf", "mass", False),
       ("k0_bump_point_diff", 1, 128, "t", 0, 1, "point", "diff", False),
       ("inverse_s_bump", 1, 128, "s", 0, 1, "point", "diff", False),
       ("inverse_s_bump_div", 1, 128, "s", 0, 1, "point", "diff", True),
       ("k0_2d_leaf_mass", 2, 16, "t", 0, 1, "leaf", "mass", False)]


def make_spec(N, dim, fam, K, hk, div):
    prof = N.RadialProfile.truncated_polynomial(K) if fam == "t" else N.RadialProfile.inverse_s()
    sym = N.SymmetryClass.Divergence if div else N.SymmetryClass.NonDivergence
    return N.KernelSpec(dim, prof, N.HorizonField(N.HorizonKind(hk), 0.25), sym)


@pytest.mark.parametrize("case", ASM, ids=[c[0] for c in ASM])
def test_assembly_matches_reference(N, case):
    tag, dim, n, fam, K, hk, rule, form, div = case
    spec = make_spec(N, dim, fam, K, hk, div)
    g = N.Grid.make(dim, n)
    a = N.assemble_dense_matrix(spec, g, N.InclusionRule.Leaf if rule == "leaf" else N.InclusionRule.Point,
                                N.ApplyForm.Mass if form == "mass" else N.ApplyForm.Difference)
    ref = golden("assemble_dense")[tag]
    assert np.max(np.abs(a - ref)) <= 1e-13 * np.max(np.abs(ref))
    assert np.array_equal(a != 0.0, ref != 0.0)            # identical sparsity (inclusion sets)


@pytest.mark.parametrize("case", ASM, ids=[c[0] for c in ASM])
def test_transpose_is_the_adjoint(N, case):
    tag, dim, n, fam, K, hk, rule, form, div = case
    spec = make_spec(N, dim, fam, K, hk, div)
    g = N.Grid.make(dim, n)
    ref = golden("assemble_dense")[tag].reshape(g.total, g.total)
    if fam == "t":
        p = N.Plan(dim=dim, n=n, family=N.A.TRUNCATED, route=N.A.ROUTE_TRUNCATED, poly=spec.profile.poly,
                   rule=N.A.LEAF if rule == "leaf" else N.A.POINT, form=N.A.MASS if form == "mass" else N.A.DIFFERENCE,
                   delta=spec.horizon.nodes(g), delta0=0.25)
    else:
        p = N.Plan(dim=dim, n=n, route=N.A.ROUTE_FULL, rule=N.A.POINT, form=N.A.DIFFERENCE, divergence=div,
                   delta=spec.horizon.nodes(g), delta0=0.25, reach=spec.horizon.max_radius(),
                   **N._profile_args(spec.profile))
    rng = np.random.default_rng(3)
    u, v = rng.standard_normal(g.total), rng.standard_normal(g.total)
    at = p.apply_transpose(v)
    assert rel_inf(at, ref.T @ v) <= 1e-12
    au, _ = p.apply_direct(u)
    assert abs(np.dot(au, v) - np.dot(u, at)) <= 1e-12 * np.linalg.norm(au) * np.linalg.norm(v)


def test_transpose_fractional_variable_delta_collar(N):
    """BASELINE fractional operator (kappa, variable delta, zero collar): the
    transpose is the adjoint of the direct apply."""
    n = 96
    h = 1.0 / n
    rng = np.random.default_rng(5)
    delta = h * (3 + 5 * rng.random(n * n))
    op = N.NonlocalOperator(2, n, alpha=2.8, delta=delta, coeff=0.5 + rng.random(n * n),
                            kappa=np.exp(0.3 * rng.standard_normal(n * n)), exterior=N.Exterior.Collar)
    u, v = rng.standard_normal(n * n), rng.standard_normal(n * n)
    au, _ = op.apply_direct(u)
    at = op.plan.apply_transpose(v)
    assert abs(np.dot(au, v) - np.dot(u, at)) <= 1e-12 * np.linalg.norm(au) * np.linalg.norm(v)


def test_device_cg_fast_operator_matches_reference(N):     # test_solve.cpp:73-116
    G = golden("solve_dirichlet")
    n = 512
    g = N.Grid.make(1, n)
    op = N.TruncatedOperator(spec_t(N, 0, N.HorizonKind.Constant, 0.25), g)
    f, ustar = G["cg_n512_f"], G["cg_n512_ustar"]
    rep = op.solve_dirichlet(f, 1e-10, 10 * n)
    assert rep.method == N.SolveMethod.CG and rep.converged and rep.final_residual <= 1e-10
    assert rel_inf(rep.solution, ustar) <= 1e-8
    assert rel_inf(rep.solution, G["cg_n512_u"]) <= 1e-8
    assert abs(rep.iterations - int(G["cg_n512_iters"])) <= 1
    assert rel_inf(rep.solution, G["cg_n512_direct"]) <= 1e-8
    # residual certificate through the independent dense apply
    au = N.apply_truncated_dense(op.spec(), g, N.InclusionRule.Leaf, rep.solution)
    assert np.sqrt(np.sum((f + au) ** 2) / np.sum(f * f)) <= 10 * max(rep.final_residual, 1e-16)


def test_device_cg_direct_apply(N):                       # "dense matvec" subcase
    G = golden("solve_dirichlet")
    n = 512
    g = N.Grid.make(1, n)
    spec = spec_t(N, 0, N.HorizonKind.Constant, 0.25)
    p = N.Plan(dim=1, n=n, family=N.A.TRUNCATED, route=N.A.ROUTE_TRUNCATED, poly=spec.profile.poly,
               rule=N.A.LEAF, form=N.A.MASS, delta0=0.25)
    rep = p.solve_dirichlet(G["cg_n512_f"], 1e-10, 10 * n, direct=True)
    assert rep.converged and rel_inf(rep.solution, G["cg_n512_dense_u"]) <= 1e-8
    assert abs(rep.iterations - int(G["cg_n512_dense_iters"])) <= 1


def test_device_cgnr_variable_horizon(N):                 # test_solve.cpp:118-145
    G = golden("solve_dirichlet")
    n = 256
    g = N.Grid.make(1, n)
    spec = spec_t(N, 0, N.HorizonKind.GaussianBump, 0.25)
    assert N.choose_method(spec) == N.SolveMethod.CGNR
    op = N.TruncatedOperator(spec, g)
    rep = op.solve_dirichlet(G["cgnr_n256_bump_f"], 1e-10, 10 * n)
    assert rep.method == N.SolveMethod.CGNR and rep.converged
    assert rep.iterations <= 10 * n
    assert rel_inf(rep.solution, G["cgnr_n256_bump_direct"]) <= 1e-6
    assert rel_inf(rep.solution, G["cgnr_n256_bump_u"]) <= 1e-6


def test_device_non_convergence_reported(N):              # test_solve.cpp:147-158
    G = golden("solve_dirichlet")
    n = 128
    op = N.TruncatedOperator(spec_t(N, 0, N.HorizonKind.Constant, 0.25), N.Grid.make(1, n))
    rep = op.solve_dirichlet(G["cg_n128_2it_f"], 1e-14, 2)
    assert not rep.converged and rep.iterations == 2
    assert abs(rep.final_residual - float(G["cg_n128_2it_residual"])) <= 1e-10


def test_device_nan_is_a_hard_error(N):                   # test_solve.cpp:160-170
    n = 128
    op = N.TruncatedOperator(spec_t(N, 0, N.HorizonKind.Constant, 0.25), N.Grid.make(1, n))
    f = np.ones(n)
    f[3] = np.nan
    with pytest.raises(RuntimeError):
        op.solve_dirichlet(f, 1e-10, 10)
    rep = op.solve_dirichlet(np.zeros(n), 1e-10, 10)
    assert rep.converged and rep.iterations == 0 and np.all(rep.solution == 0.0)


def test_device_cg_2d_fast(N):
    """2-D constant horizon (symmetric): device CG with the span fast apply
    recovers a manufactured solution."""
    n = 64
    g = N.Grid.make(2, n)
    spec = spec_t(N, 0, N.HorizonKind.Constant, 0.125, dim=2)
    op = N.TruncatedOperator(spec, g)
    k = np.arange(n * n)
    x0, x1 = (k // n + 0.5) / n, (k % n + 0.5) / n
    ustar = np.sin(np.pi * x0) * np.sin(2 * np.pi * x1)
    f = -N.apply_truncated_dense(spec, g, N.InclusionRule.Leaf, ustar)
    rep = op.solve_dirichlet(f, 1e-11, 2000)
    assert rep.converged and rel_inf(rep.solution, ustar) <= 1e-8
