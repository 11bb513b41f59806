"""2-D/3-D fast path (offset-table stencil, method 3) on the BASELINE cfg2/3/4
operators at reduced sizes: fast vs GPU direct vs restated oracle. Inclusion
sets are checked exactly through the direct pair counts; fast vs direct within
the north-star 1e-10 (FAST_TOL)."""
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


CASES = [("cfg2", 128), ("cfg2", 256), ("cfg3", 128), ("cfg4", 48), ("cfg4b", 40), ("cfg4", 32)]


@pytest.mark.parametrize("name,n", CASES)
@pytest.mark.parametrize("exterior", [0, 1])
def test_stencil_fast_vs_direct_vs_oracle(N, orc, name, n, exterior):
    from paper_1905_08375_b200 import configs
    w = configs.WORKLOADS[name](n)
    w.exterior = exterior
    op = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
    assert op.info.fast_method == 3
    fast = op.apply(w.u)
    direct, pairs = op.apply_direct(w.u)
    assert orc.rel_inf(fast, direct) <= FAST_TOL
    comps = 2 if w.kernel == "peridynamic" else 1
    tg = np.unique(np.random.default_rng(0).integers(0, w.N, 300))
    ref, _ = orc.apply(w.dim, w.n, w.u, targets=tg, **w.oracle_kwargs())
    got = fast.reshape(comps, -1)[:, tg].reshape(-1)
    assert orc.rel_inf(got, ref) <= FAST_TOL
    d = direct.reshape(comps, -1)[:, tg].reshape(-1)
    assert orc.rel_inf(d, ref) <= 1e-13


def test_stencil_constants_and_linearity(N):
    from paper_1905_08375_b200 import configs
    w = configs.cfg2(128)
    op = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
    sc = np.max(np.abs(op.apply(w.u)))
    assert np.max(np.abs(op.apply(np.ones(w.N)))) <= 1e-13 * sc      # clip: exact annihilation
    v = np.random.default_rng(4).standard_normal(w.N)
    lhs = op.apply(2.0 * w.u - 0.5 * v)
    rhs = 2.0 * op.apply(w.u) - 0.5 * op.apply(v)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(lhs))


def test_peridynamics_known_answers(N):
    """Rigid translation -> 0 and infinitesimal rotation -> 0 at every node
    (clip); linear strain -> 0 at interior nodes (odd stencil symmetry) for
    constant c and delta."""
    n = 64
    h = 1.0 / n
    op = N.NonlocalOperator(2, n, kernel="peridynamic", delta0=5.5 * h, coeff0=2.0)
    k = np.arange(n * n)
    x0, x1 = (k // n + 0.5) * h, (k % n + 0.5) * h
    rng = np.random.default_rng(1)
    sc = np.max(np.abs(op.apply(rng.standard_normal(2 * n * n))))
    assert np.max(np.abs(op.apply(np.concatenate([np.full(n * n, 0.7), np.full(n * n, -0.2)])))) <= 1e-13 * sc
    assert np.max(np.abs(op.apply(np.concatenate([-x1, x0])))) <= 1e-12 * sc
    E = np.array([[0.3, 0.1], [0.1, -0.4]])
    out = op.apply(np.concatenate([E[0, 0] * x0 + E[0, 1] * x1, E[1, 0] * x0 + E[1, 1] * x1])).reshape(2, n, n)
    assert np.max(np.abs(out[:, 8:-8, 8:-8])) <= 1e-11 * sc
