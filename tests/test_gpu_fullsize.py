"""BASELINE configurations at their full sizes (cfg2/cfg3 4096², cfg4 768³ with
constant and variable horizon): the fast apply against the GPU direct
quadrature on sampled targets (interior, every face / edge layer, and for cfg3
the inclusion interface), plus size-independent properties of the whole
output: linearity and exact annihilation of constants (clip exterior).
Tolerance: the north-star 1e-10 relative to the output's L-inf scale."""
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


def _targets(w, count=3000, seed=5):
    rng = np.random.default_rng(seed)
    n, d = w.n, w.dim
    tg = [rng.integers(0, w.N, count)]
    # boundary layers: one coordinate pinned near a face
    for j in range(d):
        idx = rng.integers(0, n, (count // 4, d))
        idx[:, j] = rng.choice(np.r_[0:12, n - 12:n], count // 4)
        flat = np.zeros(count // 4, dtype=np.int64)
        for k in range(d):
            flat = flat * n + idx[:, k]
        tg.append(flat)
    return np.unique(np.concatenate(tg))


def _check(N, w, tg_extra=None):
    op = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
    fast = op.apply(w.u)
    comps = 2 if w.kernel == "peridynamic" else 1
    tg = _targets(w) if tg_extra is None else np.unique(np.concatenate([_targets(w), tg_extra]))
    ref = op.apply_direct_at(w.u, tg).reshape(comps, -1)
    got = fast.reshape(comps, -1)[:, tg]
    scale = np.max(np.abs(fast))
    err = np.max(np.abs(got - ref)) / scale
    assert err <= FAST_TOL, err
    return op, fast, scale


@pytest.mark.parametrize("name", ["cfg2", "cfg4", "cfg4b"])
def test_full_size_fractional(N, name):
    from paper_1905_08375_b200 import configs
    w = configs.WORKLOADS[name]()
    op, fast, scale = _check(N, w)
    # constants are annihilated exactly (clip) and the apply is linear, on the whole grid
    assert np.max(np.abs(op.apply(np.ones(w.N)))) <= 1e-12 * scale
    v = np.random.default_rng(9).standard_normal(w.N)
    lhs = op.apply(2.0 * w.u - 0.5 * v)
    rhs = 2.0 * fast - 0.5 * op.apply(v)
    assert np.max(np.abs(lhs - rhs)) <= 1e-11 * np.max(np.abs(lhs))


def test_full_size_peridynamics(N):
    from paper_1905_08375_b200 import configs
    w = configs.cfg3()
    # extra targets along the inclusion interface, where delta and c jump
    h = 1.0 / w.n
    d = w.delta.reshape(w.n, w.n)
    jump = np.abs(np.diff(d, axis=1)) > 0.5 * h
    ii, jj = np.nonzero(jump)
    rng = np.random.default_rng(3)
    pick = rng.choice(len(ii), min(2000, len(ii)), replace=False)
    extra = ii[pick].astype(np.int64) * w.n + jj[pick]
    op, fast, scale = _check(N, w, extra)
    rigid = np.concatenate([np.full(w.N, 0.3), np.full(w.N, -1.1)])
    assert np.max(np.abs(op.apply(rigid))) <= 1e-12 * scale
