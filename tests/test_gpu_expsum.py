"""1-D fast path (exponential-sum scans) vs the direct quadrature and the
restated oracle, on the BASELINE cfg0/cfg1 operators. North-star tolerance:
fast vs direct within 1e-10 relative L-inf (written here as FAST_TOL)."""
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


def op_for(N, w, **kw):
    return N.NonlocalOperator(w.dim, w.n, **{**w.op_kwargs(), **kw})


@pytest.mark.parametrize("n", [1 << 15, 1 << 16, 1 << 18])
@pytest.mark.parametrize("exterior", [0, 1])
def test_cfg1_family_fast_vs_direct(N, orc, n, exterior):
    from paper_1905_08375_b200 import configs
    w = configs.cfg1(n, exterior=exterior)
    op = op_for(N, w)
    assert op.info.fast_method == 2, "wide horizons must take the scan path"
    fast = op.apply(w.u)
    direct, pairs = op.apply_direct(w.u)
    assert orc.rel_inf(fast, direct) <= FAST_TOL
    # restated oracle on sampled nodes (includes both boundaries)
    tg = np.unique(np.concatenate([np.arange(0, 40), np.arange(n - 40, n),
                                   np.random.default_rng(0).integers(0, n, 200)]))
    ref, _ = orc.apply(1, n, w.u, targets=tg, **w.oracle_kwargs())
    assert orc.rel_inf(direct[tg], ref) <= 1e-13
    assert orc.rel_inf(fast[tg], ref) <= FAST_TOL


def test_cfg1_full_size_fast_vs_direct(N, orc):
    from paper_1905_08375_b200 import configs
    w = configs.cfg1()
    op = op_for(N, w)
    info = op.info
    assert info.fast_method == 2 and info.far_rel_err <= 1e-9   # tail fit (FFT mode) or whole far field
    fast = op.apply(w.u)
    direct, pairs = op.apply_direct(w.u)
    assert pairs > 3e11
    assert orc.rel_inf(fast, direct) <= FAST_TOL
    tg = np.random.default_rng(1).integers(0, w.N, 64)
    ref, _ = orc.apply(1, w.n, w.u, targets=tg, **w.oracle_kwargs())
    assert orc.rel_inf(fast[tg], ref) <= FAST_TOL * max(1.0, np.max(np.abs(fast)) / np.max(np.abs(ref)))


def test_cfg0_fast_vs_oracle(N, orc):
    from paper_1905_08375_b200 import configs
    w = configs.cfg0()
    op = op_for(N, w)
    ref, _ = orc.apply(1, w.n, w.u, **w.oracle_kwargs())
    assert orc.rel_inf(op.apply(w.u), ref) <= FAST_TOL
    assert orc.rel_inf(op.apply_direct(w.u)[0], ref) <= 1e-13


def test_expsum_linearity_and_constants(N, orc):
    from paper_1905_08375_b200 import configs
    w = configs.cfg1(1 << 16, exterior=0)
    op = op_for(N, w)
    one = op.apply(np.ones(w.N))
    # clip + difference form annihilates constants (test_operators.cpp:235-246 analogue)
    sc = np.max(np.abs(op.apply(w.u)))
    assert np.max(np.abs(one)) <= 1e-12 * sc
    v = np.random.default_rng(3).standard_normal(w.N)
    a, b = 0.3, -2.0
    lhs = op.apply(a * w.u + b * v)
    rhs = a * op.apply(w.u) + b * op.apply(v)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(lhs))
