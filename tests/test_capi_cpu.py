"""CPU-side checks of the native boundary: the C-ABI library loads, exports
every symbol include/nlgpu.h declares, and its host algebra (no GPU needed)
matches the reference's kernel algebra (test_kernel.cpp:78-140)."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


@pytest.fixture(scope="module")
def capi():
    from paper_1905_08375_b200 import build
    build.build()
    from paper_1905_08375_b200 import _capi
    return _capi


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "nlgpu.h")).read()
    return sorted(set(re.findall(r"\b(nlg_[a-z_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(capi):
    lib = capi.lib()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(capi.EXPORTS)
    assert lib.nlg_abi_version() == 1


def test_match_polynomial_and_split_match_reference(capi):
    from paper_1905_08375_b200 import nonloc as N
    g = golden("kernel_algebra")
    for K in range(5):
        assert np.array_equal(N.match_polynomial(K), g[f"p{K}"])
    for K in range(4):
        sk = N.split(N.RadialProfile.inverse_s(), K)
        assert np.array_equal(sk.poly, g[f"split_poly{K}"])
        assert np.array_equal(sk.tail, g[f"split_tail{K}"])
    with pytest.raises(ValueError):
        N.match_polynomial(-1)


def test_reference_error_behaviour(capi):
    from paper_1905_08375_b200 import nonloc as N
    with pytest.raises(ValueError):
        N.Grid.make(1, 3)          # geometry.cpp:14-16
    with pytest.raises(ValueError):
        N.Grid.make(4, 4)
    assert N.Grid.make(3, 768, any_n=True).total == 768 ** 3
    spec = N.KernelSpec(2, N.RadialProfile.truncated_polynomial(1))
    with pytest.raises(ValueError):
        N.TruncatedOperator(spec, N.Grid.make(2, 8))   # K > 0 in 1d only (operators.cpp:108-110)
    with pytest.raises(ValueError):
        N.apply_truncated_dense(N.KernelSpec(1, N.RadialProfile.inverse_s()), N.Grid.make(1, 8),
                                N.InclusionRule.Leaf, np.zeros(8))


def test_halo_rows(capi):
    from paper_1905_08375_b200 import nonloc as N
    # window of floor(delta/h)+2 cells, a superset of window_around (operators.cpp:31-42)
    assert N.halo_rows(dim=2, n=4096, family=capi.FRACTIONAL, delta_max=12 / 4096) == 14
    assert N.halo_rows(dim=1, n=1 << 22, family=capi.FRACTIONAL, delta_max=0.015) == 62916


def test_stage_slots_match_header():
    """nlg_stage_times fills NLG_NUM_STAGES slots; the Python stage names cover them."""
    import re
    from paper_1905_08375_b200 import _capi
    src = open(os.path.join(ROOT, "include", "nlgpu.h")).read()
    n = int(re.search(r"#define NLG_NUM_STAGES (\d+)", src).group(1))
    assert len(_capi.STAGES) == n


def test_group_argument_errors(capi):
    """nlg_group_create validates its arguments before touching a device
    (std::invalid_argument semantics): no devices, a sharded descriptor, and
    slabs thinner than the halo (which would leave neighbours' halos short)."""
    from paper_1905_08375_b200 import nonloc as N
    A = N.A
    with pytest.raises(ValueError):
        N.Group([], dim=3, n=32, family=A.FRACTIONAL, alpha=3.5, delta0=6 / 32)
    with pytest.raises(ValueError, match="slab thinner than the halo"):
        N.Group([0] * 8, dim=3, n=32, family=A.FRACTIONAL, alpha=3.5, delta0=6 / 32)
