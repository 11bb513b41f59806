"""bench.py's host-side pieces (CPU): the fixed CPU-baseline target set and
the compiled-reference legs, including the 2^L twin the reference needs for
cfg4's n = 768 (geometry.cpp:14-16)."""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def bench():
    import bench as B
    return B


def test_fixed_targets_deterministic(bench):
    a = bench._fixed_targets(10 ** 6, 512)
    b = bench._fixed_targets(10 ** 6, 512)
    assert np.array_equal(a, b) and len(np.unique(a)) == 512
    assert np.array_equal(bench._fixed_targets(10 ** 6, 4096)[:512], bench._fixed_targets(10 ** 6, 4096)[:512])


def test_direct_reference_twin(bench):
    """n = 96 (not 2^L) runs on the 64^3 twin with delta/h kept; n = 64 runs as is."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.ref_available():
        pytest.skip("compiled reference not built")
    from paper_1905_08375_b200 import configs
    bench.CPU_SAMPLE["_t"] = (16, 64)
    r = bench.DirectReference(configs.cfg4(96), "_t", 2)
    assert r.n == 64 and not r.port
    # the twin's targets see delta = 6 h_twin
    assert np.allclose(r.delta[r.tn], 6.0 / 64)
    m = r.measure()
    assert m["kind"] == "reference" and m["value"] > 0 and m["value_1core"] > 0 and m["cores"] == 2
    r2 = bench.DirectReference(configs.cfg4(64, variable=True), "_t", 2)
    assert r2.n == 64 and r2.u is not None
    assert r2.measure()["value"] > 0
