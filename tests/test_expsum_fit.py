"""Host-side exponential-sum fit (plan setup, no GPU): the far-field weights
d^-alpha are reproduced to <= 1e-11 relative on every integer offset."""
import ctypes as C

import numpy as np
import pytest


@pytest.mark.parametrize("alpha,near,dmax", [(1.8, 32, 62915), (1.8, 32, 20972), (1.5, 32, 300),
                                             (1.2, 32, 62915), (3.0, 32, 4096)])
def test_fit_accuracy(alpha, near, dmax):
    from paper_1905_08375_b200 import build
    build.build()
    from paper_1905_08375_b200 import _capi as A
    r, w = np.zeros(64), np.zeros(64)
    m, e = C.c_int(), C.c_double()
    A.check(A.lib().nlg_expsum_fit(alpha, near, dmax, A.dptr(r), A.dptr(w), C.byref(m), C.byref(e)))
    M = m.value
    assert 8 <= M <= 64 and e.value <= 1e-10
    d = np.arange(near + 1, dmax + 1, dtype=float)
    # independent re-evaluation in numpy (chunks to bound memory)
    worst = 0.0
    for ch in np.array_split(d, max(1, len(d) // 8192)):
        approx = np.exp(-np.outer(ch, r[:M])) @ w[:M]
        worst = max(worst, np.max(np.abs(approx * ch ** alpha - 1.0)))
    assert worst <= 1e-10
