"""Four-step FFT convolution of the 1-D far window (csrc/fft.cu) across its
splits L = N1 x N2: every row length N2 in {2048, 4096, 8192}, column lengths
with radix-9, radix-3 and pure power-of-two plans, the cuFFT path for lengths
outside the supported set, with and without the kappa weighting and in the
diagonal mode of the Krylov consumer. Each case checks fast vs the direct
quadrature at sampled targets (both boundaries included) within the
north-star tolerance FAST_TOL = 1e-10 relative L-inf."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
FAST_TOL = 1e-10
REPEAT_TOL = 1e-12
N1_SUPPORTED = {64, 72, 96, 128, 144, 192, 256, 288, 320, 384, 512, 576, 768, 1024, 1080, 1152, 1536}


@pytest.fixture(scope="module")
def N():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1905_08375_b200 import nonloc
    return nonloc


def expected_split(L, first=4096):
    """Mirror of fourstep_plan (fft.cu): first row length whose column length is supported."""
    if first == 0:
        return 0
    order = (first, 8192 if first == 4096 else 4096, 8192 if first == 2048 else 2048)
    for n2 in order:
        if L % n2 == 0 and L // n2 in N1_SUPPORTED:
            return n2
    return 0


def sampled_check(N, w, n, **kw):
    op = N.NonlocalOperator(w.dim, w.n, **{**w.op_kwargs(), **kw})
    info = op.info
    assert info.fast_method == 2 and info.fft_len > 0
    fast = op.apply(w.u)
    tg = np.unique(np.concatenate([np.arange(0, 50), np.arange(n - 50, n),
                                   np.random.default_rng(n).integers(0, n, 300)])).astype(np.int64)
    direct = op.plan.apply_direct_at(w.u, tg)
    err = np.max(np.abs(fast[tg] - direct)) / np.max(np.abs(direct))
    return info, err


# sizes chosen so that L = smooth(n + Dmax + 1) lands on each split
SIZES = [1 << 16, 1 << 17, 180000, 1 << 18, 393216, 1 << 19, 700000, 1 << 20]


@pytest.fixture(scope="module")
def sweep(N):
    from paper_1905_08375_b200 import configs
    out = {}
    for n in SIZES:
        out[n] = sampled_check(N, configs.cfg1(n), n)
    return out


@pytest.mark.parametrize("n", SIZES)
def test_fft_split_fast_vs_direct(sweep, n):
    info, err = sweep[n]
    assert info.fft_rows == expected_split(info.fft_len)
    assert err <= FAST_TOL, (n, info.fft_len, info.fft_rows, err)


def test_fft_splits_covered(sweep):
    rows = {info.fft_rows for info, _ in sweep.values()}
    assert {0, 2048, 4096} <= rows, rows                # 0: the cuFFT path; 8192 forced below
    n1 = [info.fft_len // info.fft_rows for info, _ in sweep.values() if info.fft_rows]
    assert any(v % 9 == 0 for v in n1) and any(v % 3 == 0 and v % 9 for v in n1) and any(v % 3 for v in n1), n1


@pytest.mark.parametrize("rows", [8192, 2048, 0])
@pytest.mark.parametrize("n", [1 << 19, 1 << 20])
def test_fft_forced_row_length(N, n, rows, monkeypatch):
    """Row kernels the default preference does not reach at test sizes
    (8192), the 2048 rows and the cuFFT path (0), forced at plan time."""
    from paper_1905_08375_b200 import configs
    monkeypatch.setenv("NLG_FS_ROWS", str(rows))
    info, err = sampled_check(N, configs.cfg1(n), n)
    assert info.fft_rows == expected_split(info.fft_len, rows)
    assert err <= FAST_TOL, (n, rows, info.fft_len, info.fft_rows, err)


@pytest.mark.parametrize("n", [1 << 19, 1 << 16])
def test_fft_without_kappa(N, n):
    from paper_1905_08375_b200 import configs
    info, err = sampled_check(N, configs.cfg1(n), n, kappa=None)
    assert err <= FAST_TOL


@pytest.mark.parametrize("n", [1 << 19, 1 << 16])
def test_fft_zero_collar(N, n):
    from paper_1905_08375_b200 import configs
    info, err = sampled_check(N, configs.cfg1(n, exterior=1), n)
    assert err <= FAST_TOL


def test_fft_repeat_and_second_plan(N):
    """Two plans of one size and repeated applies agree to rounding (the fused
    passes keep no state between calls; only the order of the tail REDs varies)."""
    from paper_1905_08375_b200 import configs
    n = 1 << 19
    w = configs.cfg1(n)
    a = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
    b = N.NonlocalOperator(w.dim, w.n, **w.op_kwargs())
    assert a.info.fft_rows > 0
    ya = a.apply(w.u)
    d1 = np.max(np.abs(ya - a.apply(w.u))) / np.max(np.abs(ya))
    yb = b.apply(w.u)
    d2 = np.max(np.abs(ya - yb)) / np.max(np.abs(ya))
    print("repeat", d1, "second plan", d2)
    # only the order of the tail REDs varies; s (X - u diag) cancels ~3 digits
    assert d1 <= REPEAT_TOL and d2 <= REPEAT_TOL
