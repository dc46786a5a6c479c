"""Host-side logic that needs no GPU: numpy's linear quantile restated for estimate_scale (index.py:123-138 calls np.quantile;
the GPU supplies the two order statistics, paper_2008_02002_b200/index.py the scalar interpolation), the R x Q grid arithmetic,
the bench's corpus chunking."""
import numpy as np

from paper_2008_02002_b200.index import _lerp, _linear_quantile_plan


def test_linear_quantile_restatement_matches_numpy_bit_for_bit():
    rng = np.random.Generator(np.random.PCG64(1))
    checked = 0
    for dtype in (np.float32, np.float64):
        for n in (1, 2, 3, 5, 10, 11, 100, 101, 999, 4097, 65_537, (1 << 24) + 3):
            x = np.abs(rng.normal(0.0, 0.06, size=n)).astype(dtype)
            if n > 1000:
                x[::7] = x[3]                                   # ties
            xs = np.sort(x)
            for p in (0.98, 1.0, 0.5, 0.01, 0.999, 1.0 / 3.0, 0.75, 1e-9):
                want = np.quantile(x, p)                        # what the reference computes
                lo, hi, gamma = _linear_quantile_plan(n, p, dtype)
                got = _lerp(xs[lo], xs[hi], gamma)
                assert got == want and got.dtype == want.dtype, (dtype, n, p)
                checked += 1
    assert checked == 2 * 12 * 8


def test_linear_quantile_ranks_are_the_float32_rounded_ones_past_2_pow_24():
    """numpy casts q to the array dtype: for float32 and n - 1 > 2^24 the virtual index is a rounded float32."""
    n = (1 << 25) + 5
    lo, hi, gamma = _linear_quantile_plan(n, 0.98, np.float32)
    vi = (n - 1) * np.float32(0.98)
    assert lo == int(np.floor(vi)) and hi == lo + 1 and gamma == np.float32(np.float64(vi) - lo)
    lo64, _, _ = _linear_quantile_plan(n, 0.98, np.float64)
    assert lo64 == int(np.floor((n - 1) * 0.98)) and lo64 != lo
