"""estimate_scale on the GPU (index.py:123-138) and the hand-written float re-rank (N2, search.py:153-157).

estimate_scale: the two order statistics numpy's "linear" quantile interpolates between come from the GPU radix
select; the result must be bit-identical to 1 / np.quantile(|x|, p) (numpy IS the reference's implementation) for
float32 and float64, odd sizes, heavy ties, percentile 1.0, and sizes past 2^24 where numpy's float32 virtual index
rounds.  Re-rank: ids equal the reference ranking recomputed in numpy float64, similarities to 1e-12 relative (the
reference's `rows @ q` goes through BLAS, whose summation order is unspecified: tolerance stated here)."""
import numpy as np
import pytest

import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_estimate_scale_bit_identical_to_numpy(dtype):
    rng = np.random.Generator(np.random.PCG64(11))
    for n in (1, 2, 3, 7, 64, 1001, 65_537, 1_000_003):
        x = rng.normal(0.0, 0.0625, size=n).astype(dtype)
        for p in (0.98, 1.0, 0.5, 0.999, 1e-3, 1.0 / 3.0):
            want = 1.0 / float(np.quantile(np.abs(x), p))
            assert xb.estimate_scale(x, p) == want, (dtype, n, p)
    # heavy ties: a handful of distinct magnitudes, both signs, zeros
    x = rng.choice(np.array([0.0, -0.0, 0.125, -0.125, 0.3, -0.7, 1e-30, 3.0], dtype=dtype), size=500_001)
    for p in (0.98, 0.5, 0.9, 1.0):
        q = float(np.quantile(np.abs(x), p))
        if q > 0:
            assert xb.estimate_scale(x, p) == 1.0 / q
    # 2-D input and CUDA tensors take the same path
    import torch
    m = rng.normal(0.0, 0.0625, size=(4097, 200)).astype(dtype)
    want = 1.0 / float(np.quantile(np.abs(m), 0.98))
    assert xb.estimate_scale(m) == want
    assert xb.estimate_scale(torch.from_numpy(m).cuda()) == want
    assert xb.estimate_scale(torch.from_numpy(m)) == want


def test_estimate_scale_float32_past_2_pow_24_and_config_sample():
    """n - 1 > 2^24: numpy computes the virtual index (n - 1) * float32(p) in float32 (rounded); the GPU path must pick
    the same two ranks.  Also the bench's own use: the first 100k rows of a 256-d corpus."""
    import torch
    rng = np.random.Generator(np.random.PCG64(12))
    x = rng.normal(0.0, 0.0625, size=(1 << 25) + 5).astype(np.float32)
    for p in (0.98, 0.75):
        want = 1.0 / float(np.quantile(np.abs(x), p))
        assert xb.estimate_scale(x, p) == want
    docs = xo.synthetic_unit_rows(100_000, 256, 4000)
    assert xb.estimate_scale(docs, 0.98) == xo.estimate_scale(docs, 0.98)
    assert xb.estimate_scale(torch.from_numpy(docs).cuda(), 0.98) == xo.estimate_scale(docs, 0.98)


def test_estimate_scale_errors_and_nan():
    with pytest.raises(xb.InvalidInputError):
        xb.estimate_scale(np.zeros((0, 4), dtype=np.float32))
    with pytest.raises(xb.InvalidInputError):
        xb.estimate_scale(np.ones((3, 4), dtype=np.float32), 0.0)
    with pytest.raises(xb.InvalidInputError):
        xb.estimate_scale(np.ones((3, 4), dtype=np.float32), 1.5)
    with pytest.raises(xb.InvalidInputError):
        xb.estimate_scale(np.zeros((3, 4), dtype=np.float32))          # selected percentile is zero
    x = np.ones(100, dtype=np.float32); x[5] = np.nan
    assert np.isnan(xb.estimate_scale(x))                               # the reference returns 1 / nan


def _reference_refine(originals, query, cand, k):
    sims = originals.astype(np.float64)[cand] @ query                   # search.py:153-157
    order = np.lexsort((cand, -sims))[:k]                               # search.py:129-131
    return cand[order], sims[order]


@pytest.mark.parametrize("resident", [False, True])
def test_k_select_with_originals_refine_kernel(resident):
    n, dim, k = 200_000, 128, 50
    docs = xo.synthetic_unit_rows(n, dim, 21)
    docs[1000:1040] = docs[7]                                           # exact float ties: ranked by id
    queries = xo.synthetic_unit_rows(8, dim, 22).astype(np.float64)
    queries[0] = docs[7].astype(np.float64)
    scale = xo.estimate_scale(docs[:50_000], 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=3, query_bits=4)
    idx = xb.build_index(docs, params)
    if resident:
        idx.originals_to_device()
    planes = xo.c_quantize_matrix(docs, 3, scale)
    for qi in range(8):
        for extra in (0, 150, 1500):
            res = xb.k_select(idx, xb.SearchRequest(query=queries[qi], k=k, extra_distance=extra))
            d = xo.c_batch_distances(planes, xo.np_quantize_vector(queries[qi], 4, scale))
            thr = int(np.sort(d)[k - 1]) + extra
            cand = np.flatnonzero(d <= thr)
            want_ids, want_sims = _reference_refine(docs, queries[qi], cand, k)
            assert res.threshold_distance == thr and res.candidate_count == cand.size and not res.approximate
            got_ids = np.array([h[0] for h in res.hits]); got_sims = np.array([h[1] for h in res.hits])
            assert np.allclose(got_sims, want_sims, rtol=1e-12, atol=1e-15)
            # ids: identical wherever the float64 similarities are separated by more than the summation-order noise
            same = got_ids == want_ids
            if not same.all():
                gaps = np.abs(np.diff(want_sims))
                bad = np.flatnonzero(~same)
                assert all(min(gaps[max(b - 1, 0)], gaps[min(b, gaps.size - 1)]) < 1e-12 for b in bad)
    # the tied block ranks by id (rows 7, 1000..1039 share one float row)
    res = xb.k_select(idx, xb.SearchRequest(query=queries[0], k=41))
    assert [h[0] for h in res.hits] == [7] + list(range(1000, 1040))


def test_k_above_max_k_and_full_range_extra():
    """k > XFBQ_MAX_K (4096) is accepted like the reference does (search.py:212), and extra_distance = the whole range
    re-ranks every row (test_search.py:158-168: full extra == float oracle)."""
    n, dim = 30_000, 64
    docs = xo.synthetic_unit_rows(n, dim, 31)
    q = xo.synthetic_unit_rows(2, dim, 32)
    scale = xo.estimate_scale(docs, 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4)
    idx = xb.build_index(docs, params)
    planes = xo.c_quantize_matrix(docs, 4, scale)
    qp = xo.c_quantize_matrix(q.astype(np.float64), 4, scale).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(planes, qp, 6000)
    s, i = xb.search(idx, q, 6000)
    assert np.array_equal(s.astype(np.uint64), want_d) and np.array_equal(i, want_i)
    upper = xb.distance_upper_bound(dim, 4, 4)
    res = xb.k_select(idx, xb.SearchRequest(query=q[0].astype(np.float64), k=10, extra_distance=upper))
    assert res.candidate_count == n
    want_ids, want_sims = _reference_refine(docs, q[0].astype(np.float64), np.arange(n), 10)
    assert [h[0] for h in res.hits] == want_ids.tolist()
    assert np.allclose([h[1] for h in res.hits], want_sims, rtol=1e-12)
    res = xb.k_select(idx, xb.SearchRequest(query=q[0].astype(np.float64), k=5000, extra_distance=0))
    assert len(res.hits) == 5000


def test_standalone_histogram_gather_refine_and_packed_distance():
    """The stand-alone stages of the reference pipeline (search.py:70-185, distance.py:32-41) on GPU kernels, against numpy
    restatements of the reference lines (pkg/tests/test_search.py:45-70, test_distance.py:30-35,114-124)."""
    import torch
    rng = np.random.Generator(np.random.PCG64(3))
    d = rng.integers(0, 5000, size=300_001).astype(np.uint64)
    ub = 6000
    h = xb.DistanceHistogram.from_distances(d, ub)
    assert np.array_equal(h.bins, np.bincount(d.astype(np.int64), minlength=ub + 1)) and h.total == d.size
    srt = np.sort(d)
    for k in (1, 2, 100, 4321, d.size, d.size + 5):
        assert h.kth_smallest(k) == int(srt[min(k, d.size) - 1])
        assert xb.histogram_kth_distance(d, k, extra=7) == int(srt[min(k, d.size) - 1]) + 7
    assert xb.histogram_kth_distance(torch.from_numpy(d.astype(np.int64)).cuda(), 10, upper_bound=ub) == int(srt[9])
    with pytest.raises(xb.InvalidInputError):
        xb.DistanceHistogram.from_distances(d, 100)
    with pytest.raises(xb.InvalidInputError):
        xb.histogram_kth_distance(np.zeros(0, dtype=np.uint64), 1)
    for thr in (0, 17, 2500, 4999, 10**9):
        assert np.array_equal(xb.gather_candidates(d, thr), np.flatnonzero(d <= thr))
    assert xb.gather_candidates(d, -1).size == 0
    # packed_distance: worked values 55 / 40 (test_distance.py:30-35) and equality with batch_distances rows
    x = xb.pack_matrix(np.array([[0b010, 0b010]], dtype=np.uint8), 3).row(0)
    y = xb.pack_matrix(np.array([[0b010, 0b111]], dtype=np.uint8), 3).row(0)
    assert xb.packed_distance(x, y) == 55 and xb.packed_distance(x, x) == 40
    docs = xo.synthetic_unit_rows(500, 200, 9)
    idx = xb.build_index(docs, xb.QuantParams(dim=200, scale=4.0, doc_bits=3, query_bits=4))
    pq = xb.quantize_vector(docs[3].astype(np.float64), 4, 4.0)
    full = xb.batch_distances(idx.packed, pq)
    assert [xb.packed_distance(idx.packed.row(r), pq) for r in (0, 3, 499)] == [int(full[r]) for r in (0, 3, 499)]
    # refine: both branches, and suggest_extra_distance
    cand = np.flatnonzero(full <= np.sort(full)[40])
    hits, approx = xb.refine(idx, docs[3].astype(np.float64), cand, 10)
    want_ids, want_sims = _reference_refine(docs, docs[3].astype(np.float64), cand, 10)
    assert not approx and [h[0] for h in hits] == want_ids.tolist() and np.allclose([h[1] for h in hits], want_sims, rtol=1e-12)
    idx2 = xb.Index(params=idx.params, packed=idx.packed, originals=None)
    hits2, approx2 = xb.refine(idx2, docs[3].astype(np.float64), cand, 10, distances=full)
    sims = xb.decode_inner_product_values(full[cand], 200, 3, 4) / 16.0
    order = np.lexsort((cand, -sims))[:10]
    assert approx2 and hits2 == [(int(cand[i]), float(sims[i])) for i in order]
    hits3, _ = xb.refine(idx2, docs[3].astype(np.float64), cand, 10)
    assert hits3 == hits2
    assert xb.suggest_extra_distance(idx, 0.05) == round(0.05 * xb.distance_upper_bound(200, 4, 3))
