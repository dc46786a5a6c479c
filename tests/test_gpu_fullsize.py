"""Full-size (BASELINE config 4: 10M x 256-d, 4-bit, top-100) checks through size-independent
properties, where the CPU oracle would take minutes: the fused scan+top-K must equal an
independent route on the GPU (distance kernel -> exact (distance, id) sort), every plan must
agree, and a strided sample of rows must match the CPU oracle's codes and distances."""
import numpy as np
import pytest

import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo

pytestmark = pytest.mark.gpu

N, DIM, WD, WQ, K = 10_000_000, 256, 4, 4, 100


@pytest.fixture(scope="module")
def corpus():
    import torch
    g = torch.Generator(device="cuda").manual_seed(4000)
    docs = torch.empty((N, DIM), dtype=torch.float32, device="cuda")
    step = 1_000_000
    for r in range(0, N, step):
        x = torch.randn((step, DIM), generator=g, device="cuda", dtype=torch.float32)
        docs[r:r + step] = x / x.norm(dim=1, keepdim=True)
    queries = torch.randn((64, DIM), generator=g, device="cuda", dtype=torch.float32)
    queries /= queries.norm(dim=1, keepdim=True)
    scale = xb.estimate_scale(docs[:100_000].cpu().numpy(), 0.98)
    params = xb.QuantParams(dim=DIM, scale=scale, doc_bits=WD, query_bits=WQ)
    idx = xb.build_index(docs, params, keep_originals=False)
    sample_rows = np.arange(0, N, 9973)
    sample = docs[torch.from_numpy(sample_rows).cuda()].cpu().numpy()
    del docs
    torch.cuda.empty_cache()
    return idx, queries, params, sample_rows, sample


def test_codes_on_row_sample_match_oracle(corpus):
    idx, queries, params, rows, sample = corpus
    assert idx.packed.nbytes == N * WD * 4 * 8 == idx.packed.device_nbytes  # no padding at this shape
    planes = idx.packed.planes
    want = xo.c_quantize_matrix(sample, WD, params.scale)
    assert np.array_equal(planes[:, :, rows], want)


def test_fused_topk_equals_distance_kernel_plus_sort(corpus):
    import torch
    idx, queries, params, rows, sample = corpus
    scores, ids = xb.search(idx, queries, K)            # CUDA tensors in -> CUDA tensors out
    assert scores.shape == (64, K)
    qhost = queries.cpu().numpy().astype(np.float64)
    planes_sample = xo.c_quantize_matrix(sample, WD, params.scale)
    for qi in range(0, 64, 7):
        pq = xb.quantize_vector(qhost[qi], WQ, params.scale)
        d = xb.distance.batch_distances_device(idx.packed, pq)                  # int64[n], independent kernel
        keys = (d << 32) | torch.arange(N, device=d.device, dtype=torch.int64)
        best = torch.sort(keys).values[:K]
        assert torch.equal(best >> 32, scores[qi]) and torch.equal(best & 0xFFFFFFFF, ids[qi])
        # distances of the sampled rows equal the CPU oracle's
        want = xo.c_batch_distances(planes_sample, xo.np_quantize_vector(qhost[qi], WQ, params.scale))
        assert np.array_equal(d[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.uint64), want)
    # sortedness + uniqueness for every query
    k64 = (scores << 32) | ids
    assert bool((k64[:, 1:] > k64[:, :-1]).all())


def test_single_query_and_other_plans_agree(corpus, monkeypatch):
    import torch
    idx, queries, params, rows, sample = corpus
    base_s, base_i = xb.search(idx, queries, K)
    s1, i1 = xb.search(idx, queries[:1], K)              # Q=1 plan (many document splits + merge)
    assert torch.equal(s1, base_s[:1]) and torch.equal(i1, base_i[:1])
    monkeypatch.setenv("XFBQ_TQ", "8")
    monkeypatch.setenv("XFBQ_SPLITS", "5")
    s2, i2 = xb.search(idx, queries, K)
    assert torch.equal(s2, base_s) and torch.equal(i2, base_i)


def test_batch_engines_agree_at_full_size(corpus, monkeypatch):
    """640 queries at full n: the tcgen05 engine (sample scan + queue kernel over document slices) equals the
    mma.sync engine and the POPC route checked above, bit for bit."""
    import torch
    idx, queries, params, rows, sample = corpus
    g = torch.Generator(device="cuda").manual_seed(4100)
    q = torch.randn((640, DIM), generator=g, device="cuda", dtype=torch.float32)
    q /= q.norm(dim=1, keepdim=True)
    monkeypatch.setenv("XFBQ_ENGINE", "umma")
    su, iu = xb.search(idx, q, K)
    monkeypatch.setenv("XFBQ_ENGINE", "imma")
    si, ii = xb.search(idx, q, K)
    assert torch.equal(su, si) and torch.equal(iu, ii)
    k64 = (su << 32) | iu
    assert bool((k64[:, 1:] > k64[:, :-1]).all())
    base_s, base_i = xb.search(idx, queries, K)
    monkeypatch.setenv("XFBQ_ENGINE", "umma")
    s2, i2 = xb.search(idx, queries, K)
    assert torch.equal(s2, base_s) and torch.equal(i2, base_i)
    # the pieces of the seeded route against their predecessors: list-keeping sample scan, tree merge
    for key in ("XFBQ_SEED_HIST", "XFBQ_MERGE_BOUNDED"):
        monkeypatch.setenv(key, "0")
        s3, i3 = xb.search(idx, q, K)
        assert torch.equal(s3, su) and torch.equal(i3, iu)
