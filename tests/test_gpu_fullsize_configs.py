"""BASELINE configs 2, 3 and a config-5 shard at their REAL sizes against the CPU oracle.

The corpora are float32 unit rows generated on the GPU (seeded), copied to the host, and quantized there
by the oracle's C restatement (quant.py:138-148 + bitplane.py:151-163): the GPU planes must equal the
oracle's for EVERY row, and the CPU search (oracle/xfbq_oracle.c: _kernels.py:56-69 pass structure +
(distance, id) order of search.py:129-131) runs on the ORACLE's planes, not on GPU output.  The GPU runs the
whole production batch (10k queries: the slice / group counts of the production plan); the oracle checks a
strided sample of those queries (pkg/tests/test_acceptance.py:124-144 is the reference's own "exhaustive ==
oracle" check, at desk size).
"""
import numpy as np
import pytest

import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo

pytestmark = pytest.mark.gpu


def _unit_rows(torch, n, dim, seed, step=500_000):
    g = torch.Generator(device="cuda").manual_seed(seed)
    out = torch.empty((n, dim), dtype=torch.float32, device="cuda")
    for r in range(0, n, step):
        m = min(step, n - r)
        x = torch.randn((m, dim), generator=g, device="cuda", dtype=torch.float32)
        out[r:r + m] = x / x.norm(dim=1, keepdim=True)
    return out


def _plan(n, dim, wd, nq, wq, k):
    plan = np.zeros(6, dtype=np.int32)
    xb._native.check(xb._native.lib().xfbq_scan_plan(n, dim, wd, nq, wq, k, 1, plan.ctypes.data))
    return plan


def _check_config(n, dim, wd, wq, k, nq, n_check, seed, expect_engine=3, small_batches=(1, 8)):
    import torch
    docs = _unit_rows(torch, n, dim, seed)
    queries = _unit_rows(torch, nq, dim, seed + 1)
    docs_host = docs.cpu().numpy()
    scale = xo.estimate_scale(docs_host[:200_000], 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=wq)
    idx = xb.build_index(docs, params, keep_originals=False)
    del docs
    torch.cuda.empty_cache()
    # (1) codes: every row, against the oracle quantizer run on the host copy of the same floats
    want_planes = xo.c_quantize_matrix(docs_host, wd, scale)
    del docs_host
    assert idx.packed.nbytes == want_planes.nbytes
    assert np.array_equal(idx.packed.planes, want_planes), "GPU planes differ from the oracle quantizer"
    # (2) the production batch on the GPU
    assert int(_plan(n, dim, wd, nq, wq, k)[4]) == expect_engine
    scores, ids = xb.search(idx, queries, k)
    scores, ids = scores.cpu().numpy(), ids.cpu().numpy()
    assert scores.shape == (nq, k)
    # (3) oracle on a strided sample of the queries, on its own planes
    pick = np.unique(np.linspace(0, nq - 1, n_check).astype(np.int64))
    q_host = queries.cpu().numpy().astype(np.float64)
    qp = xo.c_quantize_matrix(q_host[pick], wq, scale).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(want_planes, qp, k)
    assert np.array_equal(scores[pick].astype(np.uint64), want_d), "distances differ from the CPU oracle"
    assert np.array_equal(ids[pick], want_i), "row ids differ from the CPU oracle"
    # every row of the batch: strictly ascending keys (sortedness + uniqueness), ids in range
    k64 = (scores.astype(np.int64) << 32) | ids
    assert bool((k64[:, 1:] > k64[:, :-1]).all())
    assert ids.min() >= 0 and ids.max() < n
    # (4) the small-batch plans (HBM-bound mma.sync scan) answer the same queries identically
    for nb in small_batches:
        sub = pick[:nb]
        s1, i1 = xb.search(idx, queries[torch.from_numpy(sub).cuda()], k)
        assert np.array_equal(s1.cpu().numpy().astype(np.uint64), want_d[:nb])
        assert np.array_equal(i1.cpu().numpy(), want_i[:nb])
    return idx, queries, want_planes, scale


def test_config2_sift_shaped_1m_128_3bit_top100_10k_queries():
    _check_config(n=1_000_000, dim=128, wd=3, wq=4, k=100, nq=10_000, n_check=256, seed=2000)


def test_config3_glove_shaped_1p2m_200_4bit_top10_10k_queries():
    """dim 200: 56 padding bits per row (bitplane.py:41-46), C = 2 chunks."""
    _check_config(n=1_200_000, dim=200, wd=4, wq=4, k=10, nq=10_000, n_check=256, seed=3000)


def test_config4_deep_shaped_10m_256_4bit_top100_10k_queries():
    """The headline workload itself at full size against the CPU oracle (every row's codes; 48 strided queries of the 10k-query
    production batch; single queries and an 8-query batch through the single-launch path)."""
    _check_config(n=10_000_000, dim=256, wd=4, wq=4, k=100, nq=10_000, n_check=48, seed=4000)


def test_config5_shard_2p5m_512_4bit_top1000_batched_and_single_query():
    """One GPU's part of config 5 (100M x 512 over 8 GPUs = 12.5M rows each; 2.5M rows here keep the CPU side at
    seconds): top-1000, a 1 024-query batch (tcgen05 engine, k = 1000 lists) and single queries."""
    import torch
    idx, queries, planes, scale = _check_config(n=2_500_000, dim=512, wd=4, wq=4, k=1000, nq=1024, n_check=64, seed=5000,
                                                small_batches=(1, 4))
    # k_select on the same shard: hits = the oracle's top-k, threshold and candidate count by the reference's definition
    q0 = queries[0].cpu().numpy().astype(np.float64)
    res = xb.k_select(idx, xb.SearchRequest(query=q0, k=1000))
    d = xo.c_batch_distances(planes, xo.np_quantize_vector(q0, 4, scale))
    want_d, want_i = xo.c_topk(d, 1000)
    assert [h[0] for h in res.hits] == want_i.tolist()
    assert res.threshold_distance == int(want_d[-1])
    assert res.candidate_count == int((d <= want_d[-1]).sum())
