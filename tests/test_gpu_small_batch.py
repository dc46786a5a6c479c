"""The single-launch small-batch search (coop::search_kernel: quantizer + threshold seeding + HBM-bound scan + merge in one
cooperative launch, <= 16 queries, databases of >= ~600k rows) against the CPU oracle, and against the multi-launch path it
replaces (XFBQ_COOP=0).  Same contract as everywhere: distances and row ids bit-exact, ties by lower row id
(search.py:129-131); non-finite queries raise (quant.py:142-143)."""
import numpy as np
import pytest

import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo
import importlib
xsearch = importlib.import_module("paper_2008_02002_b200.search")   # the module (the package exports the function `search`)

pytestmark = pytest.mark.gpu


def _fused_available(idx, nq, k):
    L = xb._native.lib()
    p = idx.params
    return int(L.xfbq_search_small_workspace_bytes(idx.n, p.dim, p.doc_bits, nq, p.query_bits, k)) > 0


@pytest.mark.parametrize("dim,wd,wq", [(128, 4, 4), (200, 3, 4), (384, 4, 7), (512, 2, 4)])
def test_fused_small_batch_matches_oracle(dim, wd, wq, monkeypatch):
    import torch
    n = 700_000
    docs = xo.synthetic_unit_rows(n, dim, 900 + dim)
    docs[5000:5200] = docs[17]                       # a block of exact ties among the best hits of query 0
    queries = xo.synthetic_unit_rows(16, dim, 901 + dim)
    queries[0] = docs[17]
    scale = xo.estimate_scale(docs[:20_000], 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=wq)
    idx = xb.build_index(docs, params, keep_originals=False)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), wq, scale).transpose(2, 0, 1)
    for k in (10, 100, 1000):
        assert _fused_available(idx, 1, k) and _fused_available(idx, 16, k)
        want_d, want_i = xo.c_search(planes, qp, k)
        for nq in (1, 3, 16):
            for q in (queries[:nq], queries[:nq].astype(np.float64), torch.from_numpy(queries[:nq]).cuda(),
                      torch.from_numpy(queries[:nq].astype(np.float64)).cuda(), torch.from_numpy(queries[:nq]).pin_memory()):
                s, i = xb.search(idx, q, k)
                if hasattr(s, "cpu"):
                    s, i = s.cpu().numpy(), i.cpu().numpy()
                assert np.array_equal(s.astype(np.uint64), want_d[:nq]), (dim, k, nq, type(q))
                assert np.array_equal(i, want_i[:nq]), (dim, k, nq, type(q))
        # the multi-launch path it replaces, and k_select through the quantized-planes entry of the same kernel
        monkeypatch.setenv("XFBQ_COOP", "0")
        s, i = xb.search(idx, queries[:5], k)
        monkeypatch.delenv("XFBQ_COOP")
        assert np.array_equal(s.astype(np.uint64), want_d[:5]) and np.array_equal(i, want_i[:5])
        res = xb.k_select(idx, xb.SearchRequest(query=queries[1].astype(np.float64), k=k))
        assert [h[0] for h in res.hits] == want_i[1].tolist()
    # with a row offset (shards) and ids past 2^31
    keys = xb.search_device(idx, torch.from_numpy(queries[:2]).cuda(), 10, row_offset=(1 << 32) - n)
    assert np.array_equal((keys.cpu().numpy() & 0xFFFFFFFF), xo.c_search(planes, qp[:2], 10)[1] + ((1 << 32) - n))


def test_fused_small_batch_non_finite_queries():
    import torch
    n, dim = 700_000, 64
    docs = xo.synthetic_unit_rows(n, dim, 77)
    scale = xo.estimate_scale(docs[:20_000], 0.98)
    idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4), keep_originals=False)
    assert _fused_available(idx, 2, 5)
    good = xo.synthetic_unit_rows(2, dim, 78)
    bad = good.copy()
    bad[1, 3] = np.nan
    for q in (bad, bad.astype(np.float64), torch.from_numpy(bad).cuda(), torch.from_numpy(bad).pin_memory()):
        with pytest.raises(xb.InvalidInputError):
            xb.search(idx, q, 5)
    assert xsearch.pending_nonfinite() == 0                     # raising cleared the counter
    # asynchronous pipelines: no synchronisation, the bad query comes back empty, the good one is answered, the counter reports it
    ref = xb.search_device(idx, torch.from_numpy(good).cuda(), 5)
    keys = xb.search_device(idx, torch.from_numpy(bad).cuda(), 5, check=False)
    assert bool((keys[1] == -1).all()) and torch.equal(keys[0], ref[0])
    assert xsearch.pending_nonfinite() == 1
    with pytest.raises(xb.InvalidInputError):                   # the next checked call (or an explicit check) reports it
        xb.search_device(idx, torch.from_numpy(good).cuda(), 5)
    assert xsearch.pending_nonfinite() == 0
    xsearch.raise_pending_nonfinite()                           # nothing pending: no error
