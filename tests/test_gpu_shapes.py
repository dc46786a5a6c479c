"""Tensor-engine shape coverage: every dim up to 512 (C = 1..4 chunks of 128 dims, incl. the three-chunk tiles of
257..384-d) on the tcgen05 and mma.sync engines against the CPU oracle, bit for bit.  The reference accepts any dim and
any widths 1..8 (quant.py:23-31, pkg/tests/test_distance.py:127-140); shapes outside the tensor engines take the POPC
kernels (covered by tests/test_gpu_parity.py::test_small_cases_everything_bit_exact)."""
import numpy as np
import pytest

import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo

pytestmark = pytest.mark.gpu


def _engine(n, dim, wd, nq, wq, k):
    plan = np.zeros(6, dtype=np.int32)
    xb._native.check(xb._native.lib().xfbq_scan_plan(n, dim, wd, nq, wq, k, 1, plan.ctypes.data))
    return int(plan[4])


@pytest.mark.parametrize("dim,wd", [(257, 4), (300, 3), (384, 4), (320, 2), (129, 4), (500, 4)])
def test_dims_on_tensor_engines(dim, wd, monkeypatch):
    n, k, wq = 70_000, 50, 4
    docs = xo.synthetic_unit_rows(n, dim, 300 + dim)
    queries = xo.synthetic_unit_rows(200, dim, 301 + dim)
    scale = xo.estimate_scale(docs[:20_000], 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=wq)
    idx = xb.build_index(docs, params, keep_originals=False)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    assert np.array_equal(idx.packed.planes, planes)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), wq, scale).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(planes, qp, k)
    assert _engine(n, dim, wd, 200, wq, k) == 3 and _engine(n, dim, wd, 5, wq, k) == 2   # tcgen05 / mma.sync by default
    for env in ({}, {"XFBQ_ENGINE": "umma"}, {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE": "0"},
                {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_SAMPLE": "4096"}, {"XFBQ_ENGINE": "imma"}):
        for key, val in env.items():
            monkeypatch.setenv(key, val)
        for nq in (200, 5, 1):
            scores, ids = xb.search(idx, queries[:nq], k)
            assert np.array_equal(scores.astype(np.uint64), want_d[:nq]), (dim, env, nq)
            assert np.array_equal(ids, want_i[:nq]), (dim, env, nq)
        for key in env:
            monkeypatch.delenv(key)


@pytest.mark.parametrize("wd,wq,dim", [(5, 3, 200), (8, 4, 256), (6, 7, 128), (8, 7, 512), (1, 7, 300), (7, 1, 96), (3, 7, 384)])
def test_wide_codes_on_the_tcgen05_engine(wd, wq, dim, monkeypatch):
    """doc_bits up to 8 (document codes are the UNSIGNED 8-bit operand of tcgen05.mma kind::i8) and query_bits up to 7
    (|2y - Aq| <= 127 fits the signed operand) at >= 50k rows with the tensor engine forced -- the widths of
    pkg/tests/test_distance.py:127-140 that fit it; query_bits = 8 (weights up to +-255) stays on the POPC kernels."""
    n, k = 60_000, 40
    docs = xo.synthetic_unit_rows(n, dim, 500 + 10 * wd + wq)
    queries = xo.synthetic_unit_rows(150, dim, 501 + 10 * wd + wq)
    scale = xo.estimate_scale(docs[:20_000], 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=wq)
    idx = xb.build_index(docs, params, keep_originals=False)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    assert np.array_equal(idx.packed.planes, planes)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), wq, scale).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(planes, qp, k)
    assert _engine(n, dim, wd, 150, wq, k) == 3
    for env in ({}, {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE": "0"}, {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_SAMPLE": "4096"},
                {"XFBQ_ENGINE": "popc"}):
        for key, val in env.items():
            monkeypatch.setenv(key, val)
        scores, ids = xb.search(idx, queries, k)
        assert np.array_equal(scores.astype(np.uint64), want_d), (wd, wq, env)
        assert np.array_equal(ids, want_i), (wd, wq, env)
        for key in env:
            monkeypatch.delenv(key)
    # small batches: the mma.sync engine for codes that fit a nibble; wider codes stay on the tcgen05 engine down to a
    # single query
    assert _engine(n, dim, wd, 3, wq, k) == (2 if wd <= 4 else 3)
    assert _engine(n, dim, wd, 1, wq, k) == (2 if wd <= 4 else 3)   # single queries too: the POPC kernels pay per code byte and query
    for nb in (3, 1):
        scores, ids = xb.search(idx, queries[:nb], k)
        assert np.array_equal(scores.astype(np.uint64), want_d[:nb]) and np.array_equal(ids, want_i[:nb])


def test_query_bits_8_stays_exact_on_popc():
    n, dim, k = 50_000, 128, 20
    docs = xo.synthetic_unit_rows(n, dim, 808)
    queries = xo.synthetic_unit_rows(40, dim, 809)
    scale = xo.estimate_scale(docs[:20_000], 0.98)
    for wd in (8, 1):
        params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=8)
        idx = xb.build_index(docs, params, keep_originals=False)
        planes = xo.c_quantize_matrix(docs, wd, scale)
        qp = xo.c_quantize_matrix(queries.astype(np.float64), 8, scale).transpose(2, 0, 1)
        want_d, want_i = xo.c_search(planes, qp, k)
        assert _engine(n, dim, wd, 40, 8, k) <= 1
        scores, ids = xb.search(idx, queries, k)
        assert np.array_equal(scores.astype(np.uint64), want_d) and np.array_equal(ids, want_i)


@pytest.mark.parametrize("dim,wd", [(513, 4), (640, 3), (768, 4), (1000, 4), (1024, 4), (768, 8)])
def test_dims_513_to_1024_on_two_part_tiles(dim, wd, monkeypatch):
    """513..1024 dims: byte tiles of two K parts (3 or 4 chunks of 128 dims each, padded to an even chunk count) that
    accumulate into one tensor-memory accumulator; the reference accepts any dim (pkg/tests/test_distance.py:50-59 goes to 513)."""
    n, k, wq = 60_000, 30, 4
    docs = xo.synthetic_unit_rows(n, dim, 700 + dim)
    queries = xo.synthetic_unit_rows(160, dim, 701 + dim)
    scale = xo.estimate_scale(docs[:10_000], 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=wq)
    idx = xb.build_index(docs, params, keep_originals=False)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    assert np.array_equal(idx.packed.planes, planes)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), wq, scale).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(planes, qp, k)
    assert _engine(n, dim, wd, 160, wq, k) == 3 and _engine(n, dim, wd, 2, wq, k) == 3 and _engine(n, dim, wd, 1, wq, k) == 3
    for env in ({}, {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE": "0"}, {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_SAMPLE": "4096"},
                {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_SAMPLE": "4096", "XFBQ_UMMA_SLICES": "3"}):
        for key, val in env.items():
            monkeypatch.setenv(key, val)
        for nq in (160, 5, 1):
            scores, ids = xb.search(idx, queries[:nq], k)
            assert np.array_equal(scores.astype(np.uint64), want_d[:nq]), (dim, wd, env, nq)
            assert np.array_equal(ids, want_i[:nq]), (dim, wd, env, nq)
        for key in env:
            monkeypatch.delenv(key)


def test_derived_layouts_are_built_on_demand_and_legacy_buffer_still_works():
    """A batch server never builds the nibble layout, a single-query server never the byte tiles; releasing one frees it
    until the next search that needs it.  The one-buffer form of ABI revision 1 (xfbq_build_derived + xfbq_scan_topk)
    gives the same keys."""
    import torch
    n, dim, k = 80_000, 256, 20
    docs = xo.synthetic_unit_rows(n, dim, 1234)
    queries = xo.synthetic_unit_rows(64, dim, 1235)
    scale = xo.estimate_scale(docs[:20_000], 0.98)
    idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4), keep_originals=False)
    pm = idx.packed
    assert pm.derived_nbytes == {"nibbles": 0, "tiles": 0}
    s64, i64 = xb.search(idx, queries, k)
    assert pm.derived_nbytes["nibbles"] == 0 and pm.derived_nbytes["tiles"] == 2 * pm.nbytes    # tcgen05 engine: tiles only
    s3, i3 = xb.search(idx, queries[:3], k)
    assert pm.derived_nbytes["nibbles"] == pm.nbytes                                              # mma.sync engine
    assert np.array_equal(s3, s64[:3]) and np.array_equal(i3, i64[:3])
    pm.release_layout("tiles")
    assert pm.derived_nbytes["tiles"] == 0
    s3b, i3b = xb.search(idx, queries[:3], k)                                                      # list-keeping seed without tiles
    assert np.array_equal(s3b, s3) and np.array_equal(i3b, i3) and pm.derived_nbytes["tiles"] == 0
    # ABI revision 1: one derived buffer
    L = xb._native.lib()
    st = torch.cuda.current_stream().cuda_stream
    derived = torch.empty(int(L.xfbq_derived_bytes(n, dim, 4)), dtype=torch.uint8, device="cuda")
    xb._native.check(L.xfbq_build_derived(pm.codes.data_ptr(), n, dim, 4, derived.data_ptr(), st))
    qwords = xb.quantize_queries(queries, 4, scale)
    for nq in (64, 3):
        ws = torch.empty(max(int(L.xfbq_scan_workspace_bytes(n, dim, 4, nq, 4, k, 1)), 16), dtype=torch.uint8, device="cuda")
        keys = torch.empty((nq, k), dtype=torch.int64, device="cuda")
        xb._native.check(L.xfbq_scan_topk(pm.codes.data_ptr(), derived.data_ptr(), n, dim, 4, qwords.data_ptr(), nq, 4, k, 0,
                                          keys.data_ptr(), ws.data_ptr(), ws.numel(), st))
        assert np.array_equal((keys.cpu().numpy() >> 32), s64[:nq]) and np.array_equal(keys.cpu().numpy() & 0xFFFFFFFF, i64[:nq])


@pytest.mark.parametrize("n,dim,wd", [(70_001, 256, 4), (50_000, 200, 3), (40_000, 768, 4), (30_000, 128, 7)])
def test_release_codes_and_rebuild_from_derived_layouts(n, dim, wd, monkeypatch):
    """The packed codes may be freed while a derived layout holds the same information (a batch server keeps the byte tiles
    alone, a single-query server the nibbles alone): searches that read the layout run without them, and everything that
    reads bit planes gets them back bit for bit (xfbq_restore_codes_from_tiles / _nibbles)."""
    docs = xo.synthetic_unit_rows(n, dim, 31)
    queries = xo.synthetic_unit_rows(40, dim, 32)
    scale = xo.estimate_scale(docs[:20_000], 0.98)
    idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=4), keep_originals=False)
    packed = idx.packed
    planes = xo.c_quantize_matrix(docs, wd, scale)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(planes, qp, 10)
    codes0 = packed.codes.clone()
    with pytest.raises(xb.InvalidInputError):
        packed.release_codes()                       # nothing to rebuild them from yet
    monkeypatch.setenv("XFBQ_ENGINE", "umma")
    s, i = xb.search(idx, queries, 10)               # builds the byte tiles
    assert np.array_equal(i, want_i) and packed.derived_nbytes["tiles"] > 0
    packed.release_codes()
    assert packed.device_nbytes == 0 and packed.codes_ptr is None
    s, i = xb.search(idx, queries, 10)               # tiles only: no packed codes in HBM
    assert np.array_equal(s.astype(np.uint64), want_d) and np.array_equal(i, want_i)
    assert packed.codes_ptr is None
    monkeypatch.delenv("XFBQ_ENGINE")
    with pytest.raises(xb.InvalidInputError):
        packed.release_layout("tiles")               # the only copy left
    assert torch_equal(packed.codes, codes0)         # rebuilt from the tiles
    packed._planes = None
    assert np.array_equal(packed.planes, planes)
    if wd <= 4 and dim <= 512:
        assert packed.nibble_layout is not None
        packed.release_layout("tiles")
        packed.release_codes()
        s1, i1 = xb.search(idx, queries[:3], 10)     # nibbles only (single-launch search or the mma.sync plan)
        assert np.array_equal(i1, want_i[:3]) and np.array_equal(s1.astype(np.uint64), want_d[:3])
        assert torch_equal(packed.codes, codes0)     # rebuilt from the nibbles
    monkeypatch.setenv("XFBQ_ENGINE", "popc")        # the XOR/POPC kernels read the packed codes: rebuilt on demand
    packed.tile_layout
    packed.release_codes()
    s2, i2 = xb.search(idx, queries[:5], 10)
    assert np.array_equal(i2, want_i[:5]) and np.array_equal(s2.astype(np.uint64), want_d[:5])


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))
