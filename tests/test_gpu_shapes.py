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
    for env in ({}, {"XFBQ_ENGINE": "umma"}, {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_SAMPLE": "4096"},
                {"XFBQ_ENGINE": "imma"}):
        for key, val in env.items():
            monkeypatch.setenv(key, val)
        for nq in (200, 5, 1):
            scores, ids = xb.search(idx, queries[:nq], k)
            assert np.array_equal(scores.astype(np.uint64), want_d[:nq]), (dim, env, nq)
            assert np.array_equal(ids, want_i[:nq]), (dim, env, nq)
        for key in env:
            monkeypatch.delenv(key)
