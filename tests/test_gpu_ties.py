"""Tie torture: corpora with 1, 8 and 1 000 DISTINCT rows repeated over >= 70k documents, so that far more
candidates than any list, ring or merge buffer holds share the k-th distance.  The reference order is
(distance asc, row id asc) (search.py:129-131, pinned by pkg/tests/test_search.py:93-97 at desk size); every
engine, the counted seed, the global candidate histogram ("bins >= b hold >= k candidates") and the bounded
merge cut must reproduce it bit for bit.  Expected results come from the CPU oracle on the oracle's planes.
"""
import numpy as np
import pytest

import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo

pytestmark = pytest.mark.gpu

DIM, WD, WQ = 256, 4, 4


def _corpus(n, distinct, seed):
    base = xo.synthetic_unit_rows(distinct, DIM, seed)
    rng = np.random.Generator(np.random.PCG64(seed + 7))
    pick = rng.integers(0, distinct, size=n)
    return base[pick]


def _expected(planes, queries, scale, k):
    qp = xo.c_quantize_matrix(queries.astype(np.float64), WQ, scale).transpose(2, 0, 1)
    return xo.c_search(planes, qp, k)


@pytest.mark.parametrize("distinct", [1, 8, 1000])
def test_ties_on_every_engine(distinct, monkeypatch):
    n = 300_000
    docs = _corpus(n, distinct, 900 + distinct)
    queries = xo.synthetic_unit_rows(300, DIM, 77)
    scale = xo.estimate_scale(xo.synthetic_unit_rows(20_000, DIM, 5), 0.98)
    params = xb.QuantParams(dim=DIM, scale=scale, doc_bits=WD, query_bits=WQ)
    idx = xb.build_index(docs, params, keep_originals=False)
    planes = xo.c_quantize_matrix(docs, WD, scale)
    assert np.array_equal(idx.packed.planes, planes)
    for k in (10, 100, 1000):
        want_d, want_i = _expected(planes, queries, scale, k)
        if distinct == 1:  # every distance equal: the answer is rows 0 .. k-1
            assert np.array_equal(want_i, np.tile(np.arange(k), (300, 1)))
        routes = [
            {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1"},                                  # counted seed + queue kernel + bounded merge
            {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_UMMA_SLICES": "9"},        # several document slices per group
            {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_UMMA_STAGES": "2"},        # two-tile operand ring: the issuer's "next group not ready" path
            {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_MERGE_BUF": "2048" if k > 512 else "1024"},  # merge overflow path
            {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_UMMA_HIST": "0"},          # no candidate histogram
            {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_SEED_HIST": "0"},          # list-keeping sample scan
            {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_SAMPLE": "0"},             # open thresholds
            {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE": "0"},                                          # list-owning epilogue kernel
            {"XFBQ_ENGINE": "umma"},                                                                  # the default plan of the tcgen05 engine
            {"XFBQ_ENGINE": "imma"},
            {"XFBQ_ENGINE": "popc"},
        ]
        for env in routes:
            for key, val in env.items():
                monkeypatch.setenv(key, val)
            scores, ids = xb.search(idx, queries, k)
            for key in env:
                monkeypatch.delenv(key)
            assert np.array_equal(scores.astype(np.uint64), want_d), (distinct, k, env)
            assert np.array_equal(ids, want_i), (distinct, k, env)
        # small batches (mma.sync HBM-bound plan, counted seed, two merge levels) and a single query
        for nb in (1, 16):
            scores, ids = xb.search(idx, queries[:nb], k)
            assert np.array_equal(scores.astype(np.uint64), want_d[:nb]) and np.array_equal(ids, want_i[:nb]), (distinct, k, nb)


def test_ties_at_two_million_rows_default_plan():
    """n = 2.1M rows with 8 distinct values: the production plan (queue kernel, counted seed spread over the database,
    shared thresholds, global histogram) with ~260k-way ties at every distance."""
    n = 2_100_000
    docs = _corpus(n, 8, 4242)
    queries = xo.synthetic_unit_rows(520, DIM, 78)
    scale = xo.estimate_scale(xo.synthetic_unit_rows(20_000, DIM, 5), 0.98)
    params = xb.QuantParams(dim=DIM, scale=scale, doc_bits=WD, query_bits=WQ)
    idx = xb.build_index(docs, params, keep_originals=False)
    planes = xo.c_quantize_matrix(docs, WD, scale)
    for k in (10, 100, 1000):
        want_d, want_i = _expected(planes, queries[:64], scale, k)
        scores, ids = xb.search(idx, queries, k)
        assert np.array_equal(scores[:64].astype(np.uint64), want_d), k
        assert np.array_equal(ids[:64], want_i), k
        k64 = (scores.astype(np.int64) << 32) | ids
        assert bool((k64[:, 1:] > k64[:, :-1]).all())
