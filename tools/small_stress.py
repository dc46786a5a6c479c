"""Randomised stress of the small-batch paths (1-16 queries: the single-launch coop::search_kernel on corpora large enough for
it, the multi-launch mma.sync / XOR-POPC paths below that) against the CPU oracle: search() and k_select() without originals
(hits, threshold_distance, candidate_count with an extra distance), every width pair the reference accepts.
Usage: python tools/small_stress.py [seed] [shapes]"""
import os, sys
os.environ.setdefault('XFBQ_ENV_LIVE', '1')
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    n = int(rng.choice([1, 33, 1000, 20_000, 150_001, 640_000, 700_001, 1_500_000]))
    dim = int(rng.choice([1, 7, 64, 100, 128, 200, 256, 300, 384, 512, 513, 768]))
    wd = int(rng.integers(1, 9))
    wq = int(rng.integers(1, 9))
    if rng.random() < 0.6:      # the shapes the single-launch kernel takes
        wd, wq, dim = min(wd, 4), min(wq, 7), min(dim, 512)
    nq = int(rng.choice([1, 2, 5, 8, 15, 16]))
    k = int(rng.choice([1, 10, 100, 1000]))
    docs = xo.synthetic_unit_rows(n, dim, 500 + it)
    if n > 1000 and rng.random() < 0.5:     # blocks of exact ties among the best hits
        docs[n // 3: n // 3 + int(rng.choice([40, 300, 3000]))] = docs[17]
    queries = xo.synthetic_unit_rows(nq, dim, 600 + it)
    if n > 1000:
        queries[0] = docs[17]
    scale = xo.estimate_scale(docs[:20000], 0.98)
    idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=wq), keep_originals=False)
    s, i = xb.search(idx, queries, k)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), wq, scale).transpose(2, 0, 1)
    kk = min(k, n)
    want_d, want_i = xo.c_search(planes, qp, kk)
    ok = np.array_equal(s.astype(np.uint64), want_d) and np.array_equal(i, want_i)
    # k_select: ids, threshold and candidate count with an extra distance (search.py:206-216)
    extra = int(rng.choice([0, 0, 3, 50]))
    qi = int(rng.integers(0, nq))
    res = xb.k_select(idx, xb.SearchRequest(query=queries[qi].astype(np.float64), k=k, extra_distance=extra))
    d = xo.c_batch_distances(planes, np.ascontiguousarray(qp[qi]))
    thr = int(np.sort(d)[kk - 1]) + extra
    cand = np.flatnonzero(d <= thr)
    order = np.lexsort((cand, d[cand]))[:kk]
    ok2 = (res.threshold_distance == thr and res.candidate_count == cand.size
           and [h[0] for h in res.hits] == cand[order].tolist())
    bad += 0 if (ok and ok2) else 1
    tag = "ok" if (ok and ok2) else f"MISMATCH search={ok} k_select={ok2}"
    print(f"{tag} n={n} dim={dim} wd={wd} wq={wq} nq={nq} k={k} extra={extra}", flush=True)
print("ALL OK" if bad == 0 else f"{bad} MISMATCHES")
sys.exit(1 if bad else 0)
