import os, sys
os.environ.setdefault('XFBQ_ENV_LIVE', '1')
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo
"""One tcgen05-engine search against the oracle, small enough for compute-sanitizer.
Usage: python tools/umma_one.py [seeded]   seeded: the full-size route (counted seed, queue kernel, bounded merge,
candidate gather) forced onto a 40k-row corpus."""
os.environ["XFBQ_ENGINE"] = "umma"
n, dim, wd, nq, k = 6000, 256, 4, 300, 20
if len(sys.argv) > 1 and sys.argv[1] == "seeded":
    os.environ.update({"XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_SAMPLE": "2048", "XFBQ_UMMA_SLICES": "3"})
    n, nq, k = 40000, 300, 20
docs = xo.synthetic_unit_rows(n, dim, 5); queries = xo.synthetic_unit_rows(nq, dim, 6)
scale = xo.estimate_scale(docs, 0.98)
idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=4), keep_originals=False)
s, i = xb.search(idx, queries, k)
planes = xo.c_quantize_matrix(docs, wd, scale)
qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
d_, i_ = xo.c_search(planes, qp, k)
print("match", np.array_equal(s.astype(np.uint64), d_) and np.array_equal(i, i_))
if len(sys.argv) > 1 and sys.argv[1] == "seeded":
    r = xb.k_select(idx, xb.SearchRequest(query=queries[0].astype(np.float64), k=k))
    print("k_select", [h[0] for h in r.hits] == i_[0].tolist(), r.candidate_count)
    del os.environ["XFBQ_ENGINE"]
    s1, i1 = xb.search(idx, queries[:3], k)   # small batch: mma.sync engine with the counted seed
    print("small batch match", np.array_equal(i1, i_[:3]))
