"""One single-launch small-batch search (coop::search_kernel) and one fused k_select against the oracle, sized for
compute-sanitizer: 640k x 64-d (the smallest database that takes the cooperative path), 3 queries."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo
n, dim, k = 640_000, 64, 20
docs = xo.synthetic_unit_rows(n, dim, 5); queries = xo.synthetic_unit_rows(3, dim, 6)
scale = xo.estimate_scale(docs[:20000], 0.98)
idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4), keep_originals=False)
assert int(xb._native.lib().xfbq_search_small_workspace_bytes(n, dim, 4, 3, 4, k)) > 0
s, i = xb.search(idx, queries, k)
planes = xo.c_quantize_matrix(docs, 4, scale)
qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
d_, i_ = xo.c_search(planes, qp, k)
print("match", np.array_equal(s.astype(np.uint64), d_) and np.array_equal(i, i_))
r = xb.k_select(idx, xb.SearchRequest(query=queries[0].astype(np.float64), k=k, extra_distance=40))
d0 = xo.c_batch_distances(planes, xo.np_quantize_vector(queries[0].astype(np.float64), 4, scale))
print("k_select", [h[0] for h in r.hits] == i_[0].tolist(), r.candidate_count == int((d0 <= d_[0, -1] + 40).sum()))
