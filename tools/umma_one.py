import os, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo
os.environ["XFBQ_ENGINE"] = "umma"
n, dim, wd, nq, k = 6000, 256, 4, 300, 20
docs = xo.synthetic_unit_rows(n, dim, 5); queries = xo.synthetic_unit_rows(nq, dim, 6)
scale = xo.estimate_scale(docs, 0.98)
idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=4), keep_originals=False)
s, i = xb.search(idx, queries, k)
planes = xo.c_quantize_matrix(docs, wd, scale)
qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
d_, i_ = xo.c_search(planes, qp, k)
print("match", np.array_equal(s.astype(np.uint64), d_) and np.array_equal(i, i_))
