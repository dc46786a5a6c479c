"""Randomised small-shape stress of the tcgen05 engine against the CPU oracle (tiny n, k up to n, ragged dims)."""
import os, sys
os.environ.setdefault('XFBQ_ENV_LIVE', '1')
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
os.environ["XFBQ_ENGINE"] = "umma"
bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 60):
    n = int(rng.choice([1, 2, 31, 33, 127, 128, 129, 200, 1000, 4097, 20000]))
    dim = int(rng.choice([1, 7, 64, 100, 128, 129, 200, 256, 300, 384, 512, 513, 700, 1024]))
    wd = int(rng.integers(1, 9))
    nq = int(rng.choice([17, 40, 128, 129, 256, 257, 700]))
    k = int(rng.choice([1, 5, 100, 1000]))
    docs = xo.synthetic_unit_rows(n, dim, 100 + it)
    queries = xo.synthetic_unit_rows(nq, dim, 200 + it)
    scale = xo.estimate_scale(docs, 0.98)
    idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=4), keep_originals=False)
    s, i = xb.search(idx, queries, k)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
    wd_, wi_ = xo.c_search(planes, qp, min(k, n))
    ok = np.array_equal(s.astype(np.uint64), wd_) and np.array_equal(i, wi_)
    bad += 0 if ok else 1
    if not ok:
        print(f"MISMATCH n={n} dim={dim} wd={wd} nq={nq} k={k}", flush=True)
print("FAILED" if bad else "ALL OK", flush=True)
sys.exit(1 if bad else 0)
