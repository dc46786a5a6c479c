"""Randomised stress of the tcgen05 QUEUE kernel (counted seed, document slices, operand-ring depths, in-place / emitted lists)
against the CPU oracle: the full-size route forced onto corpora of 20k-400k rows.  Usage: python tools/queue_stress.py [seed] [shapes]"""
import os, sys
os.environ.setdefault('XFBQ_ENV_LIVE', '1')
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
os.environ["XFBQ_ENGINE"] = "umma"
os.environ["XFBQ_UMMA_QUEUE_MIN_N"] = "1"
DEFAULT_PLANS = os.environ.get("QS_DEFAULT_PLANS", "0") == "1"   # no plan overrides: the planner's own sample, slices and ring depth
bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    n = int(rng.choice([20_000, 33_333, 70_001, 150_000, 400_000] + ([40_000, 100_000, 250_000, 900_000] if DEFAULT_PLANS else [])))
    dim = int(rng.choice([64, 128, 200, 256, 300, 384, 512, 700, 1024]))
    wd = int(rng.integers(1, 9))
    nq = int(rng.choice([17, 100, 128, 129, 256, 257, 520, 700]))
    k = int(rng.choice([1, 10, 100, 1000]))
    env = {"XFBQ_UMMA_SLICES": str(int(rng.choice([0, 1, 2, 3, 7, 20]))), "XFBQ_UMMA_STAGES": str(int(rng.choice([2, 3, 5]))),
           "XFBQ_SAMPLE": str(int(rng.choice([2048, 8192])))}
    if env["XFBQ_UMMA_SLICES"] == "0":
        del env["XFBQ_UMMA_SLICES"]
    for key in ("XFBQ_UMMA_SLICES", "XFBQ_UMMA_STAGES", "XFBQ_SAMPLE"):
        os.environ.pop(key, None)
    if DEFAULT_PLANS:
        env = {}
    os.environ.update(env)
    docs = xo.synthetic_unit_rows(n, dim, 300 + it)
    queries = xo.synthetic_unit_rows(nq, dim, 400 + it)
    scale = xo.estimate_scale(docs[:20000], 0.98)
    idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=4), keep_originals=False)
    s, i = xb.search(idx, queries, k)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
    wd_, wi_ = xo.c_search(planes, qp, min(k, n))
    ok = np.array_equal(s.astype(np.uint64), wd_) and np.array_equal(i, wi_)
    bad += 0 if ok else 1
    print(("ok      " if ok else "MISMATCH") + f" n={n} dim={dim} wd={wd} nq={nq} k={k} {env}", flush=True)
print("FAILED" if bad else "ALL OK", flush=True)
sys.exit(1 if bad else 0)
