"""GPU bring-up check for the tcgen05 engine: XFBQ_ENGINE=umma vs the IMMA engine vs the CPU oracle
on ragged shapes.  Usage (under gpurun): timeout 600 python tools/umma_check.py"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb  # noqa: E402
from oracle import xfbq_oracle as xo  # noqa: E402

CASES = [
    # n, dim, wd, nq, k
    (5000, 256, 4, 40, 10),
    (20000, 256, 4, 300, 100),
    (33333, 128, 3, 130, 7),
    (12345, 200, 4, 257, 33),
    (9000, 512, 4, 150, 100),
    (70000, 256, 4, 1000, 100),
    (3000, 100, 4, 20, 1000),
    (40000, 64, 2, 600, 1),
]


def run(engine, idx, queries, k, extra=None):
    os.environ["XFBQ_ENGINE"] = engine
    for key, val in (extra or {}).items():
        os.environ[key] = val
    try:
        return xb.search(idx, queries, k)
    finally:
        os.environ.pop("XFBQ_ENGINE", None)
        for key in (extra or {}):
            os.environ.pop(key, None)


def main():
    bad = 0
    for (n, dim, wd, nq, k) in CASES:
        docs = xo.synthetic_unit_rows(n, dim, 11 + n)
        queries = xo.synthetic_unit_rows(nq, dim, 12 + n)
        scale = xo.estimate_scale(docs, 0.98)
        params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=4)
        idx = xb.build_index(docs, params, keep_originals=False)
        planes = xo.c_quantize_matrix(docs, wd, scale)
        qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
        want_d, want_i = xo.c_search(planes, qp, k)
        for extra in ({}, {"XFBQ_GRID": "3"}, {"XFBQ_SAMPLE": "0"}, {"XFBQ_SAMPLE": "2048", "XFBQ_GRID": "5"}, {"XFBQ_UMMA_STAGES": "2"}):
            t0 = time.time()
            s, i = run("umma", idx, queries, k, extra)
            ok = np.array_equal(s.astype(np.uint64), want_d) and np.array_equal(i, want_i)
            bad += 0 if ok else 1
            nbad = int((s.astype(np.uint64) != want_d).sum()) if s.shape == want_d.shape else -1
            print(f"n={n} dim={dim} wd={wd} nq={nq} k={k} {extra}: {'OK' if ok else 'MISMATCH'} (bad dists {nbad}) {time.time() - t0:.2f}s", flush=True)
    print("FAILED" if bad else "ALL OK", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
