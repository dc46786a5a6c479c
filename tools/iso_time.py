"""Isolated kernel time of the 10k-query scan (spaced launches, no power-cap effects).  Usage: python tools/iso_time.py"""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb
from paper_2008_02002_b200 import _native
nq, n, dim, k = 10000, 10_000_000, 256, 100
g = torch.Generator(device="cuda").manual_seed(1)
docs = torch.randn((n, dim), generator=g, device="cuda"); docs /= docs.norm(dim=1, keepdim=True)
q = torch.randn((nq, dim), generator=g, device="cuda"); q /= q.norm(dim=1, keepdim=True)
import numpy as _np; scale = 1.0 / float(_np.quantile(_np.abs(docs[:100000].cpu().numpy()), 0.98))
idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4), keep_originals=False)
del docs
_native.set_timing(True)
ts = []
for i in range(8):
    xb.search_device(idx, q, k); ts.append(_native.last_scan_ms()); time.sleep(0.4)
print("main scan kernel ms:", " ".join(f"{t:.2f}" for t in ts))
