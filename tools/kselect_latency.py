"""Latency of the reference-shaped single-query call k_select (quantize, fused scan + top-K, candidate gather,
optional float64 re-rank) on the headline shape.  Usage: python tools/kselect_latency.py [n] [originals 0/1]"""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
keep = bool(int(sys.argv[2])) if len(sys.argv) > 2 else False
dim, k = 256, 100
g = torch.Generator(device="cuda").manual_seed(1)
docs = torch.randn((n, dim), generator=g, device="cuda"); docs /= docs.norm(dim=1, keepdim=True)
q = torch.randn((64, dim), generator=g, device="cuda"); q /= q.norm(dim=1, keepdim=True)
qh = q.cpu().numpy().astype(np.float64)
scale = xb.estimate_scale(docs[:100000].cpu().numpy(), 0.98)
idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4), keep_originals=keep)
for i in range(4):
    xb.k_select(idx, xb.SearchRequest(query=qh[i], k=k))
t0 = time.perf_counter()
for i in range(4, 64):
    r = xb.k_select(idx, xb.SearchRequest(query=qh[i], k=k))
ms = (time.perf_counter() - t0) / 60 * 1e3
r = xb.k_select(idx, xb.SearchRequest(query=qh[0], k=k), collect_timing=True)
print(f"k_select n={n} originals={keep}: {ms:.3f} ms per query; candidates {r.candidate_count}, stages (synchronised): "
      + ", ".join(f"{a}={b * 1e3:.3f} ms" for a, b in r.stage_seconds.items()))
