"""Phase time stamps of the single-launch small-batch search (coop::search_kernel, xfbq_debug_profile).
Usage (under gpurun): python tools/coop_profile.py [nq] [n] [dim] [k]"""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench
import paper_2008_02002_b200 as xb
from paper_2008_02002_b200 import _native

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 256
k = int(sys.argv[4]) if len(sys.argv) > 4 else 100
docs = bench.gen_rows_gpu(torch, 0, n, n, dim)
scale = xb.estimate_scale(docs[:100_000], 0.98)
idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4), keep_originals=False)
del docs
q = torch.from_numpy(bench.gen_queries(64, dim)).cuda()
for _ in range(3):
    xb.search_device(idx, q[:nq], k)
prof = torch.zeros(8 + 2 * 148, dtype=torch.int64, device="cuda")
_native.check(_native.lib().xfbq_debug_profile(prof.data_ptr()))
for rep in range(3):
    xb.search_device(idx, q[rep * nq:(rep + 1) * nq], k)
    torch.cuda.synchronize()
    t = prof.cpu().numpy().astype(np.int64)
    t0 = t[0]
    names = ["prep+zero -> sync", "sample hist -> sync", "thresholds -> sync", "scan (all CTAs) -> sync", "merge"]
    print(" | ".join(f"{nm} {(t[i + 1] - t[i]) / 1e3:.1f} us" for i, nm in enumerate(names)), f"| total {(t[5] - t0) / 1e3:.1f} us, merged entries {t[6]}")
    ends = (t[8:8 + 148] - t[3]) / 1e3
    print(f"   per-CTA scan end after phase 3: min {ends.min():.1f} median {np.median(ends):.1f} max {ends.max():.1f} us")
_native.check(_native.lib().xfbq_debug_profile(0))
