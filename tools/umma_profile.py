"""Per-role wait-cycle breakdown of the tcgen05 scan kernel (xfbq_debug_profile counters).
Usage (under gpurun): python tools/umma_profile.py [nq] [n] [dim]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb  # noqa: E402
from paper_2008_02002_b200 import _native  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 256
k = int(sys.argv[4]) if len(sys.argv) > 4 else 100
g = torch.Generator(device="cuda").manual_seed(1)
docs = torch.randn((n, dim), generator=g, device="cuda")
docs /= docs.norm(dim=1, keepdim=True)
q = torch.randn((nq, dim), generator=g, device="cuda")
q /= q.norm(dim=1, keepdim=True)
import numpy as _np; scale = 1.0 / float(_np.quantile(_np.abs(docs[:100000].cpu().numpy()), 0.98))
idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4), keep_originals=False)
del docs
for _ in range(2):
    xb.search(idx, q, k)
prof = torch.zeros((148 * 60,), dtype=torch.int64, device="cuda")
_native.check(_native.lib().xfbq_debug_profile(prof.data_ptr()))
_native.set_timing(True)
xb.search(idx, q, k)
ms = _native.last_scan_ms()
_native.set_timing(False)
_native.check(_native.lib().xfbq_debug_profile(0))
allc = prof.cpu().numpy().astype(np.float64)
c = allc[:148 * 8].reshape(148, 8)
x = allc[148 * 8:148 * 12].reshape(148, 4)
per_warp = allc[148 * 12:148 * 24].reshape(148, 12)
ring_full = allc[148 * 24:148 * 36].reshape(148, 12)
park = allc[148 * 36:].reshape(148, 2, 12)
tot = c[:, 6].mean()
st = c[:, 7].mean()
print(f"kernel {ms:.3f} ms; per CTA: {tot / 1e6:.2f} Mclk, {st:.0f} stages, {tot / st:.0f} clk/stage")
names = ["epi wait acc_full", "epi slow-path chunks (warp 0)", "mma wait b_full", "mma wait acc_empty", "prod wait b_empty",
         "drain wait ring full (warp 0)"]
for i, nm in enumerate(names):
    if i == 1:
        print(f"  {nm:34s} {c[:, i].mean():12.0f}  ({c[:, i].mean() / (st * 4) * 100:.1f}% of chunks)")
    else:
        print(f"  {nm:34s} {c[:, i].mean() / 1e6:9.2f} Mclk  {c[:, i].mean() / tot * 100:5.1f}%  min {c[:, i].min() / tot * 100:5.1f}% max {c[:, i].max() / tot * 100:5.1f}%")
print(f"  epi warp0 compactions {x[:, 2].mean():.0f}")
print(f"  issuer probes that failed (per CTA): second query tile {x[:, 0].mean():.0f}, next document tile {x[:, 1].mean():.0f} of {st:.0f} tiles (16-bit counters)")
print("  drain warps waiting for an accumulator, % of the kernel (warp = 4 * set + lane quarter): " + " ".join(f"{v / tot * 100:.0f}" for v in per_warp.mean(axis=0)))
print("  drain warps waiting for room in their ring, clk per tile: " + " ".join(f"{v / st:.1f}" for v in ring_full.mean(axis=0)) + f"  (sum {ring_full.mean(axis=0).sum() / st:.1f})")
print(f"  park path: {park[:, 1, :].sum() / 148 / st:.2f} chunks per tile park a row, {park[:, 0, :].sum() / max(park[:, 1, :].sum(), 1):.0f} clk each (ring waits included)")
if len(sys.argv) > 5:
    print("per CTA: stages, total Mclk, clk/stage, mma wait acc_empty %, mma wait b_full %, drain w0 wait acc_full %, ring-full %")
    for b in range(148):
        print(b, int(c[b, 7]), round(c[b, 6] / 1e6, 2), int(c[b, 6] / max(c[b, 7], 1)), round(100 * c[b, 3] / c[b, 6], 1), round(100 * c[b, 2] / c[b, 6], 1),
              round(100 * c[b, 0] / c[b, 6], 1), round(100 * c[b, 5] / c[b, 6], 1))
