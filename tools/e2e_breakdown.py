"""Where the end-to-end time of ShardedIndex.search goes (host buffers in, numpy out)."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb
import importlib; xs = importlib.import_module("paper_2008_02002_b200.search")

n, dim, nq, k = 10_000_000, 256, 10000, 100
g = torch.Generator(device="cuda").manual_seed(1)
docs = torch.randn((n, dim), generator=g, device="cuda"); docs /= docs.norm(dim=1, keepdim=True)
q = torch.randn((nq, dim), generator=g, device="cuda"); q /= q.norm(dim=1, keepdim=True)
scale = xb.estimate_scale(docs[:100000].cpu().numpy(), 0.98)
params = xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4)
sh = xb.ShardedIndex.build(docs, params, n_total=n, row_offset=0)
del docs
qp = q.cpu().pin_memory()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, r
ms, _ = t(lambda: sh.search(qp, k)); print(f"ShardedIndex.search (pinned in, numpy out): {ms:.2f} ms")
ms, keys = t(lambda: sh.search_keys(q, k)); print(f"search_keys, device queries: {ms:.2f} ms")
ms, _ = t(lambda: sh.search_keys(qp, k)); print(f"search_keys, pinned host queries: {ms:.2f} ms")
ms, _ = t(lambda: qp.cuda()); print(f"H2D queries: {ms:.2f} ms")
ms, kc = t(lambda: keys.cpu()); print(f"keys.cpu(): {ms:.2f} ms")
kn = kc.numpy().view(np.uint64)
ms, _ = t(lambda: ((kn >> np.uint64(32)).astype(np.int64), (kn & np.uint64(0xFFFFFFFF)).astype(np.int64))); print(f"numpy unpack: {ms:.2f} ms")
ms, _ = t(lambda: xs.unpack_keys_device(keys)); print(f"device unpack: {ms:.2f} ms")
d, i = xs.unpack_keys_device(keys)
ms, _ = t(lambda: (d.cpu(), i.cpu())); print(f"d.cpu(), i.cpu(): {ms:.2f} ms")
# per-call times: outliers point at the host side (allocator, scheduler), not at the kernels
import gc
times = []
for _ in range(40):
    t0 = time.perf_counter(); r = sh.search(qp, k); times.append((time.perf_counter() - t0) * 1e3)
print("per-call ms:", " ".join(f"{x:.1f}" for x in times))
gc.disable()
times = []
for _ in range(40):
    t0 = time.perf_counter(); r = sh.search(qp, k); times.append((time.perf_counter() - t0) * 1e3)
print("per-call ms, gc off:", " ".join(f"{x:.1f}" for x in times))
