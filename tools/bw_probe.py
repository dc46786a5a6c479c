"""HBM read-bandwidth probe on the config-4 database + sensitivity of the single-query scan to
ring depth / grid (env knobs).  Usage: python tools/bw_probe.py"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
import paper_2008_02002_b200 as xb

n, dim = 10_000_000, 256
head = bench.gen_chunk_gpu(torch, 0, bench.CHUNK, dim)[:100_000].cpu().numpy()
scale = xb.estimate_scale(head, 0.98)
params = xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4)
docs = bench.gen_rows_gpu(torch, 0, n, n, dim)
index = xb.build_index(docs, params, keep_originals=False)
del docs
nib = index.packed.nibble_layout
q = torch.from_numpy(bench.gen_queries(64, dim)).cuda()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us

v = nib.view(torch.int64)
t = timeit(lambda: v.sum())
print(f"torch int64 sum over {nib.numel()/1e9:.2f} GB: {t:.1f} us -> {nib.numel()/t/1e3:.0f} GB/s")
dst = torch.empty_like(nib)
t = timeit(lambda: dst.copy_(nib))
print(f"torch copy (read+write) : {t:.1f} us -> {2*nib.numel()/t/1e3:.0f} GB/s")
del dst
for env in [{}, {"XFBQ_RAW_STAGES": "2"}, {"XFBQ_RAW_STAGES": "3"}, {"XFBQ_NO_WIDE": "1"}, {"XFBQ_NO_WIDE": "1", "XFBQ_RAW_STAGES": "3"},
            {"XFBQ_GRID": "74"}, {"XFBQ_GRID": "296", "XFBQ_RAW_STAGES": "2"}, {"XFBQ_ENGINE": "popc"}]:
    for k in ("XFBQ_RAW_STAGES", "XFBQ_NO_WIDE", "XFBQ_GRID", "XFBQ_ENGINE"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for nq in (1, 8):
        t = timeit(lambda: xb.search_device(index, q[:nq], 100), reps=10)
        print(f"{env} nq={nq}: {t:.1f} us per search")
