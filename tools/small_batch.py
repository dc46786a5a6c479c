"""Small-batch driver for profiling: build the config-4 index once, then run nq-query searches.
Usage: python tools/small_batch.py [nq] [reps]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
import paper_2008_02002_b200 as xb

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n, dim = 10_000_000, 256
head = bench.gen_chunk_gpu(torch, 0, bench.CHUNK, dim)[:100_000].cpu().numpy()
scale = xb.estimate_scale(head, 0.98)
params = xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4)
docs = bench.gen_rows_gpu(torch, 0, n, n, dim)
index = xb.build_index(docs, params, keep_originals=False)
del docs
q = torch.from_numpy(bench.gen_queries(1024, dim)).cuda()
for r in range(3):
    xb.search_device(index, q[:nq], 100)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for r in range(reps):
    xb.search_device(index, q[(r * nq) % 512:(r * nq) % 512 + nq], 100)
e1.record(); torch.cuda.synchronize()
print(f"nq={nq}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us per search")
