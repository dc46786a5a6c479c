"""QPS / latency over the batch size on one corpus (default config 4: 10M x 256, top-100): call time (CUDA events around
search_device, device-resident queries), the dominant kernel's time, the plan.  Usage: python tools/batch_sweep.py [n] [dim] [k] [nq,nq,...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import json
import numpy as np
import torch
import bench
import paper_2008_02002_b200 as xb
from paper_2008_02002_b200 import _native

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 256
k = int(sys.argv[3]) if len(sys.argv) > 3 else 100
nqs = [int(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1, 4, 8, 16, 24, 32, 48, 64, 128, 256, 512, 1024, 1250, 2500, 5000, 10000]
head = bench.gen_chunk_gpu(torch, 0, min(bench.CHUNK, n), dim)[:100_000].cpu().numpy()
scale = xb.estimate_scale(head, 0.98)
params = xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4)
docs = bench.gen_rows_gpu(torch, 0, n, n, dim)
index = xb.build_index(docs, params, keep_originals=False)
del docs
torch.cuda.empty_cache()
q = torch.from_numpy(bench.gen_queries(max(nqs), dim)).cuda()
db_bytes = index.packed.nbytes
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for nq in nqs:
    plan = np.zeros(6, dtype=np.int32)
    _native.check(_native.lib().xfbq_scan_plan(n, dim, 4, nq, 4, k, 1, plan.ctypes.data))
    for _ in range(3):
        xb.search_device(index, q[:nq], k)
    torch.cuda.synchronize()
    reps = 20 if nq <= 1024 else 5
    e0.record()
    for r in range(reps):
        xb.search_device(index, q[:nq], k, check=False)   # pipelined: no host synchronisation between the calls
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    import time as _t
    torch.cuda.synchronize(); t0 = _t.perf_counter()
    for r in range(reps):
        xb.search_device(index, q[:nq], k); torch.cuda.synchronize()   # one search at a time, host-synchronous
    sync_ms = (_t.perf_counter() - t0) / reps * 1e3
    _native.set_timing(True)
    kms = []
    for r in range(3):
        xb.search_device(index, q[:nq], k); kms.append(_native.last_scan_ms())
    _native.set_timing(False)
    kms = sorted(kms)[1]
    tensor_ms = 2.0 * n * nq * ((dim + 127) // 128 * 128) / 4762.5e12 * 1e3
    hbm_ms = db_bytes / 6538.6e9 * 1e3
    bound = max(tensor_ms, hbm_ms)
    print(json.dumps({"nq": nq, "call_ms": round(ms, 4), "sync_call_ms": round(sync_ms, 4), "kernel_ms": round(kms, 4), "qps": round(nq / ms * 1e3, 1),
                      "engine": int(plan[4]), "q_per_cta": int(plan[0]), "groups": int(plan[1]), "parts": int(plan[2]),
                      "bound_ms": round(bound, 4), "frac_of_bound": round(bound / ms, 3)}), flush=True)
