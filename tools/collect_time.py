import sys; sys.path.insert(0,'.')
import numpy as np, torch, bench
import paper_2008_02002_b200 as xb
from paper_2008_02002_b200 import _native
n, dim = 10_000_000, 256
docs = bench.gen_rows_gpu(torch, 0, n, n, dim)
scale = xb.estimate_scale(docs[:100000], 0.98)
idx = xb.build_index(docs, xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4), keep_originals=False)
del docs
q = torch.from_numpy(bench.gen_queries(4, dim)).cuda()
qw = xb.quantize_queries(q[:1], 4, scale)
L = _native.lib(); pm = idx.packed
nib = pm.nibble_layout
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, ptr in (("planes/POPC", L.xfbq_collect_candidates, pm.codes.data_ptr()), ("nibbles/dp4a", L.xfbq_collect_candidates_nibbles, nib.data_ptr())):
    for thr in (20000, 30000):
        for _ in range(3): fn(ptr, n, dim, 4, qw.data_ptr(), 4, thr, None, 0, cnt.data_ptr(), st)
        e0.record()
        for _ in range(10): fn(ptr, n, dim, 4, qw.data_ptr(), 4, thr, None, 0, cnt.data_ptr(), st)
        e1.record(); torch.cuda.synchronize()
        print(name, thr, "count", int(cnt.item()), f"{e0.elapsed_time(e1)/10*1e3:.1f} us")
