import sys, time; sys.path.insert(0, ".")
import torch, bench, numpy as np, paper_2008_02002_b200 as xb
x = bench.gen_rows_gpu(torch, 0, 4_000_000, 4_000_000, 256)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); s = xb.estimate_scale(x, 0.98); torch.cuda.synchronize()
    print("estimate_scale 4M x 256 float32 on device:", round((time.perf_counter() - t0) * 1e3, 2), "ms, scale", s)
print("numpy:", 1.0 / float(np.quantile(np.abs(x[:1_000_000].cpu().numpy()), 0.98)), xb.estimate_scale(x[:1_000_000], 0.98))
