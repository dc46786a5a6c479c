"""Fast float32 quantizer vs the float64 kernel on adversarial inputs (values on and next to code boundaries,
denormals, +-0, huge values) and on random data; prints kernel timings."""
import os, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb

def planes(x, w, scale, slow):
    os.environ["XFBQ_QUANT_SLOW"] = "1" if slow else "0"
    return xb.quantize_matrix(x, w, scale)

rng = np.random.default_rng(5)
bad = 0
for w in range(1, 9):
    for scale in (1.0, 0.7310585786300049, 3.3333333333333335, 12.345, 1e-3):
        half = 2.0 ** (w - 1)
        grid = (np.arange(-half - 3, half + 4) / (scale * half))               # exact boundaries in x space (as f64)
        g32 = grid.astype(np.float32)
        near = np.concatenate([g32, np.nextafter(g32, np.float32(np.inf)), np.nextafter(g32, np.float32(-np.inf)),
                               np.nextafter(np.nextafter(g32, np.float32(np.inf)), np.float32(np.inf))])
        bits = g32.view(np.int32)[None, :] + np.arange(-40, 41, dtype=np.int32)[:, None]   # every float32 within 40 ulps of a boundary
        sweep = bits.astype(np.int32).view(np.float32).ravel()
        near = np.concatenate([near, sweep[np.isfinite(sweep)]])
        special = np.array([0.0, -0.0, 1e-45, -1e-45, 1e-38, -1e-38, 3e38, -3e38, 1.0, -1.0, 0.5, -0.5], dtype=np.float32)
        rnd = rng.uniform(-2, 2, size=20000).astype(np.float32) / np.float32(scale)
        vals = np.concatenate([near, special, rnd]).astype(np.float32)
        pad = (-len(vals)) % 128
        vals = np.concatenate([vals, np.zeros(pad, np.float32)]).reshape(-1, 128)
        xd = torch.from_numpy(vals).cuda()
        a = planes(xd, w, scale, False).planes
        b = planes(xd, w, scale, True).planes
        if not np.array_equal(a, b):
            bad += 1
            print("MISMATCH", w, scale, int((a != b).sum()))
print("FAILED" if bad else "ALL OK")
x = torch.randn((2_000_000, 256), device="cuda"); x /= x.norm(dim=1, keepdim=True)
for slow in (True, False):
    os.environ["XFBQ_QUANT_SLOW"] = "1" if slow else "0"
    xb.quantize_matrix(x, 4, 14.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): p = xb.quantize_matrix(x, 4, 14.0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"slow={slow}: {ms:.3f} ms per 2M x 256 ({x.numel() * 4 / ms / 1e6:.0f} GB/s read)")
os.environ.pop("XFBQ_QUANT_SLOW", None)

# zero-heavy rows (x = 0 sits exactly on a code boundary: the fast path re-examines those groups without float64)
xz = x * (torch.rand_like(x) < 0.5)
xb.quantize_matrix(xz, 4, 14.0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): p = xb.quantize_matrix(xz, 4, 14.0)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"half zeros: {ms:.3f} ms per 2M x 256 ({x.numel() * 4 / ms / 1e6:.0f} GB/s read)")
for w in (1, 2, 3, 5, 8):
    xb.quantize_matrix(x, w, 14.0)
    e0.record()
    for _ in range(5): p = xb.quantize_matrix(x, w, 14.0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"width {w}: {ms:.3f} ms per 2M x 256 ({x.numel() * 4 / ms / 1e6:.0f} GB/s read)")
