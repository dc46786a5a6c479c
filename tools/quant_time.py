"""Kernel-level timing of the document quantizer through the C ABI (no allocation or host synchronisation between launches).
Usage (under gpurun): python tools/quant_time.py [n] [dim]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_02002_b200 import _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 256
L = _native.lib()
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.randn((n, dim), generator=g, device="cuda")
x /= x.norm(dim=1, keepdim=True)
bad = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def run(label, src, width, scale=14.0, reps=10):
    out = torch.empty(int(L.xfbq_db_bytes(n, dim, width)), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        _native.check(L.xfbq_quantize_pack_f32(src.data_ptr(), n, dim, dim, scale, width, out.data_ptr(), bad.data_ptr(), st))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _native.check(L.xfbq_quantize_pack_f32(src.data_ptr(), n, dim, dim, scale, width, out.data_ptr(), bad.data_ptr(), st))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rd, wr = src.numel() * 4, out.numel()
    print(f"{label:28s} width {width}: {ms:7.3f} ms  read {rd / ms / 1e6:6.0f} GB/s  read+write {(rd + wr) / ms / 1e6:6.0f} GB/s", flush=True)


for w in (4, 1, 2, 3, 5, 6, 7, 8):
    run("unit-norm rows", x, w)
xz = x * (torch.rand_like(x) < 0.5)
run("half of the values zero", xz, 4)
xs = x * 10.0
run("40 % of the values clipped", xs, 4)
print("nonfinite counter", int(bad.item()))
