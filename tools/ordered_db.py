"""Search time on a database stored in an order that makes its head unrepresentative (two clusters stored one
after the other, queries from the second), with the counted threshold sample taken from the head (XFBQ_SEED_SPREAD=0) or
spread over the whole database (default).  Usage: python tools/ordered_db.py [n] [nq]"""
import os, sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dim, k = 256, 100
g = torch.Generator(device="cuda").manual_seed(5)
c1 = torch.randn(dim, generator=g, device="cuda"); c2 = torch.randn(dim, generator=g, device="cuda")
docs = torch.randn((n, dim), generator=g, device="cuda")
docs[: n // 2] += 0.25 * c1
docs[n // 2:] += 0.25 * c2
docs /= docs.norm(dim=1, keepdim=True)
q = torch.randn((nq, dim), generator=g, device="cuda") + 0.25 * c2
q /= q.norm(dim=1, keepdim=True)
docs_sorted = docs                                         # cluster 1 first: the head holds nothing like the queries
docs = docs[torch.randperm(n, generator=g, device="cuda")].contiguous()
scale = xb.estimate_scale(docs[:100000].cpu().numpy(), 0.98)
params = xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4)
for name, d in (("random order", docs), ("sorted", docs_sorted)):
    sh = xb.ShardedIndex.build(d, params, n_total=n, row_offset=0)
    for spread in ("1", "0"):
        os.environ["XFBQ_SEED_SPREAD"] = spread
        for _ in range(2): sh.search_keys(q, k)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(3): keys = sh.search_keys(q, k)
        torch.cuda.synchronize()
        print(f"{name:13s} spread={spread}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms per {nq} queries", flush=True)
    del sh
