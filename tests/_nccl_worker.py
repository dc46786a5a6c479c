"""torchrun worker of tests/test_gpu_nccl.py: R x Q sharded search on real CUDA kernels + NCCL, checked against the CPU oracle
on every rank.  Usage: torchrun --nproc-per-node G tests/_nccl_worker.py <query_shards>"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2008_02002_b200 as xb  # noqa: E402
from oracle import xfbq_oracle as xo  # noqa: E402
from paper_2008_02002_b200.sharded import grid_of  # noqa: E402


def main():
    query_shards = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        n, dim, k = 300_000, 256, 100
        docs = xo.synthetic_unit_rows(n, dim, 41)
        queries = xo.synthetic_unit_rows(333, dim, 42)
        scale = xo.estimate_scale(docs[:50_000], 0.98)
        params = xb.QuantParams(dim=dim, scale=scale, doc_bits=4, query_bits=4)
        R, r, _ = grid_of(world, rank, query_shards)
        lo, hi = xb.shard_bounds(n, R, r)
        shard = xb.ShardedIndex.build(docs[lo:hi], params, n_total=n, row_offset=lo, world=world, rank=rank,
                                      query_shards=query_shards)
        shard.always_gather = True
        planes = xo.c_quantize_matrix(docs, 4, scale)
        for nq in (333, 5, 1):
            qp = xo.c_quantize_matrix(queries[:nq].astype(np.float64), 4, scale).transpose(2, 0, 1)
            want_d, want_i = xo.c_search(planes, qp, k)
            scores, ids = shard.search(queries[:nq], k)
            assert np.array_equal(scores.astype(np.uint64), want_d), (rank, nq, "distances")
            assert np.array_equal(ids, want_i), (rank, nq, "ids")
            keys = shard.search_keys(torch.from_numpy(queries[:nq]).cuda(), k)      # device-resident queries
            assert np.array_equal((keys.cpu().numpy() & 0xFFFFFFFF), want_i)
        print(f"rank {rank}/{world} grid {R}x{query_shards}: ok", flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
