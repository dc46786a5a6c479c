"""Row-sharded search across the GPUs of one box (no reference code -- the paper
only states "QPS increases linearly").

Rank g holds rows [g*ceil(n/G), min(n, (g+1)*ceil(n/G))) of the database, queries are
replicated, every rank produces its local top-k keys (distance << 32 | GLOBAL row id) with the
fused scan, and ONE collective follows: an all-gather of the [nq, k] uint64 keys over
NCCL/NVLink (8 MB per GPU at nq=10k, k=100), then the G-way merge kernel.  The key order is
total, so the result is bit-identical for every G.

One process per GPU (`torch.distributed`, backend nccl).  The scan and merge callables are
injectable so the partition/gather logic is testable with gloo on CPU against the oracle;
the defaults are the CUDA kernels and there is no host fallback.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import InvalidInputError
from .index import Index, QuantParams, build_index


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range of `rank`: per = ceil(n / world); [rank*per, min(n, (rank+1)*per))."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidInputError(f"bad rank {rank} of {world}")
    per = -(-int(n) // world) if n else 0
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def _cuda_scan(index: Index, queries, k: int, row_offset: int):
    from .search import search_device
    return search_device(index, queries, k, row_offset=row_offset)


def _cuda_merge(stacked, k: int):
    """stacked: int64 CUDA tensor [parts, nq, k] -> [nq, k]."""
    torch = _native.require_cuda()
    L = _native.lib()
    parts, nq, kk = stacked.shape
    with torch.cuda.device(stacked.device):
        out = torch.empty((nq, kk), dtype=torch.int64, device=stacked.device)
        if nq and kk:
            _native.check(L.xfbq_merge_topk(stacked.data_ptr(), parts, nq, kk, out.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream))
    return out


@dataclass
class ShardedIndex:
    """This rank's shard of a row-partitioned database."""

    local: object            # Index (CUDA) -- or any object the injected scan_fn understands
    row_offset: int          # global id of local row 0
    n_total: int
    world: int = 1
    rank: int = 0
    group: object = None
    scan_fn: object = None   # (local, queries, k_local, row_offset) -> int64 tensor [nq, k_local] of keys
    merge_fn: object = None  # (stacked [parts, nq, k], k) -> [nq, k]

    @classmethod
    def build(cls, local_vectors, params: QuantParams, n_total: int, row_offset: int, world: int = 1,
              rank: int = 0, group=None, **kw) -> "ShardedIndex":
        """Quantize this rank's rows (already the [lo, hi) slice of the corpus) on its GPU."""
        idx = build_index(local_vectors, params, keep_originals=False, **kw)
        return cls(local=idx, row_offset=int(row_offset), n_total=int(n_total), world=world, rank=rank,
                   group=group)

    def search_keys(self, queries, k: int):
        """Local scan -> all-gather -> merge.  Every rank returns the same [nq, min(k, n_total)]
        key tensor (int64 holding the uint64 keys; empty slots are all-ones)."""
        import torch
        import torch.distributed as dist
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        scan = self.scan_fn or _cuda_scan
        merge = self.merge_fn or _cuda_merge
        kk = min(int(k), self.n_total)
        n_local = self.local.n
        k_local = min(kk, n_local)
        nq = queries.shape[0]
        if k_local == kk:
            pad = scan(self.local, queries, k_local, self.row_offset)
        else:  # short (or empty) shard: all-ones = empty slot
            pad = torch.full((nq, kk), -1, dtype=torch.int64, device="cpu" if self.scan_fn else "cuda")
            if k_local > 0:
                local = scan(self.local, queries, k_local, self.row_offset)
                pad = pad.to(local.device)
                pad[:, :k_local] = local
        if self.world == 1:
            return pad
        gathered = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(gathered, pad, group=self.group)
        return merge(torch.stack(gathered).contiguous(), kk)

    def search(self, queries, k: int):
        """(scores, indices) as int64 numpy arrays [nq, min(k, n_total)], identical on all ranks."""
        keys = self.search_keys(queries, k)
        if not keys.is_cuda:  # CPU hooks (tests/test_sharded_gloo.py): unpack on the host
            kn = keys.numpy().view(np.uint64)
            return (kn >> np.uint64(32)).astype(np.int64), (kn & np.uint64(0xFFFFFFFF)).astype(np.int64)
        from .search import to_host_arrays, unpack_keys_device
        d, i = unpack_keys_device(keys)  # empty slots come back as -1
        d, i = to_host_arrays(d, i)
        return d, i
