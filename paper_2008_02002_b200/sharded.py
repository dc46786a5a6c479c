"""Sharded search across the GPUs of one box (no reference code -- the paper only states "QPS increases
linearly").

The G ranks form an R x Q grid (G = R * Q): rank g holds ROW shard r = g // Q of the database -- rows
[r*ceil(n/R), min(n, (r+1)*ceil(n/R))) -- and answers QUERY block c = g % Q of every batch -- queries
[c*ceil(nq/Q), ...).  Every rank scans its rows for its queries with the fused scan (keys carry GLOBAL row ids), then ONE
collective follows: an all-gather of the [ceil(nq/Q), k] uint64 keys over NCCL/NVLink (8 MB in total at nq=10k, k=100),
and the R partial results of every query are merged by the merge kernel.  The key order is total, so the result is
bit-identical for every grid.

  Q = 1 (rows only): the database is split G ways -- what a database larger than one GPU needs (config 5) and what
      single queries want (each GPU streams 1/G of the codes).
  R = 1 (queries only): the database is replicated, no merge at all.  For large batches this is what scales: the
      per-shard fixed work of a row split (every shard must find its own top-k: seed, lists, merge) does not shrink with
      the shard, while a query block is simply a smaller batch.  Measured on one B200 (10M x 256, top-100): a 1.25M-row
      shard takes 3.37 ms per 10k queries (predicts 4.4x at 8 GPUs), a 1 250-query block over all 10M rows 2.37 ms
      (predicts 7.0x); DESIGN.md section 6.

One process per GPU (`torch.distributed`, backend nccl).  The scan and merge callables are injectable so the
partition / gather logic is testable with gloo on CPU against the oracle; the defaults are the CUDA kernels and there is
no host fallback.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import InvalidInputError
from .index import Index, QuantParams, build_index


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous range of `rank` when n items are cut into `world` parts: per = ceil(n / world);
    [rank*per, min(n, (rank+1)*per))."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidInputError(f"bad rank {rank} of {world}")
    per = -(-int(n) // world) if n else 0
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def grid_of(world: int, rank: int, query_shards: int) -> tuple[int, int, int]:
    """(row shards R, row shard of this rank, query block of this rank) for a world of R x query_shards ranks."""
    if query_shards < 1 or world % query_shards:
        raise InvalidInputError(f"query_shards={query_shards} does not divide the world size {world}")
    if not 0 <= rank < world:
        raise InvalidInputError(f"bad rank {rank} of {world}")
    return world // query_shards, rank // query_shards, rank % query_shards


def choose_query_shards(world: int, n: int, dim: int, doc_bits: int, nq_hint: int, hbm_bytes: int = 180 << 30) -> int:
    """Grid for a typical batch of nq_hint queries: replicate the database (queries only) when the batch gives every GPU at
    least two 128-query tiles and a replica with its derived layouts (4x the packed codes) takes less than half of HBM;
    otherwise split rows as far as needed for it to fit, queries for the rest."""
    packed = -(-n // 32) * 32 * doc_bits * (-(-dim // 128)) * 16
    q = world
    while q > 1 and (4 * packed * q // world > hbm_bytes // 2 or nq_hint < 256 * q):
        q //= 2
        while q > 1 and world % q:
            q -= 1
    return max(q, 1)


def _cuda_scan(index: Index, queries, k: int, row_offset: int):
    from .search import search_device
    # device-resident queries stay asynchronous (search_keys is the pipeline entry point): a non-finite query comes back as
    # empty keys and search.pending_nonfinite() reports it; ShardedIndex.search() -- host results -- raises
    return search_device(index, queries, k, row_offset=row_offset, check=False)


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
    """This rank's part of an R x Q sharded search (see the module docstring)."""

    local: object            # Index (CUDA) -- or any object the injected scan_fn understands
    row_offset: int          # global id of local row 0
    n_total: int
    world: int = 1
    rank: int = 0
    group: object = None
    scan_fn: object = None   # (local, queries, k_local, row_offset) -> int64 tensor [nq, k_local] of keys
    merge_fn: object = None  # (stacked [parts, nq, k], k) -> [nq, k]
    query_shards: int = 1    # Q; the ranks r*Q .. r*Q + Q-1 hold the same rows
    always_gather: bool = False  # run the collective and the merge even when world == 1 (tests: the NCCL path on one GPU)

    @classmethod
    def build(cls, local_vectors, params: QuantParams, n_total: int, row_offset: int, world: int = 1,
              rank: int = 0, group=None, query_shards: int = 1, **kw) -> "ShardedIndex":
        """Quantize this rank's rows (already the slice `shard_bounds(n_total, R, rank // Q)` of the corpus) on its GPU."""
        grid_of(world, rank, query_shards)
        idx = build_index(local_vectors, params, keep_originals=False, **kw)
        return cls(local=idx, row_offset=int(row_offset), n_total=int(n_total), world=world, rank=rank,
                   group=group, query_shards=int(query_shards))

    def _local_keys(self, queries, kk: int):
        """Keys of this rank's rows for `queries`, [nq, kk] (short or empty shard: all-ones = empty slot)."""
        import torch
        scan = self.scan_fn or _cuda_scan
        k_local = min(kk, self.local.n)
        nq = queries.shape[0]
        if k_local == kk:
            return scan(self.local, queries, k_local, self.row_offset)
        pad = torch.full((nq, kk), -1, dtype=torch.int64, device="cpu" if self.scan_fn else "cuda")
        if k_local > 0 and nq > 0:
            local = scan(self.local, queries, k_local, self.row_offset)
            pad = pad.to(local.device)
            pad[:, :k_local] = local
        return pad

    def search_keys(self, queries, k: int):
        """Local scan -> all-gather -> merge.  Every rank returns the same [nq, min(k, n_total)] key tensor (int64 holding
        the uint64 keys; empty slots are all-ones)."""
        import torch
        import torch.distributed as dist
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        merge = self.merge_fn or _cuda_merge
        kk = min(int(k), self.n_total)
        nq = int(queries.shape[0])
        if self.world == 1 and not self.always_gather:
            return self._local_keys(queries, kk)
        R, _, c = grid_of(self.world, self.rank, self.query_shards)
        Q = self.query_shards
        per = -(-nq // Q) if nq else 0               # queries per block (the last blocks may be short or empty)
        q_lo, q_hi = min(nq, c * per), min(nq, (c + 1) * per)
        mine = self._local_keys(queries[q_lo:q_hi], kk)
        if mine.shape[0] < per:                      # pad the block: equal shapes for the collective
            pad = torch.full((per, kk), -1, dtype=torch.int64, device=mine.device)
            pad[: mine.shape[0]] = mine
            mine = pad
        gathered = torch.empty((self.world * per, kk), dtype=torch.int64, device=mine.device)  # rank-major concatenation
        if per and kk:
            dist.all_gather_into_tensor(gathered, mine.contiguous(), group=self.group)
        # rank g = r * Q + c: [R, Q * per, kk] is, for every row shard, the whole (padded) batch in query order
        parts = gathered.view(R, Q * per, kk)
        out = parts[0] if R == 1 else merge(parts, kk)
        return out[:nq]

    def search(self, queries, k: int):
        """(scores, indices) as int64 numpy arrays [nq, min(k, n_total)], identical on all ranks."""
        keys = self.search_keys(queries, k)
        if not keys.is_cuda:  # CPU hooks (tests/test_sharded_gloo.py): unpack on the host
            kn = keys.contiguous().numpy().view(np.uint64)
            return (kn >> np.uint64(32)).astype(np.int64), (kn & np.uint64(0xFFFFFFFF)).astype(np.int64)
        from .search import raise_pending_nonfinite, to_host_arrays, unpack_keys_device
        d, i = unpack_keys_device(keys.contiguous())  # empty slots come back as -1
        d, i = to_host_arrays(d, i)
        raise_pending_nonfinite(keys.device)
        return d, i
