"""world_size-2 (and 3) gloo runs of the shard -> local top-k -> all-gather -> merge logic on
CPU.  The CUDA scan/merge kernels are replaced by the oracle (test infrastructure) through the
injectable hooks of ShardedIndex; what is under test is the partition arithmetic, global row
ids, padding of short shards, the collective and that every rank ends with the reference answer."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


class _HostShard:
    def __init__(self, planes, dim, wq, scale):
        self.planes, self.dim, self.wq, self.scale = planes, dim, wq, scale
        self.n = planes.shape[2]


def _oracle_scan(local, queries, k, row_offset):
    from oracle import xfbq_oracle as xo
    qp = xo.c_quantize_matrix(np.asarray(queries, dtype=np.float64), local.wq, local.scale).transpose(2, 0, 1)
    d, i = xo.c_search(local.planes, qp, k, row_offset=row_offset, threads=1)
    keys = (d << np.uint64(32)) | i.astype(np.uint64)
    return torch.from_numpy(keys.view(np.int64))


def _oracle_merge(stacked, k):
    a = stacked.numpy().view(np.uint64)
    parts, nq, kk = a.shape
    return torch.from_numpy(np.sort(a.transpose(1, 0, 2).reshape(nq, parts * kk), axis=1)[:, :kk].view(np.int64).copy())


def _worker(rank, world, port, case, k, out_dir, query_shards=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import xfbq_oracle as xo
        from paper_2008_02002_b200.sharded import ShardedIndex, grid_of, shard_bounds
        from tests._golden import synth_case, small_cases
        if case == "tiny":
            c = next(x for x in small_cases() if x["n"] >= 3 and x["dim"] == 65 and x["wd"] == 4)
            docs, queries, n = c["docs"], c["queries"], c["n"]
            want_d = None
        else:
            c = synth_case(case)
            docs, queries, n = c["docs"], c["queries"][:6], c["n"]
            want_d, want_i = c["z"]["dists"][:6], c["z"]["ids"][:6]
        R, r, _ = grid_of(world, rank, query_shards)   # R row shards x query_shards query blocks
        lo, hi = shard_bounds(n, R, r)
        planes = xo.c_quantize_matrix(docs[lo:hi], c["wd"], c["scale"]) if hi > lo else np.zeros((c["wd"], (c["dim"] + 63) // 64, 0), np.uint64)
        shard = ShardedIndex(local=_HostShard(planes, c["dim"], c["wq"], c["scale"]), row_offset=lo, n_total=n,
                             world=world, rank=rank, scan_fn=_oracle_scan, merge_fn=_oracle_merge, query_shards=query_shards)
        scores, ids = shard.search(queries, k)
        if want_d is None:
            full = xo.c_quantize_matrix(docs, c["wd"], c["scale"])
            qp = xo.c_quantize_matrix(np.asarray(queries, np.float64), c["wq"], c["scale"]).transpose(2, 0, 1)
            want_d, want_i = xo.c_search(full, qp, k)
        ok = np.array_equal(scores.astype(np.uint64), want_d[:, :scores.shape[1]]) and np.array_equal(ids, want_i[:, :ids.shape[1]])
        ok = ok and scores.shape[1] == min(k, n)
        Path(out_dir, f"rank{rank}.txt").write_text("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,query_shards,case,k", [
    (2, 1, "cfg1_100k_128_w4", 10), (3, 1, "cfg2_60k_128_w3", 100), (2, 1, "tiny", 50),   # rows only
    (2, 2, "cfg1_100k_128_w4", 10),                                                         # queries only (replicated database, no merge)
    (4, 2, "cfg2_60k_128_w3", 100), (4, 2, "tiny", 50),                                     # 2 row shards x 2 query blocks (6 and 3 queries: ragged blocks)
])
def test_sharded_search_gloo(world, query_shards, case, k, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), case, k, str(tmp_path), query_shards), nprocs=world, join=True)
    for r in range(world):
        assert Path(tmp_path, f"rank{r}.txt").read_text() == "ok"


def test_grid_and_layout_choice():
    from paper_2008_02002_b200.errors import InvalidInputError
    from paper_2008_02002_b200.sharded import choose_query_shards, grid_of
    assert grid_of(8, 5, 4) == (2, 1, 1) and grid_of(8, 7, 1) == (8, 7, 0) and grid_of(8, 3, 8) == (1, 0, 3)
    with pytest.raises(InvalidInputError):
        grid_of(8, 0, 3)
    assert choose_query_shards(8, 10_000_000, 256, 4, 10_000) == 8        # config 4: replicate, 1 250 queries per GPU
    assert choose_query_shards(8, 10_000_000, 256, 4, 1) == 1             # single queries: split the rows
    assert choose_query_shards(8, 100_000_000, 512, 4, 10_000) == 4       # config 5: a replica does not fit in half of HBM
    assert choose_query_shards(1, 10_000_000, 256, 4, 10_000) == 1


def test_shard_bounds_cover_rows_exactly():
    from paper_2008_02002_b200.sharded import shard_bounds
    for n in (0, 1, 7, 8, 9, 100, 10_000_000):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(hi >= lo for lo, hi in spans)
