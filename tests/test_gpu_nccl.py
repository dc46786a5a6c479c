"""The NCCL path of the sharded search on real CUDA kernels: scan -> all_gather_into_tensor -> merge.
World 1 always runs (the collective and the gathered-layout arithmetic execute on NCCL with one rank); worlds of 2 and 4
run under torchrun when the box has that many GPUs (skipped otherwise -- the multi-rank host logic is covered on CPU by
tests/test_sharded_gloo.py)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _torchrun(world: int, query_shards: int):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(ROOT / "tests" / "_nccl_worker.py"), str(query_shards)]
    env = dict(os.environ)
    env.pop("XFBQ_ENGINE", None)
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-4000:]
    assert proc.stdout.count(": ok") == world


def test_nccl_world1_through_collective():
    _torchrun(1, 1)


@pytest.mark.parametrize("world,query_shards", [(2, 1), (2, 2), (4, 2)])
def test_nccl_multi_gpu(world, query_shards):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, this box has {torch.cuda.device_count()}")
    _torchrun(world, query_shards)
