"""World-size-2 gloo test of the multi-GPU host logic (sharding + max-over-ranks)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2511_01927_b200.dist import max_over_ranks, shard, sum_over_ranks  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard(256, rank, world)
    assert max_over_ranks(float(rank + 1)) == float(world)
    total = sum_over_ranks(float(len(mine)))
    out[rank] = (mine[0], mine[-1], total)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_partition():
    for world in (1, 2, 3, 8):
        parts = [shard(256, r, world) for r in range(world)]
        assert sorted(sum(parts, [])) == list(range(256))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_gloo_world2():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == (0, 127, 256.0) and out[1] == (128, 255, 256.0)
