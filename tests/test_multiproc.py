"""World-size-2 gloo test of the multi-GPU host logic (sharding + max-over-ranks)."""
import os
import socket

import numpy as np

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2511_01927_b200.dist import max_over_ranks, shard, solve_multi_batch_sharded, sum_over_ranks  # noqa: E402


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


def _oracle_batch(pencils, contours, cfg, solver, seeds):
    """solve_multi_batch stand-in for CPU ranks: the oracle's solve_multi per GEP."""
    from oracle import cirr as O

    out = []
    for (a, b), cs, sd in zip(pencils, contours, seeds):
        m = O.solve_multi(O.Pencil(a, b, True), cs, cfg, seed=sd, solver=solver)
        out.append([None if r is None else np.sort(np.real(r.eigenvalues)) for r in m.results])
    return out


def _small_geps(count):
    rng = np.random.default_rng(11)
    geps = []
    for _ in range(count):
        n = 40
        a = np.diag(np.linspace(0.05, 2.0, n)) + 1e-3 * rng.standard_normal((n, n))
        a = (a + a.T) / 2
        geps.append((a, np.eye(n)))
    return geps


def _contours(count):
    from paper_2511_01927_b200 import Contour

    return [[Contour("circle", center=0.3 + 0.2 * g, radius=0.15)] for g in range(count)]


def _shard_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import cirr as O

    geps = _small_geps(5)
    cons = _contours(len(geps))
    cfg = O.OracleConfig(n_q=16, source_cols=8, n_moments=2)
    allres = solve_multi_batch_sharded(geps, cons, cfg, seeds=list(range(len(geps))), solve_fn=_oracle_batch)
    idx, mine = solve_multi_batch_sharded(geps, cons, cfg, seeds=list(range(len(geps))), solve_fn=_oracle_batch,
                                          gather=False)
    out[rank] = (allres, idx, mine)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_batch_world2():
    """solve_multi_batch_sharded over two gloo ranks (the oracle stands in for
    the device solve): each rank solves its contiguous block, every rank gets
    all results in input order, equal to one unsharded call."""
    from oracle import cirr as O

    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(2, port, out), nprocs=2, join=True)
    geps = _small_geps(5)
    cons = _contours(len(geps))
    cfg = O.OracleConfig(n_q=16, source_cols=8, n_moments=2)
    want = _oracle_batch(geps, cons, cfg, "cirr", list(range(len(geps))))
    for r in (0, 1):
        allres, idx, mine = out[r]
        assert idx == shard(5, r, 2)
        assert len(allres) == 5
        for g in range(5):
            for x, y in zip(allres[g], want[g]):
                assert (x is None) == (y is None)
                if x is not None:
                    np.testing.assert_array_equal(x, y)
        for i, res in zip(idx, mine):
            for x, y in zip(res, want[i]):
                if x is not None:
                    np.testing.assert_array_equal(x, y)


def _node_worker(rank, world, port, out):
    """Node split of one GEP: each rank's partial centred moments over its interleaved
    node share, summed by the dist module's all-reduce, equal the full moment blocks (oracle arithmetic)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import cirr as O
    from paper_2511_01927_b200.contours import Contour
    from paper_2511_01927_b200.dist import _allreduce

    rng = np.random.default_rng(0)
    n = 40
    a = np.diag(np.arange(1.0, n + 1)) + 0.01 * rng.standard_normal((n, n))
    a = (a + a.T) / 2
    p = O.Pencil(a, np.eye(n), True)
    c = Contour(shape="circle", center=5.0 + 0j, radius=2.6, expected_count=5)
    cfg = O.OracleConfig(n_q=16, source_cols=6, n_moments=4)
    nodes, weights = O.quadrature(c, cfg.n_q)
    frame = (5.0 + 0j, 2.6)   # centred, scaled moments (DESIGN.md section 3 item 1)
    v = rng.standard_normal((n, 6))
    ids = np.arange(rank, len(nodes), world)
    part = O.Projector(p, nodes[ids], weights[ids], cfg, frame).apply(v, 4)
    t = torch.from_numpy(np.stack(part))
    _allreduce()(t, "sum")
    full = np.stack(O.Projector(p, nodes, weights, cfg, frame).apply(v, 4))
    err = float(np.abs(t.numpy() - full).max() / np.abs(full).max())
    first = torch.tensor([7 if rank == 1 else np.iinfo(np.int64).max], dtype=torch.int64)
    _allreduce()(first, "min")
    out[rank] = (err, int(first[0]), len(ids))
    dist.barrier()
    dist.destroy_process_group()


def test_node_split_moments_world2():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_node_worker, args=(2, port, out), nprocs=2, join=True)
    for r in (0, 1):
        err, first, cnt = out[r]
        assert err < 1e-13 and first == 7 and cnt == 8
