"""Multi-rank host logic on CPU with torch.distributed gloo at world_size 2:
replica streams (bench.py: disjoint core slices per rank, whole-job
aggregation = sum of tokens, max of device time over ranks) and the
tensor-parallel handle exchange (tp_connect_group: every rank opens every
rank's handle, in rank order)."""
import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", init_method="env://")
    import bench
    core, dcores = bench.core_slice(rank, world)
    tok = torch.tensor([100.0 * (rank + 1), 10.0], dtype=torch.float64)
    ms = torch.tensor([50.0 + rank, 1.0], dtype=torch.float64)
    dist.all_reduce(tok, op=dist.ReduceOp.SUM)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    q.put((rank, core, dcores, tok.tolist(), ms.tolist()))
    dist.destroy_process_group()


def test_two_rank_aggregation():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    (r0, c0, d0, t0, m0), (r1, c1, d1, t1, m1) = out
    assert t0 == t1 == [300.0, 20.0]
    assert m0 == m1 == [51.0, 1.0]
    s0, s1 = {c0, *d0}, {c1, *d1}
    if len(os.sched_getaffinity(0)) >= 4:
        assert not (s0 & s1), "draft core slices of the two streams overlap"


def test_prompt_generator_known_answer():
    import bench
    p = bench.make_prompt(1, 4)
    assert p == [0x910A2DEC89025CC1 % 32000, 0xBEEB8DA1658EEC67 % 32000,
                 0xF893A2EEFB32555E % 32000, 0x71C18690EE42C90B % 32000]


class _FakeRank:
    """Stands in for a Target rank: the exchange logic needs no GPU."""

    def __init__(self, rank, world):
        self.tp_rank, self.tp_size = rank, world
        self.connected = None

    def tp_handle(self):
        return bytes([self.tp_rank]) * 64

    def tp_connect(self, handles):
        self.connected = list(handles)


def _tp_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", init_method="env://")
    from paper_2503_00784_b200 import ConfigError, tp_connect_group
    t = _FakeRank(rank, world)
    tp_connect_group(t)
    bad = _FakeRank((rank + 1) % world, world)  # rank mismatch must be refused
    try:
        tp_connect_group(bad)
        refused = False
    except ConfigError:
        refused = True
    q.put((rank, t.connected, refused))
    dist.destroy_process_group()


def test_tp_handle_exchange_rank_order():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_tp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, handles, refused in out:
        assert handles == [bytes([0]) * 64, bytes([1]) * 64], rank
        assert refused
