"""The data-parallel communication path (one all-reduce per weight-gradient
tensor, launched from the backward's grad_ready hook) on 2 CPU ranks with
gloo, plus prefill's no-communication sharding contract."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_16672_b200.dp import GradAllReducer, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, h = 8, 16
        gen = torch.Generator().manual_seed(rank)
        dw2 = torch.randn(h, d, generator=gen)
        dw1 = torch.randn(d, h, generator=gen)
        mine = (dw2.clone(), dw1.clone())
        red = GradAllReducer()
        red("d_w2", dw2)  # launched as soon as final, like ffn_backward does
        red("d_w1", dw1)
        out = red.wait()
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        exp2 = sum(g[0] for g in gathered)
        exp1 = sum(g[1] for g in gathered)
        ok = torch.allclose(out["d_w2"], exp2) and torch.allclose(out["d_w1"], exp1)
        n = 64
        a, b = shard_bounds(n, world, rank)
        q.put((rank, ok, a, b))
    finally:
        dist.destroy_process_group()


def test_grad_allreduce_two_ranks_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    assert all(ok for _, ok, _, _ in res)
    assert [(a, b) for _, _, a, b in res] == [(0, 32), (32, 64)]
