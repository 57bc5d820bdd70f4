"""Data-parallel training and prefill with two real ranks:
two processes on cuda:0 with the gloo backend (it accepts CUDA tensors; this
pool has one GPU per job, so NCCL over NVLink cannot run here). This checks
the multi-process code path of dp.train_step / dp.prefill -- the counts
all-reduce that gives every rank the global plan, the per-tensor gradient
all-reduces launched from the backward's hook -- not performance.

* training: the all-reduced [dW1, dW2] equal, bit for bit, the sum of the two
  shards' gradients computed in one process with the same global plan (the
  kernels are deterministic; a sum of two fp32 terms does not depend on
  order), and the global plan equals partition_features of the summed counts;
* prefill: the ranks' outputs concatenate to the single-process output bit
  for bit (no communication in the step).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    from oracle import srelu24_np as O

    n, d, h = 2048, 256, 1024
    return (n, d, h) + O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=61)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2503_16672_b200 as s24
    from paper_2503_16672_b200 import dp

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, d, h, x, w1, w2, dy = _inputs()
        p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
        a, b = dp.shard_bounds(n, world, rank)
        tx = torch.from_numpy(x[a:b]).cuda().bfloat16()
        tg = torch.from_numpy(dy[a:b]).cuda().bfloat16()
        out, grads = dp.train_step(tx, tg, p, s24.RECIPE)
        pre = dp.prefill(tx, p, s24.RECIPE)
        torch.cuda.synchronize()
        # (numpy: pickled by value, no shared-memory handle outliving this process)
        q.put((rank,) + tuple(t.float().cpu().numpy() for t in (out, grads.d_w1, grads.d_w2, grads.d_x, pre)))
    finally:
        dist.destroy_process_group()


def test_train_step_and_prefill_two_ranks():
    import paper_2503_16672_b200 as s24
    from paper_2503_16672_b200 import dp

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda t: t[0])
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0

    # single process: both shards with the global plan
    n, d, h, x, w1, w2, dy = _inputs()
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    shards = [dp.shard_bounds(n, world, r) for r in range(world)]
    counts = sum(s24.ffn_forward(torch.from_numpy(x[a:b]).cuda(), p, s24.RECIPE)[1].counts.long()
                 for a, b in shards)
    plan = s24.partition_features(counts, s24.RECIPE.split_ratio)
    dw1 = torch.zeros(d, h, device="cuda")
    dw2 = torch.zeros(h, d, device="cuda")
    for r, (a, b) in enumerate(shards):
        out, cache = s24.ffn_forward(torch.from_numpy(x[a:b]).cuda(), p, s24.RECIPE, plan=plan)
        g = s24.ffn_backward(torch.from_numpy(dy[a:b]).cuda(), cache, p, s24.RECIPE)
        assert np.array_equal(res[r][1], out.float().cpu().numpy())
        assert np.array_equal(res[r][4], g.d_x.float().cpu().numpy())
        dw1 += g.d_w1
        dw2 += g.d_w2
    for r in range(world):
        assert np.array_equal(res[r][2], dw1.cpu().numpy()) and np.array_equal(res[r][3], dw2.cpu().numpy())
    full, _ = s24.ffn_forward(torch.from_numpy(x).cuda(), p, s24.RECIPE, for_backward=False)
    assert np.array_equal(np.concatenate([res[r][5] for r in range(world)]), full.float().cpu().numpy())
