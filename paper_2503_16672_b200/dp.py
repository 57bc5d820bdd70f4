"""Token-sharded data parallelism for the FFN (one process per GPU).

The FFN is per-token, so both inference prefill and training shard tokens:
  * prefill: each rank runs ffn_forward on its own token shard, no
    communication (outputs concatenate to the single-GPU result);
  * training: each rank runs the full recipe on its shard (its own permutation
    of n/G tokens and its own split plan, i.e. the reference applied per shard)
    and the weight gradients are summed with ONE all-reduce bucket per tensor
    over NCCL / NVLink. With the hook the backward runs dW2, dW1, then dX:
    each all-reduce is launched (async, NCCL's own stream) as soon as its
    gradient is final, dW2's overlapping dW1 and dX, dW1's overlapping dX.

Nothing here is in the reference (distributed training is a reference
non-goal, ref SPEC.md:486); it is the multi-GPU plumbing the north star asks
for. The communication half (GradAllReducer) is device-agnostic so it is
exercised with the gloo backend on CPU in tests/test_dp_gloo.py.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n_tokens: int, world: int, rank: int, multiple: int = 4) -> tuple[int, int]:
    """Contiguous token shard of rank `rank`: every shard but the last is a
    multiple of `multiple` tokens (2:4 groups never straddle ranks)."""
    if n_tokens % multiple:
        raise ValueError(f"token count {n_tokens} must be a multiple of {multiple}")
    units = n_tokens // multiple
    per = units // world
    extra = units % world
    start = rank * per + min(rank, extra)
    stop = start + per + (1 if rank < extra else 0)
    return start * multiple, stop * multiple


class GradAllReducer:
    """Sums gradients across ranks as they become final.

    Use as the `grad_ready` hook of ffn_backward: each call launches an async
    all-reduce (SUM) of that tensor; wait() completes them all. With NCCL the
    collective is ordered after the producing kernels on the current stream
    and overlaps whatever the caller launches next."""

    def __init__(self, group=None, average: bool = False):
        self.group = group
        self.average = average
        self.pending: list[tuple[str, torch.Tensor, object]] = []

    def __call__(self, name: str, tensor: torch.Tensor) -> None:
        work = dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        self.pending.append((name, tensor, work))

    def wait(self) -> dict[str, torch.Tensor]:
        out = {}
        world = dist.get_world_size(self.group)
        for name, tensor, work in self.pending:
            work.wait()
            if self.average and world > 1:
                tensor.div_(world)
            out[name] = tensor
        self.pending.clear()
        return out


def train_step(x_shard, g_shard, params, cfg, group=None, global_plan: bool = True, average: bool = False):
    """Forward + backward on this rank's token shard, weight gradients summed
    over the group. Returns (out_shard, FfnGrads with global d_w1 / d_w2).

    global_plan=True all-reduces K1's per-feature nonzero counts (h int32,
    one small collective between K1 and the plan) so every rank splits the
    same features dense / sparse: the plan of the global batch, as a
    single-GPU run over all tokens would choose it. The feature-wise 2:4
    groups themselves stay per shard (groups of 4 consecutive tokens of the
    rank's own permutation), i.e. the reference applied per shard.

    The backward hands d_w2 to the all-reducer as soon as it is final (right
    after K3) and computes dW1 before dX, so both all-reduces overlap compute
    (dW2's overlaps dW1 and dX, dW1's overlaps dX)."""
    from .ffn import ffn_backward, ffn_forward

    hook = None
    if global_plan and cfg.backward_mode == "split_masked":
        def hook(counts):
            dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)

    out, cache = ffn_forward(x_shard, params, cfg, counts_hook=hook)
    reducer = GradAllReducer(group, average=average)
    grads = ffn_backward(g_shard, cache, params, cfg, grad_ready=reducer)
    reducer.wait()
    return out, grads


def prefill(x_shard, params, cfg):
    """Inference prefill on this rank's tokens: no communication."""
    from .ffn import ffn_forward

    out, _ = ffn_forward(x_shard, params, cfg, for_backward=False)
    return out
