"""CUDA-graph capture of a whole FFN training (or prefill) step.

The recipe step is ~20 kernel launches on two streams (main + the side stream
that carries K4, the plan and the permuted copies). Captured once, the step is
replayed as a single graph launch: no per-kernel host work, no launch gaps, the
side-stream fork/join kept as graph edges. Every libs24 launch is a plain
stream operation (tensor maps are kernel parameters, the tile-scheduler
counters reset themselves), so the captured graph is replay-safe.

Usage:
    step = FfnStepGraph(params, cfg, n)          # static [n, d] input buffers
    step.x.copy_(x_batch); step.dy.copy_(dy_batch)
    step.replay()                                # out / d_w1 / d_w2 / d_x updated
"""

from __future__ import annotations

import torch

from ._tensors import BF16, require_cuda
from .ffn import FfnConfig, FfnParams, ffn_backward, ffn_forward


class FfnStepGraph:
    """Forward + backward of one token batch, captured as a CUDA graph.

    Inputs live in the static buffers `x` and `dy` (bf16 [n, d]); after
    `replay()` the results are in `out`, `d_w1`, `d_w2`, `d_x` (the same
    tensors every replay). backward=False captures the forward only (prefill).
    """

    def __init__(self, params: FfnParams, cfg: FfnConfig, n: int, backward: bool = True, warmup: int = 2,
                 grad_bucket: bool = False):
        require_cuda()
        d = params.model_dim
        dev = params.w1.device
        self.params, self.cfg, self.backward = params, cfg, backward
        # grad_bucket=True: d_w1 and d_w2 live in one flat fp32 buffer
        # (self.bucket), so the data-parallel step all-reduces them in one call
        self.bucket = (torch.empty(2 * d * params.hidden_dim, dtype=torch.float32, device=dev)
                       if grad_bucket and backward else None)
        self.x = torch.zeros(n, d, dtype=BF16, device=dev)
        self.dy = torch.zeros(n, d, dtype=BF16, device=dev)
        self.pool = torch.cuda.graph_pool_handle()
        # warm up on a side stream first: one-time work (kernel attributes,
        # occupancy queries, scheduler counters, permutation upload) must not
        # happen inside the capture
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(max(1, warmup)):
                self._step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, pool=self.pool):
            self.out, self.cache, self.grads = self._step()
        torch.cuda.synchronize()

    def _step(self):
        out, cache = ffn_forward(self.x, self.params, self.cfg, for_backward=self.backward)
        grads = ffn_backward(self.dy, cache, self.params, self.cfg, grad_bucket=self.bucket) if self.backward else None
        return out, cache, grads

    @property
    def d_w1(self):
        return self.grads.d_w1

    @property
    def d_w2(self):
        return self.grads.d_w2

    @property
    def d_x(self):
        return self.grads.d_x

    def replay(self) -> None:
        self.graph.replay()
