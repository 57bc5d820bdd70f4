"""torch.nn / autograd integration of the FFN (SURVEY 8b "who calls the
C-ABI": the training-harness entry point).

    ffn = SquaredReluFFN24(d_model, d_hidden)          # recipe config by default
    y = ffn(x)                                          # x [..., d], bf16 or fp32
    y.float().pow(2).mean().backward()                  # dX, dW1, dW2 through ffn_backward

The forward is ffn_forward (K1 -> plan -> K2, K4 next to it), the backward is
ffn_backward (K3, dX, the grouped split weight-gradient GEMM). Weights may be
fp32 master copies (their bf16 images are made per call) or bf16; weight
gradients come back in the parameters' dtype. Token counts that are not a
multiple of 4 are padded with zero rows (they contribute nothing).
"""

from __future__ import annotations

import math

import torch

from ._tensors import BF16
from .ffn import RECIPE, FfnConfig, FfnParams, ffn_backward, ffn_forward


class _FfnFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w1, w2, cfg):
        params = FfnParams(w1=w1.detach(), w2=w2.detach())
        out, cache = ffn_forward(x.detach(), params, cfg)
        ctx.cache, ctx.params, ctx.cfg = cache, params, cfg
        ctx.wdtypes = (w1.dtype, w2.dtype)
        return out

    @staticmethod
    def backward(ctx, g):
        grads = ffn_backward(g.contiguous().to(BF16), ctx.cache, ctx.params, ctx.cfg)
        ctx.cache = None
        return grads.d_x, grads.d_w1.to(ctx.wdtypes[0]), grads.d_w2.to(ctx.wdtypes[1]), None


def squared_relu_ffn(x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor, cfg: FfnConfig = RECIPE) -> torch.Tensor:
    """relu(x W1)^2 W2 with the 2:4 recipe, differentiable (x [n, d] bf16)."""
    return _FfnFunction.apply(x, w1, w2, cfg)


class SquaredReluFFN24(torch.nn.Module):
    """Squared-ReLU FFN layer on the B200 2:4 activation-sparse path."""

    def __init__(self, d_model: int, d_hidden: int, cfg: FfnConfig = RECIPE, device=None,
                 dtype: torch.dtype = torch.float32):
        super().__init__()
        self.cfg = cfg
        dev = device or "cuda"
        # the reference's init: W1 ~ N(0, 1/d), W2 ~ N(0, 1/h) (ref ffn.py:104-126)
        self.w1 = torch.nn.Parameter(torch.randn(d_model, d_hidden, device=dev, dtype=dtype) / math.sqrt(d_model))
        self.w2 = torch.nn.Parameter(torch.randn(d_hidden, d_model, device=dev, dtype=dtype) / math.sqrt(d_hidden))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        shape = x.shape
        xf = x.reshape(-1, shape[-1]).to(BF16)
        n = xf.shape[0]
        pad = (-n) % 4
        if pad:
            xf = torch.cat([xf, xf.new_zeros(pad, xf.shape[1])])
        y = squared_relu_ffn(xf.contiguous(), self.w1, self.w2, self.cfg)
        if pad:
            y = y[:n]
        return y.reshape(shape).to(x.dtype)
