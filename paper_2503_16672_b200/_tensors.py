"""Device-tensor plumbing shared by the API modules (torch is plumbing only:
allocation, streams, host<->device copies; all math runs in libs24.so)."""

from __future__ import annotations

import numpy as np
import torch

from . import errors

BF16 = torch.bfloat16
F32 = torch.float32


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise errors.BackendError("the B200 backend needs a CUDA device; there is no CPU fallback")


def ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def as_matrix(a, name: str = "a", dtype: torch.dtype | None = None) -> torch.Tensor:
    """2-D contiguous CUDA tensor (fp32 or bf16). numpy inputs are uploaded.
    float64 is rejected: the device path works in bf16 operands / fp32
    accumulation (the reference's "oracle" precision stays on the CPU)."""
    require_cuda()
    if isinstance(a, np.ndarray):
        if a.dtype == np.float64:
            raise errors.PrecisionError(f"{name}: float64 (oracle precision) is not a device precision")
        if a.dtype not in (np.float32,):
            raise errors.PrecisionError(f"{name} has unsupported dtype {a.dtype}")
        a = torch.from_numpy(np.ascontiguousarray(a))
    if not isinstance(a, torch.Tensor) or a.dim() != 2:
        raise errors.DimensionError(f"{name} must be a 2-D array")
    if a.dtype not in (F32, BF16):
        raise errors.PrecisionError(f"{name} has unsupported dtype {a.dtype}")
    if not a.is_cuda:
        a = a.cuda(non_blocking=True)
    if dtype is not None and a.dtype != dtype:
        a = a.to(dtype)
    return a.contiguous()


def dtype_code(t: torch.Tensor) -> int:
    return 0 if t.dtype == F32 else 1


def pad128(n: int) -> int:
    return (n + 127) // 128 * 128
