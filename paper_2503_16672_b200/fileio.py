"""On-disk formats of the reference: the S24C compressed
2:4 file and the S24M dense matrix file, byte-compatible with
ref sparse24.py:224-291 (write_sparse / read_sparse) and
ref matcore.py:310-361 (write_matrix / read_matrix).

S24C: magic "S24C", version u32, orientation u8 (0 token, 1 feature), rows
u32, cols u32; then 2*groups float32 kept values in storage order ([rows,
cols/4, 2] token-wise, [rows/4, cols, 2] feature-wise) and ceil(groups/2)
metadata bytes, each group's positions packed as i0 | i1 << 2, two groups per
byte, lower group in the low nibble.
S24M: magic "S24M", version u32, rows u32, cols u32, rows*cols float32
row-major.

The byte layout work (header, nibble packing, validation with the
reference's error messages and byte offsets) is host code on numpy arrays;
write_sparse / read_sparse move a device Sparse24Matrix through it (the device
metadata is converted with the s24_meta_hw_to_ref / ref_to_hw kernels).
Values are stored as float32: a bf16 device matrix writes exactly, a file
written from float32 values reads back rounded to bf16 (the device
precision).
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from . import _lib
from ._tensors import BF16, pad128, ptr, require_cuda, stream
from .errors import DimensionError, FormatError, NonFiniteError, PrecisionError
from .sparse24 import FEATURE_WISE, TOKEN_WISE, Sparse24Matrix

SPARSE_MAGIC = b"S24C"
SPARSE_VERSION = 1
MATRIX_MAGIC = b"S24M"
MATRIX_VERSION = 1
_SPARSE_HEADER = struct.Struct("<4sIBII")  # 17 bytes
_MATRIX_HEADER = struct.Struct("<4sIII")  # 16 bytes


# --------------------------------------------------------------------- S24C bytes
def encode_sparse(orientation: str, rows: int, cols: int, values: np.ndarray, meta: np.ndarray) -> bytes:
    """S24C bytes of a 2:4 matrix given in the reference layout (host arrays)."""
    if values.dtype != np.float32:
        raise PrecisionError("sparse files store working precision (float32) only")
    orient = 0 if orientation == TOKEN_WISE else 1
    nib = (meta[..., 0] | (meta[..., 1] << 2)).ravel().astype(np.uint8)
    if len(nib) % 2:
        nib = np.append(nib, np.uint8(0))
    packed = (nib[0::2] | (nib[1::2] << 4)).astype(np.uint8)
    return (_SPARSE_HEADER.pack(SPARSE_MAGIC, SPARSE_VERSION, orient, rows, cols)
            + np.ascontiguousarray(values, dtype="<f4").tobytes() + packed.tobytes())


def decode_sparse(blob: bytes):
    """(orientation, rows, cols, values, meta) from S24C bytes, validated as
    the reference validates them (same messages and byte offsets)."""
    if len(blob) < 17:
        raise FormatError("file shorter than the 17-byte header", offset=len(blob))
    if blob[:4] != SPARSE_MAGIC:
        raise FormatError(f"bad magic {blob[:4]!r}, expected {SPARSE_MAGIC!r}", offset=0)
    _, version, orient, rows, cols = _SPARSE_HEADER.unpack(blob[:17])
    if version != SPARSE_VERSION:
        raise FormatError(f"unsupported version {version}", offset=4)
    if orient not in (0, 1):
        raise FormatError(f"unknown orientation byte {orient}", offset=8)
    orientation = TOKEN_WISE if orient == 0 else FEATURE_WISE
    if orientation == TOKEN_WISE and cols % 4 != 0:
        raise FormatError(f"token-wise file with cols = {cols}", offset=13)
    if orientation == FEATURE_WISE and rows % 4 != 0:
        raise FormatError(f"feature-wise file with rows = {rows}", offset=9)
    groups = rows * cols // 4
    values_bytes = 2 * groups * 4
    meta_bytes = (groups + 1) // 2
    if len(blob) != 17 + values_bytes + meta_bytes:
        raise FormatError(f"expected {17 + values_bytes + meta_bytes} bytes, got {len(blob)}", offset=len(blob))
    shape = (rows, cols // 4, 2) if orientation == TOKEN_WISE else (rows // 4, cols, 2)
    values = np.frombuffer(blob[17:17 + values_bytes], dtype="<f4").reshape(shape).astype(np.float32)
    packed = np.frombuffer(blob[17 + values_bytes:], dtype=np.uint8)
    nib = np.empty(2 * len(packed), dtype=np.uint8)
    nib[0::2] = packed & 0x0F
    nib[1::2] = packed >> 4
    nib = nib[:groups]
    meta = np.stack([nib & 0x3, (nib >> 2) & 0x3], axis=-1).reshape(shape).astype(np.uint8)
    if groups and not np.all(meta[..., 0] < meta[..., 1]):
        raise FormatError("metadata positions not strictly increasing", offset=17 + values_bytes)
    return orientation, rows, cols, values, meta


# --------------------------------------------------------------------- S24M bytes
def encode_matrix(a: np.ndarray) -> bytes:
    if a.ndim != 2:
        raise DimensionError("matrix files hold 2-D arrays")
    if a.dtype != np.float32:
        raise PrecisionError("matrix files store working precision (float32) only")
    if not np.all(np.isfinite(a)):
        raise NonFiniteError("matrix contains NaN or Inf")
    return _MATRIX_HEADER.pack(MATRIX_MAGIC, MATRIX_VERSION, *a.shape) + np.ascontiguousarray(a, "<f4").tobytes()


def decode_matrix(blob: bytes) -> np.ndarray:
    if len(blob) < 16:
        raise FormatError("file shorter than the 16-byte header", offset=len(blob))
    if blob[:4] != MATRIX_MAGIC:
        raise FormatError(f"bad magic {blob[:4]!r}, expected {MATRIX_MAGIC!r}", offset=0)
    _, version, rows, cols = _MATRIX_HEADER.unpack(blob[:16])
    if version != MATRIX_VERSION:
        raise FormatError(f"unsupported version {version}", offset=4)
    expected = rows * cols * 4
    if len(blob) - 16 < expected:
        raise FormatError(f"payload truncated: need {expected} bytes for {rows}x{cols}", offset=len(blob))
    if len(blob) - 16 > expected:
        raise FormatError("trailing bytes after payload", offset=16 + expected)
    data = np.frombuffer(blob[16:], dtype="<f4").reshape(rows, cols).astype(np.float32)
    bad = ~np.isfinite(data)
    if bad.any():
        first = int(np.flatnonzero(bad.ravel())[0])
        raise FormatError("non-finite value in payload", offset=16 + 4 * first)
    return data


# --------------------------------------------------------------------- files
def write_matrix(path, a) -> None:
    """ref matcore.py:321-333. Accepts numpy float32 or a torch tensor
    (bf16 tensors are written exactly as float32)."""
    if isinstance(a, torch.Tensor):
        if a.dtype not in (torch.float32, BF16):
            raise PrecisionError(f"unsupported dtype {a.dtype}")
        a = a.detach().float().cpu().numpy()
    with open(path, "wb") as f:
        f.write(encode_matrix(np.asarray(a)))


def read_matrix(path) -> np.ndarray:
    """ref matcore.py:336-361: a float32 numpy matrix."""
    with open(path, "rb") as f:
        return decode_matrix(f.read())


def write_sparse(path, s: Sparse24Matrix) -> None:
    """ref sparse24.py:233-247, from a device Sparse24Matrix."""
    values = s.values.float().cpu().numpy()
    meta = s.meta.cpu().numpy()
    with open(path, "wb") as f:
        f.write(encode_sparse(s.orientation, s.rows, s.cols, values, meta))


def read_sparse(path, device=None) -> Sparse24Matrix:
    """ref sparse24.py:250-291, into a device Sparse24Matrix (bf16 values,
    tcgen05 metadata when the grouped axis is a multiple of 128)."""
    require_cuda()
    with open(path, "rb") as f:
        orientation, rows, cols, values, meta = decode_sparse(f.read())
    dev = torch.device(device or "cuda")
    tv = torch.from_numpy(values).to(dev)
    tm = torch.from_numpy(meta).to(dev)
    if orientation == TOKEN_WISE:
        data = torch.zeros(pad128(rows), cols // 2, dtype=BF16, device=dev)
        data[:rows] = tv.reshape(rows, cols // 2).to(BF16)
        hw = None
        if rows and cols % 128 == 0:
            hw = torch.full((_lib.meta_hw_bytes(rows, cols),), 0x44, dtype=torch.uint8, device=dev)
            _lib.call("s24_meta_ref_to_hw", ptr(tm.contiguous()), rows, cols, ptr(hw), stream())
        return Sparse24Matrix(rows, cols, TOKEN_WISE, data, hw, tm)
    # feature-wise: the device operand is the transposed (per-feature) layout
    data = torch.zeros(pad128(cols), rows // 2, dtype=BF16, device=dev)
    data[:cols] = tv.permute(1, 0, 2).reshape(cols, rows // 2).to(BF16)
    hw = None
    if cols and rows % 128 == 0:
        hw = torch.full((_lib.meta_hw_bytes(cols, rows),), 0x44, dtype=torch.uint8, device=dev)
        _lib.call("s24_meta_ref_to_hw", ptr(tm.permute(1, 0, 2).contiguous()), cols, rows, ptr(hw), stream())
    return Sparse24Matrix(rows, cols, FEATURE_WISE, data, hw, tm)
