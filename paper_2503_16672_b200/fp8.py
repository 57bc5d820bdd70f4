"""e4m3 (fp8) path on the kind::f8f6f4 tensor cores.

The reference emulates 8-bit storage on the CPU (ref matcore.py:113-261,
ffn.py:206-268): per-row / per-column amax/448 scales, e4m3 codes, an fp32 sum
over the decoded codes with the scales applied outside it. Here the codes are
real e4m3 operands of tcgen05 MMAs (dense and 2:4), produced by the
quantization kernels of csrc/fp8.cu and consumed K-major:

  _mm(a, b)       a per row  -> codes [M, K];  b per column -> codes_t [N, K]
  _mm_at(a, b)    a, b per column, both transposed (K = tokens)
  _sp_mm(s, b)    token-wise 2:4 values per row (metadata converted to the
                  e4m3 operand-E layout), b per column
  split / naive   the feature-wise split operand (csrc/k4*.cuh) quantized per
                  row -- per feature; a dense feature's two 2:4 rows share one
                  scale -- times b per column

Codes and scales are bit-identical to the reference given identical fp32
inputs (tests/test_gpu_fp8.py). Inside the FFN the inputs are the bf16
activations of the device path, so FFN results agree with the reference's
emulation to a tolerance (tests/test_gpu_ffn_fp8.py), not bitwise.

Public API mirrors ref matcore.py: E4M3_MAX, Fp8Rowwise, e4m3_encode,
e4m3_decode, fp8_quantize_rowwise, fp8_dequantize, fp8_gemm_rowwise.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._tensors import BF16, F32, as_matrix, pad128, ptr, require_cuda, stream
from .errors import DimensionError, NonFiniteError, OrientationError

E4M3_MAX = 448.0
U8 = torch.uint8


def _dtype_code(t: torch.Tensor) -> int:
    return _lib.F32 if t.dtype == F32 else _lib.BF16


def _decode_table(device) -> torch.Tensor:
    """float32 value of every e4m3 code (ref matcore.py:128-145)."""
    c = torch.arange(256, device=device)
    e, m = (c >> 3) & 0xF, c & 7
    mag = torch.where(e == 0, m.double() * 2.0**-9, torch.ldexp(1.0 + m.double() / 8.0, (e - 7).double()))
    v = torch.where((c & 0x80) != 0, -mag, mag)
    v = torch.where((e == 15) & (m == 7), torch.full_like(v, float("nan")), v)
    return v.float()


# ---------------------------------------------------------------- kernels


def quant_rows(a: torch.Tensor, rows: int | None = None, pair_rows: int = 0, amax: torch.Tensor | None = None,
               codes: torch.Tensor | None = None, deq: torch.Tensor | None = None,
               raw: torch.Tensor | None = None, scales: torch.Tensor | None = None,
               st=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Per-row e4m3 codes [R, C] and scales of the first `rows` rows of a
    (bf16 or fp32). Rows past `rows` in a preallocated `codes` / `scales` are
    left as they are. deq / raw: optional bf16 outputs (dequantized /
    unquantized images). Outputs are allocated on the current stream; st
    (a torch stream) launches the kernel elsewhere."""
    R = a.shape[0] if rows is None else rows
    C = a.shape[1]
    if codes is None:
        codes = torch.empty(a.shape[0], C, dtype=U8, device=a.device)
    if scales is None:
        scales = torch.empty(codes.shape[0], dtype=F32, device=a.device)
    _lib.call("s24_fp8_quant_rows", ptr(a), _dtype_code(a), R, C, a.stride(0), ptr(amax), pair_rows, ptr(codes),
              codes.stride(0), ptr(scales), ptr(deq), deq.stride(0) if deq is not None else 0, ptr(raw),
              raw.stride(0) if raw is not None else 0, st.cuda_stream if st is not None else stream())
    return codes, scales


def quant_cols_t(a: torch.Tensor, codes_t: torch.Tensor | None = None, scales: torch.Tensor | None = None,
                 st=None, keep: list | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Per-column codes of a [R, C] (bf16 or fp32), transposed: ([C, R16]
    codes with R16 = R rounded up to 16, zero beyond R; scales [C]). With st
    (another stream) the workspace is appended to `keep`, to stay alive until
    that stream's work has been joined."""
    R, C = a.shape
    ld = (R + 15) // 16 * 16
    if codes_t is None:
        codes_t = torch.empty(C, ld, dtype=U8, device=a.device)
        if ld > R:
            codes_t[:, R:].zero_()
    if scales is None:
        scales = torch.empty(C, dtype=F32, device=a.device)
    ws = torch.empty(max(C, 1), dtype=torch.int32, device=a.device)
    if keep is not None:
        keep.append(ws)
    _lib.call("s24_fp8_quant_cols_t", ptr(a), _dtype_code(a), R, C, a.stride(0), ptr(codes_t), codes_t.stride(0),
              ptr(scales), ptr(ws), st.cuda_stream if st is not None else stream())
    return codes_t, scales


def meta_to_f8(meta_hw: torch.Tensor, rows: int, kdim: int, out: torch.Tensor | None = None,
               st=None) -> torch.Tensor:
    out = torch.empty_like(meta_hw) if out is None else out
    _lib.call("s24_meta_hw_to_f8", ptr(meta_hw), rows, kdim, ptr(out), st.cuda_stream if st is not None else stream())
    return out


def _t_codes(R: int, C: int, dev) -> tuple[torch.Tensor, torch.Tensor]:
    """Output buffers of quant_cols_t for an [R, C] operand (padding zeroed)."""
    ld = (R + 15) // 16 * 16
    codes_t = torch.empty(C, ld, dtype=U8, device=dev)
    if ld > R:
        codes_t[:, R:].zero_()
    return codes_t, torch.empty(C, dtype=F32, device=dev)


class _Overlap:
    """Side-stream work next to the main-stream GEMMs (as in the bf16 path):
    outputs are allocated on the main stream before the side stream is
    forked, temporaries are kept alive in `keep` until the main stream has
    joined the side stream's event."""

    def __init__(self, dev, enabled: bool):
        from .splitgemm import side_stream

        self.main = torch.cuda.current_stream(dev)
        self.side = side_stream(dev) if enabled else None
        self.keep: list = []

    @property
    def st(self):
        return self.side if self.side is not None else self.main

    def fork(self, ev=None) -> None:
        """The side stream waits for the main stream's work so far (or ev)."""
        if self.side is not None:
            if ev is not None:
                self.side.wait_event(ev)
            else:
                self.side.wait_stream(self.main)

    def record(self, stream=None):
        ev = torch.cuda.Event()
        ev.record(stream or self.st)
        return ev

    def join(self, ev) -> None:
        if ev is not None and self.side is not None:
            self.main.wait_event(ev)


def gemm_f8(aq, sa, bq, sb, M, N, K, out, row_map=None, transposed=False, rows_valid=-1) -> torch.Tensor:
    """out = (sa x sb) * (aq [M, K] . bq [N, K]^T) on e4m3 codes."""
    _lib.call("s24_gemm_f8", ptr(aq), aq.stride(0), ptr(bq), bq.stride(0), M, N, K, ptr(sa), ptr(sb), ptr(out),
              _dtype_code(out), out.stride(0), ptr(row_map), int(transposed), rows_valid, stream())
    return out


def spmm_f8(aq, meta8, sa, bq, sb, M, N, K, out, row_map=None, transposed=False, rows_valid=-1, row_valid=None,
            pair_rows=0) -> torch.Tensor:
    """out = (sa x sb) * (2:4 aq [M, K/2] . bq [N, K]^T)."""
    _lib.call("s24_spmm_f8", ptr(aq), ptr(meta8), ptr(bq), bq.stride(0), M, N, K, ptr(sa), ptr(sb), ptr(out),
              _dtype_code(out), out.stride(0), ptr(row_map), int(transposed), rows_valid, ptr(row_valid), pair_rows,
              stream())
    return out


def mm_f8(a: torch.Tensor, bt: torch.Tensor, out: torch.Tensor, row_map=None, rows: int | None = None):
    """ref _mm(a, b) with b given as its transpose bt [N, K] (the stored
    weight): a per row, b per column = bt per row (ref ffn.py:206-209)."""
    M = a.shape[0] if rows is None else rows
    aq, sa = quant_rows(a, rows=M)
    bq, sb = quant_rows(bt)
    return gemm_f8(aq, sa, bq, sb, M, bt.shape[0], a.shape[1], out, row_map, rows_valid=M)


def mm_at_f8(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, transposed: bool = False):
    """ref _mm_at(a, b) = a^T b, both per column (ref ffn.py:212-218); K =
    rows of a and b (zero rows past the logical count are harmless)."""
    aq, sa = quant_cols_t(a)
    bq, sb = quant_cols_t(b)
    return gemm_f8(aq, sa, bq, sb, a.shape[1], b.shape[1], aq.shape[1], out, transposed=transposed)


# ---------------------------------------------------------------- reference-facing API


@dataclass(frozen=True)
class Fp8Rowwise:
    """e4m3 matrix with one positive scale per row or column (ref
    matcore.py:200-207), on the device. For axis "cols" the codes are stored
    transposed (K-major for the GEMM); .codes is the [rows, cols] view."""

    rows: int
    cols: int
    storage: torch.Tensor  # uint8 [rows, cols] ("rows") or [cols, >= rows] ("cols")
    scales: torch.Tensor  # float32 [rows] or [cols]
    axis: str

    @property
    def codes(self) -> torch.Tensor:
        return self.storage if self.axis == "rows" else self.storage[:, :self.rows].t()


def e4m3_encode(x) -> torch.Tensor:
    """Nearest e4m3 codes of finite input, ties to even, saturating (ref
    matcore.py:155-197); device uint8 of the same shape."""
    require_cuda()
    t = torch.as_tensor(x, dtype=F32)
    t = t.cuda() if not t.is_cuda else t
    if not bool(torch.isfinite(t).all()):
        raise NonFiniteError("e4m3_encode requires finite input")
    flat = t.contiguous().view(-1)
    codes = torch.empty(flat.numel(), dtype=U8, device=t.device)
    _lib.call("s24_e4m3_encode", ptr(flat), flat.numel(), ptr(codes), stream())
    return codes.view(t.shape)


def e4m3_decode(code) -> torch.Tensor:
    """Exact value (float32) of e4m3 bit patterns (ref matcore.py:148-152)."""
    require_cuda()
    c = torch.as_tensor(code).cuda().to(torch.long)
    return _decode_table(c.device)[c]


def fp8_quantize_rowwise(a, axis: str = "rows") -> Fp8Rowwise:
    """ref matcore.py:210-230: amax/448 scales per row or column (1 for an
    all-zero slice), e4m3 codes of a / scale."""
    require_cuda()
    if axis not in ("rows", "cols"):
        raise OrientationError(f"axis must be 'rows' or 'cols', got {axis!r}")
    a = as_matrix(a, "a")  # fp32 or bf16, quantized as given
    if not bool(torch.isfinite(a).all()):
        raise NonFiniteError("quantization requires finite input")
    rows, cols = a.shape
    if cols % 8 or (axis == "cols" and a.dtype == BF16 and a.stride(0) % 8):
        a_in = torch.zeros(rows, (cols + 7) // 8 * 8, dtype=a.dtype, device=a.device)
        a_in[:, :cols] = a
    else:
        a_in = a
    if axis == "rows":
        codes, scales = quant_rows(a_in)
        return Fp8Rowwise(rows, cols, codes[:, :cols], scales, axis)
    codes_t, scales = quant_cols_t(a_in)
    return Fp8Rowwise(rows, cols, codes_t[:cols], scales[:cols], axis)


def fp8_dequantize(q: Fp8Rowwise) -> torch.Tensor:
    """scale * decode(code), float32 (ref matcore.py:233-238)."""
    vals = _decode_table(q.scales.device)[q.codes.long()]
    return vals * (q.scales[:, None] if q.axis == "rows" else q.scales[None, :])


def fp8_gemm_rowwise(a: Fp8Rowwise, b: Fp8Rowwise) -> torch.Tensor:
    """c = (scaleA x scaleB) * (decode(a) @ decode(b)) with fp32 accumulation on
    the e4m3 tensor cores (ref matcore.py:241-261)."""
    if a.axis != "rows":
        raise OrientationError("first operand must carry per-row scales")
    if b.axis != "cols":
        raise OrientationError("second operand must carry per-column scales")
    if a.cols != b.rows:
        raise DimensionError(f"inner dimensions differ: {a.rows}x{a.cols} x {b.rows}x{b.cols}")
    M, K, N = a.rows, a.cols, b.cols
    out = torch.empty(M, N, dtype=F32, device=a.scales.device)
    if M == 0 or N == 0:
        return out
    Kp = (K + 15) // 16 * 16
    aq = a.storage
    if aq.shape[1] != Kp or aq.stride(0) % 16:
        aq = torch.zeros(M, Kp, dtype=U8, device=out.device)
        aq[:, :K] = a.storage[:, :K]
    bq = b.storage
    if bq.shape[1] < Kp or bq.stride(0) % 16:
        bq = torch.zeros(N, Kp, dtype=U8, device=out.device)
        bq[:, :K] = b.storage[:, :K]
    Np = (N + 31) // 32 * 32
    if Np != N:
        bq = torch.cat([bq, torch.zeros(Np - N, bq.shape[1], dtype=U8, device=out.device)])
        sb = torch.cat([b.scales, torch.ones(Np - N, dtype=F32, device=out.device)])
        full = torch.empty(M, Np, dtype=F32, device=out.device)
        gemm_f8(aq, a.scales, bq, sb, M, Np, Kp, full)
        return full[:, :N].contiguous()
    return gemm_f8(aq, a.scales, bq, b.scales, M, N, Kp, out)


# ---------------------------------------------------------------- FFN


def ffn_forward_f8(x: torch.Tensor, p, cfg, plan, keep_pre_act: bool, for_backward: bool, h_valid=None,
                   counts_hook=None):
    """ffn_forward under fp8_emulation (ref ffn.py:276-363 with fp8=True): the
    two forward GEMMs on e4m3 operands. Sparse forward: K1 on e4m3 codes
    selects on the fp32 scaled pre-activation (selection before quantization,
    ref tests/test_ffn.py:360-367), the kept values are quantized per token,
    fwd.out is the e4m3 2:4 MMA. The cache holds the dequantized activation
    (what the backward of the reference sees) and, for K3, the unquantized one."""
    from .ffn import FfnCache, GemmEvent, _frame_rows, _plan_split
    from .matcore import device_permutation, gemm_macs
    from .sparse24 import SparsifyStats, sp_gemm_macs

    n, d = x.shape
    h = p.hidden_dim
    dev = x.device
    npad = pad128(n)
    census = []
    sparse_fwd = cfg.forward_mode == "sparse24"
    perm_dev = inv_dev = None
    if cfg.permute_tokens and sparse_fwd and for_backward:  # (inference: see ffn.ffn_forward)
        perm_dev, inv_dev = device_permutation(cfg.permute_seed, n, dev)
    out = torch.empty(n, d, dtype=BF16, device=dev)
    if not sparse_fwd:
        x_in = _frame_rows(x, npad, None)
        xq, sx = quant_rows(x_in)
        w1q, s1 = quant_cols_t(p.w1)  # [h, d] (d % 32 == 0)
        pre = gemm_f8(xq, sx, w1q, s1, n, h, d, torch.empty(n, h, dtype=F32, device=dev), rows_valid=n)
        census.append(GemmEvent("fwd.pre_act", False, gemm_macs(n, d, h)))
        r = torch.clamp_min(pre, 0)
        act = r * r
        w2q, s2 = quant_cols_t(p.w2)  # [d, h]
        aq, sa = quant_rows(act)
        gemm_f8(aq, sa, w2q, s2, n, d, h, out, rows_valid=n)
        census.append(GemmEvent("fwd.out", False, gemm_macs(n, h, d)))
        return out, FfnCache(n, cfg, census, _x_in=x_in, act_dense=act.to(BF16), pre_act=pre, act_f32=act)

    from .ffn import _all_sparse_plan
    from .splitgemm import alloc_feature_split, run_feature_split

    ov = _Overlap(dev, True)
    fp8b = cfg.fp8_backward and for_backward
    split_bwd = for_backward and cfg.backward_mode != "dense"
    # W2 codes for fwd.out -- and the backward's weight codes -- on the side
    # stream while the main stream gathers / quantizes x and runs K1
    w2q, s2 = _t_codes(h, d, dev)  # [d, h]
    wb = None
    if fp8b:
        wb = {"w2r": torch.empty(h, d, dtype=U8, device=dev), "s2r": torch.empty(h, dtype=F32, device=dev),
              "w1r": torch.empty(d, h, dtype=U8, device=dev), "s1r": torch.empty(d, dtype=F32, device=dev)}
    ov.fork()
    quant_cols_t(p.w2, w2q, s2, st=ov.st, keep=ov.keep)
    if wb is not None:
        quant_rows(p.w2, codes=wb["w2r"], scales=wb["s2r"], st=ov.st)  # w2t per column (K3 B)
        quant_rows(p.w1, codes=wb["w1r"], scales=wb["s1r"], st=ov.st)  # w1t per column (dX B)
    ev_w = ov.record()

    x_in = _frame_rows(x, npad, inv_dev)
    # x_in^T codes (the dW1 GEMM's B operand) on a stream of their own, from
    # here on: off the chain of plan / K4(act) / split codes of the side stream,
    # so neither waits for the other (their events are merged into side_ready)
    xt = sxt = ev_xt = None
    if split_bwd and fp8b:
        from .splitgemm import side_stream

        xt = torch.empty(d, npad, dtype=U8, device=dev)  # npad % 128 == 0: no padding columns
        sxt = torch.empty(d, dtype=F32, device=dev)
        st_x = side_stream(dev, 2)
        st_x.wait_stream(ov.main)
        quant_cols_t(x_in, xt, sxt, st=st_x, keep=ov.keep)
        ev_xt = ov.record(st_x)
    xq, sx = quant_rows(x_in)
    w1q, s1 = quant_cols_t(p.w1)  # [h, d] (d % 32 == 0)
    vals32 = torch.empty(npad, h // 2, dtype=F32, device=dev)
    amax = torch.zeros(npad, dtype=torch.int32, device=dev)
    act_meta = torch.empty(_lib.meta_hw_bytes(n, h), dtype=U8, device=dev)
    act_vals = torch.empty(npad, h // 2, dtype=BF16, device=dev)  # dequantized (the reference's act_sparse)
    act_raw = torch.empty(npad, h // 2, dtype=BF16, device=dev)  # unquantized, for K3
    aq = torch.empty(npad, h // 2, dtype=U8, device=dev)
    if npad > n:
        act_vals[n:].zero_()
        act_raw[n:].zero_()
        aq[n:].zero_()
        act_meta[(n // 128) * (h // 128) * 2048:].fill_(0x44)
    counts = torch.zeros(h, dtype=torch.int32, device=dev)
    stats_dev = torch.zeros(3, dtype=torch.int64, device=dev)
    need_pre = keep_pre_act or not cfg.mask_grad_with_fwd
    pre = torch.empty(n, h, dtype=F32, device=dev) if need_pre else None
    _lib.call("s24_fwd_gemm1_f8", ptr(xq), xq.stride(0), ptr(w1q), w1q.stride(0), n, h, d, ptr(sx),
              ptr(s1), ptr(vals32), ptr(amax), ptr(act_meta), ptr(counts), ptr(stats_dev), ptr(pre), stream())
    census.append(GemmEvent("fwd.pre_act", False, gemm_macs(n, d, h)))
    _, sa = quant_rows(vals32, rows=n, amax=amax, codes=aq, deq=act_vals, raw=act_raw)
    meta8 = meta_to_f8(act_meta, n, h)
    if plan is not None and plan.hidden_dim != (h_valid or h):
        raise DimensionError(f"plan built for {plan.hidden_dim} features, FFN has {h_valid or h}")

    # backward operands that depend only on the forward, prepared on the side
    # stream next to fwd.out: the plan, the feature-wise split of act (K4),
    # and under fp8_backward its e4m3 codes plus the codes of x_in^T (dW1's B).
    # Everything the side stream reads or writes is allocated (and, with
    # kernels, initialised) on the main stream before the fork point ev_k1.
    naive_plan = _all_sparse_plan(h, dev) if cfg.backward_mode == "naive_sparse" else None
    ev_k1 = ov.record(ov.main)
    ov.fork(ev_k1)
    if counts_hook is not None:
        with torch.cuda.stream(ov.st):  # (a collective here overlaps fwd.out, as in ffn.py)
            counts_hook(counts)
    plan_api = plan_out = plan
    if cfg.backward_mode == "split_masked" or plan is not None:  # (allocations only here)
        plan_api, plan_out = _plan_split(counts, cfg.split_ratio, plan, h, h_valid, ov.st)
    bplan = naive_plan if naive_plan is not None else plan_out
    fa = f8 = None
    if split_bwd:
        fa = alloc_feature_split(act_vals, act_meta, npad, h, bplan)
    if split_bwd and fp8b:
        f8 = dict(wb, vq_a=torch.empty(fa.vs.shape, dtype=U8, device=dev),
                  sv_a=torch.empty(fa.vs.shape[0], dtype=F32, device=dev), e8_a=torch.empty_like(fa.es),
                  rows_a=fa.rows(bplan), xt=xt, sxt=sxt, keep=ov.keep)
    elif wb is not None:
        f8 = dict(wb, keep=ov.keep)
    ov.join(ev_w)
    spmm_f8(aq, meta8, sa, w2q, s2, n, d, h, out, row_map=inv_dev, rows_valid=n)
    census.append(GemmEvent("fwd.out", True, sp_gemm_macs(n, h, d)))
    ev_side = None
    if split_bwd:
        with torch.cuda.stream(ov.st):
            run_feature_split(fa, act_vals, act_meta, npad, h, bplan, nonneg=True)
            if f8 is not None and "vq_a" in f8:
                f8["vq_a"].zero_()  # (padding rows of the operand)
        if f8 is not None and "vq_a" in f8:
            quant_rows(fa.vs, rows=f8["rows_a"], pair_rows=fa.pair_rows, codes=f8["vq_a"], scales=f8["sv_a"],
                       st=ov.st)
            meta_to_f8(fa.es, f8["rows_a"], npad, out=f8["e8_a"], st=ov.st)
        if ev_xt is not None:
            ov.st.wait_event(ev_xt)  # (side_ready covers the x_in^T codes too)
        ev_side = ov.record()
    elif ov.side is not None and plan_out is not None and plan_out is not plan:
        ev_side = ov.record()
    if ov.side is None:
        ev_side = None
    elif ev_side is None:
        ev_side = ev_w
    cache = FfnCache(n, cfg, census, _x_in=x_in if for_backward else None, act_vals=act_vals, act_meta=act_meta,
                     pre_act=pre, perm_dev=perm_dev, inv_dev=inv_dev, _plan=plan_out,
                     stats=SparsifyStats(n * h, stats_dev[:2]), counts=counts, stats_dev=stats_dev, act_split=fa,
                     side_ready=ev_side, act_raw=act_raw, act_meta8=meta8, f8=f8,
                     plan_valid=plan_api if h_valid is not None else None)
    if ov.side is not None and not for_backward:
        ov.join(ev_side)
    return out, cache


def _split_grad_f8(fs, plan, b: torch.Tensor, npad: int, out: torch.Tensor, transposed: bool) -> None:
    """split / naive weight gradient on e4m3 operands: the feature-wise split
    (paired layout) quantized per feature, b per column (ref ffn.py:258-270)."""
    rows, rmap, valid = fs.rows(plan), plan.paired_row_map, None
    if not rows:
        return
    vq = torch.zeros(fs.vs.shape[0], fs.vs.shape[1], dtype=U8, device=b.device)
    _, sv = quant_rows(fs.vs, rows=rows, pair_rows=max(fs.pair_rows, 0), codes=vq)
    e8 = meta_to_f8(fs.es, rows, npad)
    bq, sb = quant_cols_t(b)  # [d, npad]
    spmm_f8(vq, e8, sv, bq, sb, rows, b.shape[1], npad, out, row_map=rmap, transposed=transposed, rows_valid=rows,
            row_valid=valid, pair_rows=max(fs.pair_rows, 0))


def ffn_backward_f8(g_out: torch.Tensor, cache, p, cfg, grad_ready=None, grad_bucket=None):
    """ffn_backward under fp8_backward (ref ffn.py:366-451 with fp8b=True):
    every backward GEMM on e4m3 operands."""
    from .ffn import FfnGrads, GemmEvent, _all_sparse_plan, _frame_rows, weight_grad_buffers
    from .matcore import gemm_macs
    from .sparse24 import sp_gemm_macs, sparsify_feature_wise
    from .splitgemm import feature_split, split_gemm_macs

    n = cache.n
    x_in = cache._x_in
    d = x_in.shape[1]
    h = p.hidden_dim
    dev = g_out.device
    npad = pad128(n)
    s = stream()
    census = []
    notify = grad_ready or (lambda name, t: None)
    d_w1, d_w2 = weight_grad_buffers(d, h, dev, grad_bucket)
    d_x = torch.empty(n, d, dtype=BF16, device=dev)
    g_c = _frame_rows(g_out, npad, cache.inv_dev)

    if cfg.forward_mode == "dense":
        G = mm_f8(g_c, p.w2, torch.empty(n, h, dtype=F32, device=dev), rows=n)  # g_out_c . w2t
        census.append(GemmEvent("bwd.d_act", False, gemm_macs(n, d, h)))
        g_pre = G * (2 * torch.clamp_min(cache.pre_act, 0))
        mm_at_f8(cache.act_f32, g_c[:n], d_w2)
        census.append(GemmEvent("bwd.d_w2", False, gemm_macs(h, n, d)))
        notify("d_w2", d_w2)
        mm_at_f8(x_in[:n], g_pre, d_w1)
        census.append(GemmEvent("bwd.d_w1", False, gemm_macs(d, n, h)))
        notify("d_w1", d_w1)
        mm_f8(g_pre, p.w1, d_x)
        census.append(GemmEvent("bwd.d_x", False, gemm_macs(n, h, d)))
        return FfnGrads(d_w1, d_w2, d_x, None, census)

    # ---------------------------------------------------------- sparse forward
    from .splitgemm import alloc_feature_split, run_feature_split

    f8 = cache.f8 or {}
    ov = _Overlap(dev, True)
    mode = cfg.backward_mode
    raw_naive = mode == "naive_sparse" and not cfg.mask_grad_with_fwd
    split = mode != "dense" and not raw_naive and cache.act_split is not None
    # weight codes: prepared by the forward on its side stream (joined before
    # fwd.out), else here
    if "w2r" in f8:
        w2q, s2, w1r, s1r = f8["w2r"], f8["s2r"], f8["w1r"], f8["s1r"]
    else:
        w2q, s2 = quant_rows(p.w2)  # w2t per column = w2 per row: [h, d]
        w1r, s1r = quant_rows(p.w1)  # w1t per column = w1 per row: [d, h]
    gt = sgt = ev_gt = None
    if split:
        # g_c^T codes (dW2's B operand) on a stream of their own (not queued
        # behind the forward's side work), next to K3
        from .splitgemm import side_stream

        gt = torch.empty(d, npad, dtype=U8, device=dev)
        sgt = torch.empty(d, dtype=F32, device=dev)
        st_g = side_stream(dev, 3)
        st_g.wait_stream(ov.main)
        quant_cols_t(g_c, gt, sgt, st=st_g, keep=ov.keep)
        ev_gt = ov.record(st_g)
    # K3 on e4m3 codes: g_pre on the forward keep pattern (relu from the
    # unquantized activation), compressed
    gq, sg = quant_rows(g_c)
    g_vals = torch.empty(npad, h // 2, dtype=BF16, device=dev)
    if npad > n:
        g_vals[n:].zero_()
    _lib.call("s24_bwd_dact_f8", ptr(gq), gq.stride(0), ptr(w2q), w2q.stride(0), n, h, d, ptr(sg), ptr(s2),
              ptr(cache.act_raw), ptr(cache.act_meta), ptr(g_vals), s)
    census.append(GemmEvent("bwd.d_act", False, gemm_macs(n, d, h)))
    g_pre_dense = None
    if not cfg.mask_grad_with_fwd:
        G = gemm_f8(gq, sg, w2q, s2, n, h, d, torch.empty(n, h, dtype=F32, device=dev), rows_valid=n)
        g_pre_dense = G * (2 * torch.clamp_min(cache.pre_act, 0))

    # K4 of g_pre and its codes on the side stream, next to the dX GEMM
    ev_g = None
    if split:
        plan = _all_sparse_plan(h, dev) if mode == "naive_sparse" else cache._plan
        fg = alloc_feature_split(g_vals, cache.act_meta, npad, h, plan)
        rows_g = fg.rows(plan)
        vq_g = torch.empty(fg.vs.shape, dtype=U8, device=dev)
        sv_g = torch.empty(fg.vs.shape[0], dtype=F32, device=dev)
        e8_g = torch.empty_like(fg.es)
        ov.fork()
        with torch.cuda.stream(ov.st):
            run_feature_split(fg, g_vals, cache.act_meta, npad, h, plan)
            vq_g.zero_()
        quant_rows(fg.vs, rows=rows_g, pair_rows=fg.pair_rows, codes=vq_g, scales=sv_g, st=ov.st)
        meta_to_f8(fg.es, rows_g, npad, out=e8_g, st=ov.st)
        ev_g = ov.record()

    # dX (main stream)
    if cfg.mask_grad_with_fwd:
        gsq = torch.empty(npad, h // 2, dtype=U8, device=dev)
        if npad > n:
            gsq[n:].zero_()
        _, sgs = quant_rows(g_vals, rows=n, codes=gsq)
        spmm_f8(gsq, cache.act_meta8, sgs, w1r, s1r, n, d, h, d_x, row_map=cache.inv_dev, rows_valid=n)
        ev_dx = GemmEvent("bwd.d_x", True, sp_gemm_macs(n, h, d))
    else:
        aq, sa = quant_rows(g_pre_dense)
        gemm_f8(aq, sa, w1r, s1r, n, d, h, d_x, row_map=cache.inv_dev, rows_valid=n)
        ev_dx = GemmEvent("bwd.d_x", False, gemm_macs(n, h, d))

    stats_a = stats_g = None
    if mode == "dense":
        act = torch.empty(n, h, dtype=BF16, device=dev)
        _lib.call("s24_decompress_token", ptr(cache.act_vals), None, ptr(cache.act_meta), n, h, ptr(act), _lib.BF16,
                  h, s)
        mm_at_f8(act, g_c[:n], d_w2)
        census.append(GemmEvent("bwd.d_w2", False, gemm_macs(h, n, d)))
        notify("d_w2", d_w2)
        if g_pre_dense is None:
            gp = torch.empty(n, h, dtype=BF16, device=dev)
            _lib.call("s24_decompress_token", ptr(g_vals), None, ptr(cache.act_meta), n, h, ptr(gp), _lib.BF16, h, s)
        else:
            gp = g_pre_dense
        ov.join(cache.side_ready)
        mm_at_f8(x_in[:n], gp, d_w1)
        census.append(GemmEvent("bwd.d_w1", False, gemm_macs(d, n, h)))
        notify("d_w1", d_w1)
    else:
        plan = _all_sparse_plan(h, dev) if mode == "naive_sparse" else cache._plan
        macs_w = sp_gemm_macs(n, h, d) if mode == "naive_sparse" else split_gemm_macs(n, d, plan)
        # the forward's side work (act split, its codes, x_in^T codes) and ours
        if cache.side_ready is not None:
            torch.cuda.current_stream().wait_event(cache.side_ready)
        ov.join(ev_g)
        ov.join(ev_gt)
        fa = cache.act_split
        if fa is None:
            fa = feature_split(cache.act_vals, cache.act_meta, npad, h, plan)
        if "vq_a" in f8 and ev_g is not None and grad_ready is None and gt is not None and "xt" in f8:
            # both split weight gradients in one grouped e4m3 launch (no
            # per-gradient hook to serve): dW2 = split(act)^T g_c, dW1^T = split(g_pre)^T x_in
            rows_a, rmap, valid = fa.rows(plan), plan.paired_row_map, None
            _lib.call("s24_spmm_pair_f8", rows_a, d, npad, _lib.F32,
                      ptr(f8["vq_a"]), ptr(f8["e8_a"]), ptr(gt), gt.stride(0), ptr(f8["sv_a"]), ptr(sgt), ptr(d_w2),
                      d_w2.stride(0), ptr(rmap), 0, ptr(valid),
                      ptr(vq_g), ptr(e8_g), ptr(f8["xt"]), f8["xt"].stride(0), ptr(sv_g), ptr(f8["sxt"]), ptr(d_w1),
                      d_w1.stride(0), ptr(rmap), 1, ptr(valid), max(fa.pair_rows, 0), s)
            census.append(GemmEvent("bwd.d_w2", True, macs_w))
            census.append(GemmEvent("bwd.d_w1", True, macs_w))
            census.append(ev_dx)
            return FfnGrads(d_w1, d_w2, d_x, None, census, fa.stats, fg.stats)
        if "vq_a" in f8:
            if gt is None:
                gt, sgt = quant_cols_t(g_c)
            rows_a, rmap, valid = fa.rows(plan), plan.paired_row_map, None
            spmm_f8(f8["vq_a"], f8["e8_a"], f8["sv_a"], gt, sgt, rows_a, d, npad, d_w2, row_map=rmap,
                    rows_valid=rows_a, row_valid=valid, pair_rows=max(fa.pair_rows, 0))
        else:
            _split_grad_f8(fa, plan, g_c, npad, d_w2, transposed=False)
        stats_a = fa.stats
        census.append(GemmEvent("bwd.d_w2", True, macs_w))
        notify("d_w2", d_w2)
        if raw_naive:
            gpad = torch.zeros(npad, h, dtype=F32, device=dev)
            gpad[:n] = g_pre_dense
            sgw, _, stats_g = sparsify_feature_wise(gpad)
            vq = torch.zeros(sgw.data.shape, dtype=U8, device=dev)
            _, sv = quant_rows(sgw.data, rows=h, codes=vq)
            bq, sb = quant_cols_t(x_in)
            spmm_f8(vq, meta_to_f8(sgw.meta_hw, h, npad), sv, bq, sb, h, d, npad, d_w1, transposed=True, rows_valid=h)
        elif ev_g is not None:
            rmap, valid = plan.paired_row_map, None
            xt, sxt = (f8["xt"], f8["sxt"]) if "xt" in f8 else quant_cols_t(x_in)
            spmm_f8(vq_g, e8_g, sv_g, xt, sxt, rows_g, d, npad, d_w1, row_map=rmap, transposed=True,
                    rows_valid=rows_g, row_valid=valid, pair_rows=max(fg.pair_rows, 0))
            stats_g = fg.stats
        else:
            fg = feature_split(g_vals, cache.act_meta, npad, h, plan)
            _split_grad_f8(fg, plan, x_in, npad, d_w1, transposed=True)
            stats_g = fg.stats
        census.append(GemmEvent("bwd.d_w1", True, macs_w))
        notify("d_w1", d_w1)
    census.append(ev_dx)
    return FfnGrads(d_w1, d_w2, d_x, None, census, stats_a, stats_g)
