"""Squared-ReLU FFN with the 2:4 activation-sparsity recipe on B200 -- drop-in
for the reference's pkg/src/srelu24/ffn.py (ffn_forward / ffn_backward and
their dataclasses; activation = squared_relu).

Recipe forward (ref ffn.py:276-363), one device pass each:
  K6  x_in = permute_rows(x, perm)                     (row gather, padded to 128 rows)
  K1  Y1 = x_in . W1 -> relu^2 -> token-wise 2:4       (tcgen05 GEMM, fused epilogue:
      compressed act + hw metadata + per-feature counts + drop stats)
  K2  out = inverse_permute_rows(act_sp . W2)          (tcgen05.mma.sp, row map epilogue)
  side stream, next to K2:
  K7  plan = partition_features(counts, ratio)         (device radix select)
  K4  feature-wise 2:4 split of act (sparse features) + dense features as row pairs
Recipe backward (ref ffn.py:366-451):
  K6  g_c = permute_rows(dY, perm)
  K3  g_pre = (g_c . W2^T) * 2 relu(y1) on the forward keep pattern (fused, compressed)
  K2  dX = inverse_permute_rows(g_pre_sp . W1^T)       (exact: forward metadata)
      side stream, next to it: K4 split of g_pre
  K5  dW2 = split(act)^T g_c ; dW1 = (split(g_pre)^T x_in)^T  (one grouped 2:4 launch,
      feature-index scatter / transpose in the epilogue)
Dense mode runs the same GEMM kernels with dense operands (the "dense twin").

Tensors are bf16 on the device (numpy float32 inputs are uploaded and rounded
to bf16). Weight gradients are fp32, activations/outputs bf16.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import torch

from . import _lib
from ._tensors import BF16, F32, as_matrix, pad128, ptr, require_cuda, stream
from .errors import ConfigError, DimensionError, StateError
from .matcore import device_permutation, gather_rows, gemm_macs
from .sparse24 import (
    TOKEN_WISE,
    Sparse24Matrix,
    SparsifyStats,
    sp_gemm_macs,
)
from .splitgemm import (
    FeatureSplit,
    SplitPlan,
    alloc_feature_split,
    feature_split,
    pad_plan,
    partition_features,
    partition_features_padded,
    run_feature_split,
    side_stream,
    split_gemm_macs,
    split_weight_grad,
)

ACTIVATIONS = ("squared_relu", "swiglu")
FORWARD_MODES = ("dense", "sparse24")
BACKWARD_MODES = ("dense", "naive_sparse", "split_masked")


@dataclass(frozen=True)
class FfnConfig:
    """Same fields, defaults and cross-field validation as ref ffn.py:58-101."""

    activation: str = "squared_relu"
    forward_mode: str = "dense"
    backward_mode: str = "dense"
    mask_grad_with_fwd: bool = False
    permute_tokens: bool = False
    permute_seed: int = 0
    split_ratio: float = 0.95
    fp8_emulation: bool = False
    fp8_backward: bool = False

    def __post_init__(self):
        if self.activation not in ACTIVATIONS:
            raise ConfigError(f"unknown activation {self.activation!r}")
        if self.forward_mode not in FORWARD_MODES:
            raise ConfigError(f"unknown forward_mode {self.forward_mode!r}")
        if self.backward_mode not in BACKWARD_MODES:
            raise ConfigError(f"unknown backward_mode {self.backward_mode!r}")
        sparse_any = self.forward_mode != "dense" or self.backward_mode != "dense" or self.mask_grad_with_fwd
        if sparse_any and self.activation != "squared_relu":
            raise ConfigError("sparse modes are defined only for squared_relu")
        if self.backward_mode != "dense" and self.forward_mode != "sparse24":
            raise ConfigError("sparse backward modes need the sparse forward")
        if self.mask_grad_with_fwd and self.forward_mode != "sparse24":
            raise ConfigError("mask_grad_with_fwd needs the sparse forward")
        if not 0.0 <= self.split_ratio <= 1.0:
            raise ConfigError(f"split_ratio must be in [0, 1], got {self.split_ratio}")
        if self.fp8_backward and not self.fp8_emulation:
            raise ConfigError("fp8_backward requires fp8_emulation")

    def densified(self) -> "FfnConfig":
        """Same config with every sparsity feature off (ref ffn.py:93-101)."""
        return replace(self, forward_mode="dense", backward_mode="dense", mask_grad_with_fwd=False,
                       permute_tokens=False)


RECIPE = FfnConfig(forward_mode="sparse24", backward_mode="split_masked", mask_grad_with_fwd=True,
                   permute_tokens=True)


@dataclass(frozen=True)
class FfnParams:
    """w1 [d, h], w2 [h, d] (ref ffn.py:104-126), held as bf16 device tensors.
    Both GEMM orientations read the weights in place (no transposed copies)."""

    w1: torch.Tensor
    w2: torch.Tensor
    w3: torch.Tensor | None = None
    beta: float = 1.0

    def __post_init__(self):
        w1 = as_matrix(self.w1, "w1", BF16)
        w2 = as_matrix(self.w2, "w2", BF16)
        object.__setattr__(self, "w1", w1)
        object.__setattr__(self, "w2", w2)
        d, h = w1.shape
        if tuple(w2.shape) != (h, d):
            raise DimensionError(f"w2 shape {tuple(w2.shape)} does not match w1 {tuple(w1.shape)}")
        if h % 4 != 0:
            raise DimensionError(f"hidden width must be a multiple of 4, got {h}")
        if self.w3 is not None:
            w3 = as_matrix(self.w3, "w3", BF16)
            if tuple(w3.shape) != (d, h):
                raise DimensionError(f"w3 shape {tuple(w3.shape)} does not match w1 {tuple(w1.shape)}")
            object.__setattr__(self, "w3", w3)

    @property
    def model_dim(self) -> int:
        return self.w1.shape[0]

    @property
    def hidden_dim(self) -> int:
        return self.w1.shape[1]


@dataclass(frozen=True)
class GemmEvent:
    name: str
    sparse: bool
    macs: int


@dataclass
class FfnCache:
    """What the backward reads (ref ffn.py:136-150), kept compressed.

    x_in      bf16 [pad128(n), d] compute-frame input (zero padding rows)
    act_vals  bf16 [pad128(n), h/2] kept relu^2 values (sparse forward)
    act_meta  uint8 hw metadata of the forward keep pattern
    act_dense bf16 [n, h] activation (dense forward only)
    pre_act   fp32 [n, h] pre-activation, kept only when the backward needs
              relu(y1) outside the keep mask (mask_grad_with_fwd=False) or the
              caller asked for it (keep_pre_act, parity checks)
    perm / inv_dev : the permutation and its inverse (int32 device tensors)

    The split plan, x_in's permuted copy and the feature-wise split of act are
    produced on a side stream next to fwd.out; `plan` and `x_in` make the
    caller's current stream wait for that work before handing them out, so
    reading them right after ffn_forward is safe. The backward uses the raw
    fields and joins the side stream only where it consumes them.
    """

    n: int
    config: FfnConfig
    census: list[GemmEvent]
    _x_in: torch.Tensor | None = None
    act_vals: torch.Tensor | None = None
    act_meta: torch.Tensor | None = None
    act_dense: torch.Tensor | None = None
    pre_act: torch.Tensor | None = None
    perm_dev: torch.Tensor | None = None
    inv_dev: torch.Tensor | None = None
    _plan: SplitPlan | None = None
    stats: SparsifyStats | None = None
    counts: torch.Tensor | None = None
    stats_dev: torch.Tensor | None = None  # int64 [3]: K1's nonzeros before / after, NaN-kept flag
    act_split: FeatureSplit | None = None  # feature-wise split of act (K4, run next to fwd.out)
    side_ready: object = None  # CUDA event after which the side-stream work of the forward is complete
    # fp8_emulation (fp8.py): act_vals holds the dequantized activation (the
    # reference's act_sparse); K3 recovers relu(y1) from the unquantized one
    act_raw: torch.Tensor | None = None
    act_meta8: torch.Tensor | None = None  # act metadata in the e4m3 operand-E layout
    act_f32: torch.Tensor | None = None  # dense fp8 forward: the fp32 activation
    f8: dict | None = None  # e4m3 backward operands prepared next to the forward GEMMs (fp8.py)
    # padded FFN (model dim % 32 or hidden width % 128 != 0, see ffn_forward):
    # this cache is the caller's view of d_valid x h_valid features; `core` is
    # the device cache of the zero-padded FFN the backward runs on. On a core
    # cache, plan_valid is the plan of the real features (_plan: the padded one).
    core: "FfnCache | None" = None
    d_valid: int | None = None
    h_valid: int | None = None
    plan_valid: SplitPlan | None = None

    def _join(self) -> None:
        if self.side_ready is not None:
            torch.cuda.current_stream().wait_event(self.side_ready)

    @property
    def x_in(self) -> torch.Tensor | None:
        self._join()
        return self._x_in

    @property
    def plan(self) -> SplitPlan | None:
        self._join()
        return self._plan

    @property
    def perm(self) -> torch.Tensor | None:
        return self.perm_dev

    # Side-stream work of the forward reads and writes tensors allocated on
    # the main stream (no record_stream: its deferred frees stall the caching
    # allocator). The backward joins that work before its first use; a cache
    # dropped without a backward joins it here, so the memory is never handed
    # to new main-stream work while the side stream still uses it.
    def __del__(self):
        try:
            if self.side_ready is not None and torch.cuda.is_initialized():
                torch.cuda.current_stream(self.side_ready_device).wait_event(self.side_ready)
        except Exception:  # interpreter shutdown
            pass

    @property
    def side_ready_device(self):
        t = self.act_vals if self.act_vals is not None else self._x_in
        return t.device if t is not None else None

    @property
    def act_sparse(self) -> Sparse24Matrix | None:
        """The compressed activation in the compute frame (ref FfnCache.act_sparse)."""
        if self.act_vals is None:
            return None
        h = self.act_vals.shape[1] * 2
        if self.core is not None and self.h_valid != h:
            # padded hidden width: the first h_valid features (whole groups of 4)
            full = self.core.act_sparse
            hv = self.h_valid
            return Sparse24Matrix(self.n, hv, TOKEN_WISE, full.data[:, : hv // 2].contiguous(), None,
                                  meta_ref_cache=full.meta[:, : hv // 4].contiguous())
        return Sparse24Matrix(self.n, h, TOKEN_WISE, self.act_vals, self.act_meta)

    @property
    def fwd_mask(self) -> torch.Tensor | None:
        s = self.act_sparse
        if s is None:
            return None
        m = torch.zeros(self.n, s.cols // 4, 4, dtype=torch.bool, device=self.act_vals.device)
        m.scatter_(2, s.meta.long(), True)
        return m.view(self.n, s.cols)


@dataclass
class FfnGrads:
    d_w1: torch.Tensor
    d_w2: torch.Tensor
    d_x: torch.Tensor
    d_w3: torch.Tensor | None = None
    census: list[GemmEvent] = field(default_factory=list)
    stats_act: SparsifyStats | None = None  # feature-wise drops of the act split (dW2)
    stats_grad: SparsifyStats | None = None  # feature-wise drops of the g_pre split (dW1)
    # diagnostic views (parity checks): g_pre as K3 stored it (token-wise, on
    # the forward metadata, compute frame; built on first read for a padded
    # FFN) and the feature-wise split of it the dW1 GEMM consumed (the act
    # split is FfnCache.act_split)
    _g_pre: object = None
    g_split: FeatureSplit | None = None

    @property
    def g_pre_sparse(self) -> Sparse24Matrix | None:
        if callable(self._g_pre):
            self._g_pre = self._g_pre()
        return self._g_pre


def act_squared_relu(pre):
    """relu(pre)^2 (ref ffn.py:167-169)."""
    r = torch.clamp_min(pre, 0)
    return r * r


def act_squared_relu_grad(pre):
    """2 relu(pre) (ref ffn.py:172-173)."""
    return 2 * torch.clamp_min(pre, 0)


def _unsupported(cfg: FfnConfig) -> None:
    if cfg.activation != "squared_relu":
        raise ConfigError("the B200 backend implements the squared_relu FFN only (SwiGLU is the "
                          "reference's dense Table-1 baseline, out of scope)")


def _check_dims(n: int, d: int, h: int) -> None:
    if d % 32 != 0:
        raise DimensionError(f"model dim {d} must be a multiple of 32 on the device path (GEMM N tiles)")
    if h % 128 != 0:
        raise DimensionError(f"hidden width {h} must be a multiple of 128 on the device path")


def _pad_to(v: int, m: int) -> int:
    return (v + m - 1) // m * m


def _pad_cols(a: torch.Tensor, cols: int) -> torch.Tensor:
    if a.shape[1] == cols:
        return a
    out = torch.zeros(a.shape[0], cols, dtype=a.dtype, device=a.device)
    out[:, : a.shape[1]] = a
    return out


def _pad_params(p: FfnParams, dp: int, hp: int) -> FfnParams:
    d, h = p.model_dim, p.hidden_dim
    w1 = torch.zeros(dp, hp, dtype=BF16, device=p.w1.device)
    w1[:d, :h] = p.w1
    w2 = torch.zeros(hp, dp, dtype=BF16, device=p.w2.device)
    w2[:h, :d] = p.w2
    w3 = None
    if p.w3 is not None:
        w3 = torch.zeros(dp, hp, dtype=BF16, device=p.w3.device)
        w3[:d, :h] = p.w3
    return FfnParams(w1, w2, w3, p.beta)


def _plan_split(counts, ratio: float, plan: SplitPlan | None, h: int, h_valid: int | None, launch_stream=None):
    """(plan of the real features, device plan of all h features): computed
    from K1's counts (plan None) or the caller's plan, padded when h_valid < h."""
    if plan is None:
        if h_valid is None:
            pl = partition_features(counts, ratio, launch_stream=launch_stream)
            return pl, pl
        return partition_features_padded(counts, ratio, h_valid, launch_stream)
    return plan, pad_plan(plan, h, launch_stream)


def ffn_forward(x, p: FfnParams, cfg: FfnConfig, plan: SplitPlan | None = None, keep_pre_act: bool = False,
                for_backward: bool = True, counts_hook=None):
    """Run the forward pass; returns (out [n, d] bf16, FfnCache) (ref ffn.py:276-363).
    keep_pre_act=True also stores the fp32 pre-activation in the cache (parity
    tests use it to replay the selection on identical inputs). for_backward=False
    (inference prefill) skips what only the backward needs: the token
    permutation (every forward stage maps one token row to one output row, so
    the output is the same bits), x_in and the feature-wise split.
    counts_hook(counts): called right after K1 with the int32 per-feature
    nonzero counts, before the split plan is computed from them, with the
    side stream that computes the plan current: data parallelism all-reduces
    them here (every rank then uses the plan of the global batch) while fwd.out
    runs on the caller's stream.

    Any d and h % 4 == 0 (the reference's shapes): the device GEMMs tile the
    model dim by 32 and the hidden width by 128, so other sizes run on the FFN
    zero-padded to those multiples. Padding features have zero pre-activation
    (no kept values, count 0) and are appended to the plan's sparse list after
    the real ones, so the real features' selection, plan, statistics, outputs
    and gradients are those of the unpadded FFN."""
    require_cuda()
    _unsupported(cfg)
    x = as_matrix(x, "x", BF16)
    d, h = p.model_dim, p.hidden_dim
    dp, hp = _pad_to(d, 32), _pad_to(h, 128)
    if (dp, hp) == (d, h):
        return _ffn_forward(x, p, cfg, plan, keep_pre_act, for_backward, counts_hook=counts_hook)
    if x.shape[1] != d:
        raise DimensionError(f"input width {x.shape[1]} does not match w1 {tuple(p.w1.shape)}")
    if plan is not None and plan.hidden_dim != h:
        raise DimensionError(f"plan built for {plan.hidden_dim} features, FFN has {h}")
    hook = None if counts_hook is None else (lambda c: counts_hook(c[:h]))
    out, core = _ffn_forward(_pad_cols(x, dp), _pad_params(p, dp, hp), cfg, plan, keep_pre_act, for_backward,
                             h_valid=h, counts_hook=hook)
    n = core.n
    stats = None
    if core.stats is not None:
        def real_feature_stats():
            # nonzeros before / after over the real features (the padding
            # features are zero unless the input carries NaN / Inf)
            before = core.counts[:h].sum(dtype=torch.int64)
            vals = core.act_vals[:n].view(n, hp // 4, 2)[:, : h // 4]
            return torch.stack([before, (vals != 0).sum(dtype=torch.int64)])

        stats = SparsifyStats(n * h, real_feature_stats if hp != h else core.stats._dev)
    view = replace(core, pre_act=core.pre_act[:, :h] if core.pre_act is not None else None,
                   counts=core.counts[:h] if core.counts is not None else None,
                   _plan=core.plan_valid if core.plan_valid is not None else core._plan,
                   stats=stats,
                   census=_census_real(core.census, n, d, h, core.plan_valid, cfg),
                   core=core, d_valid=d, h_valid=h, plan_valid=None)
    return (out[:, :d].contiguous() if dp != d else out), view


def _census_real(events, n: int, d: int, h: int, plan: SplitPlan | None, cfg: FfnConfig) -> list:
    """The GEMM census of a padded run restated at the real (n, d, h)."""
    out = []
    for ev in events:
        if ev.name in ("bwd.d_w2", "bwd.d_w1") and ev.sparse:
            m = split_gemm_macs(n, d, plan) if (cfg.backward_mode == "split_masked" and plan is not None) \
                else sp_gemm_macs(n, h, d)
        else:
            m = sp_gemm_macs(n, h, d) if ev.sparse else gemm_macs(n, d, h)
        out.append(GemmEvent(ev.name, ev.sparse, m))
    return out


def _all_sparse_plan(h: int, dev) -> SplitPlan:
    """naive_sparse: every feature feature-wise 2:4 (ref ffn.py:430-437)."""
    pos = torch.arange(h, dtype=torch.int32, device=dev)
    return SplitPlan(h, 1.0, torch.zeros(h, dtype=torch.int64, device=dev), pos,
                     torch.empty(0, dtype=torch.int32, device=dev), pos)


def _frame_rows(a: torch.Tensor, npad: int, src_rows, fill: bool = True) -> torch.Tensor:
    """The compute-frame copy of a [n, d] input: rows permuted (out[i] =
    a[src_rows[i]]) and zero-padded to npad rows. Returns `a` itself when
    neither applies. fill=False only allocates (fill with _fill_frame_rows)."""
    n = a.shape[0]
    if src_rows is None and npad == n:
        return a
    out = torch.empty(npad, a.shape[1], dtype=a.dtype, device=a.device)
    if fill:
        _fill_frame_rows(out, a, src_rows)
    return out


def _fill_frame_rows(out: torch.Tensor, a: torch.Tensor, src_rows) -> None:
    """Fill a _frame_rows buffer on the current stream (K6 gather or copy)."""
    n = a.shape[0]
    if out.shape[0] > n:
        out[n:].zero_()
    if src_rows is not None:
        gather_rows(a, src_rows, out)
    else:
        out[:n].copy_(a)


def _ffn_forward(x, p: FfnParams, cfg: FfnConfig, plan: SplitPlan | None, keep_pre_act: bool, for_backward: bool,
                 h_valid: int | None = None, counts_hook=None):
    """ffn_forward on device-tileable sizes (d % 32 == 0, h % 128 == 0).
    h_valid: the FFN is zero-padded beyond its first h_valid features."""
    require_cuda()
    _unsupported(cfg)
    x = as_matrix(x, "x", BF16)
    n, d = x.shape
    if d != p.model_dim:
        raise DimensionError(f"input width {d} does not match w1 {tuple(p.w1.shape)}")
    if (p.w3 is not None) != (cfg.activation == "swiglu"):
        raise ConfigError("gate weight w3 must be present exactly for swiglu")
    sparse_fwd = cfg.forward_mode == "sparse24"
    if sparse_fwd and n % 4 != 0:
        raise DimensionError(f"sparse modes need token count % 4 == 0, got {n}")
    h = p.hidden_dim
    _check_dims(n, d, h)
    if plan is not None and plan.hidden_dim != (h_valid or h):
        raise DimensionError(f"plan built for {plan.hidden_dim} features, FFN has {h_valid or h}")
    if cfg.fp8_emulation:
        # e4m3 operands on the kind::f8f6f4 tensor cores (fp8.py)
        from .fp8 import ffn_forward_f8

        return ffn_forward_f8(x, p, cfg, plan, keep_pre_act, for_backward, h_valid=h_valid,
                              counts_hook=counts_hook)
    dev = x.device
    s = stream()
    npad = pad128(n)
    census: list[GemmEvent] = []

    out = torch.empty(n, d, dtype=BF16, device=dev)
    if not sparse_fwd:
        # ------------------------------------------------------------ dense twin
        act = torch.empty(n, h, dtype=BF16, device=dev)
        _lib.call("s24_gemm_relu2", ptr(x), d, ptr(p.w1), h, n, h, d, ptr(act), h, s)
        census.append(GemmEvent("fwd.pre_act", False, gemm_macs(n, d, h)))
        _lib.call("s24_gemm", ptr(act), 0, h, ptr(p.w2), 1, d, n, d, h, ptr(out), _lib.BF16, d, None, 0, -1, None, s)
        census.append(GemmEvent("fwd.out", False, gemm_macs(n, h, d)))
        x_in = _frame_rows(x, npad, None) if for_backward else None
        return out, FfnCache(n, cfg, census, _x_in=x_in, act_dense=act)

    # The compute frame is the token-permuted order (ref ffn.py:297-303). The
    # permutation only shapes the feature-wise groups of the backward, so an
    # inference forward skips it.
    perm_dev = inv_dev = None
    if cfg.permute_tokens and for_backward:
        perm_dev, inv_dev = device_permutation(cfg.permute_seed, n, dev)
    act_vals = torch.empty(npad, h // 2, dtype=BF16, device=dev)
    act_meta = torch.empty(_lib.meta_hw_bytes(n, h), dtype=torch.uint8, device=dev)
    if npad > n:
        act_vals[n:].zero_()
        act_meta[(n // 128) * (h // 128) * 2048:].fill_(0x44)
    counts = torch.zeros(h, dtype=torch.int32, device=dev)
    stats_dev = torch.zeros(3, dtype=torch.int64, device=dev)
    need_pre = keep_pre_act or not cfg.mask_grad_with_fwd
    pre = torch.empty(n, h, dtype=F32, device=dev) if need_pre else None
    # K1 reads the permuted copy x_in (K6 gather on the main stream); without
    # a permutation x itself, and the padded copy the dW1 GEMM reads is made on
    # the side stream
    x_in = None
    k1_in = x
    if perm_dev is not None:
        x_in = k1_in = _frame_rows(x, npad, inv_dev)
    elif for_backward:
        x_in = _frame_rows(x, npad, None, fill=False)
    _lib.call("s24_fwd_gemm1_fused", ptr(k1_in), d, ptr(p.w1), h, n, h, d, ptr(act_vals), ptr(act_meta),
              ptr(counts), ptr(stats_dev), ptr(pre), s)
    census.append(GemmEvent("fwd.pre_act", False, gemm_macs(n, d, h)))

    # fwd.out on tensor cores (inverse permutation as its epilogue row map)
    # and next to it, on the side stream: the split plan (K7, one small CTA
    # that fits beside a GEMM CTA), x_in's padded copy and -- when the
    # backward will need it -- K4, the feature-wise split of act. Their
    # outputs are allocated here, on the main stream.
    main = torch.cuda.current_stream()
    side = side_stream(dev)
    side.wait_stream(main)
    if counts_hook is not None:
        with torch.cuda.stream(side):  # (a collective here overlaps fwd.out)
            counts_hook(counts)
    _lib.call("s24_spmm", ptr(act_vals), ptr(act_meta), ptr(p.w2), 1, d, n, d, h, ptr(out), _lib.BF16, d,
              ptr(inv_dev), 0, -1, None, 0, s)
    census.append(GemmEvent("fwd.out", True, sp_gemm_macs(n, h, d)))
    plan_api = plan_out = plan
    if cfg.backward_mode == "split_masked" or plan is not None:
        plan_api, plan_out = _plan_split(counts, cfg.split_ratio, plan, h, h_valid, side)
    act_split = None
    split = for_backward and cfg.backward_mode != "dense"
    bplan = plan_out if cfg.backward_mode == "split_masked" else _all_sparse_plan(h, dev)
    if split:
        act_split = alloc_feature_split(act_vals, act_meta, npad, h, bplan)
    with torch.cuda.stream(side):
        if split:
            bplan.paired_row_map  # (the weight-gradient row map, built on the side stream)
        if x_in is not None and x_in is not k1_in and x_in is not x:
            _fill_frame_rows(x_in, x, None)
        if split:  # (relu^2: >= 0; NaN-aware only if K1 kept a NaN)
            run_feature_split(act_split, act_vals, act_meta, npad, h, bplan, nonneg=True, nan_flag=stats_dev[2:])
        ev = torch.cuda.Event()
        ev.record(side)
    if not for_backward:
        main.wait_event(ev)  # (inference: no backward will join the side stream)
        ev = None
    if x_in is None and for_backward:
        x_in = x
    cache = FfnCache(n, cfg, census, _x_in=x_in, act_vals=act_vals, act_meta=act_meta, pre_act=pre,
                     perm_dev=perm_dev, inv_dev=inv_dev, _plan=plan_out, stats=SparsifyStats(n * h, stats_dev[:2]),
                     counts=counts, stats_dev=stats_dev, act_split=act_split, side_ready=ev,
                     plan_valid=plan_api if h_valid is not None else None)
    return out, cache


def weight_grad_buffers(d: int, h: int, dev, bucket: torch.Tensor | None = None):
    """(d_w1 [d, h], d_w2 [h, d]) fp32: fresh tensors, or views into bucket."""
    if bucket is None:
        return torch.empty(d, h, dtype=F32, device=dev), torch.empty(h, d, dtype=F32, device=dev)
    if bucket.dtype != F32 or bucket.numel() != 2 * d * h or not bucket.is_contiguous():
        raise DimensionError(f"grad_bucket must be a contiguous fp32 buffer of {2 * d * h} elements")
    return bucket[: d * h].view(d, h), bucket[d * h:].view(h, d)


def ffn_backward(g_out, cache: FfnCache, p: FfnParams, cfg: FfnConfig, grad_ready=None,
                 grad_bucket: torch.Tensor | None = None) -> FfnGrads:
    """Backward matching the cached forward (ref ffn.py:366-451).

    grad_ready(name, tensor), if given, is called as soon as d_w2 and then
    d_w1 are final on the current stream (the data-parallel step launches
    their all-reduce there). The recipe runs dW2 right after K3, then dX and
    dW1, so that dW2's all-reduce overlaps the rest of the backward.
    grad_bucket: optional fp32 buffer of 2*d*h elements; d_w1 and d_w2 are then
    written as views into it ([d_w1 | d_w2]), so one collective covers both.
    A padded forward (see ffn_forward) runs the padded backward and returns
    the gradients of the real d x h parameters."""
    if cache.core is None:
        gr = _ffn_backward(g_out, cache, p, cfg, grad_ready, grad_bucket)
        gr.stats_act, gr.stats_grad = (_token_total(st, cache.n, 0) for st in (gr.stats_act, gr.stats_grad))
        return gr
    if cache.config != cfg:
        raise StateError("cache was produced under a different configuration")
    d, h, n = cache.d_valid, cache.h_valid, cache.n
    if (p.model_dim, p.hidden_dim) != (d, h):
        raise DimensionError(f"parameters {tuple(p.w1.shape)} do not match the cached FFN {(d, h)}")
    g_out = as_matrix(g_out, "g_out", BF16)
    if tuple(g_out.shape) != (n, d):
        raise StateError(f"gradient shape {tuple(g_out.shape)} does not match cached input {(n, d)}")
    dp, hp = _pad_to(d, 32), _pad_to(h, 128)
    gr = _ffn_backward(_pad_cols(g_out, dp), cache.core, _pad_params(p, dp, hp), cfg)
    d_w1, d_w2 = weight_grad_buffers(d, h, g_out.device, grad_bucket)
    notify = grad_ready or (lambda name, t: None)
    d_w2.copy_(gr.d_w2[:h, :d])
    notify("d_w2", d_w2)
    d_w1.copy_(gr.d_w1[:d, :h])
    notify("d_w1", d_w1)
    d_x = gr.d_x[:, :d].contiguous() if dp != d else gr.d_x

    def g_pre_view():  # (diagnostic: the real features of the padded FFN's stored g_pre)
        full = gr.g_pre_sparse
        if full is None:
            return None
        if hp == h:
            return full
        return Sparse24Matrix(n, h, TOKEN_WISE, full.data[:, : h // 2].contiguous(), None,
                              meta_ref_cache=full.meta[:, : h // 4].contiguous())

    return FfnGrads(d_w1, d_w2, d_x, None, _census_real(gr.census, n, d, h, cache._plan, cfg),
                    _token_total(gr.stats_act, n, hp - h), _token_total(gr.stats_grad, n, hp - h), g_pre_view)


def _token_total(st: SparsifyStats | None, n: int, pad_features: int) -> SparsifyStats | None:
    """Feature-wise split statistics over the caller's n tokens and real
    features: the device splits count pad128(n) token rows (zero padding rows)
    and, in a padded FFN, pad_features all-zero features; the reference's
    total is n x (sparse features) (ref splitgemm.py:75, sparse24.py:50-69)."""
    if st is None:
        return None
    return SparsifyStats(st.total_entries // pad128(n) * n - n * pad_features, st._dev)


def _ffn_backward(g_out, cache: FfnCache, p: FfnParams, cfg: FfnConfig, grad_ready=None,
                  grad_bucket: torch.Tensor | None = None) -> FfnGrads:
    """ffn_backward on a device-tileable cache (see _ffn_forward)."""
    if cache.config != cfg:
        raise StateError("cache was produced under a different configuration")
    _unsupported(cfg)
    n = cache.n
    x_in = cache._x_in
    if x_in is None:
        raise StateError("cache comes from an inference forward (for_backward=False)")
    d = x_in.shape[1]
    g_out = as_matrix(g_out, "g_out", BF16)
    if tuple(g_out.shape) != (n, d):
        raise StateError(f"gradient shape {tuple(g_out.shape)} does not match cached input {(n, d)}")
    sparse_fwd = cfg.forward_mode == "sparse24"
    if sparse_fwd and cache.act_vals is None:
        raise StateError("sparse forward cache is missing the compressed activation")
    if not sparse_fwd and cache.act_dense is None:
        raise StateError("dense forward cache is missing the activation")
    if cfg.backward_mode == "split_masked" and cache._plan is None:
        raise StateError("split backward needs the plan computed in forward")
    h = p.hidden_dim
    if cfg.fp8_backward:
        from .fp8 import ffn_backward_f8

        return ffn_backward_f8(g_out, cache, p, cfg, grad_ready, grad_bucket)
    dev = g_out.device
    s = stream()
    npad = pad128(n)
    census: list[GemmEvent] = []
    notify = grad_ready or (lambda name, t: None)
    d_w1, d_w2 = weight_grad_buffers(d, h, dev, grad_bucket)
    d_x = torch.empty(n, d, dtype=BF16, device=dev)
    main = torch.cuda.current_stream()

    if not sparse_fwd:
        # ------------------------------------------------------------ dense twin
        act = cache.act_dense
        g_pre = torch.empty(n, h, dtype=BF16, device=dev)
        _lib.call("s24_gemm_dact", ptr(g_out), d, ptr(p.w2), d, n, h, d, ptr(act), h, ptr(g_pre), h, s)
        census.append(GemmEvent("bwd.d_act", False, gemm_macs(n, d, h)))
        _lib.call("s24_gemm", ptr(act), 1, h, ptr(g_out), 1, d, h, d, n, ptr(d_w2), _lib.F32, d, None, 0, -1, None, s)
        census.append(GemmEvent("bwd.d_w2", False, gemm_macs(h, n, d)))
        notify("d_w2", d_w2)
        _lib.call("s24_gemm", ptr(g_pre), 1, h, ptr(x_in), 1, d, h, d, n, ptr(d_w1), _lib.F32, h, None, 1, -1, None, s)
        census.append(GemmEvent("bwd.d_w1", False, gemm_macs(d, n, h)))
        notify("d_w1", d_w1)
        _lib.call("s24_gemm", ptr(g_pre), 0, h, ptr(p.w1), 0, h, n, d, h, ptr(d_x), _lib.BF16, d, None, 0, -1, None, s)
        census.append(GemmEvent("bwd.d_x", False, gemm_macs(n, h, d)))
        return FfnGrads(d_w1, d_w2, d_x, None, census)

    # -------------------------------------------------------------- sparse forward
    # g_c = permute_rows(dY) padded to npad rows: K3's A operand and dW2's B
    g_c = _frame_rows(g_out, npad, cache.inv_dev)
    # K3: g_pre on the forward keep pattern, compressed (exact; ref ffn.py:415-417, 443)
    g_vals = torch.empty(npad, h // 2, dtype=BF16, device=dev)
    if npad > n:
        g_vals[n:].zero_()
    # (fp8 forward: relu(y1) comes from the unquantized activation)
    k3_act = cache.act_raw if cache.act_raw is not None else cache.act_vals
    _lib.call("s24_bwd_dact_fused", ptr(g_c), d, ptr(p.w2), d, n, h, d, ptr(k3_act), ptr(cache.act_meta),
              ptr(g_vals), s)
    census.append(GemmEvent("bwd.d_act", False, gemm_macs(n, d, h)))
    g_pre_dense = None
    if not cfg.mask_grad_with_fwd:
        # unmasked derivative: needs relu(y1) everywhere (fp32 pre-activation kept by the forward)
        G = torch.empty(n, h, dtype=F32, device=dev)
        _lib.call("s24_gemm", ptr(g_c), 0, d, ptr(p.w2), 0, d, n, h, d, ptr(G), _lib.F32, h, None, 0, -1, None, s)
        G *= act_squared_relu_grad(cache.pre_act)  # g_pre in fp32 (the reference's precision)
        g_pre_dense = G.to(BF16)

    mode = cfg.backward_mode
    if mode == "dense":
        if cache.side_ready is not None:
            main.wait_event(cache.side_ready)
        act = torch.empty(n, h, dtype=BF16, device=dev)
        _lib.call("s24_decompress_token", ptr(cache.act_vals), None, ptr(cache.act_meta), n, h, ptr(act), _lib.BF16, h, s)
        gp = g_pre_dense
        if gp is None:
            gp = torch.empty(n, h, dtype=BF16, device=dev)
            _lib.call("s24_decompress_token", ptr(g_vals), None, ptr(cache.act_meta), n, h, ptr(gp), _lib.BF16, h, s)
        _dx(cfg, g_vals, g_pre_dense, cache, p, d_x, n, d, h, s, census)
        _lib.call("s24_gemm", ptr(act), 1, h, ptr(g_c), 1, d, h, d, n, ptr(d_w2), _lib.F32, d, None, 0, -1, None, s)
        census.insert(1, GemmEvent("bwd.d_w2", False, gemm_macs(h, n, d)))
        notify("d_w2", d_w2)
        _lib.call("s24_gemm", ptr(gp), 1, h, ptr(x_in), 1, d, h, d, n, ptr(d_w1), _lib.F32, h, None, 1, -1, None, s)
        census.insert(2, GemmEvent("bwd.d_w1", False, gemm_macs(d, n, h)))
        notify("d_w1", d_w1)
        return FfnGrads(d_w1, d_w2, d_x, None, census)

    # split_masked / naive_sparse: the weight gradients are feature-wise 2:4
    # GEMMs over the split operands (K4 in the paired layout)
    plan = _all_sparse_plan(h, dev) if mode == "naive_sparse" else cache._plan
    macs_w = sp_gemm_macs(n, h, d) if mode == "naive_sparse" else split_gemm_macs(n, d, plan)
    fa = cache.act_split
    if fa is None:
        raise StateError("cache is missing the feature-wise split of the activation")
    raw_naive = mode == "naive_sparse" and not cfg.mask_grad_with_fwd
    side = side_stream(dev)
    if raw_naive:
        # naive_sparse without the mask sparsifies the raw g_pre feature-wise
        # (ref ffn.py:430-437); the split path always sees the masked g_pre
        from .sparse24 import sparsify_feature_wise

        # (the selection ranks the fp32 g_pre, as the reference does; a bf16
        # copy would turn near-ties into ties that break toward lower tokens)
        gpad = torch.zeros(npad, h, dtype=F32, device=dev)
        gpad[:n] = G
        sg, _, stats_g = sparsify_feature_wise(gpad)
        _dx(cfg, g_vals, g_pre_dense, cache, p, d_x, n, d, h, s, census)
        main.wait_event(cache.side_ready)
        split_weight_grad(fa, plan, g_c, npad, d_w2, transposed=False)
        census.insert(1, GemmEvent("bwd.d_w2", True, macs_w))
        notify("d_w2", d_w2)
        _lib.call("s24_spmm", ptr(sg.data), ptr(sg.meta_hw), ptr(x_in), 1, d, h, d, npad, ptr(d_w1), _lib.F32, h,
                  None, 1, -1, None, 0, s)
        census.insert(2, GemmEvent("bwd.d_w1", True, macs_w))
        notify("d_w1", d_w1)
        return FfnGrads(d_w1, d_w2, d_x, None, census, fa.stats, stats_g)

    # K4 of g_pre on a second side stream (not queued behind the forward's
    # K4 of act), next to the next main-stream GEMM
    fg = alloc_feature_split(g_vals, cache.act_meta, npad, h, plan)
    side = side_stream(dev, 1)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        run_feature_split(fg, g_vals, cache.act_meta, npad, h, plan)
        ev_g = torch.cuda.Event()
        ev_g.record(side)
    # dW2 first (it needs only the forward's split of act, ready long before),
    # with K4(g_pre) next to it. Alone: dX, then dW1, so K4(g_pre) has two
    # GEMMs to hide under. With a grad_ready hook (data parallel): dW1 before
    # dX, so both weight-gradient all-reduces overlap compute (dW2's overlaps
    # dW1 and dX, dW1's overlaps dX) instead of dW1's trailing the step. On one
    # GPU the two orders take the same time (1.837 vs 1.844 ms median, 1.814
    # both min, 16 interleaved blocks, scripts/ab_step.py); K4(g_pre) ends
    # before dW2 does (profiles/r02/timeline_queued_c2.txt).
    main.wait_event(cache.side_ready)
    split_weight_grad(fa, plan, g_c, npad, d_w2, transposed=False)
    notify("d_w2", d_w2)
    if grad_ready is not None:
        main.wait_event(ev_g)
        split_weight_grad(fg, plan, x_in, npad, d_w1, transposed=True)
        notify("d_w1", d_w1)
        _dx(cfg, g_vals, g_pre_dense, cache, p, d_x, n, d, h, s, census)
    else:
        _dx(cfg, g_vals, g_pre_dense, cache, p, d_x, n, d, h, s, census)
        main.wait_event(ev_g)
        split_weight_grad(fg, plan, x_in, npad, d_w1, transposed=True)
        notify("d_w1", d_w1)
    census.insert(1, GemmEvent("bwd.d_w2", True, macs_w))
    census.insert(2, GemmEvent("bwd.d_w1", True, macs_w))
    return FfnGrads(d_w1, d_w2, d_x, None, census, fa.stats, fg.stats,
                    Sparse24Matrix(n, h, TOKEN_WISE, g_vals, cache.act_meta), fg)


def _dx(cfg, g_vals, g_pre_dense, cache, p, d_x, n, d, h, s, census) -> None:
    """bwd.d_x: the 2:4 GEMM on g_pre's forward keep pattern (exact, ref
    ffn.py:440-445), or dense on the unmasked derivative (:446-447); the
    inverse permutation is its epilogue row map."""
    if cfg.mask_grad_with_fwd:
        _lib.call("s24_spmm", ptr(g_vals), ptr(cache.act_meta), ptr(p.w1), 0, h, n, d, h, ptr(d_x), _lib.BF16, d,
                  ptr(cache.inv_dev), 0, -1, None, 0, s)
        census.append(GemmEvent("bwd.d_x", True, sp_gemm_macs(n, h, d)))
    else:
        _lib.call("s24_gemm", ptr(g_pre_dense), 0, h, ptr(p.w1), 0, h, n, d, h, ptr(d_x), _lib.BF16, d,
                  ptr(cache.inv_dev), 0, -1, None, s)
        census.append(GemmEvent("bwd.d_x", False, gemm_macs(n, h, d)))
