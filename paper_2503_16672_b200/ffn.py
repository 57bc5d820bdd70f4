"""Squared-ReLU FFN with the 2:4 activation-sparsity recipe on B200 -- drop-in
for the reference's pkg/src/srelu24/ffn.py (ffn_forward / ffn_backward and
their dataclasses; activation = squared_relu).

Recipe forward (ref ffn.py:276-363), one device pass each:
  K1  Y1 = x . W1 -> relu^2 -> token-wise 2:4          (tcgen05 GEMM, fused epilogue:
      compressed act + hw metadata + per-feature counts + drop stats; input row
      r is written as act row perm[r], i.e. permute_rows folded into the store)
  K2  out = inverse_permute_rows(act_sp . W2)          (tcgen05.mma.sp, row map epilogue)
  side stream, next to K2:
  K7  plan = partition_features(counts, ratio)         (device radix select)
  K6  x_in = permute_rows(x, perm)                     (row gather, dW1 operand)
  K4  feature-wise 2:4 split of act (sparse features) + dense columns
Recipe backward (ref ffn.py:366-451):
  K3  g_pre = (dY . W2^T) * 2 relu(y1) on the forward keep pattern (fused,
      compressed, rows paired with act row perm[r])
  K2  dX = inverse_permute_rows(g_pre_sp . W1^T)       (exact: forward metadata)
  side stream: K6 g_c = permute_rows(dY, perm); K4 split of g_pre (next to dX)
  K5  dW2 = split(act)^T g_c ; dW1 = (split(g_pre)^T x_in)^T  (one grouped sparse
      launch + dense remainders, feature-index scatter / transpose in the epilogue)
Dense mode runs the same GEMM kernels with dense operands (the "dense twin").

Tensors are bf16 on the device (numpy float32 inputs are uploaded and rounded
to bf16). Weight gradients are fp32, activations/outputs bf16.
"""

from __future__ import annotations

import os
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
    FusedFeatureOperand,
    alloc_feature_split,
    k4_job_args,
    run_feature_split,
    side_stream,
    SplitPlan,
    feature_split,
    fused_weight_grad,
    pad_plan,
    partition_features,
    partition_features_padded,
    split_gemm_macs,
    split_weight_grad,
    split_weight_grad_pair,
    run_feature_split_dual,
)

ACTIVATIONS = ("squared_relu", "swiglu")

# Where the feature-wise 2:4 operands of the split weight-gradient GEMMs come
# from: False (default) = the standalone K4 kernel after the plan is known;
# True = fused into the K1 / K3 epilogues for every feature (csrc/fwsel.cuh).
# Both are bit-identical; on B200 the fused variant currently makes the K1/K3
# epilogues the bottleneck, so it is opt-in.
FUSED_FEATURE_SPLIT = os.environ.get("S24_FUSED_FW", "0") == "1"

# How the standalone K4 runs next to the sparse GEMM that precedes its use
# (fwd.out for the activation split, bwd.d_x for the g_pre split):
#   "side"       -- on a side stream, co-resident with the GEMM (the sparse
#                   GEMMs cap their registers to leave room for it)  [default]
#   "background" -- inside the GEMM, in its idle epilogue warps (s24_spmm_bg)
#   "inline"     -- serialized on the main stream
#   "gemm"       -- inside the GEMM, by extra warps that split its own A
#                   pipeline stages (s24_spmm_fs, csrc/k4s.cuh)
K4_MODE = os.environ.get("S24_K4_MODE", "side")
# Both split weight gradients in one grouped sparse launch (s24_spmm_pair)
# when no per-gradient hook needs dW2 early. S24_PAIRED_WGRAD=0 disables.
PAIRED_WEIGHT_GRADS = os.environ.get("S24_PAIRED_WGRAD", "1") == "1"
# Gather the permuted copies x_in / g_c (weight-gradient operands only) on the
# side stream next to the GEMMs ("1") or on the main stream right before
# their first use ("0").
SIDE_GATHERS = os.environ.get("S24_SIDE_GATHERS", "1") == "1"
# K1 / K3 read x / dY unpermuted and apply the permutation as an epilogue row
# map ("1"), or read the gathered copies x_in / g_c ("0").
ROWMAP_GEMMS = os.environ.get("S24_ROWMAP", "0") == "1"
# K3 alone row-mapped (dY read as is; its epilogue reads / writes the act and
# g_pre rows perm[r] with whole-sector stores): the g_c gather leaves the
# critical path for the side stream (dW2's B operand only)
ROWMAP_K3 = os.environ.get("S24_ROWMAP_K3", os.environ.get("S24_ROWMAP", "0")) == "1"
# Feature-wise split in the paired layout: the dense features travel inside
# the 2:4 weight-gradient operand as fixed-selector row pairs, so no dense
# remainder GEMM / split-K reduction runs ("1"); "0": separate dense operand.
PAIRED_DENSE = os.environ.get("S24_PAIRED_DENSE", "1") == "1"
# ... and in the identity layout (coalesced K4, csrc/k4id.cuh): rows in
# feature order after the dense pairs ("1"), or rank order ("0").
IDENTITY_LAYOUT = os.environ.get("S24_IDENTITY_LAYOUT", "0") == "1"
# Where the feature-wise split of act (K4) runs on the side stream: next to
# fwd.out in the forward ("0"), or next to K3 at the start of the backward
# ("1": K3 is tensor/epilogue-bound and leaves room for it, fwd.out is
# operand-feed-bound).
ACT_SPLIT_IN_BWD = os.environ.get("S24_ACT_SPLIT_IN_BWD", "0") == "1"
# One K4 pass for the activation and g_pre together (shared metadata work),
# next to the dX GEMM in the backward ("1"), instead of two passes.
DUAL_K4 = os.environ.get("S24_DUAL_K4", "0") == "1"
# Backward tail order: dW2 on the main stream next to K4(g_pre) on the side
# stream, then dW1 (side, after K4) and dX (third stream, after K3), so each
# persistent GEMM's last partial wave is filled by the next one's CTAs ("1");
# or dX next to K4(g_pre), then both weight gradients in one grouped launch ("0").
WGRAD_OVERLAP = os.environ.get("S24_WGRAD_OVERLAP", "0") == "1"
# Token-order storage ("1"): the recipe's activations stay in the caller's
# token order -- K1 reads x and fwd.out writes out without row maps, K3 reads
# dY and dX is written without one -- and the compute frame's permutation is
# applied only where the backward needs it: inside K4 (row-mapped reads) and
# in the permuted copies x_in / g_c that feed the weight-gradient GEMMs, both
# on the side stream. "0": gather x / dY into the permuted frame before K1 / K3.
# Measured slower on B200 (2.06 vs 1.99 ms at c2: row-mapped K4 reads scatter
# over the whole activation, and the overlapped gathers slow K1 / K3 more than
# the serialized ones cost), so opt-in.
TOKEN_ORDER_STORAGE = os.environ.get("S24_TOKEN_ORDER", "0") == "1"
# Side-stream start in the forward: right after K1 ("0": K4(act) co-runs with
# fwd.out, a 2:4 GEMM) or after fwd.out ("1": K4(act) co-runs with K3, dense).
K4_AFTER_FWD_OUT = os.environ.get("S24_K4_LATE", "0") == "1"


def _dual_k4() -> bool:
    lay = _layout()
    return DUAL_K4 and K4_MODE == "side" and lay["paired"] and not lay["identity"]


def _layout() -> dict:
    """Layout of the feature-wise split operands (see splitgemm.FeatureSplit)."""
    paired = PAIRED_DENSE and K4_MODE != "background"  # the in-GEMM K4 job writes the separate layout
    return {"paired": paired, "identity": paired and IDENTITY_LAYOUT}
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
              relu(y1) outside the keep mask (mask_grad_with_fwd=False)
    perm / perm_dev / inv_dev : host permutation and its device copies
    """

    x_in: torch.Tensor
    n: int
    act_vals: torch.Tensor | None
    act_meta: torch.Tensor | None
    act_dense: torch.Tensor | None
    pre_act: torch.Tensor | None
    perm: object
    perm_dev: torch.Tensor | None
    inv_dev: torch.Tensor | None
    plan: SplitPlan | None
    stats: SparsifyStats | None
    counts: torch.Tensor | None
    census: list[GemmEvent]
    config: FfnConfig
    gate: torch.Tensor | None = None
    act_fw: FusedFeatureOperand | None = None  # feature-wise 2:4 act of all features (from K1)
    act_split: FeatureSplit | None = None  # feature-wise split of act (K4, run during fwd.out)
    act_split_ready: object = None  # CUDA event after which act_split is complete (side-stream K4)
    x_in_ready: object = None  # CUDA event after which x_in is complete (gathered on the side stream)
    # fp8_emulation (fp8.py): act_vals holds the dequantized activation (the
    # reference's act_sparse); K3 recovers relu(y1) from the unquantized one
    act_raw: torch.Tensor | None = None
    act_meta8: torch.Tensor | None = None  # act metadata in the e4m3 operand-E layout
    act_f32: torch.Tensor | None = None  # dense fp8 forward: the fp32 activation
    f8: dict | None = None  # e4m3 backward operands prepared next to the forward GEMMs (fp8.py)
    # token-order storage (TOKEN_ORDER_STORAGE): act_vals / act_meta rows are in
    # the caller's token order; compute-frame token j is storage row row_frame[j]
    row_frame: torch.Tensor | None = None
    # padded FFN (model dim % 32 or hidden width % 128 != 0, see ffn_forward):
    # this cache is the caller's view of d_valid x h_valid features; `core` is
    # the device cache of the zero-padded FFN the backward runs on. On a core
    # cache, plan_valid is the plan of the real features (plan: the padded one).
    core: "FfnCache | None" = None
    d_valid: int | None = None
    h_valid: int | None = None
    plan_valid: SplitPlan | None = None

    # Side-stream work of the forward reads and writes tensors allocated on
    # the main stream (no record_stream: its deferred frees stall the caching
    # allocator). The backward joins that work before its first use; a cache
    # dropped without a backward joins it here, so the memory is never handed
    # to new main-stream work while the side stream still uses it.
    def __del__(self):
        try:
            ev = self.act_split_ready or self.x_in_ready
            if ev is not None and torch.cuda.is_initialized():
                torch.cuda.current_stream(self.act_vals.device if self.act_vals is not None else None).wait_event(ev)
        except Exception:  # interpreter shutdown
            pass

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
        stored = Sparse24Matrix(self.n, h, TOKEN_WISE, self.act_vals, self.act_meta)
        if self.row_frame is None:
            return stored
        # token-order storage: gather the rows into the compute frame (API view only)
        from .splitgemm import frame_rows_compressed

        data, hw = frame_rows_compressed(self.act_vals, self.act_meta, self.row_frame, self.n, h)
        return Sparse24Matrix(self.n, h, TOKEN_WISE, data, hw)

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
                for_backward: bool = True):
    """Run the forward pass; returns (out [n, d] bf16, FfnCache) (ref ffn.py:276-363).
    keep_pre_act=True also stores the fp32 pre-activation in the cache (parity
    tests use it to replay the selection on identical inputs). for_backward=False
    (inference prefill) skips the feature-wise split the backward would need.

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
        return _ffn_forward(x, p, cfg, plan, keep_pre_act, for_backward)
    if x.shape[1] != d:
        raise DimensionError(f"input width {x.shape[1]} does not match w1 {tuple(p.w1.shape)}")
    if plan is not None and plan.hidden_dim != h:
        raise DimensionError(f"plan built for {plan.hidden_dim} features, FFN has {h}")
    out, core = _ffn_forward(_pad_cols(x, dp), _pad_params(p, dp, hp), cfg, plan, keep_pre_act, for_backward,
                             h_valid=h)
    n = core.n
    view = replace(core, pre_act=core.pre_act[:, :h] if core.pre_act is not None else None,
                   counts=core.counts[:h] if core.counts is not None else None,
                   plan=core.plan_valid if core.plan_valid is not None else core.plan,
                   stats=SparsifyStats(n * h, core.stats._dev) if core.stats is not None else None,
                   census=_census_real(core.census, n, d, h, core.plan_valid, cfg),
                   act_split_ready=None, x_in_ready=None, core=core, d_valid=d, h_valid=h, plan_valid=None)
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


def _ffn_forward(x, p: FfnParams, cfg: FfnConfig, plan: SplitPlan | None, keep_pre_act: bool, for_backward: bool,
                 h_valid: int | None = None):
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
    if cfg.fp8_emulation:
        # e4m3 operands on the kind::f8f6f4 tensor cores (fp8.py)
        from .fp8 import ffn_forward_f8

        return ffn_forward_f8(x, p, cfg, plan, keep_pre_act, for_backward, h_valid=h_valid)
    dev = x.device
    s = stream()
    npad = pad128(n)
    census: list[GemmEvent] = []

    perm = perm_dev = inv_dev = None
    # The token permutation only shapes the feature-wise groups of the
    # backward; every forward stage maps one token row to one output row, so an
    # inference forward (for_backward=False) skips it: same bits, no gathers.
    permute = cfg.permute_tokens and sparse_fwd and for_backward
    if permute:
        perm_dev, inv_dev = device_permutation(cfg.permute_seed, n, dev)
        perm = perm_dev

    out = torch.empty(n, d, dtype=BF16, device=dev)
    if not sparse_fwd:
        act = torch.empty(n, h, dtype=BF16, device=dev)
        _lib.call("s24_gemm_relu2", ptr(x), d, ptr(p.w1), h, n, h, d, ptr(act), h, s)
        census.append(GemmEvent("fwd.pre_act", False, gemm_macs(n, d, h)))
        _lib.call("s24_gemm", ptr(act), 0, h, ptr(p.w2), 1, d, n, d, h, ptr(out), _lib.BF16, d, None, 0, -1, None, s)
        census.append(GemmEvent("fwd.out", False, gemm_macs(n, h, d)))
        cache = FfnCache(x, n, None, None, act, None, None, None, None, None, None, None, census, cfg)
        return out, cache

    act_vals = torch.empty(npad, h // 2, dtype=BF16, device=dev)
    act_meta = torch.empty(_lib.meta_hw_bytes(n, h), dtype=torch.uint8, device=dev)
    if npad > n:
        act_vals[n:].zero_()
        act_meta[(n // 128) * (h // 128) * 2048:].fill_(0x44)
    counts = torch.zeros(h, dtype=torch.int32, device=dev)
    stats_dev = torch.zeros(2, dtype=torch.int64, device=dev)
    need_pre = keep_pre_act or not cfg.mask_grad_with_fwd
    pre = torch.empty(n, h, dtype=F32, device=dev) if need_pre else None
    # the split / naive weight-gradient GEMMs read the activation feature-wise
    # 2:4 compressed; K1's epilogue produces that operand for every feature
    act_fw = FusedFeatureOperand.alloc(h, npad, dev) if (FUSED_FEATURE_SPLIT and cfg.backward_mode != "dense") else None
    fw_args = act_fw.args() if act_fw is not None else (None, None, None, 0)

    # The compute frame is the token-permuted order (ref ffn.py:297-303). K1
    # reads x as is and writes input row r as activation row perm[r] (row map
    # in its epilogue); the permuted copy x_in (zero rows up to a multiple of
    # 128) is only the B operand of the dW1 GEMM, so it is gathered off the
    # critical path. The fused feature-wise epilogue needs permuted input rows.
    side = side_stream(dev) if (for_backward and K4_MODE == "side") else None
    # (inference prefill, for_backward=False, needs no x_in at all)
    x_in = _frame_rows(x, npad, inv_dev if permute else None, defer=True) if for_backward else None
    k1_in, k1_map = x, (perm_dev if permute else None)
    row_frame = None
    if (TOKEN_ORDER_STORAGE and permute and side is not None and cfg.mask_grad_with_fwd and act_fw is None
            and cfg.backward_mode in ("split_masked", "naive_sparse") and _layout()["paired"]
            and not _layout()["identity"] and not _dual_k4() and not ACT_SPLIT_IN_BWD):
        # token-order storage: K1 on x as is; the permutation is applied by K4
        # and by the side-stream gathers (see TOKEN_ORDER_STORAGE)
        row_frame = inv_dev if npad == n else torch.cat(
            [inv_dev, torch.arange(n, npad, dtype=inv_dev.dtype, device=dev)])
        k1_map = None
    elif (act_fw is not None or not ROWMAP_GEMMS) and permute:
        if x_in is None:
            x_in = _frame_rows(x, npad, inv_dev, defer=True)
        _fill_frame_rows(x_in, x, inv_dev)
        k1_in, k1_map = x_in, None
    _lib.call("s24_fwd_gemm1_fused", ptr(k1_in), d, ptr(p.w1), h, n, h, d, ptr(act_vals), ptr(act_meta),
              ptr(counts), ptr(stats_dev), ptr(pre), *fw_args, ptr(k1_map), s)
    census.append(GemmEvent("fwd.pre_act", False, gemm_macs(n, d, h)))
    if plan is not None and plan.hidden_dim != (h_valid or h):
        raise DimensionError(f"plan built for {plan.hidden_dim} features, FFN has {h_valid or h}")
    need_plan = cfg.backward_mode == "split_masked"
    plan_api = plan

    # fwd.out on tensor cores (inverse permutation as its epilogue row map).
    # Next to it, on a side stream: the split plan (K7), x_in, and -- when the
    # backward will need it -- K4, the feature-wise split of act.
    act_split = None
    split_ready = x_in_ready = None
    plan_out = plan
    want_split = for_backward and cfg.backward_mode != "dense" and act_fw is None
    defer_split = want_split and side is not None and (ACT_SPLIT_IN_BWD or _dual_k4())
    want_split = want_split and not defer_split

    def fwd_out(st):
        _lib.call("s24_spmm", ptr(act_vals), ptr(act_meta), ptr(p.w2), 1, d, n, d, h, ptr(out), _lib.BF16, d,
                  ptr(inv_dev if row_frame is None else None), 0, -1, None, 0, st)

    if side is not None:
        main = torch.cuda.current_stream()
        if not K4_AFTER_FWD_OUT:
            side.wait_stream(main)  # K1's outputs are ready; the side work must not wait for fwd.out
        fwd_out(s)
        if K4_AFTER_FWD_OUT:
            side.wait_stream(main)
        if need_plan or plan is not None:
            plan_api, plan_out = _plan_split(counts, cfg.split_ratio, plan, h, h_valid, side)
        bg_plan = plan_out if need_plan else _all_sparse_plan(h, dev)
        if want_split:
            act_split = alloc_feature_split(act_vals, act_meta, npad, h, bg_plan, row_map=row_frame, **_layout())
        with torch.cuda.stream(side):
            if SIDE_GATHERS and x_in is not None and x_in is not x and k1_in is not x_in:
                _fill_frame_rows(x_in, x, inv_dev)
            if want_split:  # (relu^2: >= 0)
                run_feature_split(act_split, act_vals, act_meta, npad, h, bg_plan, nonneg=True, row_map=row_frame)
                if act_split.pair_rows >= 0 and not act_split.identity:
                    bg_plan.paired_row_map  # (the weight-gradient row map, built here off the main stream)
            ev = torch.cuda.Event()
            ev.record(side)
        split_ready = x_in_ready = ev
        if not SIDE_GATHERS and x_in is not None and x_in is not x and k1_in is not x_in:
            _fill_frame_rows(x_in, x, inv_dev)
    else:
        if need_plan or plan is not None:
            plan_api, plan_out = _plan_split(counts, cfg.split_ratio, plan, h, h_valid)
        if x_in is not None and x_in is not x and k1_in is not x_in:
            _fill_frame_rows(x_in, x, inv_dev)
        bg_plan = plan_out if need_plan else _all_sparse_plan(h, dev)
        if want_split:
            act_split = alloc_feature_split(act_vals, act_meta, npad, h, bg_plan, **_layout())
        if want_split and K4_MODE == "gemm" and _layout()["paired"] and not _layout()["identity"]:
            # fwd.out whose CTAs also split their act stages feature-wise
            _lib.call("s24_spmm_fs", ptr(act_vals), ptr(act_meta), ptr(p.w2), 1, d, n, d, h, ptr(out), _lib.BF16, d,
                      ptr(inv_dev), 0, -1, None, npad, ptr(bg_plan.feat_pos), bg_plan.n_sparse, bg_plan.n_dense,
                      ptr(act_split.vs), ptr(act_split.es), 1, s)
        elif want_split and K4_MODE == "background":
            counter = torch.empty(1, dtype=torch.int32, device=dev)
            _lib.call("s24_spmm_bg", ptr(act_vals), ptr(act_meta), ptr(p.w2), 1, d, n, d, h, ptr(out), _lib.BF16,
                      d, ptr(inv_dev), 0, -1, None,
                      *k4_job_args(act_vals, act_meta, npad, h, bg_plan, act_split, counter), s)
        else:
            fwd_out(s)
            if want_split:
                run_feature_split(act_split, act_vals, act_meta, npad, h, bg_plan, nonneg=True)
    census.append(GemmEvent("fwd.out", True, sp_gemm_macs(n, h, d)))
    if row_frame is not None and pre is not None:
        pre = pre[row_frame[:n].long()]  # (debug / parity view: the compute frame)
    cache = FfnCache(x_in, n, act_vals, act_meta, None, pre, perm, perm_dev, inv_dev, plan_out,
                     SparsifyStats(n * h, stats_dev), counts, census, cfg, act_fw=act_fw, act_split=act_split,
                     act_split_ready=split_ready, x_in_ready=x_in_ready, row_frame=row_frame,
                     plan_valid=plan_api if h_valid is not None else None)
    return out, cache


def _frame_rows(a: torch.Tensor, npad: int, src_rows, defer: bool = False) -> torch.Tensor:
    """The compute-frame copy of a [n, d] input: rows permuted (out[i] =
    a[src_rows[i]]) and zero-padded to npad rows. Returns `a` itself when
    neither applies. defer=True only allocates (fill with _fill_frame_rows)."""
    n = a.shape[0]
    if src_rows is None and npad == n:
        return a
    out = torch.empty(npad, a.shape[1], dtype=a.dtype, device=a.device)
    if not defer:
        _fill_frame_rows(out, a, src_rows)
    return out


def _fill_frame_rows(out: torch.Tensor, a: torch.Tensor, src_rows) -> None:
    """Fill a _frame_rows buffer on the current stream."""
    n = a.shape[0]
    if out.shape[0] > n:
        out[n:].zero_()
    if src_rows is not None:
        gather_rows(a, src_rows, out)
    else:
        out[:n].copy_(a)





def _spmm_with_split(launch_gemm, k4_work):
    """Launch a sparse GEMM on the current stream and the K4 job `k4_work()`
    next to it (K4_MODE "side": side stream, co-resident; "inline": after it).
    Returns the CUDA event after which the K4 outputs are complete (None if
    inline)."""
    main = torch.cuda.current_stream()
    if K4_MODE != "side":
        launch_gemm(main.cuda_stream)
        k4_work()
        return None
    side = side_stream(main.device)
    side.wait_stream(main)  # K4's inputs are ready; it must not wait for the GEMM
    launch_gemm(main.cuda_stream)
    with torch.cuda.stream(side):
        k4_work()
        ev = torch.cuda.Event()
        ev.record(side)
    return ev


def _act_split(cache: FfnCache, npad: int, h: int, plan: SplitPlan):
    """The feature-wise split of the cached activation (made by the forward
    next to fwd.out when K4 runs on the side stream, else here)."""
    if cache.act_split is None:
        if cache.row_frame is not None:
            fs = alloc_feature_split(cache.act_vals, cache.act_meta, npad, h, plan, paired=True,
                                     row_map=cache.row_frame)
            run_feature_split(fs, cache.act_vals, cache.act_meta, npad, h, plan, nonneg=True, row_map=cache.row_frame)
            return fs
        return feature_split(cache.act_vals, cache.act_meta, npad, h, plan, nonneg=True, **_layout())
    if cache.act_split_ready is not None:
        torch.cuda.current_stream().wait_event(cache.act_split_ready)
    return cache.act_split


def weight_grad_buffers(d: int, h: int, dev, bucket: torch.Tensor | None = None):
    """(d_w1 [d, h], d_w2 [h, d]) fp32: fresh tensors, or views into bucket."""
    if bucket is None:
        return torch.empty(d, h, dtype=F32, device=dev), torch.empty(h, d, dtype=F32, device=dev)
    if bucket.dtype != F32 or bucket.numel() != 2 * d * h or not bucket.is_contiguous():
        raise DimensionError(f"grad_bucket must be a contiguous fp32 buffer of {2 * d * h} elements")
    return bucket[: d * h].view(d, h), bucket[d * h:].view(h, d)


_third_streams: dict = {}


def _third_stream(device) -> torch.cuda.Stream:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    st = _third_streams.get(idx)
    if st is None:
        st = _third_streams[idx] = torch.cuda.Stream(device=device)
    return st


def _all_sparse_plan(h: int, dev) -> SplitPlan:
    pos = torch.arange(h, dtype=torch.int32, device=dev)
    return SplitPlan(h, 1.0, torch.zeros(h, dtype=torch.int64, device=dev), pos,
                     torch.empty(0, dtype=torch.int32, device=dev), pos)


def ffn_backward(g_out, cache: FfnCache, p: FfnParams, cfg: FfnConfig, grad_ready=None,
                 grad_bucket: torch.Tensor | None = None) -> FfnGrads:
    """Backward matching the cached forward (ref ffn.py:366-451).

    grad_ready(name, tensor), if given, is called as soon as d_w2 and then
    d_w1 are final on the current stream (used by the data-parallel step to
    launch their all-reduce while the rest of the backward runs).
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
    return FfnGrads(d_w1, d_w2, d_x, None, _census_real(gr.census, n, d, h, cache.plan, cfg),
                    _token_total(gr.stats_act, n, hp - h), _token_total(gr.stats_grad, n, hp - h))


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
    if cache.x_in is None:
        raise StateError("cache comes from an inference forward (for_backward=False)")
    d = cache.x_in.shape[1]
    g_out = as_matrix(g_out, "g_out", BF16)
    if tuple(g_out.shape) != (n, d):
        raise StateError(f"gradient shape {tuple(g_out.shape)} does not match cached input {(n, d)}")
    sparse_fwd = cfg.forward_mode == "sparse24"
    if sparse_fwd and cache.act_vals is None:
        raise StateError("sparse forward cache is missing the compressed activation")
    if not sparse_fwd and cache.act_dense is None:
        raise StateError("dense forward cache is missing the activation")
    if cfg.backward_mode == "split_masked" and cache.plan is None:
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
    stats_a = stats_g = None

    if not sparse_fwd:
        # ---------------------------------------------------------- dense twin
        act = cache.act_dense
        g_pre = torch.empty(n, h, dtype=BF16, device=dev)
        _lib.call("s24_gemm_dact", ptr(g_out), d, ptr(p.w2), d, n, h, d, ptr(act), h, ptr(g_pre), h, s)
        census.append(GemmEvent("bwd.d_act", False, gemm_macs(n, d, h)))
        _lib.call("s24_gemm", ptr(act), 1, h, ptr(g_out), 1, d, h, d, n, ptr(d_w2), _lib.F32, d, None, 0, -1, None, s)
        census.append(GemmEvent("bwd.d_w2", False, gemm_macs(h, n, d)))
        notify("d_w2", d_w2)
        _lib.call("s24_gemm", ptr(g_pre), 1, h, ptr(cache.x_in), 1, d, h, d, n, ptr(d_w1), _lib.F32, h, None, 1, -1, None, s)
        census.append(GemmEvent("bwd.d_w1", False, gemm_macs(d, n, h)))
        notify("d_w1", d_w1)
        _lib.call("s24_gemm", ptr(g_pre), 0, h, ptr(p.w1), 0, h, n, d, h, ptr(d_x), _lib.BF16, d, None, 0, -1, None, s)
        census.append(GemmEvent("bwd.d_x", False, gemm_macs(n, h, d)))
        return FfnGrads(d_w1, d_w2, d_x, None, census)

    # -------------------------------------------------------------- sparse forward
    # g_pre on the forward keep pattern, compressed (exact; ref ffn.py:415-417, 443)
    g_vals = torch.empty(npad, h // 2, dtype=BF16, device=dev)
    if npad > n:
        g_vals[n:].zero_()
    # K3's epilogue also emits the feature-wise 2:4 g_pre operand of the dW1
    # GEMM when the split path will consume it
    fused_g = FUSED_FEATURE_SPLIT and (
        cfg.backward_mode == "split_masked" or (cfg.backward_mode == "naive_sparse" and cfg.mask_grad_with_fwd))
    raw_naive = cfg.backward_mode == "naive_sparse" and not cfg.mask_grad_with_fwd
    g_fw = FusedFeatureOperand.alloc(h, npad, dev) if fused_g else None
    fw_args = g_fw.args() if g_fw is not None else (None, None, None, 0)
    # The permuted, padded copy g_c of dY is only an operand of the weight
    # gradients (B of dW2) and of the unmasked-derivative path, so it is
    # gathered on the side stream while K3 reads dY as is (row map).
    main = torch.cuda.current_stream()
    side = side_stream(dev) if K4_MODE == "side" else None
    g_c = _frame_rows(g_out, npad, cache.inv_dev, defer=True)
    g_ready = None
    rowmap = ROWMAP_K3 and g_fw is None
    stored = cache.row_frame is not None  # token-order storage: K3 / dX need no frame rows
    if stored and (side is None or g_fw is not None or not cfg.mask_grad_with_fwd):
        raise StateError("token-order storage needs the side-stream backward with mask_grad_with_fwd")
    if g_c is not g_out:
        if not rowmap and cache.perm_dev is not None and not stored:
            _fill_frame_rows(g_c, g_out, cache.inv_dev)  # K3 reads g_c
        elif side is not None and SIDE_GATHERS:
            side.wait_stream(main)
            with torch.cuda.stream(side):
                _fill_frame_rows(g_c, g_out, cache.inv_dev)
                g_ready = torch.cuda.Event()
                g_ready.record(side)
        elif side is None:
            _fill_frame_rows(g_c, g_out, cache.inv_dev)
    late_g_c = g_c is not g_out and side is not None and not SIDE_GATHERS and rowmap

    def need_frame_inputs():
        """Main-stream consumers of g_c / x_in wait for their side-stream gathers."""
        nonlocal g_ready, late_g_c
        if late_g_c:
            _fill_frame_rows(g_c, g_out, cache.inv_dev)
            late_g_c = False
        if g_ready is not None:
            main.wait_event(g_ready)
            g_ready = None
        if cache.x_in_ready is not None:
            main.wait_event(cache.x_in_ready)

    # the feature-wise split of act, when the forward left it for here: on the
    # side stream next to K3
    if cache.act_split is None and cache.act_fw is None and side is not None and \
            cfg.backward_mode != "dense" and ACT_SPLIT_IN_BWD and not _dual_k4():
        plan_a = _all_sparse_plan(h, dev) if cfg.backward_mode == "naive_sparse" else cache.plan
        fa_b = alloc_feature_split(cache.act_vals, cache.act_meta, npad, h, plan_a, **_layout())
        side.wait_stream(main)
        with torch.cuda.stream(side):
            run_feature_split(fa_b, cache.act_vals, cache.act_meta, npad, h, plan_a, nonneg=True)
            ev_a = torch.cuda.Event()
            ev_a.record(side)
        cache.act_split, cache.act_split_ready = fa_b, ev_a

    # K3 reads dY unpermuted and pairs input row r with act / g_pre row
    # perm[r]; the fused feature-wise epilogue needs the permuted rows
    k3_in, k3_map = g_out, cache.perm_dev
    if stored:
        k3_in, k3_map = g_out, None  # dY rows pair with the stored act rows as they are
    elif not rowmap and cache.perm_dev is not None:
        need_frame_inputs()
        k3_in, k3_map = g_c, None
    # (fp8 forward: relu(y1) comes from the unquantized activation)
    k3_act = cache.act_raw if cache.act_raw is not None else cache.act_vals
    _lib.call("s24_bwd_dact_fused", ptr(k3_in), d, ptr(p.w2), d, n, h, d, ptr(k3_act), ptr(cache.act_meta),
              ptr(g_vals), *fw_args, ptr(k3_map), s)
    census.append(GemmEvent("bwd.d_act", False, gemm_macs(n, d, h)))
    g_pre_dense = None
    if not cfg.mask_grad_with_fwd:
        # unmasked derivative: needs relu(y1) everywhere (fp32 pre-activation kept by the forward)
        need_frame_inputs()
        G = torch.empty(n, h, dtype=F32, device=dev)
        _lib.call("s24_gemm", ptr(g_c), 0, d, ptr(p.w2), 0, d, n, h, d, ptr(G), _lib.F32, h, None, 0, -1, None, s)
        g_pre_dense = (G * act_squared_relu_grad(cache.pre_act)).to(BF16)

    mode = cfg.backward_mode
    ev_dx = None
    if mode != "dense":
        plan = _all_sparse_plan(h, dev) if mode == "naive_sparse" else cache.plan
        macs_w = sp_gemm_macs(n, h, d) if mode == "naive_sparse" else split_gemm_macs(n, d, plan)
    fg = None
    fg_ready = None
    if (WGRAD_OVERLAP and side is not None and cfg.mask_grad_with_fwd and mode != "dense" and g_fw is None
            and not raw_naive and grad_ready is None and cache.act_fw is None and _layout()["paired"]
            and not _dual_k4()):
        # dW2 (main) || K4(g_pre) (side) ; then dW1 (side) || dX (third stream)
        ev_k3 = torch.cuda.Event()
        ev_k3.record(main)
        fa = _act_split(cache, npad, h, plan)
        fg = alloc_feature_split(g_vals, cache.act_meta, npad, h, plan, row_map=cache.row_frame, **_layout())
        need_frame_inputs()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            run_feature_split(fg, g_vals, cache.act_meta, npad, h, plan, row_map=cache.row_frame)
        split_weight_grad(fa, plan, g_c, npad, d_w2, transposed=False)
        with torch.cuda.stream(side):
            split_weight_grad(fg, plan, cache.x_in, npad, d_w1, transposed=True)
            ev_w1 = torch.cuda.Event()
            ev_w1.record(side)
        third = _third_stream(dev)
        third.wait_event(ev_k3)
        with torch.cuda.stream(third):
            _lib.call("s24_spmm", ptr(g_vals), ptr(cache.act_meta), ptr(p.w1), 0, h, n, d, h, ptr(d_x), _lib.BF16,
                      d, ptr(None if stored else cache.inv_dev), 0, -1, None, 0, third.cuda_stream)
            ev_x = torch.cuda.Event()
            ev_x.record(third)
        main.wait_event(ev_w1)
        main.wait_event(ev_x)
        census.append(GemmEvent("bwd.d_w2", True, macs_w))
        census.append(GemmEvent("bwd.d_w1", True, macs_w))
        census.append(GemmEvent("bwd.d_x", True, sp_gemm_macs(n, h, d)))
        return FfnGrads(d_w1, d_w2, d_x, None, census, fa.stats, fg.stats)
    if cfg.mask_grad_with_fwd and mode != "dense" and g_fw is None and not raw_naive:
        # dX first: its sparse GEMM carries the feature-wise split of g_pre (K4)
        # as background work in its idle epilogue warps
        fg = alloc_feature_split(g_vals, cache.act_meta, npad, h, plan, row_map=cache.row_frame, **_layout())
        if K4_MODE == "gemm" and fg.pair_rows >= 0 and not fg.identity:
            # dX whose CTAs also split their g_pre stages feature-wise
            _lib.call("s24_spmm_fs", ptr(g_vals), ptr(cache.act_meta), ptr(p.w1), 0, h, n, d, h, ptr(d_x), _lib.BF16,
                      d, ptr(cache.inv_dev), 0, -1, None, npad, ptr(plan.feat_pos), plan.n_sparse, plan.n_dense,
                      ptr(fg.vs), ptr(fg.es), 0, s)
        elif K4_MODE == "background":
            counter = torch.empty(1, dtype=torch.int32, device=dev)
            _lib.call("s24_spmm_bg", ptr(g_vals), ptr(cache.act_meta), ptr(p.w1), 0, h, n, d, h, ptr(d_x),
                      _lib.BF16, d, ptr(cache.inv_dev), 0, -1, None,
                      *k4_job_args(g_vals, cache.act_meta, npad, h, plan, fg, counter), s)
        else:
            dual = cache.act_split is None and cache.act_fw is None and _dual_k4()
            fa = alloc_feature_split(cache.act_vals, cache.act_meta, npad, h, plan, **_layout()) if dual else None

            def k4_side():
                if dual:  # act (>= 0) and g_pre share the keep pattern: one pass for both
                    run_feature_split_dual(fa, fg, cache.act_vals, g_vals, cache.act_meta, npad, h, plan)
                else:
                    run_feature_split(fg, g_vals, cache.act_meta, npad, h, plan, row_map=cache.row_frame)

            fg_ready = _spmm_with_split(
                lambda st: _lib.call("s24_spmm", ptr(g_vals), ptr(cache.act_meta), ptr(p.w1), 0, h, n, d, h,
                                     ptr(d_x), _lib.BF16, d, ptr(None if stored else cache.inv_dev), 0, -1, None,
                                     0, st),
                k4_side)
            if dual:
                cache.act_split, cache.act_split_ready = fa, fg_ready
        ev_dx = GemmEvent("bwd.d_x", True, sp_gemm_macs(n, h, d))

    need_frame_inputs()
    if mode == "dense":
        act = torch.empty(n, h, dtype=BF16, device=dev)
        _lib.call("s24_decompress_token", ptr(cache.act_vals), None, ptr(cache.act_meta), n, h, ptr(act), _lib.BF16, h, s)
        if g_pre_dense is None:
            gp = torch.empty(n, h, dtype=BF16, device=dev)
            _lib.call("s24_decompress_token", ptr(g_vals), None, ptr(cache.act_meta), n, h, ptr(gp), _lib.BF16, h, s)
        else:
            gp = g_pre_dense
        _lib.call("s24_gemm", ptr(act), 1, h, ptr(g_c), 1, d, h, d, n, ptr(d_w2), _lib.F32, d, None, 0, -1, None, s)
        census.append(GemmEvent("bwd.d_w2", False, gemm_macs(h, n, d)))
        notify("d_w2", d_w2)
        _lib.call("s24_gemm", ptr(gp), 1, h, ptr(cache.x_in), 1, d, h, d, n, ptr(d_w1), _lib.F32, h, None, 1, -1, None, s)
        census.append(GemmEvent("bwd.d_w1", False, gemm_macs(d, n, h)))
        notify("d_w1", d_w1)
    elif (grad_ready is None and cache.act_fw is None and g_fw is None and not raw_naive
          and PAIRED_WEIGHT_GRADS):
        # both split weight gradients in one grouped launch: dW2 = split(act)^T g_c
        # and dW1^T = split(g_pre)^T x_in share (M, N, K) = (|S|, d, n), so the
        # second fills the first one's partial last wave (no per-gradient hook
        # to serve, hence only without grad_ready)
        fa = _act_split(cache, npad, h, plan)
        if fg is None:
            fg = feature_split(g_vals, cache.act_meta, npad, h, plan, **_layout())
        elif fg_ready is not None:
            torch.cuda.current_stream().wait_event(fg_ready)
        split_weight_grad_pair(fa, fg, plan, g_c, cache.x_in, npad, d_w2, d_w1)
        stats_a, stats_g = fa.stats, fg.stats
        census.append(GemmEvent("bwd.d_w2", True, macs_w))
        census.append(GemmEvent("bwd.d_w1", True, macs_w))
    else:
        # dW2 = split(act)^T g_c  (act is already restricted to the mask)
        if cache.act_fw is not None:
            fused_weight_grad(cache.act_fw, cache.act_vals, cache.act_meta, h, plan, g_c, d_w2, transposed=False)
            stats_a = cache.act_fw.stats(plan)
        else:
            fa = _act_split(cache, npad, h, plan)
            split_weight_grad(fa, plan, g_c, npad, d_w2, transposed=False)
            stats_a = fa.stats
        census.append(GemmEvent("bwd.d_w2", True, macs_w))
        notify("d_w2", d_w2)
        # dW1 = (split(g_pre)^T x_in)^T. The split path always sees the masked
        # g_pre (ref splitgemm.py:72, even with mask_grad_with_fwd off);
        # naive_sparse without the mask sparsifies the raw g_pre feature-wise.
        if raw_naive:
            from .sparse24 import sparsify_feature_wise

            gpad = torch.zeros(npad, h, dtype=BF16, device=dev)
            gpad[:n] = g_pre_dense
            sg, _, stats_g = sparsify_feature_wise(gpad)
            _lib.call("s24_spmm", ptr(sg.data), ptr(sg.meta_hw), ptr(cache.x_in), 1, d, h, d, npad, ptr(d_w1),
                      _lib.F32, h, None, 1, -1, None, 0, s)
        elif g_fw is not None:
            fused_weight_grad(g_fw, g_vals, cache.act_meta, h, plan, cache.x_in, d_w1, transposed=True)
            stats_g = g_fw.stats(plan)
        else:
            if fg is None:
                fg = feature_split(g_vals, cache.act_meta, npad, h, plan, **_layout())
            elif fg_ready is not None:
                torch.cuda.current_stream().wait_event(fg_ready)
            split_weight_grad(fg, plan, cache.x_in, npad, d_w1, transposed=True)
            stats_g = fg.stats
        census.append(GemmEvent("bwd.d_w1", True, macs_w))
        notify("d_w1", d_w1)

    if ev_dx is not None:
        census.append(ev_dx)
    elif cfg.mask_grad_with_fwd:
        _lib.call("s24_spmm", ptr(g_vals), ptr(cache.act_meta), ptr(p.w1), 0, h, n, d, h, ptr(d_x), _lib.BF16, d,
                  ptr(cache.inv_dev), 0, -1, None, 0, s)
        census.append(GemmEvent("bwd.d_x", True, sp_gemm_macs(n, h, d)))
    else:
        _lib.call("s24_gemm", ptr(g_pre_dense), 0, h, ptr(p.w1), 0, h, n, d, h, ptr(d_x), _lib.BF16, d,
                  ptr(cache.inv_dev), 0, -1, None, s)
        census.append(GemmEvent("bwd.d_x", False, gemm_macs(n, h, d)))
    return FfnGrads(d_w1, d_w2, d_x, None, census, stats_a, stats_g)
