"""Routing strategies on the B200 path: the reference's ``baselines`` surface.

Mirrors /root/reference/pkg/src/beamoe/baselines.py: ``KINDS`` (:37-46),
``RoutingStrategy`` (:51-103), ``build_block`` (:106-113), ``RouteResult``
(:116-129), ``temperature_at`` (:146-149), ``route`` (:158-283) and
``block_forward`` (:286-323), inference branch.  Every strategy reduces to the
same kernels as BEAM: one routing rule in the gating kernel
(``beam_route_t``), then the masked permute, the grouped experts and the
ordered combine — skipped slots (masked, pruned, null, outside the dynamic
prefix) cost neither bytes nor FLOPs.

``training=True`` is out of scope on the GPU path and raises.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, _runtime
from .beam import MaskRouter
from .moe import MoEBlock, MoEBlockConfig
from .tensor import ContractError, ShapeError, as_torch

KINDS = (
    "vanilla_topk",
    "topk_reduced",
    "topk_pruning",
    "moe_dynamic",
    "ada_moe",
    "beam",
    "soft_mask",
    "soft_mask_tempered",
)

_MASKED_KINDS = {"beam", "soft_mask", "soft_mask_tempered"}


@dataclass
class RoutingStrategy:
    """baselines.py:51-103 (same parameter names and validation messages)."""

    kind: str
    params: dict = field(default_factory=dict)

    def validate(self, cfg: MoEBlockConfig) -> None:
        if self.kind not in KINDS:
            raise ContractError(f"unknown routing strategy {self.kind!r}")
        p = dict(self.params)
        known = {
            "vanilla_topk": set(),
            "topk_reduced": {"k_small"},
            "topk_pruning": {"k_infer"},
            "moe_dynamic": {"phi"},
            "ada_moe": {"null_count"},
            "beam": {"tau"},
            "soft_mask": {"tau"},
            "soft_mask_tempered": {"tau", "temp_floor"},
        }[self.kind]
        unknown = set(p) - known
        if unknown:
            raise ContractError(f"{self.kind}: unknown params {sorted(unknown)}")
        if self.kind == "topk_reduced":
            if not 1 <= p.get("k_small", cfg.top_k) <= cfg.num_experts:
                raise ContractError("k_small out of range")
        elif self.kind == "topk_pruning":
            if not 1 <= p.get("k_infer", cfg.top_k) <= cfg.top_k:
                raise ContractError("k_infer must satisfy 1 <= K_infer <= K_train")
        elif self.kind == "moe_dynamic":
            if not 0.0 < p.get("phi", 0.5) <= 1.0:
                raise ContractError("phi must lie in (0, 1]")
        elif self.kind == "ada_moe":
            if p.get("null_count", 0) < 0:
                raise ContractError("null_count must be >= 0")
        if self.kind in _MASKED_KINDS:
            if not 0.0 < p.get("tau", 0.5) < 1.0:
                raise ContractError("tau must lie in (0, 1)")
        if self.kind == "soft_mask_tempered" and p.get("temp_floor", 0.1) <= 0:
            raise ContractError("temp_floor must be positive")

    @property
    def needs_mask_router(self) -> bool:
        return self.kind in _MASKED_KINDS

    @property
    def extra_router_cols(self) -> int:
        return self.params.get("null_count", 0) if self.kind == "ada_moe" else 0


def build_block(cfg: MoEBlockConfig, strategy: RoutingStrategy, rng: np.random.Generator, **kw) -> MoEBlock:
    """baselines.py:106-113 (same parameter draws as the reference)."""
    strategy.validate(cfg)
    block = MoEBlock(cfg, rng, extra_router_cols=strategy.extra_router_cols, **kw)
    if strategy.needs_mask_router:
        block.mask_router = MaskRouter.zero_init(cfg.d_h, cfg.num_experts, strategy.params.get("tau", 0.5),
                                                 device=block.device)
    return block


@dataclass
class RouteResult:
    """baselines.py:116-129 — the fields the inference path produces."""

    weights_hat: torch.Tensor  # (T, N) final expert weights
    logits: torch.Tensor  # (T, N) or (T, N + nulls)
    balance_active: torch.Tensor  # bool, same width as logits
    candidate_ids: torch.Tensor  # (T, K); -1 marks a null slot
    active_bits: torch.Tensor  # (T, K) 0/1 per candidate slot
    active_counts: torch.Tensor  # (T,)
    raw_mask: torch.Tensor | None = None
    reg_indices: torch.Tensor | None = None
    compute_ids: torch.Tensor | None = None
    kept_ids: torch.Tensor | None = None


def temperature_at(step: int, total_steps: int, floor: float = 0.1) -> float:
    """baselines.py:146-149 — geometric decay 1.0 -> floor, reaching the floor halfway."""
    half = max(1, total_steps // 2)
    return max(floor, float(floor ** (min(step, half) / half)))


def _route_desc(block: MoEBlock, strategy: RoutingStrategy, binarize_soft: bool) -> _lib.RouteDesc:
    cfg = block.cfg
    p = strategy.params
    r = _lib.RouteDesc()
    r.k, r.null_count, r.phi, r.temp, r.tau, r.binarize = cfg.top_k, 0, 0.5, 1.0, 0.5, 1
    kind = strategy.kind
    if kind in ("vanilla_topk", "topk_reduced", "topk_pruning"):  # :173-190
        r.kind = _lib.BEAM_ROUTE_TOPK
        if kind == "topk_reduced":
            r.k = p.get("k_small", cfg.top_k)
        elif kind == "topk_pruning":
            r.k = p.get("k_infer", cfg.top_k)
    elif kind == "moe_dynamic":  # :192-210
        r.kind = _lib.BEAM_ROUTE_DYNAMIC
        r.phi = p.get("phi", 0.5)
    elif kind == "ada_moe":  # :212-225
        r.kind = _lib.BEAM_ROUTE_ADA
        r.null_count = block.router_w.shape[1] - cfg.num_experts
    elif kind == "beam":  # :230-247
        r.kind = _lib.BEAM_ROUTE_BEAM
    else:  # soft variants :250-283 (inference: temp = floor for the tempered kind)
        r.kind = _lib.BEAM_ROUTE_SOFT
        r.tau = block.mask_router.tau
        r.temp = p.get("temp_floor", 0.1) if kind == "soft_mask_tempered" else 1.0
        r.binarize = 1 if (kind == "soft_mask_tempered" or binarize_soft) else 0
    return r


def block_forward(h, block: MoEBlock, strategy: RoutingStrategy, training: bool, step: int = 0,
                  total_steps: int = 1, binarize_soft: bool = False, block_size: int = 16):
    """baselines.py:286-323 with training=False -> (h', RouteResult), one C-ABI
    call (``beam_layer_forward_routed``)."""
    if training:
        raise ContractError("training-mode routing is out of scope of the B200 path (inference only)")
    strategy.validate(block.cfg)
    if strategy.needs_mask_router and block.mask_router is None:
        raise ContractError("block has no mask router (build it with baselines.build_block)")
    if strategy.kind == "beam" and block.mask_router.tau != 0.5:
        raise ContractError("beam routing keeps ids with a >= 0 (tau = 0.5); the reference rejects other tau")
    if block_size < 1:
        raise ContractError("block_size must be >= 1")
    cfg = block.cfg
    x = as_torch(h)
    if x.ndim != 2 or x.shape[1] != cfg.d_h:
        raise ShapeError("h must be [tokens, d_h]")
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    host = not x.is_cuda
    dev = block.device
    xd = x.to(dev).contiguous()
    rd = _route_desc(block, strategy, binarize_soft)
    t = xd.shape[0]
    k, n = rd.k, cfg.num_experts
    nr = block.router_w.shape[1]
    out = torch.empty(t, cfg.d_h, dtype=xd.dtype, device=dev)
    ids = torch.empty(t, k, dtype=torch.int64, device=dev)
    kept = torch.empty(t, k, dtype=torch.int64, device=dev)
    logits = torch.empty(t, nr, dtype=torch.float32, device=dev)
    weights_hat = torch.empty(t, n, dtype=torch.float32, device=dev)
    masked = strategy.needs_mask_router
    raw = torch.empty(t, n, dtype=torch.float32, device=dev) if masked else None
    hard = torch.empty(t, n, dtype=torch.float32, device=dev) if strategy.kind == "beam" else None
    if t > 0:
        desc = block.layer_desc(0.0)
        o = _lib.Outputs()
        o.out, o.topk_ids, o.masked_ids = out.data_ptr(), ids.data_ptr(), kept.data_ptr()
        o.logits, o.weights = logits.data_ptr(), weights_hat.data_ptr()
        if masked:
            o.raw_mask = raw.data_ptr()
        if hard is not None:
            o.mask = hard.data_ptr()
        lib = _lib.load()
        ws_bytes = lib.beam_workspace_bytes_routed(ctypes.byref(desc), ctypes.byref(rd), t, block_size)
        if ws_bytes == 0:
            raise ContractError("routing strategy not supported for this block")
        ws = _runtime.workspace(ws_bytes, dev)
        _lib.check(lib.beam_layer_forward_routed(ctypes.byref(desc), ctypes.byref(rd), xd.data_ptr(),
                                                 _lib.BEAM_BF16 if xd.dtype == torch.bfloat16 else _lib.BEAM_F32,
                                                 t, block_size, ctypes.byref(o), ws.data_ptr(), ws.numel(),
                                                 _runtime.stream_handle(dev)),
                   "beam_layer_forward_routed")
    if hard is not None:  # beam: the kernel reports RouterDecision.weights; weights_hat = g * m (beam.py:159)
        weights_hat = weights_hat * hard
    bits = (kept >= 0).to(torch.int64)
    # balance sets: the experts that took load (moe_dynamic: the active prefix; the
    # others: the candidates; ada_moe's null columns are not reported)
    sel = kept if strategy.kind == "moe_dynamic" else ids
    balance = torch.zeros(t, nr, dtype=torch.bool, device=dev)
    if t > 0:
        balance.scatter_(1, sel.clamp(min=0), sel >= 0)
    rr = RouteResult(weights_hat=weights_hat, logits=logits, balance_active=balance, candidate_ids=ids,
                     active_bits=bits, active_counts=bits.sum(dim=-1), raw_mask=raw,
                     reg_indices=ids if masked else None, compute_ids=None, kept_ids=kept)
    if host:
        torch.cuda.current_stream(dev).synchronize()
        out = out.cpu()
        rr = RouteResult(**{k2: (v.cpu() if isinstance(v, torch.Tensor) else v) for k2, v in rr.__dict__.items()})
    return out, rr
