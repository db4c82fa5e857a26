"""Masked expert dispatch on B200.

Mirrors /root/reference/pkg/src/beamoe/dispatch/__init__.py: ``mask_route``
(:55-62), ``DispatchPlan`` (:65-86), ``align_block`` (:89-126),
``grouped_execute`` (:129-157), ``naive_execute`` (:160-174),
``bench_dispatch`` (:189-245) and the backend registry (:21-52).

There is exactly one backend, the sm_100a CUDA library (the north star bans
multi-backend dispatch and CPU fallbacks); ``backend=`` arguments are accepted
for signature compatibility and must name it (or be None).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, _runtime
from .moe import Expert, ExpertBank, MoEBlock, MoEBlockConfig, _default_device, topk_select
from .tensor import ContractError, ShapeError, as_torch

BACKEND_NAME = "cuda-sm100a"


def active_backend() -> str:
    return BACKEND_NAME


def available_backends() -> list:
    return [BACKEND_NAME]


def _check_backend(backend):
    if backend not in (None, BACKEND_NAME):
        raise ContractError(f"dispatch backend {backend!r} unavailable; have {available_backends()}")


def _to_device(x, dtype=None):
    t = as_torch(x, dtype)
    host = not t.is_cuda
    dev = _default_device() if host else t.device
    return t.to(dev).contiguous(), host


def mask_route(topk_ids, mask_pre_activations, backend: str | None = None):
    """_kernels.pyx:17-34: keep id when 0 <= id < N and a[t, id] >= 0, else -1.
    fp64 pre-activations are compared in fp64 (bit-exact with the reference)."""
    _check_backend(backend)
    ids, host = _to_device(topk_ids, torch.int64)
    a = getattr(mask_pre_activations, "data", mask_pre_activations)
    if not isinstance(a, torch.Tensor):
        a = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
    if a.dtype not in (torch.float32, torch.float64):
        a = a.to(torch.float32)
    a = a.to(ids.device).contiguous()
    if ids.ndim != 2 or a.ndim != 2 or a.shape[0] != ids.shape[0]:
        raise ShapeError("mask_route expects ids [T, K] and pre-activations [T, N]")
    t, k = ids.shape
    n = a.shape[1]
    out = torch.empty_like(ids)
    if n < 1:
        out.fill_(-1)
    else:
        lib = _lib.load()
        _lib.check(lib.beam_mask_route(ids.data_ptr(), a.data_ptr(),
                                       _lib.BEAM_F64 if a.dtype == torch.float64 else _lib.BEAM_F32,
                                       t, k, n, out.data_ptr(), _runtime.stream_handle(ids.device)),
                   "beam_mask_route")
    return out.cpu() if host else out


class DispatchPlan:
    """dispatch/__init__.py:65-86 — expert-grouped, block-aligned slot layout,
    backed by flat int32 device buffers (``counts``, ``offsets`` = padded
    exclusive scan, ``flat_tokens``/``flat_slots``, ``active``, ``meta``).
    ``tokens[e]`` / ``slots[e]`` / ``real_counts`` materialise reference-style
    per-expert int64 arrays on first access (one device->host copy)."""

    def __init__(self, block_size, num_experts, T, K, counts, offsets, flat_tokens, flat_slots,
                 active, meta, host=False):
        self.block_size = block_size
        self.num_experts = num_experts
        self.T, self.K = T, K
        self.counts = counts
        self.offsets = offsets
        self.flat_tokens = flat_tokens
        self.flat_slots = flat_slots
        self.active = active
        self.meta = meta
        self._host = host
        self._cache = None

    def _materialize(self):
        if self._cache is None:
            meta = self.meta.cpu()
            total = int(meta[1])
            offs = self.offsets.cpu().to(torch.int64)
            toks = self.flat_tokens[:total].cpu().to(torch.int64)
            slots = self.flat_slots[:total].cpu().to(torch.int64)
            dev = None if self._host else self.counts.device
            tok_l, slot_l = [], []
            for e in range(self.num_experts):
                a, b = int(offs[e]), int(offs[e + 1])
                tok_l.append(toks[a:b] if dev is None else toks[a:b].to(dev))
                slot_l.append(slots[a:b] if dev is None else slots[a:b].to(dev))
            counts = self.counts.cpu().to(torch.int64)
            self._cache = (tok_l, slot_l, counts if dev is None else counts.to(dev), int(meta[2]))
        return self._cache

    @property
    def tokens(self):
        return self._materialize()[0]

    @property
    def slots(self):
        return self._materialize()[1]

    @property
    def real_counts(self):
        return self._materialize()[2]

    @property
    def total_real(self) -> int:
        return self._materialize()[3]

    def padded_count(self, expert: int) -> int:
        return len(self.tokens[expert])


def align_block(ids, block_size: int, num_experts: int | None = None, backend: str | None = None) -> DispatchPlan:
    """dispatch/__init__.py:89-126: group the surviving (id >= 0) slots by expert
    in ascending (token, slot) order and pad each run with -1 to a multiple of
    block_size.  A deterministic counting sort on the GPU: one CTA for small
    inputs, the layer's multi-CTA permute (two grid-wide passes) above 16384
    slots."""
    _check_backend(backend)
    if block_size < 1:
        raise ContractError("block_size must be >= 1")
    idt, host = _to_device(ids, torch.int64)
    if idt.ndim != 2:
        raise ShapeError("ids must be [T, K]")
    t, k = idt.shape
    if num_experts is None:
        mx = int(idt.max()) if idt.numel() else -1
        num_experts = mx + 1 if mx >= 0 else 0
    dev = idt.device
    cap = t * k + num_experts * (block_size - 1)
    buf = torch.empty(2 * num_experts + 1 + 4 + 2 * max(cap, 1), dtype=torch.int32, device=dev)
    counts = buf[:num_experts]
    offsets = buf[num_experts : 2 * num_experts + 1]
    meta = buf[2 * num_experts + 1 : 2 * num_experts + 5]
    rest = buf[2 * num_experts + 5 :]
    flat_tokens, flat_slots = rest[:cap], rest[max(cap, 1) : max(cap, 1) + cap]
    active = torch.empty(max(num_experts, 1), dtype=torch.int32, device=dev)
    lib = _lib.load()
    ws = _runtime.workspace(lib.beam_group_by_expert_workspace_bytes(t, k, num_experts), dev)
    _lib.check(lib.beam_group_by_expert(idt.data_ptr(), t, k, num_experts, block_size,
                                        counts.data_ptr(), offsets.data_ptr(), flat_tokens.data_ptr(),
                                        flat_slots.data_ptr(), active.data_ptr(), meta.data_ptr(),
                                        ws.data_ptr(), ws.numel(), _runtime.stream_handle(dev)),
               "beam_group_by_expert")
    return DispatchPlan(block_size, num_experts, t, k, counts, offsets, flat_tokens, flat_slots,
                        active, meta, host=host)


def _experts_layer(experts, activation: str, d: int, dtype_hint=None):
    """A beam_layer_t over the given experts (an ExpertBank of a block, or a list
    of reference-layout Expert/triples, packed on the fly)."""
    if isinstance(experts, ExpertBank) and experts._start == 0:
        blk = experts._block
        cfg = blk.cfg
        if cfg.activation != activation:
            cfg = MoEBlockConfig(cfg.d_h, cfg.d_ff, cfg.num_experts, cfg.top_k, 0, False, activation)
        return blk, cfg
    experts = list(experts)
    if not experts:
        raise ContractError("need at least one expert")
    e0 = experts[0]
    g0 = as_torch(e0.w_gate if isinstance(e0, Expert) else e0[0])
    d_h, d_ff = g0.shape
    if d_h != d:
        raise ShapeError("expert d_h does not match h")
    dtype = dtype_hint or (torch.bfloat16 if g0.dtype == torch.bfloat16 else torch.float32)
    cfg = MoEBlockConfig(d_h, d_ff, len(experts), 1, 0, False, activation)
    blk = MoEBlock.from_weights(cfg, torch.zeros(d_h, len(experts)), experts, dtype=dtype)
    return blk, cfg


def _desc_for(blk: MoEBlock, cfg: MoEBlockConfig):
    desc = blk.layer_desc(0.0)
    desc.activation = _lib.BEAM_ACT_SILU if cfg.activation == "silu" else _lib.BEAM_ACT_IDENTITY
    return desc


def grouped_execute(h, plan: DispatchPlan, experts, weights_hat, activation: str = "silu", *,
                    check: bool = True):
    """dispatch/__init__.py:129-157: run each planned expert once over its real
    slots and scatter the ghat-weighted outputs, per token in ascending expert id.
    Raises ContractError exactly where the reference does (:143-144, :152-153);
    the check reads two device flags (one device->host sync), so ``check=False``
    skips it for timing loops (bench_dispatch) and CUDA-graph capture.
    Returns fp32 [T, d] (on the host if h was on the host)."""
    x, host = _to_device(h)
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    t, d = x.shape
    blk, cfg = _experts_layer(experts, activation, d)
    w = as_torch(weights_hat).to(x.device, torch.float32).contiguous()
    if w.shape != (t, plan.num_experts) or plan.T != t:
        raise ShapeError("weights_hat must be [T, num_experts] matching the plan")
    if plan.num_experts > cfg.num_experts:
        raise ShapeError("plan routes to more experts than provided")
    y = torch.empty(t, d, dtype=torch.float32, device=x.device)
    flags = torch.zeros(2, dtype=torch.int32, device=x.device) if check else None
    if t > 0:
        desc = _desc_for(blk, cfg)
        lib = _lib.load()
        ws_bytes = lib.beam_workspace_bytes(ctypes.byref(desc), t, plan.K, plan.block_size)
        ws = _runtime.workspace(ws_bytes, x.device)
        _lib.check(lib.beam_grouped_execute(
            ctypes.byref(desc), x.data_ptr(), _lib.BEAM_BF16 if x.dtype == torch.bfloat16 else _lib.BEAM_F32,
            t, plan.K, plan.block_size, plan.counts.data_ptr(), plan.offsets.data_ptr(),
            plan.flat_tokens.data_ptr(), plan.flat_slots.data_ptr(), plan.active.data_ptr(),
            plan.meta.data_ptr(), w.data_ptr(), y.data_ptr(), flags.data_ptr() if check else None,
            ws.data_ptr(), ws.numel(), _runtime.stream_handle(x.device)), "beam_grouped_execute")
        if check:
            f = flags.cpu()
            if int(f[0]) != 0:
                raise ContractError("weights_hat nonzero count disagrees with plan slots")
            if int(f[1]) != 0:
                raise ContractError("plan routes a zero-weight slot to an expert")
    elif check:
        if int(torch.count_nonzero(w)) != 0:
            raise ContractError("weights_hat nonzero count disagrees with plan slots")
    return y.cpu() if host else y


def naive_execute(h, masked_ids, experts, weights_hat, activation: str = "silu"):
    """dispatch/__init__.py:160-174 semantics (per token, its surviving experts in
    ascending id) through the per-pair entry ``beam_moe_execute`` (no grouping
    plan from the caller, no contract checks)."""
    x, host = _to_device(h)
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    t, d = x.shape
    ids = as_torch(masked_ids, torch.int64).to(x.device)
    w = as_torch(weights_hat).to(x.device, torch.float32)
    blk, cfg = _experts_layer(experts, activation, d)
    k = ids.shape[1]
    ids32 = ids.clamp(min=-1).to(torch.int32).contiguous()
    wk = torch.where(ids >= 0, torch.gather(w, 1, ids.clamp(min=0)), torch.zeros((), device=x.device))
    wk = wk.to(torch.float32).contiguous()
    y = execute_routed(blk, x, ids32, wk, cfg=cfg)
    return y.cpu() if host else y


def execute_routed(blk: MoEBlock, x: torch.Tensor, ids32: torch.Tensor, w: torch.Tensor, cfg=None) -> torch.Tensor:
    """y[t] = sum_k (ascending id) w[t,k] * E_{ids[t,k]}(x[t]) via beam_moe_execute."""
    cfg = cfg or blk.cfg
    t = x.shape[0]
    k = ids32.shape[1]
    y = torch.empty(t, cfg.d_h, dtype=torch.float32, device=x.device)
    if t == 0:
        return y
    desc = _desc_for(blk, cfg)
    lib = _lib.load()
    ws_bytes = lib.beam_workspace_bytes(ctypes.byref(desc), t, k, 1)
    ws = _runtime.workspace(ws_bytes, x.device)
    _lib.check(lib.beam_moe_execute(ctypes.byref(desc), x.data_ptr(),
                                    _lib.BEAM_BF16 if x.dtype == torch.bfloat16 else _lib.BEAM_F32,
                                    t, k, ids32.data_ptr(), w.data_ptr(), y.data_ptr(), ws.data_ptr(),
                                    ws.numel(), _runtime.stream_handle(x.device)), "beam_moe_execute")
    return y


@dataclass
class BenchRow:
    """dispatch/__init__.py:177-183."""

    active_fraction: float
    slots_executed: int
    wall_time_ns_min: int
    wall_time_ns_mean: float
    backend: str


BENCH_CSV_HEADER = "active_fraction,slots_executed,wall_time_ns_min,wall_time_ns_mean"


def bench_dispatch(num_tokens, num_experts, top_k, d_h, d_ff, active_fractions, repetitions,
                   block_size: int = 16, seed: int = 0, backend: str | None = None,
                   dtype=torch.bfloat16) -> list:
    """dispatch/__init__.py:189-245: time grouped_execute at synthetic activity
    levels — exactly round(fraction*T*K) surviving slots, plans built outside the
    timed region, min over repetitions.  Timed with CUDA events on the stream."""
    _check_backend(backend)
    for f in active_fractions:
        if not 0.0 < f <= 1.0:
            raise ContractError("active fractions must lie in (0, 1]")
    rng = np.random.default_rng(seed)
    dev = _default_device()
    h = torch.from_numpy(rng.normal(0.0, 1.0, (num_tokens, d_h))).to(dev, torch.float32)
    cfg = MoEBlockConfig(d_h, d_ff, num_experts, top_k, has_norm=False)
    experts = [Expert.init_random(d_h, d_ff, rng) for _ in range(num_experts)]
    blk = MoEBlock.from_weights(cfg, np.zeros((d_h, num_experts)), experts, dtype=dtype)
    base_ids = topk_select(torch.from_numpy(rng.normal(0.0, 1.0, (num_tokens, num_experts))).float(), top_k).cpu().numpy()
    base_weights = rng.uniform(0.1, 1.0, (num_tokens, top_k))
    rows = []
    for fraction in active_fractions:
        keep_count = int(round(fraction * num_tokens * top_k))
        keep_flat = np.zeros(num_tokens * top_k, dtype=bool)
        keep_flat[rng.permutation(num_tokens * top_k)[:keep_count]] = True
        keep = keep_flat.reshape(num_tokens, top_k)
        masked_ids = np.where(keep, base_ids, np.int64(-1))
        weights_hat = np.zeros((num_tokens, num_experts))
        r_idx = np.repeat(np.arange(num_tokens), top_k)[keep_flat]
        c_idx = base_ids.reshape(-1)[keep_flat]
        weights_hat[r_idx, c_idx] = base_weights.reshape(-1)[keep_flat]
        plan = align_block(torch.from_numpy(masked_ids).to(dev), block_size, num_experts)
        w = torch.from_numpy(weights_hat).to(dev, torch.float32)
        grouped_execute(h, plan, blk.experts, w)  # warm-up (with the contract checks)
        timings = []
        for _ in range(repetitions):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            grouped_execute(h, plan, blk.experts, w, check=False)
            e.record()
            e.synchronize()
            timings.append(int(s.elapsed_time(e) * 1e6))
        rows.append(BenchRow(fraction, plan.total_real, min(timings), float(np.mean(timings)), BACKEND_NAME))
    return rows
