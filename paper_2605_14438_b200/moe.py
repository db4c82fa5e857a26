"""MoE block: configuration, expert container, routing (B200, CUDA only).

Mirrors the reference's public surface in /root/reference/pkg/src/beamoe/moe.py:
``MoEBlockConfig`` (:45-65), ``Expert`` (:68-87), ``RouterDecision`` (:103-113),
``topk_select`` (:116-119), ``topk_route`` (:122-137) and ``MoEBlock``
(:161-220), with parameters held on the GPU in the packed layouts the sm_100a
kernels read (``include/beam_b200.h``, ``beam_layer_t``):

* ``gate_wT``  f32  [2N, d_pad]        router_w^T stacked over mask_w^T
* ``w_gu``     bf16 [E, 2 f_pad, d_pad] gate/up rows interleaved in 32-row groups
* ``w_down``   bf16 [E, d_pad, f_pad]  w_down^T (row = output channel)

``MoEBlock(cfg, rng)`` draws its parameters with the reference's numpy
generator in the reference's order (router, then gate/up/down per expert, then
shared experts; moe.py:177-191), so a reference block built from the same seed
holds the same values (before the bf16 cast of the experts).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, _runtime
from .tensor import ContractError, ShapeError, as_torch

ACTIVATIONS = ("silu", "identity")
_ACT_CODE = {"silu": _lib.BEAM_ACT_SILU, "identity": _lib.BEAM_ACT_IDENTITY}


def _default_device():
    if not torch.cuda.is_available():
        raise _lib.BeamNativeError("no CUDA device visible: the BEAM B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class MoEBlockConfig:
    """moe.py:45-65 (same fields, defaults and validation)."""

    d_h: int
    d_ff: int
    num_experts: int
    top_k: int
    num_shared: int = 0
    has_norm: bool = True
    activation: str = "silu"

    def __post_init__(self):
        if self.d_h < 1 or self.d_ff < 1:
            raise ContractError("d_h and d_ff must be positive")
        if self.num_experts < 1:
            raise ContractError("need at least one expert")
        if not 1 <= self.top_k <= self.num_experts:
            raise ContractError("top_k must satisfy 1 <= K <= N")
        if self.num_shared < 0:
            raise ContractError("num_shared must be non-negative")
        if self.activation not in ACTIVATIONS:
            raise ContractError(f"unknown activation {self.activation!r}")

    @property
    def d_pad(self) -> int:
        return (self.d_h + 7) // 8 * 8

    @property
    def f_pad(self) -> int:
        return (self.d_ff + 15) // 16 * 16


@dataclass
class Expert:
    """One gated-linear-unit expert in the reference layout (moe.py:68-87):
    w_gate [d, f], w_up [d, f], w_down [f, d]."""

    w_gate: torch.Tensor
    w_up: torch.Tensor
    w_down: torch.Tensor

    @classmethod
    def init_random(cls, d_h: int, d_ff: int, rng: np.random.Generator, std: float = 0.02) -> "Expert":
        """moe.py:76-84 — same draws, same order."""
        return cls(
            w_gate=torch.from_numpy(rng.normal(0.0, std, (d_h, d_ff))),
            w_up=torch.from_numpy(rng.normal(0.0, std, (d_h, d_ff))),
            w_down=torch.from_numpy(rng.normal(0.0, std, (d_ff, d_h))),
        )

    def tensors(self) -> list:
        return [self.w_gate, self.w_up, self.w_down]


@dataclass
class RouterDecision:
    """moe.py:103-113: logits [T, N] f32, topk_indices [T, K] int64 (rank order),
    weights [T, N] f32 (softmax over the top-K set, exactly 0 elsewhere)."""

    logits: torch.Tensor
    topk_indices: torch.Tensor
    weights: torch.Tensor


# ---------------------------------------------------------------------------
# packing
# ---------------------------------------------------------------------------


def pack_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor, d_pad: int, f_pad: int) -> torch.Tensor:
    """[E, d, f] x2 -> [E, 2 f_pad, d_pad]; packed row 32b+i = gate feature 16b+i,
    32b+16+i = up feature 16b+i (zero padding)."""
    e, d, f = w_gate.shape
    out = torch.zeros(e, f_pad // 16, 2, 16, d_pad, dtype=w_gate.dtype, device=w_gate.device)
    g = torch.zeros(e, f_pad, d_pad, dtype=w_gate.dtype, device=w_gate.device)
    g[:, :f, :d] = w_gate.transpose(1, 2)
    out[:, :, 0] = g.view(e, f_pad // 16, 16, d_pad)
    g.zero_()
    g[:, :f, :d] = w_up.transpose(1, 2)
    out[:, :, 1] = g.view(e, f_pad // 16, 16, d_pad)
    return out.view(e, 2 * f_pad, d_pad)


def unpack_gate_up(w_gu: torch.Tensor, d: int, f: int):
    e, two_f, d_pad = w_gu.shape
    v = w_gu.view(e, two_f // 32, 2, 16, d_pad)
    gate = v[:, :, 0].reshape(e, -1, d_pad)[:, :f, :d].transpose(1, 2)
    up = v[:, :, 1].reshape(e, -1, d_pad)[:, :f, :d].transpose(1, 2)
    return gate, up


def pack_down(w_down: torch.Tensor, d_pad: int, f_pad: int) -> torch.Tensor:
    """[E, f, d] -> [E, d_pad, f_pad] (transposed, zero padding)."""
    e, f, d = w_down.shape
    out = torch.zeros(e, d_pad, f_pad, dtype=w_down.dtype, device=w_down.device)
    out[:, :d, :f] = w_down.transpose(1, 2)
    return out


class ExpertBank:
    """The routed (and shared) experts of a block, stored packed on the GPU.

    Indexing returns an ``Expert`` view in the reference layout (unpacked
    copy); assigning ``bank[i] = Expert(...)`` repacks that expert."""

    def __init__(self, block: "MoEBlock", start: int, count: int):
        self._block = block
        self._start = start
        self._count = count

    def __len__(self) -> int:
        return self._count

    def _index(self, i: int) -> int:
        if i < 0:
            i += self._count
        if not 0 <= i < self._count:
            raise IndexError(i)
        return self._start + i

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(self._count))]
        b = self._block
        j = self._index(i)
        g, u = unpack_gate_up(b.w_gu[j : j + 1], b.cfg.d_h, b.cfg.d_ff)
        d = b.w_down[j, : b.cfg.d_h, : b.cfg.d_ff].transpose(0, 1)
        return Expert(w_gate=g[0].contiguous(), w_up=u[0].contiguous(), w_down=d.contiguous())

    def __setitem__(self, i: int, expert: Expert) -> None:
        self._block._set_expert(self._index(i), expert)

    def __iter__(self):
        return (self[i] for i in range(self._count))


class MoEBlock:
    """Parameter container for one MoE layer (moe.py:161-220), on the GPU.

    ``dtype`` is the expert weight / expert-input dtype (bf16 or fp32); routers
    and the norm weight are fp32.  ``mask_router`` (``beam.MaskRouter``) is
    attached by the caller, as in the reference."""

    def __init__(self, cfg: MoEBlockConfig, rng: np.random.Generator | None = None,
                 extra_router_cols: int = 0, init_std: float = 0.02, *,
                 dtype: torch.dtype = torch.bfloat16, device=None, _empty: bool = False,
                 _router_only: bool = False):
        if extra_router_cols < 0:
            raise ContractError("extra_router_cols must be >= 0")
        if dtype not in (torch.bfloat16, torch.float32):
            raise ContractError("expert dtype must be torch.bfloat16 or torch.float32")
        self.cfg = cfg
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else _default_device()
        n_all = cfg.num_experts + cfg.num_shared
        if _router_only:
            # gating only (expert-parallel ranks): the gate kernels never read the
            # expert weights, so none are allocated (placeholders keep the
            # descriptor's pointers valid)
            self.w_gu = torch.zeros(1, dtype=dtype, device=self.device)
            self.w_down = torch.zeros(1, dtype=dtype, device=self.device)
            _empty = True
        else:
            self.w_gu = torch.zeros(n_all, 2 * cfg.f_pad, cfg.d_pad, dtype=dtype, device=self.device)
            self.w_down = torch.zeros(n_all, cfg.d_pad, cfg.f_pad, dtype=dtype, device=self.device)
        # moe.py:164-178: num_experts + extra_router_cols columns (the extra ones are the
        # null experts of ada_moe routing, baselines.py:212-225)
        self.extra_router_cols = extra_router_cols
        self.router_w = torch.zeros(cfg.d_h, cfg.num_experts + extra_router_cols, dtype=torch.float32,
                                    device=self.device)
        self.norm_w = torch.ones(cfg.d_h, dtype=torch.float32, device=self.device) if cfg.has_norm else None
        self._mask_router = None
        self._pack_key = None
        self._desc = None
        if _empty:
            return
        rng = rng if rng is not None else np.random.default_rng()
        # moe.py:177-191: router, experts (gate, up, down each), shared — same draws
        self.router_w.copy_(torch.from_numpy(
            rng.normal(0.0, init_std, (cfg.d_h, cfg.num_experts + extra_router_cols))))
        for i in range(n_all):
            self._set_expert(i, Expert.init_random(cfg.d_h, cfg.d_ff, rng, init_std))

    # -- construction helpers -------------------------------------------------
    @classmethod
    def from_weights(cls, cfg: MoEBlockConfig, router_w, experts, shared=(), norm_w=None,
                     mask_w=None, tau: float = 0.5, *, dtype=torch.bfloat16, device=None) -> "MoEBlock":
        """Build from reference-layout arrays: router_w [d, N]; experts/shared as
        (w_gate [d,f], w_up [d,f], w_down [f,d]) triples or ``Expert``s, or as
        stacked [E, d, f]/[E, d, f]/[E, f, d] tensors (3-tuple of 3-D arrays)."""
        from .beam import MaskRouter

        rw = as_torch(router_w)
        extra = rw.shape[-1] - cfg.num_experts
        if rw.ndim != 2 or rw.shape[0] != cfg.d_h or extra < 0:
            raise ShapeError("router_w must be [d_h, num_experts (+ null columns)]")
        b = cls(cfg, extra_router_cols=extra, dtype=dtype, device=device, _empty=True)
        b.router_w.copy_(rw.to(torch.float32))
        if norm_w is not None and b.norm_w is not None:
            b.norm_w.copy_(as_torch(norm_w).to(torch.float32))
        b._set_all_experts(experts, 0, cfg.num_experts)
        if cfg.num_shared:
            b._set_all_experts(shared, cfg.num_experts, cfg.num_shared)
        if mask_w is not None:
            b.mask_router = MaskRouter(as_torch(mask_w).to(torch.float32).to(b.device), tau)
        return b

    @classmethod
    def random(cls, cfg: MoEBlockConfig, seed: int = 0, init_std: float = 0.02, *,
               dtype=torch.bfloat16, device=None) -> "MoEBlock":
        """Random-init on the device (torch generator; fast for large shapes).
        Same distribution as the reference init (N(0, init_std)), not the same draws."""
        b = cls(cfg, dtype=dtype, device=device, _empty=True)
        g = torch.Generator(device=b.device)
        g.manual_seed(seed)
        n_all = cfg.num_experts + cfg.num_shared
        b.router_w.normal_(0.0, init_std, generator=g)
        for i in range(n_all):  # per expert to bound temporaries
            wg = torch.empty(1, cfg.d_h, cfg.d_ff, device=b.device).normal_(0.0, init_std, generator=g)
            wu = torch.empty(1, cfg.d_h, cfg.d_ff, device=b.device).normal_(0.0, init_std, generator=g)
            wd = torch.empty(1, cfg.d_ff, cfg.d_h, device=b.device).normal_(0.0, init_std, generator=g)
            b.w_gu[i : i + 1] = pack_gate_up(wg.to(dtype), wu.to(dtype), cfg.d_pad, cfg.f_pad)
            b.w_down[i : i + 1] = pack_down(wd.to(dtype), cfg.d_pad, cfg.f_pad)
        return b

    def _set_expert(self, i: int, e) -> None:
        if isinstance(e, Expert):
            g, u, d = e.w_gate, e.w_up, e.w_down
        else:
            g, u, d = e
        cfg = self.cfg
        g = as_torch(g).to(self.device, self.dtype)
        u = as_torch(u).to(self.device, self.dtype)
        d = as_torch(d).to(self.device, self.dtype)
        if g.shape != (cfg.d_h, cfg.d_ff) or u.shape != (cfg.d_h, cfg.d_ff) or d.shape != (cfg.d_ff, cfg.d_h):
            raise ShapeError("expert weights must be w_gate/w_up [d_h, d_ff], w_down [d_ff, d_h]")
        self.w_gu[i : i + 1] = pack_gate_up(g[None], u[None], cfg.d_pad, cfg.f_pad)
        self.w_down[i : i + 1] = pack_down(d[None], cfg.d_pad, cfg.f_pad)

    def _set_all_experts(self, experts, start: int, count: int) -> None:
        if (isinstance(experts, (tuple, list)) and len(experts) == 3
                and isinstance(experts[0], (np.ndarray, torch.Tensor)) and experts[0].ndim == 3):
            g, u, d = (as_torch(x).to(self.device, self.dtype) for x in experts)
            self.w_gu[start : start + count] = pack_gate_up(g, u, self.cfg.d_pad, self.cfg.f_pad)
            self.w_down[start : start + count] = pack_down(d, self.cfg.d_pad, self.cfg.f_pad)
            return
        experts = list(experts)
        if len(experts) != count:
            raise ShapeError(f"expected {count} experts, got {len(experts)}")
        for i, e in enumerate(experts):
            self._set_expert(start + i, e)

    # -- reference surface ------------------------------------------------------
    @property
    def experts(self) -> ExpertBank:
        return ExpertBank(self, 0, self.cfg.num_experts)

    @property
    def shared(self) -> ExpertBank:
        return ExpertBank(self, self.cfg.num_experts, self.cfg.num_shared)

    @property
    def mask_router(self):
        return self._mask_router

    @mask_router.setter
    def mask_router(self, router) -> None:
        if router is not None:
            router.weight = as_torch(router.weight).to(self.device, torch.float32).contiguous()
            if tuple(router.weight.shape) != (self.cfg.d_h, self.cfg.num_experts):
                raise ShapeError("mask router weight must be [d_h, num_experts]")
        self._mask_router = router

    def named_tensors(self, prefix: str = "") -> list:
        """moe.py:194-212 (reference layout views/copies)."""
        out = [(f"{prefix}router_w", self.router_w)]
        for i, e in enumerate(self.experts):
            out += [(f"{prefix}experts.{i}.w_gate", e.w_gate), (f"{prefix}experts.{i}.w_up", e.w_up),
                    (f"{prefix}experts.{i}.w_down", e.w_down)]
        for i, e in enumerate(self.shared):
            out += [(f"{prefix}shared.{i}.w_gate", e.w_gate), (f"{prefix}shared.{i}.w_up", e.w_up),
                    (f"{prefix}shared.{i}.w_down", e.w_down)]
        if self.norm_w is not None:
            out.append((f"{prefix}norm_w", self.norm_w))
        if self.mask_router is not None:
            out.append((f"{prefix}mask_w", self.mask_router.weight))
        return out

    def normalize(self, h) -> torch.Tensor:
        """moe.py:214-215 — RMS norm on the GPU (fp32 result)."""
        from .beam import rms_norm

        return rms_norm(h, self.norm_w) if self.norm_w is not None else as_torch(h)

    # -- kernel descriptor --------------------------------------------------------
    def layer_desc(self, mask_threshold: float = 0.0) -> _lib.LayerDesc:
        """The packed ``beam_layer_t`` (re-packed when a router weight changed)."""
        cfg = self.cfg
        mr = self._mask_router
        mw = mr.weight if mr is not None else None
        key = (self.router_w._version, id(mw), mw._version if mw is not None else -1,
               self.norm_w._version if self.norm_w is not None else -1)
        if key != self._pack_key:
            # repacked in place: captured CUDA graphs keep a valid pointer
            # rows: router [N (+ null columns)], mask router at rows [N, 2N) (beam_route_t)
            nr = self.router_w.shape[1]
            if getattr(self, "gate_wT", None) is None:
                self.gate_wT = torch.zeros(max(2 * cfg.num_experts, nr), cfg.d_pad, dtype=torch.float32,
                                           device=self.device)
            gate = self.gate_wT
            gate.zero_()
            gate[:nr, : cfg.d_h] = self.router_w.t()
            if mw is not None:
                if nr > cfg.num_experts:
                    raise ContractError("a block with null-expert router columns has no mask router")
                gate[cfg.num_experts : 2 * cfg.num_experts, : cfg.d_h] = mw.t()
            # the prefill tensor-core router's bf16 hi/mid/lo split of (norm_w o gate rows),
            # built once here instead of on every prefill call
            rows = gate.shape[0]
            if getattr(self, "gate_w3", None) is None or self.gate_w3.shape[1] != rows:
                self.gate_w3 = torch.empty(3, rows, cfg.d_pad, dtype=torch.bfloat16, device=self.device)
            if self.device.type == "cuda":
                _lib.check(_lib.load().beam_router_split(
                    gate.data_ptr(), self.norm_w.data_ptr() if self.norm_w is not None else None, rows, cfg.d_h,
                    cfg.d_pad, self.gate_w3.data_ptr(), _runtime.stream_handle(self.device)), "beam_router_split")
            self._pack_key = key
        ck = (key, mask_threshold, id(self.norm_w), id(self.w_gu), id(self.w_down), id(self.gate_wT),
              id(getattr(self, "gate_w3", None)))
        cached = getattr(self, "_desc_cache", None)
        if cached is not None and cached[0] == ck:
            return cached[1]
        d = _lib.LayerDesc()
        d.d_h, d.d_ff, d.num_experts, d.top_k = cfg.d_h, cfg.d_ff, cfg.num_experts, cfg.top_k
        d.num_shared = cfg.num_shared
        d.has_norm = 1 if self.norm_w is not None else 0
        d.activation = _ACT_CODE[cfg.activation]
        d.wdtype = _lib.BEAM_BF16 if self.dtype == torch.bfloat16 else _lib.BEAM_F32
        d.mask_threshold = mask_threshold
        d.norm_w = self.norm_w.data_ptr() if self.norm_w is not None else None
        d.gate_wT = self.gate_wT.data_ptr()
        d.w_gu = self.w_gu.data_ptr()
        d.w_down = self.w_down.data_ptr()
        if self.device.type == "cuda":
            d.gate_w3 = self.gate_w3.data_ptr()
            d.gate_w3_cols = self.gate_w3.shape[1]
        self._desc_cache = (ck, d)
        return d

    def weight_bytes(self) -> int:
        return (self.w_gu.numel() + self.w_down.numel()) * self.w_gu.element_size()


# ---------------------------------------------------------------------------
# routing
# ---------------------------------------------------------------------------


def _gate_call(x, gate_wT_rows_router, gate_wT_rows_mask, k: int, norm_w=None,
               mask_threshold: float = 0.0, want=("logits", "topk_ids", "weights")):
    """Run beam_gate with ad-hoc router/mask weights ([d, N] each or None)."""
    x = as_torch(x)
    dev = x.device if x.is_cuda else _default_device()
    x = x.to(dev)
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    x = x.contiguous()
    if x.ndim != 2:
        raise ShapeError("expected [T, d] activations")
    t, d = x.shape
    rw = gate_wT_rows_router if gate_wT_rows_router is not None else None
    n = (rw if rw is not None else gate_wT_rows_mask).shape[1]
    cfg = MoEBlockConfig(d_h=d, d_ff=16, num_experts=n, top_k=k, has_norm=norm_w is not None)
    d_pad = cfg.d_pad
    gate = torch.zeros(2 * n, d_pad, dtype=torch.float32, device=dev)
    if rw is not None:
        gate[:n, :d] = as_torch(rw).to(dev, torch.float32).t()
    if gate_wT_rows_mask is not None:
        gate[n:, :d] = as_torch(gate_wT_rows_mask).to(dev, torch.float32).t()
    dummy = torch.zeros(16, dtype=torch.float32, device=dev)
    desc = _lib.LayerDesc(d, 16, n, k, 0, 1 if norm_w is not None else 0, 0, _lib.BEAM_F32,
                          mask_threshold,
                          as_torch(norm_w).to(dev, torch.float32).contiguous().data_ptr() if norm_w is not None else None,
                          gate.data_ptr(), dummy.data_ptr(), dummy.data_ptr())
    outs = {}
    o = _lib.Outputs()
    for name in want:
        if name in ("topk_ids", "masked_ids"):
            outs[name] = torch.empty(t, k, dtype=torch.int64, device=dev)
        else:
            outs[name] = torch.empty(t, n, dtype=torch.float32, device=dev)
        setattr(o, name, outs[name].data_ptr())
    lib = _lib.load()
    ws_bytes = lib.beam_workspace_bytes(ctypes.byref(desc), t, 0, 1)
    ws = _runtime.workspace(ws_bytes, dev)
    _lib.check(lib.beam_gate(ctypes.byref(desc), x.data_ptr(),
                             _lib.BEAM_BF16 if x.dtype == torch.bfloat16 else _lib.BEAM_F32, t,
                             ctypes.byref(o), ws.data_ptr(), ws.numel(), _runtime.stream_handle(dev)),
               "beam_gate")
    return outs


def topk_route(x, router_weights, k: int) -> RouterDecision:
    """moe.py:122-137 on the GPU: fp32 logits, stable top-K (desc value, ties ->
    lower index), softmax over exactly the K kept logits."""
    n = as_torch(router_weights).shape[-1]
    if not 1 <= k <= n:
        raise ContractError("top_k must satisfy 1 <= K <= N")
    o = _gate_call(x, router_weights, None, k)
    return RouterDecision(logits=o["logits"], topk_indices=o["topk_ids"], weights=o["weights"])


def topk_select(logits, k: int) -> torch.Tensor:
    """moe.py:116-119: indices of the k largest entries per row, ties won by the
    lower index (numpy's stable argsort order on -logits: NaN last, -0.0 == +0.0).
    fp64 logits are compared in fp64 (``beam_topk_select``, one warp per row)."""
    lg = as_torch(logits)
    n = lg.shape[-1]
    if not 1 <= k <= n:
        raise ContractError("top_k must satisfy 1 <= K <= N")
    dev = lg.device if lg.is_cuda else _default_device()
    dt = torch.float64 if lg.dtype == torch.float64 else torch.float32
    x = lg.to(dev, dt).contiguous()
    lead = x.shape[:-1]
    x = x.reshape(-1, n)
    out = torch.empty(x.shape[0], k, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().beam_topk_select(x.data_ptr(), _lib.BEAM_F64 if dt == torch.float64 else _lib.BEAM_F32,
                                            x.shape[0], n, k, out.data_ptr(), _runtime.stream_handle(dev)),
               "beam_topk_select")
    return out.reshape(*lead, k)
