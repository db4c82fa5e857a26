"""Binary expert-activation masking: the BEAM layer forward on B200.

Mirrors /root/reference/pkg/src/beamoe/beam.py: ``MaskRouter`` (:33-48),
``MaskDecision`` (:51-65), ``mask_forward`` (:68-72) and
``beam_block_forward`` (:127-165).  The whole layer runs as one C-ABI call,
``beam_layer_forward`` (include/beam_b200.h), i.e. the sm_100a kernel chain
gating -> masked permute -> grouped SwiGLU experts -> weighted combine.

Threshold rule: one fp32 predicate ``a >= 0`` decides both the
mask bit and whether the routed id survives (tau = 0.5).  The reference ties
the ids to ``a >= 0`` (dispatch.mask_route) but the mask to ``sigmoid(a) >= tau``;
for tau != 0.5 the two disagree and its grouped_execute raises ContractError
(dispatch/__init__.py:143-144), so ``beam_block_forward`` rejects tau != 0.5 up
front.  ``mask_forward`` alone honours any tau via a >= logit(tau).
"""

from __future__ import annotations

import collections
import ctypes
import functools
import math
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, _runtime
from .moe import MoEBlock, RouterDecision, _default_device, _gate_call
from .tensor import ContractError, ShapeError, as_torch


@dataclass
class MaskRouter:
    """beam.py:33-48: linear mask scorer W_m [d_h, N] (fp32 on the GPU);
    zero-init opens every mask (a = 0 >= 0)."""

    weight: torch.Tensor
    tau: float = 0.5

    def __post_init__(self):
        if not 0.0 < self.tau < 1.0:
            raise ContractError("tau must lie in (0, 1)")
        self.weight = as_torch(self.weight)

    @classmethod
    def zero_init(cls, d_h: int, num_experts: int, tau: float = 0.5, device=None) -> "MaskRouter":
        dev = torch.device(device) if device is not None else _default_device()
        return cls(torch.zeros(d_h, num_experts, dtype=torch.float32, device=dev), tau)


@dataclass
class MaskDecision:
    """beam.py:51-65: pre_activation a, raw_mask sigmoid(a), mask in {0., 1.}."""

    pre_activation: torch.Tensor
    raw_mask: torch.Tensor
    mask: torch.Tensor

    @property
    def binary_mask(self) -> torch.Tensor:
        return self.mask.to(torch.int64)


def _threshold(tau: float) -> float:
    """a >= logit(tau)  <=>  sigmoid(a) >= tau (exactly 0.0 for tau = 0.5)."""
    return 0.0 if tau == 0.5 else float(np.float32(math.log(tau / (1.0 - tau))))


def mask_forward(x, router: MaskRouter) -> MaskDecision:
    """beam.py:68-72 on the GPU: a = x W_m (fp32), raw = sigmoid(a), m = a >= logit(tau)."""
    w = as_torch(router.weight)
    o = _gate_call(x, None, w, 1, mask_threshold=_threshold(router.tau),
                   want=("pre_activation", "raw_mask", "mask"))
    return MaskDecision(pre_activation=o["pre_activation"], raw_mask=o["raw_mask"], mask=o["mask"])


def rms_norm(h, weight, eps: float = 1e-6) -> torch.Tensor:
    """tensor.py:485-508 forward on the GPU (fp32 output)."""
    if eps != 1e-6:
        raise ContractError("the sm_100a kernel implements the reference eps = 1e-6")
    x = as_torch(h)
    dev = x.device if x.is_cuda else _default_device()
    x = x.to(dev)
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    x = x.contiguous()
    w = as_torch(weight).to(dev, torch.float32).contiguous()
    t, d = x.shape
    out = torch.empty(t, d, dtype=torch.float32, device=dev)
    lib = _lib.load()
    _lib.check(lib.beam_rms_norm(x.data_ptr(), _lib.BEAM_BF16 if x.dtype == torch.bfloat16 else _lib.BEAM_F32,
                                 t, d, w.data_ptr(), out.data_ptr(), _runtime.stream_handle(dev)),
               "beam_rms_norm")
    return out


# ---------------------------------------------------------------------------
# layer forward
# ---------------------------------------------------------------------------


_EXPERT_PATH = [0]  # beam_set_expert_path mode (changes the workspace layout)
_F32_FIELDS = ("logits", "weights", "pre_activation", "raw_mask", "mask")
_ID_FIELDS = ("topk_ids", "masked_ids")


@functools.lru_cache(maxsize=256)
def _outputs_layout(t: int, d: int, n: int, k: int, out_dtype: torch.dtype):
    """Byte layout of one layer's outputs in a single flat buffer: the decision
    outputs first (f32 [5, T, N] block, int64 [2, T, K] block), then `out`
    [T, d] — so the decisions are one contiguous range a host caller can copy
    while the experts still run.  Returns (total, f32_off, ids_off, out_off,
    field byte offsets)."""
    es = torch.empty(0, dtype=out_dtype).element_size()
    f32_off = 0
    ids_off = (f32_off + 5 * t * n * 4 + 255) // 256 * 256
    out_off = (ids_off + 2 * t * k * 8 + 255) // 256 * 256
    total = out_off + t * d * es
    offs = {name: f32_off + i * t * n * 4 for i, name in enumerate(_F32_FIELDS)}
    offs.update({name: ids_off + i * t * k * 8 for i, name in enumerate(_ID_FIELDS)})
    offs["out"] = out_off
    return total, f32_off, ids_off, out_off, tuple(offs.items())


class LayerOutputs:
    """All outputs of one layer call carved from ONE flat buffer, so a host
    caller pays one device->host copy for the decisions and one for `out`.
    Views are built on first use, all at once (a device-side staging copy never
    builds any)."""

    def __init__(self, t: int, d: int, n: int, k: int, out_dtype: torch.dtype, device, pin=False):
        self.shape = (t, d, n, k, out_dtype)
        self.nbytes, self._f32_off, self._ids_off, self.out_off, self._offs = _outputs_layout(t, d, n, k, out_dtype)
        kw = dict(dtype=torch.uint8, device=device)
        self.buf = torch.empty(self.nbytes, pin_memory=pin, **kw) if pin else torch.empty(self.nbytes, **kw)
        self._views = None

    def _build(self):
        t, d, n, k, dt = self.shape
        b = self.buf
        f = b[self._f32_off : self._f32_off + 5 * t * n * 4].view(torch.float32).view(5, t, n).unbind(0)
        ids = b[self._ids_off : self._ids_off + 2 * t * k * 8].view(torch.int64).view(2, t, k).unbind(0)
        v = dict(zip(_F32_FIELDS, f))
        v.update(zip(_ID_FIELDS, ids))
        v["out"] = b[self.out_off :].view(dt).view(t, d)
        self._views = v
        return v

    def __getitem__(self, name):
        v = self._views if self._views is not None else self._build()
        return v[name]

    @property
    def views(self):
        return dict(self._views if self._views is not None else self._build())

    def ctypes_outputs(self, decision_event=None, out_ptr=None) -> _lib.Outputs:
        base = self.buf.data_ptr()
        o = _lib.Outputs(**{name: base + off for name, off in self._offs})
        if decision_event is not None:
            o.decision_event = decision_event
        if out_ptr is not None:
            o.out = out_ptr
        return o

    def copy_from(self, other: "LayerOutputs") -> None:
        self.buf.copy_(other.buf, non_blocking=True)

    def copy_decisions_from(self, other: "LayerOutputs") -> None:
        self.buf[: self.out_off].copy_(other.buf[: other.out_off], non_blocking=True)

    def copy_out_from(self, other: "LayerOutputs") -> None:
        self.buf[self.out_off :].copy_(other.buf[other.out_off :], non_blocking=True)


_TLS = threading.local()


def _copy_stream(dev: torch.device):
    """(side stream, decision event) of a device for the host-output path (per
    host thread)."""
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    per = getattr(_TLS, "copy", None)
    if per is None:
        per = _TLS.copy = {}
    if key not in per:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dev))  # instantiates the CUDA event (lazy in torch)
        per[key] = (torch.cuda.Stream(dev), ev)
    return per[key]


def _check_block(block: MoEBlock):
    if block.mask_router is None:
        raise ContractError("block has no mask router (attach beam.MaskRouter)")
    if block.mask_router.tau != 0.5:
        raise ContractError(
            "beam_block_forward: mask_route keeps ids with a >= 0 (tau = 0.5) while the mask uses "
            f"sigmoid(a) >= tau = {block.mask_router.tau}; the reference rejects the mismatch "
            "(dispatch/__init__.py:143-144)")


_WS_CACHE: dict = {}


def _ws_bytes(desc, t: int, block_size: int) -> int:
    """beam_workspace_bytes, memoised on the values it depends on."""
    key = (desc.d_h, desc.d_ff, desc.num_experts, desc.top_k, desc.num_shared, desc.wdtype, desc.has_norm,
           desc.activation, t, block_size, _EXPERT_PATH[0])
    v = _WS_CACHE.get(key)
    if v is None:
        v = _WS_CACHE[key] = _lib.load().beam_workspace_bytes(ctypes.byref(desc), t, 0, block_size)
    return v


def layer_forward_into(x: torch.Tensor, block: MoEBlock, outs: LayerOutputs,
                       block_size: int = 16, decision_event=None, out_ptr=None) -> None:
    """Launch the fused layer on ``x`` (device, [T, d], bf16/f32) writing into
    preallocated ``outs`` — no allocation, no sync (CUDA-graph capturable).
    ``decision_event`` (a torch.cuda.Event): recorded once the decision outputs
    are complete; ``out_ptr``: write `out` there instead (e.g. mapped pinned
    host memory)."""
    t = x.shape[0]
    desc = block.layer_desc(0.0)
    lib = _lib.load()
    ws = _runtime.workspace(_ws_bytes(desc, t, block_size), x.device)
    o = outs.ctypes_outputs(decision_event.cuda_event if decision_event is not None else None, out_ptr)
    _lib.check(lib.beam_layer_forward(ctypes.byref(desc), x.data_ptr(),
                                      _lib.BEAM_BF16 if x.dtype == torch.bfloat16 else _lib.BEAM_F32,
                                      t, block_size, ctypes.byref(o), ws.data_ptr(), ws.numel(),
                                      _runtime.stream_handle(x.device)),
               "beam_layer_forward")


class _HostSession:
    """Host-buffer fast path of beam_block_forward for one (block, T, dtype,
    block_size): fixed device rows / outputs and the layer's kernels captured
    ONCE as a CUDA graph (workspace of a private stream).  A call is then: H2D of
    the rows, one graph launch, one D2H of all outputs into fresh pinned memory —
    the per-call host work is a few microseconds instead of the eager launch
    sequence (~35 us of Python + ctypes + 4-5 kernel launches)."""

    def __init__(self, block: MoEBlock, t: int, dtype: torch.dtype, block_size: int, dev: torch.device):
        cfg = block.cfg
        self.lock = threading.Lock()
        self.x = torch.zeros(t, cfg.d_h, dtype=dtype, device=dev)
        self.outs = LayerOutputs(t, cfg.d_h, cfg.num_experts, cfg.top_k, dtype, dev)
        self.stream = torch.cuda.Stream(dev)
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(self.stream):
            layer_forward_into(self.x, block, self.outs, block_size)  # sizes this stream's workspace
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            layer_forward_into(self.x, block, self.outs, block_size)


_SESSIONS: "collections.OrderedDict" = collections.OrderedDict()
_SESSIONS_LOCK = threading.Lock()
_MAX_SESSIONS = 16


def _host_session(block: MoEBlock, t: int, dtype: torch.dtype, block_size: int, dev: torch.device):
    key = (id(block), t, dtype, block_size, dev.index, _EXPERT_PATH[0])
    with _SESSIONS_LOCK:
        sess = _SESSIONS.get(key)
        if sess is not None and sess[0] is block:
            _SESSIONS.move_to_end(key)
            return sess[1]
    new = _HostSession(block, t, dtype, block_size, dev)
    with _SESSIONS_LOCK:
        _SESSIONS[key] = (block, new)
        while len(_SESSIONS) > _MAX_SESSIONS:
            _SESSIONS.popitem(last=False)
    return new


def _graph_host_path() -> bool:
    return os.environ.get("BEAM_HOST_GRAPH", "1") != "0"


def beam_block_forward(h, block: MoEBlock, training: bool = True, block_size: int = 16):
    """beam.py:127-165 -> (h', RouterDecision, MaskDecision).

    ``h`` is [T, d_h] (torch tensor on the GPU or host, numpy array, or a
    reference ``Tensor``); bf16 and fp32 are computed as given, fp64 as fp32.
    Host input => host outputs (one H2D copy in, one D2H copy out).
    ``training=True`` returns the same forward values (the reference pins
    training == inference to 1e-9, test_beam.py:281-292); there is no autograd
    tape on this path (training is out of scope)."""
    _check_block(block)
    if block_size < 1:
        raise ContractError("block_size must be >= 1")
    x = as_torch(h)
    if x.ndim != 2 or x.shape[1] != block.cfg.d_h:
        raise ShapeError("h must be [tokens, d_h]")
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    host = not x.is_cuda
    dev = block.device
    cfg = block.cfg
    t = x.shape[0]
    if host and t > 0 and _graph_host_path():
        block.layer_desc(0.0)  # re-packs changed router weights in place (the graph reads those buffers)
        sess = _host_session(block, t, x.dtype, block_size, dev)
        with sess.lock:
            main = torch.cuda.current_stream(dev)
            sess.x.copy_(x, non_blocking=True)
            sess.graph.replay()
            hb = LayerOutputs(t, cfg.d_h, cfg.num_experts, cfg.top_k, x.dtype, "cpu", pin=True)
            hb.buf.copy_(sess.outs.buf, non_blocking=True)
            res = _results(hb)  # views built while the GPU works
            main.synchronize()
        return res
    xd = x.to(dev, non_blocking=True).contiguous() if host else x.contiguous()
    outs = LayerOutputs(t, cfg.d_h, cfg.num_experts, cfg.top_k, xd.dtype, dev)
    if host and t > 0:
        # decisions leave the GPU on a side stream while the experts run; `out`
        # follows the layer on the compute stream
        side, ev = _copy_stream(dev)
        main = torch.cuda.current_stream(dev)
        hb = LayerOutputs(t, cfg.d_h, cfg.num_experts, cfg.top_k, xd.dtype, "cpu",
                          pin=torch.cuda.is_available())
        # `out` is written by the combine kernel straight into the (UVA-mapped)
        # pinned host buffer: no trailing device->host copy
        host_out = hb.buf.data_ptr() + hb.out_off
        direct = _lib.load().beam_host_mapped(host_out) == 1
        layer_forward_into(xd, block, outs, block_size, decision_event=ev, out_ptr=host_out if direct else None)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            hb.copy_decisions_from(outs)
        if not direct:
            hb.copy_out_from(outs)
        # result views are host-side bookkeeping: built while the GPU still works
        res = _results(hb)
        side.synchronize()
        main.synchronize()
        return res
    elif t > 0:
        layer_forward_into(xd, block, outs, block_size)
    elif host:
        outs = LayerOutputs(t, cfg.d_h, cfg.num_experts, cfg.top_k, xd.dtype, "cpu")
    return _results(outs)


def _results(outs: LayerOutputs):
    v = outs.views
    dec = RouterDecision(logits=v["logits"], topk_indices=v["topk_ids"], weights=v["weights"])
    md = MaskDecision(pre_activation=v["pre_activation"], raw_mask=v["raw_mask"], mask=v["mask"])
    return v["out"], dec, md


# ---------------------------------------------------------------------------
# mask-router training (beam.py:87-124, 146-157)
# ---------------------------------------------------------------------------


def _f32(x, dev):
    return as_torch(x).to(dev, torch.float32).contiguous()


def sparsity_loss(raw_mask, topk_indices) -> torch.Tensor:
    """beam.py:87-97: sum of raw_mask over each token's top-K candidates / (K*T)
    (0-d fp32 tensor on the GPU; fixed-order fp64 accumulation)."""
    raw = as_torch(raw_mask)
    dev = raw.device if raw.is_cuda else _default_device()
    raw = _f32(raw, dev)
    ids = as_torch(topk_indices).to(dev, torch.int64).contiguous()
    t, n = raw.shape
    k = ids.shape[1]
    out = torch.empty(1, dtype=torch.float32, device=dev)
    _lib.check(_lib.load().beam_sparsity_loss(raw.data_ptr(), ids.data_ptr(), t, n, k, out.data_ptr(),
                                              _runtime.stream_handle(dev)), "beam_sparsity_loss")
    return out[0]


def ste_backward(upstream, weights, decision: MaskDecision, beta: float, k: int) -> torch.Tensor:
    """beam.py:100-124 closed form on the GPU:
    dL/da = (upstream * g + beta/(K*T) * [g > 0]) * sigma'(a), [T, N] fp32."""
    if beta < 0:
        raise ContractError("beta must be non-negative")
    a = as_torch(decision.pre_activation)
    dev = a.device if a.is_cuda else _default_device()
    a, up, w = _f32(a, dev), _f32(upstream, dev), _f32(weights, dev)
    if up.shape != a.shape or w.shape != a.shape:
        raise ShapeError("upstream, weights and pre_activation must all be [T, N]")
    t, n = a.shape
    grad = torch.empty_like(a)
    _lib.check(_lib.load().beam_ste_backward(up.data_ptr(), w.data_ptr(), a.data_ptr(), t, n, int(k),
                                             float(beta), grad.data_ptr(), _runtime.stream_handle(dev)),
               "beam_ste_backward")
    return grad


@dataclass
class MaskGrad:
    """Mask-router gradient of one layer for L = sum(out * dy) + beta * sparsity_loss."""

    grad_pre_activation: torch.Tensor  # [T, N] (exact 0 off each token's candidates)
    grad_weight: torch.Tensor          # [d_h, N] = x_n^T grad_pre_activation
    dghat: torch.Tensor                # [T, K] dL_task/dghat at the candidates (rank order)
    loss_reg: torch.Tensor             # 0-d: sparsity_loss(raw_mask, topk_indices)
    decision: RouterDecision
    mask_decision: MaskDecision


def mask_router_backward(h, block: MoEBlock, dy, beta: float = 0.0, block_size: int = 16) -> MaskGrad:
    """Backward of beam_block_forward(training=True) (beam.py:146-157) to the mask
    router, through the closed form ste_backward (beam.py:100-124): ONE C-ABI call
    (beam_mask_backward) runs the gate, evaluates every top-K candidate on the
    expert kernels (masked ones included) and fuses the slot dots with the STE
    step; the [d_h, N] weight gradient x_n^T dA is a plain cuBLAS GEMM.  Expert
    and router weights are frozen (BEAM trains the mask router only)."""
    _check_block(block)
    if beta < 0:
        raise ContractError("beta must be non-negative")
    if block_size < 1:
        raise ContractError("block_size must be >= 1")
    dev = block.device
    x = as_torch(h)
    if x.ndim != 2 or x.shape[1] != block.cfg.d_h:
        raise ShapeError("h must be [tokens, d_h]")
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    x = x.to(dev).contiguous()
    g = _f32(dy, dev)
    if g.shape != x.shape:
        raise ShapeError("dy must be [tokens, d_h]")
    cfg = block.cfg
    t, n, k = x.shape[0], cfg.num_experts, cfg.top_k
    outs = LayerOutputs(t, cfg.d_h, n, k, x.dtype, dev)
    grad = torch.empty(t, n, dtype=torch.float32, device=dev)
    dghat = torch.empty(t, k, dtype=torch.float32, device=dev)
    loss = torch.zeros(1, dtype=torch.float32, device=dev)
    if t > 0:
        desc = block.layer_desc(0.0)
        lib = _lib.load()
        ws = _runtime.workspace(lib.beam_workspace_bytes(ctypes.byref(desc), t, 0, block_size), dev)
        o = outs.ctypes_outputs()
        _lib.check(lib.beam_mask_backward(ctypes.byref(desc), x.data_ptr(),
                                          _lib.BEAM_BF16 if x.dtype == torch.bfloat16 else _lib.BEAM_F32, t,
                                          g.data_ptr(), float(beta), block_size, ctypes.byref(o),
                                          grad.data_ptr(), dghat.data_ptr(), loss.data_ptr(), ws.data_ptr(),
                                          ws.numel(), _runtime.stream_handle(dev)),
                   "beam_mask_backward")
    x_n = block.normalize(x) if block.norm_w is not None else x.float()
    grad_w = x_n.t().matmul(grad)
    dec = RouterDecision(logits=outs["logits"], topk_indices=outs["topk_ids"], weights=outs["weights"])
    md = MaskDecision(pre_activation=outs["pre_activation"], raw_mask=outs["raw_mask"], mask=outs["mask"])
    return MaskGrad(grad, grad_w, dghat, loss[0], dec, md)


def set_expert_path(mode: str = "auto") -> None:
    """Choose the expert-stage kernels of beam_block_forward: "auto" (tcgen05
    grouped GEMM for prefill-sized batches, weight streaming for decode),
    "simt" (weight streaming always), "tc" (tcgen05 always, bf16 weights; 2-SM
    CTA pairs) or "tc1" (tcgen05 always, 1-SM kernel)."""
    code = {"auto": 0, "simt": 1, "tc": 2, "tc1": 3}[mode]
    _lib.check(_lib.load().beam_set_expert_path(code), "beam_set_expert_path")
    _EXPERT_PATH[0] = code
