"""Expert parallelism (EP) for the BEAM layer over torch.distributed.

Not in the reference (expert parallelism is listed as an open limitation,
PAPER.md:712) — this is the north star's multi-GPU row.

Rank r of P owns the contiguous expert range [r*N/P, (r+1)*N/P); only those
experts are ever allocated on it.  The router and mask router (0.5-1 MB each)
are replicated, so gating is local.  Per layer call (all data-plane work in
sm_100a kernels, csrc/ep.cu, behind the C ABI):

  1. gate the rank's own T tokens (``beam_gate``): masked ids + weights;
  2. pack (``beam_ep_pack``, ONE launch): one send row per (token, destination
     rank) with at least one surviving slot there — deduplicated; masked slots
     send nothing — holding the raw token row and a metadata row
     [K local ids | K weights | inv_rms];
  3. all-to-all of rows and metadata (NCCL over NVLink / NVSwitch);
  4. the owner runs its local experts on what it received (``beam_ep_execute``:
     unpack -> masked permute -> weight-streaming or tcgen05 experts -> ordered
     combine), applying the RMS norm itself, exactly as the single-GPU layer;
  5. all-to-all of the fp32 partial sums back;
  6. ``beam_ep_combine``: out = h + partial sums in ascending rank order
     (= ascending expert ranges, dispatch/__init__.py:145-156).

Two protocols, chosen identically on every rank:
  * FIXED capacity (decode, T <= 256 per rank): every peer gets a block of
    `cap` rows (unused rows carry id -1 and cost no expert work); no counts
    exchange and no host sync, so the whole step — collectives included —
    replays as one CUDA graph.  `cap` is the layer's ``capacity`` (a static
    serving contract, same on every rank) or, without one, the max T over the
    ranks (one all-reduce).
  * COMPACT (prefill): per-destination counts (``beam_ep_count``) are exchanged
    first (the one host sync), then variable-split all-to-alls — BEAM's masked
    slots shrink the exchange.

Output equals the single-GPU layer up to fp32 re-association of the per-token
sum across rank boundaries.  ``virtual_forward`` runs P shards in ONE process
with a loopback exchange (SURVEY §4 "virtual EP"); the host-side protocol is
covered with gloo on CPU by tests/test_ep_gloo.py (oracle kernels injected).
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, _runtime
from .tensor import ContractError, ShapeError

FIXED_CAPACITY_MAX_T = 256  # decode-sized batches use the sync-free fixed-capacity exchange


@dataclass
class Sent:
    """One rank's packed send buffers."""

    x: torch.Tensor          # [rows, d] raw token rows (h dtype)
    meta: torch.Tensor       # [rows, 2K+1] int32
    send_pos: torch.Tensor   # [P, T] int32: row of (peer, token) or -1
    cap: int                 # fixed layout: rows per peer; 0 = compact
    splits: list | None      # compact: rows per peer (host ints)


# ---------------------------------------------------------------------------
# device kernels through the C ABI (backend-independent host logic is below)
# ---------------------------------------------------------------------------


class DeviceKernels:
    """The product data plane: pack / local execute / combine on the GPU."""

    def __init__(self, layer: "EPBeamLayer"):
        self.L = layer

    def gate(self, h):
        """beam_gate with the replicated routers: (masked ids [T, K] int64,
        router weights [T, N] f32)."""
        from .beam import _threshold

        L = self.L
        blk = L.router
        desc = blk.layer_desc(_threshold(blk.mask_router.tau))
        t = h.shape[0]
        n, k = L.cfg.num_experts, L.cfg.top_k
        masked = torch.empty(t, k, dtype=torch.int64, device=h.device)
        weights = torch.empty(t, n, dtype=torch.float32, device=h.device)
        if t == 0:
            return masked, weights
        o = _lib.Outputs()
        o.masked_ids = masked.data_ptr()
        o.weights = weights.data_ptr()
        lib = _lib.load()
        ws = _runtime.workspace(lib.beam_workspace_bytes(ctypes.byref(desc), t, 0, 1), h.device)
        _lib.check(lib.beam_gate(ctypes.byref(desc), h.data_ptr(), _dt(h), t, ctypes.byref(o), ws.data_ptr(),
                                 ws.numel(), _runtime.stream_handle(h.device)), "beam_gate")
        return masked, weights

    def counts(self, masked):
        """Rows per destination rank (int64 [P], device) for the compact layout,
        and the per-tile counts the pack kernel reads."""
        L = self.L
        t = masked.shape[0]
        lib = _lib.load()
        tiles = torch.zeros(L.world, max(lib.beam_ep_tiles(t), 1), dtype=torch.int32, device=masked.device)
        if t:
            _lib.check(lib.beam_ep_count(masked.data_ptr(), t, L.cfg.top_k, L.cfg.num_experts, L.world,
                                         tiles.data_ptr(), _runtime.stream_handle(masked.device)), "beam_ep_count")
        return tiles.sum(dim=1, dtype=torch.int64), tiles

    def pack(self, h, masked, weights, cap, tiles=None, rows=None):
        L = self.L
        t, d = h.shape
        k = L.cfg.top_k
        dev = h.device
        n_rows = L.world * cap if cap > 0 else rows
        x = torch.empty(n_rows, d, dtype=h.dtype, device=dev)
        meta = torch.empty(n_rows, 2 * k + 1, dtype=torch.int32, device=dev)
        send_pos = torch.empty(L.world, t, dtype=torch.int32, device=dev)
        counts = torch.empty(L.world, dtype=torch.int32, device=dev)
        _lib.check(_lib.load().beam_ep_pack(
            h.data_ptr() if t else None, _dt(h), t, d, masked.data_ptr() if t else None,
            weights.data_ptr() if t else None, L.cfg.num_experts, k, L.world, cap,
            tiles.data_ptr() if tiles is not None else None, 1 if L.cfg.has_norm else 0, x.data_ptr(),
            meta.data_ptr(), send_pos.data_ptr() if t else None, counts.data_ptr(), _runtime.stream_handle(dev)),
            "beam_ep_pack")
        return x, meta, send_pos

    def local(self, x, meta, mode):
        """Owner side: y f32 [n, d] = this rank's experts on the received rows."""
        L = self.L
        n = x.shape[0]
        y = torch.empty(n, L.cfg.d_h, dtype=torch.float32, device=x.device)
        if n == 0:
            return y
        desc = L.local.layer_desc(0.0)
        lib = _lib.load()
        ws = _runtime.workspace(lib.beam_ep_workspace_bytes(ctypes.byref(desc), n, L.cfg.top_k, mode), x.device)
        _lib.check(lib.beam_ep_execute(ctypes.byref(desc), x.data_ptr(), _dt(x), n, L.cfg.top_k, meta.data_ptr(),
                                       mode, y.data_ptr(), ws.data_ptr(), ws.numel(),
                                       _runtime.stream_handle(x.device)), "beam_ep_execute")
        return y

    def combine(self, h, y_back, send_pos):
        out = torch.empty_like(h)
        t = h.shape[0]
        if t:
            _lib.check(_lib.load().beam_ep_combine(y_back.data_ptr() if y_back.numel() else None,
                                                   send_pos.data_ptr(), self.L.world, t, h.shape[1],
                                                   h.data_ptr(), _dt(h), out.data_ptr(),
                                                   _runtime.stream_handle(h.device)), "beam_ep_combine")
        return out


def _dt(x):
    return _lib.BEAM_BF16 if x.dtype == torch.bfloat16 else _lib.BEAM_F32


# ---------------------------------------------------------------------------
# the sharded layer
# ---------------------------------------------------------------------------


class EPBeamLayer:
    """One BEAM MoE layer sharded over ranks: this rank's experts + replicated routers.

    ``local_experts`` = (w_gate [n_local, d, f], w_up [n_local, d, f], w_down
    [n_local, f, d]) of THIS rank's expert range only (host or device tensors;
    packed straight into the rank's device layout — the full block is never
    built).  ``capacity``: static max tokens per rank per call (decode serving
    contract, identical on every rank): the fixed-capacity protocol with no host
    sync; None = agree on the protocol per call (one all-reduce)."""

    def __init__(self, cfg, router_w, mask_w, local_experts, *, norm_w=None, tau: float = 0.5, group=None,
                 rank: int | None = None, world: int | None = None, capacity: int | None = None,
                 dtype=torch.bfloat16, device=None, kernels=None):
        from .beam import MaskRouter
        from .moe import MoEBlock, MoEBlockConfig

        self.group = group
        self.world = world if world is not None else dist.get_world_size(group)
        self.rank = rank if rank is not None else dist.get_rank(group)
        if cfg.num_experts % self.world:
            raise ContractError("num_experts must divide evenly across ranks")
        if cfg.num_shared:
            raise ContractError("shared experts are not sharded by the EP path")
        if capacity is not None and not 1 <= capacity <= FIXED_CAPACITY_MAX_T:
            raise ContractError(f"capacity must lie in [1, {FIXED_CAPACITY_MAX_T}]")
        self.cfg = cfg
        self.capacity = capacity
        self.n_local = cfg.num_experts // self.world
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        # replicated gating: routers + norm, no expert storage
        self.router = MoEBlock(cfg, dtype=dtype, device=dev, _router_only=True)
        self.router.router_w.copy_(torch.as_tensor(router_w, dtype=torch.float32))
        if self.router.norm_w is not None and norm_w is not None:
            self.router.norm_w.copy_(torch.as_tensor(norm_w, dtype=torch.float32))
        self.router.mask_router = MaskRouter(torch.as_tensor(mask_w, dtype=torch.float32).to(dev), tau)
        # this rank's experts (norm weight applied by the owner, beam_ep_execute)
        lcfg = MoEBlockConfig(cfg.d_h, cfg.d_ff, self.n_local, 1, 0, cfg.has_norm, cfg.activation)
        self.local = MoEBlock(lcfg, dtype=dtype, device=dev, _empty=True)
        if self.local.norm_w is not None:
            self.local.norm_w.copy_(self.router.norm_w)
        g, u, dn = local_experts
        if g.shape[0] != self.n_local:
            raise ShapeError(f"expected {self.n_local} local experts, got {g.shape[0]}")
        self.local._set_all_experts((g, u, dn), 0, self.n_local)
        # the data-plane kernels: the CUDA library; the CPU protocol tests inject a
        # host restatement (oracle/ep_oracle.py) through this factory
        self.kernels = (kernels or DeviceKernels)(self)
        self._staged = dist.is_initialized() and dist.get_backend(group) == "gloo" and dev.type == "cuda"

    @classmethod
    def from_block(cls, block, group=None, *, rank=None, world=None, capacity=None) -> "EPBeamLayer":
        """Shard of a full single-GPU block (tests / comparisons): this rank's
        slice of its experts, its routers and norm."""
        from .moe import unpack_gate_up

        world = world if world is not None else dist.get_world_size(group)
        rank = rank if rank is not None else dist.get_rank(group)
        cfg = block.cfg
        nl = cfg.num_experts // world
        lo = rank * nl
        g, u = unpack_gate_up(block.w_gu[lo:lo + nl], cfg.d_h, cfg.d_ff)
        dn = block.w_down[lo:lo + nl, :cfg.d_h, :cfg.d_ff].transpose(1, 2)
        return cls(cfg, block.router_w, block.mask_router.weight, (g, u, dn), norm_w=block.norm_w,
                   tau=block.mask_router.tau, group=group, rank=rank, world=world, capacity=capacity,
                   dtype=block.dtype, device=block.device)

    @classmethod
    def random(cls, cfg, seed: int, *, group=None, rank=None, world=None, capacity=None, dtype=torch.bfloat16,
               device=None, mask_std: float | None = None) -> "EPBeamLayer":
        """Random-init shard (N(0, 0.02) experts, bench workloads): expert e is
        drawn from its own generator (seed, e), so every rank draws only its own
        experts and any sharding holds the same layer."""
        world = world if world is not None else dist.get_world_size(group)
        rank = rank if rank is not None else dist.get_rank(group)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        nl = cfg.num_experts // world
        d, f = cfg.d_h, cfg.d_ff
        gr = torch.Generator().manual_seed(seed)
        router = torch.empty(d, cfg.num_experts).normal_(0.0, 0.02, generator=gr)
        router[0] = 0.0
        mask = torch.empty(d, cfg.num_experts).normal_(0.0, mask_std or 1.0 / np.sqrt(d), generator=gr)
        mask[0] = 0.0
        gs, us, ds = [], [], []
        for e in range(rank * nl, (rank + 1) * nl):
            ge = torch.Generator(device=dev).manual_seed(seed * 1_000_003 + e)
            gs.append(torch.empty(d, f, device=dev).normal_(0.0, 0.02, generator=ge).to(dtype))
            us.append(torch.empty(d, f, device=dev).normal_(0.0, 0.02, generator=ge).to(dtype))
            ds.append(torch.empty(f, d, device=dev).normal_(0.0, 0.02, generator=ge).to(dtype))
        return cls(cfg, router, mask, (torch.stack(gs), torch.stack(us), torch.stack(ds)), group=group, rank=rank,
                   world=world, capacity=capacity, dtype=dtype, device=dev)

    # -- collectives (gloo process groups with CUDA tensors stage through host memory)
    def _a2a(self, out, inp, out_splits=None, in_splits=None):
        if not self._staged:
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
            return
        # gloo + CUDA tensors: through host memory, as raw bytes (gloo has no
        # bf16 / int16 all-to-all); rows stay dim 0, so the splits are unchanged
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o.view(torch.uint8), inp.cpu().contiguous().view(torch.uint8), out_splits, in_splits,
                               group=self.group)
        out.copy_(o)

    def _protocol(self, t: int):
        """(cap, fixed): the same on every rank."""
        if self.capacity is not None:
            if t > self.capacity:
                raise ContractError(f"{t} tokens exceed the layer's fixed capacity {self.capacity}")
            return self.capacity, True
        tt = torch.tensor([t], dtype=torch.int64, device="cpu" if self._staged or self.device.type != "cuda"
                          else self.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX, group=self.group)
        t_max = int(tt.item())
        if t_max <= FIXED_CAPACITY_MAX_T:
            return max(t_max, 1), True
        return 0, False

    # -- the step
    def send(self, h, cap: int) -> Sent:
        """Gate + pack into the fixed-capacity layout (`cap` rows per peer)."""
        masked, weights = self.kernels.gate(h)
        x, meta, pos = self.kernels.pack(h, masked, weights, cap)
        return Sent(x, meta, pos, cap, None)

    def forward(self, h: torch.Tensor) -> torch.Tensor:
        h = h.contiguous()
        if h.ndim != 2 or h.shape[1] != self.cfg.d_h:
            raise ShapeError("h must be [tokens, d_h]")
        cap, fixed = self._protocol(h.shape[0])
        k = self.cfg.top_k
        if fixed:
            snd = self.send(h, cap)
            x_recv, meta_recv = torch.empty_like(snd.x), torch.empty_like(snd.meta)
            self._a2a(x_recv, snd.x)
            self._a2a(meta_recv, snd.meta)
            y = self.kernels.local(x_recv, meta_recv, 1)
            y_back = torch.empty_like(y)
            self._a2a(y_back, y)
            return self.kernels.combine(h, y_back, snd.send_pos)
        masked, weights = self.kernels.gate(h)
        counts, tiles = self.kernels.counts(masked)
        counts_recv = torch.empty_like(counts)
        self._a2a(counts_recv, counts)
        send_splits = counts.tolist()           # the compact protocol's one host sync
        recv_splits = counts_recv.tolist()
        x, meta, pos = self.kernels.pack(h, masked, weights, 0, tiles=tiles, rows=int(sum(send_splits)))
        n_recv = int(sum(recv_splits))
        x_recv = torch.empty(n_recv, h.shape[1], dtype=h.dtype, device=h.device)
        meta_recv = torch.empty(n_recv, 2 * k + 1, dtype=torch.int32, device=h.device)
        self._a2a(x_recv, x, recv_splits, send_splits)
        self._a2a(meta_recv, meta, recv_splits, send_splits)
        y = self.kernels.local(x_recv, meta_recv, 0)
        y_back = torch.empty(x.shape[0], h.shape[1], dtype=y.dtype, device=h.device)
        self._a2a(y_back, y, send_splits, recv_splits)
        return self.kernels.combine(h, y_back, pos)

    __call__ = forward


def virtual_forward(layers: list, hs: list, fixed: bool | None = None) -> list:
    """SURVEY §4 "virtual EP": P shards (``layers[r]``, world = P) in ONE process
    with a loopback exchange — the pack / execute / combine kernels and the
    protocols' row bookkeeping exactly as in ``forward``, no process group.
    Returns every rank's output."""
    world = len(layers)
    t_max = max(h.shape[0] for h in hs)
    if fixed is None:
        fixed = t_max <= FIXED_CAPACITY_MAX_T
    if fixed:
        cap = max(t_max, 1)
        sent = [ly.send(h.contiguous(), cap) for ly, h in zip(layers, hs)]
        # rank r receives block r of every peer p's send buffer, in peer order
        recv = [(torch.cat([s.x[r * cap:(r + 1) * cap] for s in sent]),
                 torch.cat([s.meta[r * cap:(r + 1) * cap] for s in sent])) for r in range(world)]
        ys = [layers[r].kernels.local(x, m, 1) for r, (x, m) in enumerate(recv)]
        backs = [torch.cat([ys[r][p * cap:(p + 1) * cap] for r in range(world)]) for p in range(world)]
        return [ly.kernels.combine(h.contiguous(), yb, s.send_pos) for ly, h, yb, s in zip(layers, hs, backs, sent)]
    packs = []
    for ly, h in zip(layers, hs):
        h = h.contiguous()
        masked, weights = ly.kernels.gate(h)
        counts, tiles = ly.kernels.counts(masked)
        splits = counts.tolist()
        x, meta, pos = ly.kernels.pack(h, masked, weights, 0, tiles=tiles, rows=int(sum(splits)))
        offs = np.concatenate([[0], np.cumsum(splits)]).astype(int)
        packs.append((h, x, meta, pos, splits, offs))
    ys, src = [], []
    for r in range(world):
        xr = torch.cat([p[1][p[5][r]:p[5][r + 1]] for p in packs])
        mr = torch.cat([p[2][p[5][r]:p[5][r + 1]] for p in packs])
        ys.append(layers[r].kernels.local(xr, mr, 0))
        src.append(np.concatenate([[0], np.cumsum([p[4][r] for p in packs])]).astype(int))
    outs = []
    for p_rank, (h, x, meta, pos, splits, offs) in enumerate(packs):
        yb = torch.cat([ys[r][src[r][p_rank]:src[r][p_rank + 1]] for r in range(world)]) if world else None
        outs.append(layers[p_rank].kernels.combine(h, yb, pos))
    return outs


# ---------------------------------------------------------------------------
# bench.py --gpus N (torchrun): EP at the BASELINE shapes, T tokens per rank
# ---------------------------------------------------------------------------


def _capture_step(layer, x, dev):
    """Fixed-capacity steps (no host sync) replay as one CUDA graph, NCCL
    collectives included.  Returns (graph, graph output) or (None, None)."""
    if layer.capacity is None or os.environ.get("BEAM_EP_NO_GRAPH") == "1":
        return None, None
    try:
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(2):
                layer.forward(x)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):  # the warmed-up stream: no workspace fill captured
            y_graph = layer.forward(x)
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        ref = layer.forward(x)
        if not torch.equal(ref, y_graph):
            return None, None  # not replay-safe here: time the eager step
        return graph, y_graph
    except Exception:  # capture unsupported by this NCCL / torch combination
        torch.cuda.synchronize()
        return None, None


def _timed_total(step, steps, flush):
    """Sum of per-step CUDA-event times (ms) on this rank, L2 flushed and ranks
    barriered before every step."""
    total = 0.0
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        step()
        e.record()
        e.synchronize()
        total += s.elapsed_time(e)
    return total


def _theta_layer(layer, bench, t, s, seed=7):
    """Calibrate the mask router's row 0 to sparsity s on the rank's tokens
    (same tokens on every rank's calibration: identical routers everywhere)."""
    d, k = layer.cfg.d_h, layer.cfg.top_k
    router = layer.router.router_w.cpu()
    mask = layer.router.mask_router.weight.cpu()
    theta = bench.calibrate_theta(bench.make_tokens(t, seed, d), router, mask, k, s)
    layer.router.mask_router.weight.copy_(bench.mask_with_theta(mask, theta).to(layer.device))


def _ep_shape_points(args, bench, dev, flush, world, rank):
    """EP lines for the other BASELINE shapes (configs[3] OLMoE, configs[4]
    Qwen3-235B): device ms per step, max over ranks, T tokens per rank.  Every
    rank allocates only its own experts (EPBeamLayer.random)."""
    import paper_2605_14438_b200 as B

    rows = []
    for name, t, s in (("olmoe", 64, 0.5), ("olmoe", 8192, 0.5), ("q235", 1, 0.85), ("q235", 64, 0.85),
                       ("q235", 8192, 0.85)):
        sh = bench.SHAPES[name]
        if sh["n"] % world:
            continue
        cfg = B.MoEBlockConfig(d_h=sh["d"], d_ff=sh["f"], num_experts=sh["n"], top_k=sh["k"])
        layer = EPBeamLayer.random(cfg, 2605, rank=rank, world=world, device=dev,
                                   capacity=t if t <= FIXED_CAPACITY_MAX_T else None)
        _theta_layer(layer, bench, t, s)
        x = bench.make_tokens(t, 7 + rank, sh["d"]).to(dev)
        for _ in range(2):
            layer.forward(x)
        torch.cuda.synchronize()
        graph, _ = _capture_step(layer, x, dev)
        step = graph.replay if graph is not None else (lambda: layer.forward(x))
        steps = 10 if t <= 256 else 3
        dist.barrier()
        t_max = torch.tensor([_timed_total(step, steps, flush)], device=dev)
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        ms = float(t_max.item()) / steps
        rows.append({"shape": name, **sh, "T_per_rank": t, "s_target": s, "ep": world,
                     "experts_per_rank": sh["n"] // world, "ms_per_step": round(ms, 4),
                     "tokens_per_s": round(world * t / (ms / 1e3), 1), "graph": graph is not None,
                     "protocol": "fixed" if layer.capacity else "compact"})
        del layer, graph, step
        torch.cuda.empty_cache()
    return rows


def bench_main(args, bench):
    import json

    import paper_2605_14438_b200 as B

    # a single process without torchrun (BEAM_BENCH_FORCE_EP=1 check): rank 0 of 1
    for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29511")):
        os.environ.setdefault(k, v)
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=q["d"], d_ff=q["f"], num_experts=q["n"], top_k=q["k"])
    w = bench.make_layer0()  # host tensors; only this rank's expert slice goes to the device
    h = bench.make_tokens(args.tokens, 7 + rank)
    theta = bench.calibrate_theta(bench.make_tokens(args.tokens, 7), w["router"], w["mask"], q["k"], args.sparsity)
    nl = q["n"] // world
    sl = slice(rank * nl, (rank + 1) * nl)
    layer = EPBeamLayer(cfg, w["router"], bench.mask_with_theta(w["mask"], theta),
                        (w["wg"][sl], w["wu"][sl], w["wd"][sl]), device=dev,
                        capacity=args.tokens if args.tokens <= FIXED_CAPACITY_MAX_T else None)
    del w
    x = h.to(dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    lib = _lib.load()
    for _ in range(args.warmup):
        layer.forward(x)
    torch.cuda.synchronize()
    c0 = lib.beam_kernel_launches()
    layer.forward(x)  # launches of one step through the C ABI (gate, pack, local experts, combine)
    torch.cuda.synchronize()
    launches_per_step = int(lib.beam_kernel_launches() - c0)
    graph, y_graph = _capture_step(layer, x, dev)
    step = graph.replay if graph is not None else (lambda: layer.forward(x))
    dist.barrier()
    with bench.ClockSampler(dev.index) as clocks:
        total = _timed_total(step, args.steps, flush)
    t_max = torch.tensor([total], device=dev)
    dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item()) / args.steps
    # e2e: pinned host tokens -> device -> EP layer -> host output, every step
    h_pin = h.pin_memory()
    out_host = torch.empty(h.shape, dtype=h.dtype).pin_memory()
    e2e_total = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        if graph is not None:  # serving-style: pinned input into the graph's static buffer, replay, copy out
            x.copy_(h_pin, non_blocking=True)
            graph.replay()
            out_host.copy_(y_graph, non_blocking=True)
        else:
            y = layer.forward(h_pin.to(dev, non_blocking=True))
            out_host.copy_(y, non_blocking=True)
        torch.cuda.synchronize()
        e2e_total += time.perf_counter() - t0
    e2e_max = torch.tensor([e2e_total], device=dev)
    dist.all_reduce(e2e_max, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_max.item()) / args.steps
    shape_rows = [] if getattr(args, "no_shapes", False) else _ep_shape_points(args, bench, dev, flush, world, rank)
    if rank == 0:
        line = {
            "metric": bench.METRIC, "value": world * args.tokens / (ms / 1e3), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": bench.workload_config(args.tokens, args.sparsity),
            "measurement": {"parallelism": f"expert parallel EP{world}, T={args.tokens} tokens per rank",
                            "experts_per_rank": q["n"] // world, "l2": "flushed before every step",
                            "protocol": "fixed capacity" if layer.capacity else "compact (counts exchange)",
                            "timing": "CUDA events per step, max over ranks" + (
                                ", CUDA-graph replay of the step (NCCL collectives captured)" if graph is not None
                                else ", eager step"),
                            "exchange": "device pack/combine kernels (beam_ep_pack / beam_ep_combine) around NCCL "
                                        "all_to_all_single (rows, metadata, partial sums)"},
            "e2e": {"value": world * args.tokens / e2e_s, "unit": "tokens/s",
                    "h2d_bytes_per_step": world * int(h.numel()) * h.element_size(),
                    "d2h_bytes_per_step": world * int(h.numel()) * h.element_size(),
                    "path": "pinned host tokens -> device -> EPBeamLayer step (graph replay when captured) -> host output, "
                            "max over ranks"},
            "roofline": None,
            "clocks": clocks.summary(),
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step,
            "shapes": shape_rows,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
