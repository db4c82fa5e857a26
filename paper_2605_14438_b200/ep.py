"""Expert parallelism (EP) for the BEAM layer over torch.distributed.

Not in the reference (expert parallelism is listed as an open limitation,
PAPER.md:712) — this is the north star's multi-GPU row.

Rank r of P owns the contiguous expert range [r*N/P, (r+1)*N/P).  Every rank
holds the (small) router and mask router, so gating is replicated; per layer call:

  1. gate the rank's own T tokens (fused sm_100a gating kernel): surviving
     (token, slot) pairs with their routing weights ghat;
  2. dispatch: each token is sent ONCE to every rank that owns at least one of its
     surviving experts (dedup), with a metadata row [K local ids | K weights];
     masked slots cost no bytes — BEAM's sparsity shrinks the all-to-all;
  3. the owner runs its local experts on the received rows (beam_moe_execute:
     masked permute + weight-streaming / tcgen05 experts + combine);
  4. combine: partial sums travel back; the token's rank adds them in ascending
     rank order (= ascending expert ranges), then the residual.

Collectives: one all-to-all of P ints (counts; the only host sync) and three
all_to_all_single calls (rows, metadata, partial sums); decode-sized batches
(T <= 256) use a fixed-capacity variant with no counts exchange and no host
sync (``ep_exchange_forward_fixed``) — NCCL over NVLink /
NVSwitch on B200s, gloo in the CPU tests.  Output equals the single-GPU layer up
to fp32 re-association of the per-token sum across ranks.

The exchange logic is device-agnostic and takes the gating and local-expert
compute as callables, so tests/test_ep_gloo.py runs it with world_size 2 on CPU
with the oracle as the local compute.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, _runtime


@dataclass
class Gated:
    xn: torch.Tensor     # [T, d] normalised activations (what the experts consume)
    ids: torch.Tensor    # [T, K] int64 surviving expert ids, -1 = masked
    ghat: torch.Tensor   # [T, K] f32 routing weight of each slot (0 where masked)


FIXED_CAPACITY_MAX_T = 256  # decode-sized batches use the sync-free fixed-capacity exchange


def ep_exchange_forward_fixed(h: torch.Tensor, gated: Gated, num_experts: int, local_fn, group=None) -> torch.Tensor:
    """Steps 2-4 with a fixed-capacity protocol (no counts exchange, no host
    sync): every rank sends each peer one row per token — the rows a peer owns
    no surviving expert of carry only -1 ids, so the peer's masked permute skips
    them (no expert bytes or FLOPs; the exchange costs T rows per peer, a few MB
    at decode sizes).  Partial sums come back the same way and are added in
    ascending rank order."""
    world = dist.get_world_size(group)
    if num_experts % world:
        raise ValueError("num_experts must divide evenly across ranks")
    n_local = num_experts // world
    t, k = gated.ids.shape
    d = gated.xn.shape[1]
    dev = h.device
    ids = gated.ids
    ranks = torch.arange(world, device=dev).view(world, 1, 1)
    owner = torch.where(ids >= 0, ids // n_local, torch.full_like(ids, -1))[None]            # [1, T, K]
    mine = owner == ranks                                                                     # [P, T, K]
    loc_ids = torch.where(mine, ids[None] - ranks * n_local, torch.full_like(ids[None], -1))
    loc_w = torch.where(mine, gated.ghat[None].to(torch.float32), torch.zeros((), device=dev))
    meta = torch.cat([loc_ids.to(torch.int32), loc_w.view(torch.int32)], dim=2).reshape(world * t, 2 * k).contiguous()
    x_send = gated.xn[None].expand(world, t, d).reshape(world * t, d).contiguous()
    x_recv = torch.empty_like(x_send)
    meta_recv = torch.empty_like(meta)
    dist.all_to_all_single(x_recv, x_send, group=group)
    dist.all_to_all_single(meta_recv, meta, group=group)
    y_recv = local_fn(x_recv, meta_recv[:, :k].contiguous(), meta_recv[:, k:].contiguous().view(torch.float32))
    y_recv = y_recv.to(torch.float32).contiguous()
    y_back = torch.empty_like(y_recv)
    dist.all_to_all_single(y_back, y_recv, group=group)
    y_back = y_back.view(world, t, d)
    y = y_back[0].clone()
    for r in range(1, world):  # ascending rank == ascending expert range
        y += y_back[r]
    return (h.to(torch.float32) + y).to(h.dtype)


def ep_exchange_forward(h: torch.Tensor, gated: Gated, num_experts: int, local_fn, group=None) -> torch.Tensor:
    """Steps 2-4 above.  ``local_fn(x [n, d], ids [n, K] int32 local ids (-1 skip),
    w [n, K] f32) -> y [n, d] f32`` runs this rank's experts.  Returns h + y in
    h's dtype."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if num_experts % world:
        raise ValueError("num_experts must divide evenly across ranks")
    n_local = num_experts // world
    t, k = gated.ids.shape
    dev = h.device
    ids = gated.ids
    dest = torch.where(ids >= 0, ids // n_local, torch.full_like(ids, -1))            # [T, K]
    send_mask = torch.stack([(dest == r).any(dim=1) for r in range(world)])             # [P, T]
    pairs = send_mask.nonzero()                                                          # (r, t) rank-major
    r_idx, t_idx = pairs[:, 0], pairs[:, 1]
    counts_send = send_mask.sum(dim=1).to(torch.int64)
    # metadata: local ids of the slots that belong to the destination, and their weights
    mine = dest[t_idx] == r_idx[:, None]                                                 # [n, K]
    loc_ids = torch.where(mine, ids[t_idx] - r_idx[:, None] * n_local, torch.full_like(ids[t_idx], -1))
    loc_w = torch.where(mine, gated.ghat[t_idx], torch.zeros_like(gated.ghat[t_idx]))
    meta = torch.cat([loc_ids.to(torch.int32), loc_w.to(torch.float32).view(torch.int32)], dim=1).contiguous()
    x_send = gated.xn[t_idx].contiguous()

    counts_recv = torch.empty_like(counts_send)
    dist.all_to_all_single(counts_recv, counts_send, group=group)
    send_splits = counts_send.tolist()
    recv_splits = counts_recv.tolist()
    n_recv = int(sum(recv_splits))
    x_recv = torch.empty((n_recv, x_send.shape[1]), dtype=x_send.dtype, device=dev)
    meta_recv = torch.empty((n_recv, 2 * k), dtype=torch.int32, device=dev)
    dist.all_to_all_single(x_recv, x_send, recv_splits, send_splits, group=group)
    dist.all_to_all_single(meta_recv, meta, recv_splits, send_splits, group=group)

    ids_recv = meta_recv[:, :k].contiguous()
    w_recv = meta_recv[:, k:].contiguous().view(torch.float32)
    y_recv = local_fn(x_recv, ids_recv, w_recv) if n_recv else torch.zeros((0, x_send.shape[1]), device=dev)
    y_recv = y_recv.to(torch.float32).contiguous()

    y_back = torch.empty((int(sum(send_splits)), y_recv.shape[1]), dtype=torch.float32, device=dev)
    dist.all_to_all_single(y_back, y_recv, send_splits, recv_splits, group=group)

    # ascending rank == ascending expert range; each rank's rows have unique tokens
    y = torch.zeros((t, h.shape[1]), dtype=torch.float32, device=dev)
    start = 0
    for r in range(world):
        n = send_splits[r]
        if n:
            y[t_idx[start : start + n]] += y_back[start : start + n]
        start += n
    return (h.to(torch.float32) + y).to(h.dtype)


class EPBeamLayer:
    """One BEAM MoE layer sharded over the ranks of ``group`` (CUDA + NCCL).

    ``block`` is a full-size ``MoEBlock`` description used only for its routers /
    norm (replicated); only this rank's experts are kept on the device."""

    def __init__(self, block, group=None):
        from .moe import MoEBlock, MoEBlockConfig

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        cfg = block.cfg
        if cfg.num_experts % self.world:
            raise ValueError("num_experts must divide evenly across ranks")
        if cfg.num_shared:
            raise ValueError("shared experts are not sharded by the EP path")
        self.cfg = cfg
        self.n_local = cfg.num_experts // self.world
        self.block = block
        lo = self.rank * self.n_local
        lcfg = MoEBlockConfig(cfg.d_h, cfg.d_ff, self.n_local, 1, 0, False, cfg.activation)
        self.local = MoEBlock(lcfg, dtype=block.dtype, device=block.device, _empty=True)
        self.local.w_gu.copy_(block.w_gu[lo : lo + self.n_local])
        self.local.w_down.copy_(block.w_down[lo : lo + self.n_local])

    def gate(self, h: torch.Tensor) -> Gated:
        from .beam import _threshold
        from .moe import _gate_call  # noqa: F401  (same C entry, full router)

        blk = self.block
        desc = blk.layer_desc(_threshold(blk.mask_router.tau))
        t = h.shape[0]
        n, k = self.cfg.num_experts, self.cfg.top_k
        masked = torch.empty(t, k, dtype=torch.int64, device=h.device)
        weights = torch.empty(t, n, dtype=torch.float32, device=h.device)
        o = _lib.Outputs()
        o.masked_ids = masked.data_ptr()
        o.weights = weights.data_ptr()
        lib = _lib.load()
        ws = _runtime.workspace(lib.beam_workspace_bytes(ctypes.byref(desc), t, 0, 1), h.device)
        _lib.check(lib.beam_gate(ctypes.byref(desc), h.data_ptr(),
                                 _lib.BEAM_BF16 if h.dtype == torch.bfloat16 else _lib.BEAM_F32, t,
                                 ctypes.byref(o), ws.data_ptr(), ws.numel(), _runtime.stream_handle(h.device)),
                   "beam_gate")
        ghat = torch.where(masked >= 0, torch.gather(weights, 1, masked.clamp(min=0)), torch.zeros((), device=h.device))
        xn = blk.normalize(h).to(blk.dtype) if blk.norm_w is not None else h.to(blk.dtype)
        return Gated(xn=xn, ids=masked, ghat=ghat)

    def local_fn(self, x, ids, w):
        from .dispatch import execute_routed

        return execute_routed(self.local, x.contiguous(), ids.contiguous(), w.contiguous())

    def forward(self, h: torch.Tensor) -> torch.Tensor:
        h = h.contiguous()
        fwd = ep_exchange_forward_fixed if h.shape[0] <= FIXED_CAPACITY_MAX_T else ep_exchange_forward
        return fwd(h, self.gate(h), self.cfg.num_experts, self.local_fn, self.group)


# ---------------------------------------------------------------------------
# bench.py --gpus N (torchrun): EP at the Qwen3-30B-A3B shape, T tokens per rank
# ---------------------------------------------------------------------------


def _capture_step(layer, x, dev):
    """Decode-sized steps (fixed-capacity exchange: no host sync) replay as one
    CUDA graph, NCCL collectives included — the eager step is host-launch bound.
    Returns (graph, graph output) or (None, None) when the step is not captured."""
    if x.shape[0] > FIXED_CAPACITY_MAX_T or os.environ.get("BEAM_EP_NO_GRAPH") == "1":
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


def _ep_shape_points(args, bench, dev, flush, world, rank):
    """EP lines for the other BASELINE shapes (configs[3] OLMoE, configs[4]
    Qwen3-235B): device ms per step, max over ranks, T tokens per rank."""
    import paper_2605_14438_b200 as B

    rows = []
    for name, t, s in (("olmoe", 64, 0.5), ("olmoe", 8192, 0.5), ("q235", 1, 0.85), ("q235", 64, 0.85),
                       ("q235", 8192, 0.85)):
        sh = bench.SHAPES[name]
        if sh["n"] % world:
            continue
        w = bench.shape_layer(B, name, dev)
        blk = w["_block"]
        theta = bench.calibrate_theta(bench.make_tokens(t, 7, sh["d"]), w["router"], w["mask"], sh["k"], s)
        blk.mask_router.weight.copy_(bench.mask_with_theta(w["mask"], theta).to(dev))
        layer = EPBeamLayer(blk)
        blk.w_gu = torch.zeros(1, dtype=torch.bfloat16, device=dev)
        blk.w_down = torch.zeros(1, dtype=torch.bfloat16, device=dev)
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
                     "tokens_per_s": round(world * t / (ms / 1e3), 1), "graph": graph is not None})
        del layer, blk, w, graph, step
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
    w = bench.make_layer0()
    h = bench.make_tokens(args.tokens, 7 + rank)
    theta = bench.calibrate_theta(bench.make_tokens(args.tokens, 7), w["router"], w["mask"], q["k"], args.sparsity)
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]),
                                  mask_w=bench.mask_with_theta(w["mask"], theta), dtype=torch.bfloat16, device=dev)
    layer = EPBeamLayer(blk)
    # only the local shard stays resident (the gate never reads expert weights)
    blk.w_gu = torch.zeros(1, dtype=torch.bfloat16, device=dev)
    blk.w_down = torch.zeros(1, dtype=torch.bfloat16, device=dev)
    x = h.to(dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    lib = _lib.load()
    for _ in range(args.warmup):
        layer.forward(x)
    torch.cuda.synchronize()
    c0 = lib.beam_kernel_launches()
    layer.forward(x)  # launches of one step through the C ABI (gate + local experts)
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
            "config": {"workload": f"Qwen3-30B-A3B MoE layer, expert parallel EP{world}, T={args.tokens} tokens/rank, "
                                   f"s={args.sparsity}", **q, "parallelism": f"ep{world}",
                       "experts_per_rank": q["n"] // world, "l2": "flushed before every step",
                       "timing": "CUDA events per step, max over ranks" + (
                           ", CUDA-graph replay of the step (NCCL collectives captured)" if graph is not None
                           else ", eager step"),
                       "exchange": "NCCL all_to_all_single (counts, rows, metadata, partial sums)"},
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
