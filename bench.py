#!/usr/bin/env python
"""bench.py — BEAM MoE layer on B200 at the Qwen3-30B-A3B shape (BASELINE.json).

Workload (configs[1]): one BEAM MoE layer, 128 experts top-8, hidden 2048,
moe_ffn 768, bf16 experts / fp32 routing, decode batch T (default 64) at mask
sparsity s (default 0.5 of the T*K top-K slots masked).  A "step" is one full
layer forward (RMSnorm -> router + mask router -> top-K -> mask -> permute ->
experts -> combine -> residual) on one batch of synthetic tokens.

Lines printed (rank 0, one JSON object):
  value   tokens/s, device time of K steps (CUDA graph replay of the public
          layer call; L2 flushed before every step, flush not timed)
  e2e     the same through the public API beam_block_forward() with pinned HOST
          buffers: H2D of h and D2H of all outputs inside the timed region
  roofline  dominant kernel (experts gate/up, weight streaming): algorithmic
          bytes / its CUDA-event duration vs the measured HBM copy peak
  cpu_baseline  the reference package (oracle/_ref, numpy fp64 + Cython) on the
          host cores, same weights / tokens / mask, bounded sample
  sweep   T in {1, 8, 16, 32, 64} x s in {0, .25, .5, .75, .85} (+ prefill T=8192)

--impl reference runs the reference's own CPU implementation (beamoe, built
into oracle/_ref from /root/reference) on the same workload, rank 0 only.

Multi-GPU (torchrun, N>1): expert parallel over NCCL (paper_2605_14438_b200.ep),
T tokens per rank, experts split N/world per rank ("scaling": "weak").
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

Q30 = dict(d=2048, f=768, n=128, k=8)
METRIC = "BEAM MoE-layer tokens/s & decode µs at Qwen3-30B-A3B shape vs sparsity"
SWEEP_T = (1, 8, 16, 32, 64)
SWEEP_S = (0.0, 0.25, 0.5, 0.75, 0.85)


# ---------------------------------------------------------------------------
# synthetic workload (shared by both arms; CPU-generated so both see the same bits)
# ---------------------------------------------------------------------------


def make_layer0(seed: int = 2605, shape=None, wdtype=None):
    """Layer weights from a seeded torch CPU generator: router [d,N] fp32 with
    row 0 zeroed (constant channel carries no routing signal), experts bf16 (or
    `wdtype`), mask router rows 1.. ~ N(0, 1/d) (row 0 = theta, set per sparsity)."""
    import torch

    shape = shape or Q30
    wdtype = wdtype or torch.bfloat16
    d, f, n = shape["d"], shape["f"], shape["n"]
    g = torch.Generator().manual_seed(seed)
    router = torch.empty(d, n).normal_(0.0, 0.02, generator=g)
    router[0] = 0.0
    wg = torch.empty(n, d, f).normal_(0.0, 0.02, generator=g).to(wdtype)
    wu = torch.empty(n, d, f).normal_(0.0, 0.02, generator=g).to(wdtype)
    wd = torch.empty(n, f, d).normal_(0.0, 0.02, generator=g).to(wdtype)
    mask = torch.empty(d, n).normal_(0.0, 1.0 / math.sqrt(d), generator=g)
    mask[0] = 0.0
    return dict(router=router, wg=wg, wu=wu, wd=wd, mask=mask)


def make_tokens(t: int, seed: int, d: int = Q30["d"], dtype=None):
    """h ~ N(0,1) with channel 0 held at 8, rounded to bf16
    (or kept in `dtype`, e.g. fp32 for the tiny config)."""
    import torch

    g = torch.Generator().manual_seed(seed)
    h = torch.empty(t, d).normal_(0.0, 1.0, generator=g)
    h[:, 0] = 8.0
    return h.to(dtype if dtype is not None else torch.bfloat16)


def calibrate_theta(h_bf16, router, mask, k: int, s: float) -> float:
    """theta for mask row 0 so that a fraction s of the top-K slots has a < 0:
    a[t,e] = x_n[t,0]*theta + a_rest[t,e] with x_n[t,0] > 0, so the masked
    fraction is P(theta < -a_rest/x0) and theta is its (1-s) quantile."""
    h = h_bf16.float().double().numpy()
    ms = (h * h).mean(axis=1, keepdims=True) + 1e-6
    xn = h * ms**-0.5
    logits = xn @ router.double().numpy()
    ids = np.argsort(-logits, axis=1, kind="stable")[:, :k]
    a_rest = xn @ mask.double().numpy()
    r = -np.take_along_axis(a_rest, ids, 1) / xn[:, :1]
    r = np.sort(r.reshape(-1))
    if s <= 0.0:
        return float(r[-1] + 1.0)
    m = int(round(s * r.size))
    if m >= r.size:
        return float(r[0] - 1.0)
    return float(0.5 * (r[r.size - m - 1] + r[r.size - m]))  # exactly m slots masked (away from ties)


def workload_config(t: int, s: float) -> dict:
    """The `config` object of BOTH arms (ours and --impl reference): the same
    workload description, key for key; measurement details live elsewhere."""
    return {"workload": f"Qwen3-30B-A3B MoE layer decode T={t} s={s} (configs[1])", "T": t,
            "sparsity_target": s, **Q30, "routing_dtype": "f32", "expert_dtype": "bf16",
            "tokens": "synthetic N(0,1), channel 0 = 8, bf16; mask row 0 = theta calibrated to s",
            "parallelism": "single device"}


def mask_with_theta(mask, theta: float):
    m = mask.clone()
    m[0] = theta
    return m


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons during a timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return False
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)
        return False

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower().startswith("active")})
        busy = [x for x in sm if x > 0.5 * (max(sm) if sm else 0)]
        return {"sm_mhz": float(np.median(busy)) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    """(HBM GB/s, bf16 TFLOP/s burst, bf16 TFLOP/s sustained, kind)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        burst = float(p.get("bf16_tflops", 1628.7))
        return float(p["hbm_gbs"]), burst, float(p.get("bf16_tflops_sustained", burst)), "measured"
    return 6650.0, 1590.0, 1590.0, "fallback"


def ncu_traffic(kernel: str, workload: str):
    """DRAM bytes per launch of `kernel` from the committed ncu summary
    (profiles/ncu_summary.json, written from an `ncu --set full` capture of the
    same workload), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        rows = json.load(fh).get("kernels", [])
    for r in rows:
        if r.get("kernel") == kernel and r.get("workload") == workload:
            return r.get("dram_bytes_per_launch")
    return None


def cpu_cores_used():
    try:
        from threadpoolctl import threadpool_info

        info = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if info:
            return int(info[0]["num_threads"]), info[0].get("internal_api", "blas")
    except Exception:
        pass
    return os.cpu_count() or 1, "blas"


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the unmodified reference package)
# ---------------------------------------------------------------------------


def reference_block(w, theta: float, shape=None):
    from oracle import ref

    beamoe = ref.import_beamoe()
    from beamoe.beam import MaskRouter
    from beamoe.moe import Expert, MoEBlock, MoEBlockConfig
    from beamoe.tensor import Tensor

    shape = shape or Q30
    cfg = MoEBlockConfig(d_h=shape["d"], d_ff=shape["f"], num_experts=shape["n"], top_k=shape["k"])
    rb = MoEBlock.__new__(MoEBlock)
    rb.cfg = cfg
    rb.router_w = Tensor._raw(w["router"].double().numpy())
    wg = w["wg"].double().numpy()
    wu = w["wu"].double().numpy()
    wd = w["wd"].double().numpy()
    rb.experts = [Expert(Tensor._raw(wg[i]), Tensor._raw(wu[i]), Tensor._raw(wd[i])) for i in range(cfg.num_experts)]
    rb.shared = []
    rb.norm_w = Tensor._raw(np.ones(cfg.d_h))
    rb.mask_router = MaskRouter(Tensor._raw(mask_with_theta(w["mask"], theta).double().numpy()))
    return beamoe, rb


def time_reference(w, h_bf16, theta, budget_s: float, min_reps: int = 2, max_reps: int = 50, shape=None):
    beamoe, rb = reference_block(w, theta, shape)
    from beamoe.beam import beam_block_forward
    from beamoe.tensor import Tensor

    h64 = h_bf16.float().double().numpy()
    out, _, _ = beam_block_forward(Tensor(h64), rb, training=False)  # warm-up
    times = []
    t_start = time.perf_counter()
    while len(times) < max_reps and (len(times) < min_reps or time.perf_counter() - t_start < budget_s):
        t0 = time.perf_counter()
        out, _, _ = beam_block_forward(Tensor(h64), rb, training=False)
        times.append(time.perf_counter() - t0)
    return float(np.mean(times)), len(times), out.data


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t = args.tokens
    w = make_layer0()
    h = make_tokens(t, 7)
    theta = calibrate_theta(h, w["router"], w["mask"], Q30["k"], args.sparsity)
    beamoe, rb = reference_block(w, theta)
    from beamoe.beam import beam_block_forward
    from beamoe.tensor import Tensor

    h64 = h.float().double().numpy()
    for _ in range(args.warmup):
        beam_block_forward(Tensor(h64), rb, training=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        beam_block_forward(Tensor(h64), rb, training=False)
    dt = (time.perf_counter() - t0) / args.steps
    cores, api = cpu_cores_used()
    value = t / dt
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(t, args.sparsity),
        "measurement": {"where": "host CPU", "timing": "time.perf_counter over the steps"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} calls of beamoe.beam.beam_block_forward(training=False) "
                                   f"(numpy fp64 + Cython dispatch, {api} threads={cores}) on T={t}"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


_CAPTURE_STREAMS = {}


def _capture_stream(device):
    """One capture stream per device for every graph the bench builds (so the
    library's per-stream workspace is created once, outside any capture)."""
    import torch

    if device not in _CAPTURE_STREAMS:
        _CAPTURE_STREAMS[device] = torch.cuda.Stream(device)
    return _CAPTURE_STREAMS[device]


class GpuLayer:
    """One BEAM block on the GPU plus preallocated outputs and a captured graph."""

    def __init__(self, block, x, block_size=16):
        import torch

        from paper_2605_14438_b200.beam import LayerOutputs, layer_forward_into

        self.block, self.x, self.bs = block, x, block_size
        cfg = block.cfg
        self.outs = LayerOutputs(x.shape[0], cfg.d_h, cfg.num_experts, cfg.top_k, x.dtype, x.device)
        self._fwd = layer_forward_into
        self.eager()
        torch.cuda.synchronize()
        # warm up on the capture stream first: the library's workspace is cached
        # per stream and zero-filled once on creation — created inside the capture,
        # that fill would become part of every replay
        cap = _capture_stream(x.device)
        cap.wait_stream(torch.cuda.current_stream(x.device))
        with torch.cuda.stream(cap):
            self.eager()
        torch.cuda.current_stream(x.device).wait_stream(cap)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=cap):
            self.eager()
        torch.cuda.synchronize()

    def eager(self):
        self._fwd(self.x, self.block, self.outs, self.bs)

    def replay(self):
        self.graph.replay()


def algorithmic_bytes(t, s_real, e_act, r, d, f, n, k=Q30["k"], wbytes=2, xbytes=2):
    """Bytes the layer must move (bf16 experts, fp32 routers): activated experts'
    weights + router/mask weights + tokens in/out (+ small metadata)."""
    w_exp = e_act * 3 * d * f * wbytes
    w_gate = 2 * n * d * 4
    act = t * d * xbytes * 2
    meta = t * k * 8 * 2
    return w_exp + w_gate + act + meta


def gateup_kernel_name(t, r, e_act, f, sms=148, k=8):
    """Which gate/up kernel runs the expert stage (the host-side rule of
    experts_simt.cu: CTA items at T <= 2; the one-launch tensor-core / FFMA item
    kernel when the planned slots T*K could give every warp >= 3 tensor-core
    items (mma_possible) — the device then picks the item kind — else FFMA only)."""
    if t <= 2:
        return "gateup_cta_kernel"
    f_pad = (f + 15) // 16 * 16
    e_min = -(-3 * 2 * sms * 8 // (f_pad // 8))
    return "gateup_mix_kernel" if t * k >= 2 * e_min else "gateup_ffma_kernel"


def gateup_bytes(t, e_act, r, d, f):
    """Algorithmic bytes of the gate/up stage: the active experts' gate + up
    rows (bf16), one read of the token rows, the bf16 act rows written."""
    return e_act * 2 * f * d * 2 + t * d * 2 + r * f * 2


def timed_steps(layer, steps, flush, use_graph=True):
    """Per-step device time (ms) with an untimed L2 flush before every step."""
    import torch

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    rsweep = os.environ.get("BEAM_BENCH_FLUSH") == "rw"  # diagnostics: memset, then a read sweep (clean L2)
    for s_ev, e_ev in evs:
        flush.zero_()
        if rsweep:
            flush[: 256 << 20].view(torch.int32).sum()
        s_ev.record()
        layer.replay() if use_graph else layer.eager()
        e_ev.record()
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in evs]


def run_point(B, w, t, s, steps, warmup, flush, dev, seed=7, block_size=16):
    import torch

    blk = w["_block"]
    k = blk.cfg.top_k
    h = make_tokens(t, seed, blk.cfg.d_h, w.get("_xdtype"))
    theta = calibrate_theta(h, w["router"], w["mask"], k, s)
    blk.mask_router.weight.copy_(mask_with_theta(w["mask"], theta).to(dev))
    x = h.to(dev)
    layer = GpuLayer(blk, x, block_size)
    for _ in range(warmup):
        layer.replay()
    torch.cuda.synchronize()
    ms = timed_steps(layer, steps, flush)
    mids = layer.outs["masked_ids"]
    r = int((mids >= 0).sum())
    e_act = int(torch.unique(mids[mids >= 0]).numel())
    s_real = 1.0 - r / (t * k)
    return dict(layer=layer, theta=theta, h=h, ms=float(np.mean(ms)), r=r, e_act=e_act, s_real=s_real)


SHAPES = {  # BASELINE.json configs[0], [3], [4] (single-GPU layer; EP lines come from --gpus N)
    "tiny": dict(d=256, f=512, n=8, k=2),
    "olmoe": dict(d=2048, f=1024, n=64, k=8),
    "q235": dict(d=4096, f=1536, n=128, k=8),
}


def shape_layer(B, name, dev):
    """A block of one of the other BASELINE shapes.  tiny: fp32 experts and
    tokens from the CPU generator (so the reference can run the same weights);
    OLMoE / Q235: bf16 experts drawn on the device (MoEBlock.random, N(0, 0.02)),
    router row 0 zeroed and the mask router drawn as for Q30."""
    import torch

    sh = SHAPES[name]
    cfg = B.MoEBlockConfig(d_h=sh["d"], d_ff=sh["f"], num_experts=sh["n"], top_k=sh["k"])
    if name == "tiny":
        w = make_layer0(26050, sh, torch.float32)
        w["_block"] = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), mask_w=w["mask"],
                                              dtype=torch.float32, device=dev)
        w["_xdtype"] = torch.float32
        return w
    blk = B.MoEBlock.random(cfg, seed=2605, dtype=torch.bfloat16, device=dev)
    with torch.no_grad():
        blk.router_w[0].zero_()
    g = torch.Generator().manual_seed(2606)
    mask = torch.empty(sh["d"], sh["n"]).normal_(0.0, 1.0 / math.sqrt(sh["d"]), generator=g)
    mask[0] = 0.0
    blk.mask_router = B.MaskRouter(mask.to(dev))
    return dict(router=blk.router_w.cpu(), mask=mask, _block=blk)


def run_shapes(B, args, flush, dev, hbm_peak, tc_peak_sus):
    """Decode T in {1, 64} and prefill T = 8192 across the sparsity range for the
    OLMoE and Qwen3-235B layer shapes, and the tiny fp32 config (T = 1024) with
    the reference's own CPU time and the parity of the same call beside it."""
    import torch

    rows = []
    plan = {"tiny": [(1024, 0.0), (1024, 0.5)],
            "olmoe": [(1, 0.0), (1, 0.5), (1, 0.85), (64, 0.0), (64, 0.5), (64, 0.85), (8192, 0.0), (8192, 0.85)],
            "q235": [(1, 0.0), (1, 0.5), (1, 0.85), (64, 0.0), (64, 0.5), (64, 0.85), (8192, 0.0), (8192, 0.85)]}
    for name, points in plan.items():
        sh = SHAPES[name]
        d, f, n, k = sh["d"], sh["f"], sh["n"], sh["k"]
        w = shape_layer(B, name, dev)
        wb = 4 if name == "tiny" else 2
        for t, s in points:
            steps = args.sweep_steps if t <= 1024 else 3
            p = run_point(B, w, t, s, steps, 2, flush, dev, seed=7 if t <= 1024 else 11)
            sec = p["ms"] * 1e-3
            byt = algorithmic_bytes(t, p["s_real"], p["e_act"], p["r"], d, f, n, k, wbytes=wb, xbytes=wb)
            flops = 6 * d * f * p["r"]
            row = {"shape": name, **sh, "T": t, "s_target": s, "s_actual": round(p["s_real"], 4),
                   "E_act": p["e_act"], "us_per_step": round(p["ms"] * 1e3, 2), "tokens_per_s": round(t / sec, 1),
                   "layer_bytes": byt, "hbm_gbs": round(byt / sec / 1e9, 1),
                   "hbm_frac_of_measured": round(byt / sec / 1e9 / hbm_peak, 4),
                   "hbm_frac_of_8tbs": round(byt / sec / 1e9 / 8000.0, 4),
                   "expert_tflops": round(flops / sec / 1e12, 2),
                   "tensor_frac_of_sustained": round(flops / sec / 1e12 / tc_peak_sus, 4),
                   "dtype": "f32" if name == "tiny" else "bf16"}
            if name == "tiny" and not args.no_cpu:
                ref_s, reps, ref_out = time_reference(w, p["h"], p["theta"], budget_s=min(args.cpu_budget, 5.0),
                                                      shape=sh)
                ours = p["layer"].outs["out"].float().cpu().double().numpy()
                row["reference_cpu_us"] = round(ref_s * 1e6, 1)
                row["reference_reps"] = reps
                row["parity_vs_reference_max_rel_err"] = float(np.abs(ours - ref_out).max() / np.abs(ref_out).max())
            rows.append(row)
            del p
        del w
        torch.cuda.empty_cache()
    return rows


def run_lm_decode(args, new_tokens: int = 48):
    """trainer.sample_greedy on the GPU (KV cache, eager vs one CUDA graph per
    step) next to the reference's own sample_greedy on the host, same seed /
    BEAM strategy / prompt; ms per generated token (the window never slides)."""
    import torch

    from paper_2605_14438_b200 import lm as L
    from paper_2605_14438_b200.baselines import RoutingStrategy

    kw = dict(vocab_size=256, d_h=64, n_layers=2, n_heads=4, context_length=64, d_ff=128, num_experts=8,
              top_k=4, seed=0)
    m = L.TinyMoELM(L.ModelConfig(strategy=RoutingStrategy("beam"), **kw))
    rng = np.random.default_rng(77)
    masks = [rng.normal(0.0, 0.5, (kw["d_h"], kw["num_experts"])) for _ in range(kw["n_layers"])]
    for layer, w in zip(m.layers, masks):
        layer["block"].mask_router.weight.copy_(torch.from_numpy(w))
    prompt = np.random.default_rng(3).integers(0, kw["vocab_size"], 8)
    res = {"config": {**kw, "strategy": "beam", "prompt": 8, "new_tokens": new_tokens}}
    for g in (False, True):
        L.sample_greedy(m, prompt, 4, use_graph=g)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gen = L.sample_greedy(m, prompt, new_tokens, use_graph=g)
        res["ms_per_token_graph" if g else "ms_per_token_eager"] = round((time.perf_counter() - t0) * 1e3 / new_tokens, 3)
    if not args.no_cpu:
        try:
            from oracle import ref

            ref.import_beamoe()
            from beamoe.baselines import RoutingStrategy as RS
            from beamoe.trainer import ModelConfig as MC, TinyMoELM as TM, sample_greedy as sg

            rm = TM(MC(strategy=RS("beam"), **kw))
            for layer, w in zip(rm.layers, masks):
                layer["block"].mask_router.weight.data[...] = w
            t0 = time.perf_counter()
            rgen = sg(rm, prompt, 16)
            res["reference_ms_per_token"] = round((time.perf_counter() - t0) * 1e3 / 16, 3)
            res["tokens_match_reference"] = bool(np.array_equal(rgen, gen[:16]))
        except Exception as e:  # reference package not built on this box
            res["reference_ms_per_token"] = None
            res["reference_error"] = str(e)[:120]
    return res


def run_ours(args):
    import torch

    import paper_2605_14438_b200 as B
    from paper_2605_14438_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or os.environ.get("BEAM_BENCH_FORCE_EP") == "1":  # the EP path (forced: 1-rank check)
        from paper_2605_14438_b200 import ep

        return ep.bench_main(args, sys.modules[__name__])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    lib = _lib.load()
    hbm_peak, tc_peak, tc_peak_sus, peak_kind = measured_peaks()
    B.set_expert_path(args.expert_path)
    d, f, n, k = Q30["d"], Q30["f"], Q30["n"], Q30["k"]
    cfg = B.MoEBlockConfig(d_h=d, d_ff=f, num_experts=n, top_k=k)

    w = make_layer0()
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), norm_w=None,
                                  mask_w=w["mask"], dtype=torch.bfloat16, device=dev)
    w["_block"] = blk
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # ---- headline point -------------------------------------------------------
    t, s = args.tokens, args.sparsity
    launches0 = lib.beam_kernel_launches()
    with ClockSampler(dev.index) as clocks:
        pt = run_point(B, w, t, s, args.steps, args.warmup, flush, dev)
    ms = pt["ms"]
    c0 = lib.beam_kernel_launches()
    pt["layer"].eager()  # the graph replays exactly this launch sequence
    torch.cuda.synchronize()
    launches_per_step = int(lib.beam_kernel_launches() - c0)
    value = t / (ms / 1e3)
    layer = pt["layer"]

    # ---- stage breakdown + dominant-kernel roofline (eager, stage events) -----
    for _ in range(3):
        layer.eager()
    torch.cuda.synchronize()
    import ctypes

    lib.beam_profile_begin(args.steps)
    for _ in range(args.steps):
        flush.zero_()
        layer.eager()
    stage = (ctypes.c_float * 5)()
    ncalls = ctypes.c_int()
    lib.beam_profile_end(stage, ctypes.byref(ncalls))
    names = ("gate", "permute", "experts_gateup", "experts_down", "combine")
    stage_us = {nm: stage[i] * 1e3 / max(ncalls.value, 1) for i, nm in enumerate(names)}
    gu_bytes = gateup_bytes(t, pt["e_act"], pt["r"], d, f)
    dn_bytes = pt["e_act"] * d * f * 2 + pt["r"] * f * 2 + pt["r"] * d * 4  # W_down + bf16 act in + fp32 rows out
    gu_gbs = gu_bytes / (stage_us["experts_gateup"] * 1e-6) / 1e9
    layer_bytes = algorithmic_bytes(t, pt["s_real"], pt["e_act"], pt["r"], d, f, n)

    # ---- e2e through the public API with pinned host buffers -------------------
    h_pin = pt["h"].pin_memory()
    from paper_2605_14438_b200.beam import LayerOutputs

    probe = LayerOutputs(t, d, n, k, torch.bfloat16, "cpu")
    for _ in range(args.warmup):
        B.beam_block_forward(h_pin, blk, training=False)
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, dec, md = B.beam_block_forward(h_pin, blk, training=False)  # H2D + layer + D2H + sync
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_value = t / (np.mean(e2e_ms) / 1e3)

    # ---- parity of this exact workload vs the reference (cheap: T <= 64) ------
    parity = None
    cpu = None
    if not args.no_cpu:
        ref_s, reps, ref_out = time_reference(w, pt["h"], pt["theta"], budget_s=args.cpu_budget)
        cores, api = cpu_cores_used()
        ours = layer.outs["out"].float().cpu().double().numpy()
        parity = float(np.abs(ours - ref_out).max() / np.abs(ref_out).max())
        cpu = {"value": t / ref_s, "unit": "tokens/s", "cores": cores, "kind": "reference",
               "sample": f"{reps} calls of beamoe.beam.beam_block_forward(training=False) on the same "
                         f"T={t} tokens / weights / mask (numpy fp64 + Cython, {api} threads={cores}), "
                         f"{ref_s*1e3:.1f} ms per call"}

    # ---- sparsity sweep ------------------------------------------------------
    sweep = []
    if not args.no_sweep:
        for tt in SWEEP_T:
            for ss in SWEEP_S:
                p = run_point(B, w, tt, ss, args.sweep_steps, 2, flush, dev)
                byt = algorithmic_bytes(tt, p["s_real"], p["e_act"], p["r"], d, f, n)
                sweep.append({"T": tt, "s_target": ss, "s_actual": round(p["s_real"], 4), "E_act": p["e_act"],
                              "us_per_step": round(p["ms"] * 1e3, 2), "tokens_per_s": round(tt / (p["ms"] / 1e3), 1),
                              "layer_bytes": byt, "hbm_frac_of_measured": round(byt / (p["ms"] * 1e-3) / 1e9 / hbm_peak, 4),
                              "hbm_frac_of_8tbs": round(byt / (p["ms"] * 1e-3) / 1e9 / 8000.0, 4)})
                del p
        if not args.no_prefill:
            for ss in (0.0, 0.5, 0.85):
                p = run_point(B, w, 8192, ss, 3, 1, flush, dev, seed=11)
                r = p["r"]
                flops = 6 * d * f * r
                byt = algorithmic_bytes(8192, p["s_real"], p["e_act"], r, d, f, n)
                sec = p["ms"] * 1e-3
                sweep.append({"T": 8192, "s_target": ss, "s_actual": round(p["s_real"], 4), "E_act": p["e_act"],
                              "us_per_step": round(p["ms"] * 1e3, 1), "tokens_per_s": round(8192 / sec, 1),
                              "expert_tflops": round(flops / sec / 1e12, 2),
                              "tensor_frac_of_measured": round(flops / sec / 1e12 / tc_peak, 4),
                              "tensor_frac_of_sustained": round(flops / sec / 1e12 / tc_peak_sus, 4),
                              "hbm_frac_of_measured": round(byt / sec / 1e9 / hbm_peak, 4)})
                del p

    # ---- SPEC C9 / `beamoe bench-dispatch` defaults (cli.py:386-403): grouped
    #      execution at active fractions 1.0 / 0.5 / 0.25, min over 20 reps --------
    bench_dispatch = None
    if not args.no_sweep:
        rows = B.dispatch.bench_dispatch(num_tokens=4096, num_experts=8, top_k=4, d_h=256, d_ff=512,
                                         active_fractions=[1.0, 0.5, 0.25], repetitions=20, seed=0)
        bench_dispatch = {"config": "T=4096 N=8 K=4 d_h=256 d_ff=512 block 16 seed 0, fp32 tokens, bf16 experts "
                                    "(reference test_acceptance.py:299-313 / cli.py:386-403)",
                          "rows": [{"active_fraction": r.active_fraction, "slots_executed": r.slots_executed,
                                    "us_min": round(r.wall_time_ns_min / 1e3, 2),
                                    "us_mean": round(r.wall_time_ns_mean / 1e3, 2)} for r in rows],
                          "strictly_decreasing": bool(rows[0].wall_time_ns_min > rows[1].wall_time_ns_min
                                                      > rows[2].wall_time_ns_min)}

    # ---- the other BASELINE shapes (tiny fp32, OLMoE, Qwen3-235B) ------------------
    shapes = [] if args.no_shapes else run_shapes(B, args, flush, dev, hbm_peak, tc_peak_sus)

    # ---- mask-router training step: forward over all K candidates
    #      + fused slot-dot / closed-form STE backward + x_n^T dA (cuBLAS) ---------
    train = []
    if not args.no_train:
        for tt in (64, 8192):
            p = run_point(B, w, tt, 0.5, 2, 1, flush, dev, seed=13)
            x = p["h"].to(dev)
            dy = torch.randn(tt, d, device=dev)
            for _ in range(2):
                B.mask_router_backward(x, blk, dy, beta=0.5)
            evs = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                B.mask_router_backward(x, blk, dy, beta=0.5)
                e1.record()
                evs.append((e0, e1))
            torch.cuda.synchronize()
            us = float(np.mean([a.elapsed_time(b) for a, b in evs])) * 1e3
            train.append({"T": tt, "s_target": 0.5, "us_per_step": round(us, 1),
                          "inference_us_per_step": round(p["ms"] * 1e3, 1),
                          "candidate_expert_flops": 6 * d * f * tt * k,
                          "what": "beam.mask_router_backward: gate + every top-K candidate through the expert "
                                  "kernels + fused slot-dot/STE + grad_weight GEMM (eager)"})
            del p

    # ---- tiny MoE LM greedy decoding: ms per generated token ------
    lm_line = None
    if not args.no_train:
        lm_line = run_lm_decode(args)

    launches = lib.beam_kernel_launches() - launches0
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": workload_config(t, s),
        "measurement": {"sparsity_actual": round(pt["s_real"], 4), "E_act": pt["e_act"],
                        "surviving_slots": pt["r"], "l2": "flushed (512 MiB memset) before every timed step, not timed",
                        "timing": "CUDA events per step around a CUDA-graph replay of the public layer call"},
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": t * d * 2,
                "d2h_bytes_per_step": probe.nbytes,
                "path": "paper_2605_14438_b200.beam_block_forward(pinned host h) -> host outputs"},
        "roofline": {"bound": "hbm", "kernel": gateup_kernel_name(t, pt["r"], pt["e_act"], f) + " (experts gate/up, weight streaming)",
                     "achieved": gu_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gu_gbs / hbm_peak,
                     "frac_of_8tbs": gu_gbs / 8000.0,
                     "peak_kind": peak_kind + " (copy bandwidth, MEASURED_PEAKS.json hbm_gbs)",
                     "traffic": ncu_traffic(gateup_kernel_name(t, pt["r"], pt["e_act"], f), f"T={t} s={s}"),
                     "algorithmic_bytes_per_launch": gu_bytes,
                     "layer": {"bytes": layer_bytes, "achieved_gbs": layer_bytes / (ms * 1e-3) / 1e9,
                               "frac": layer_bytes / (ms * 1e-3) / 1e9 / hbm_peak},
                     "experts_down": {"bytes": dn_bytes, "achieved_gbs": dn_bytes / (stage_us["experts_down"] * 1e-6) / 1e9}},
        "stages_us": {k2: round(v, 2) for k2, v in stage_us.items()},
        "cpu_baseline": cpu,
        "parity_vs_reference_max_rel_err": parity,
        "clocks": clocks.summary(),
        "gpu_launches": launches_per_step * args.steps,
        "gpu_launches_per_step": launches_per_step,
        "gpu_launches_counted_total": int(launches),
        "sweep": sweep,
        "bench_dispatch": bench_dispatch,
        "shapes": shapes,
        "train_mask_router": train,
        "lm_greedy_decode": lm_line,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--tokens", type=int, default=64)
    ap.add_argument("--sparsity", type=float, default=0.5)
    ap.add_argument("--sweep-steps", type=int, default=20)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--no-shapes", action="store_true", help="skip the tiny / OLMoE / Qwen3-235B shape lines")
    ap.add_argument("--expert-path", default="auto", choices=("auto", "simt", "tc", "tc1"),
                    help="expert-stage kernels (diagnostics; default auto)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
