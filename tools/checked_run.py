"""Run the layer paths with the device-checked library (BEAM_LIB=checked) and
report the bounds-check word: the compute-sanitizer substitute on this pool.

    BEAM_LIB=checked python tools/checked_run.py [--negative]

Prints one JSON line {"build": ..., "flag": int, "cases": [...]}; with
--negative a plan with an out-of-range token index is fed to grouped_execute
and the flag must come back non-zero (the checks are live)."""

from __future__ import annotations

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_14438_b200 as B  # noqa: E402
from paper_2605_14438_b200 import _lib  # noqa: E402
from paper_2605_14438_b200.ep import EPBeamLayer, virtual_forward  # noqa: E402


def main():
    assert os.environ.get("BEAM_LIB") == "checked"
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(lib.beam_debug_checks(flag.data_ptr()), "beam_debug_checks")
    cases = []
    if "--negative" in sys.argv:
        rng = np.random.default_rng(0)
        t, n, k, d, f = 16, 8, 2, 64, 32
        big = torch.from_numpy(rng.normal(size=(t + 8, d))).float().cuda()
        ids = torch.from_numpy(np.stack([rng.permutation(n)[:k] for _ in range(t)])).cuda()
        w = torch.zeros(t, n, device=dev)
        w.scatter_(1, ids, 0.5)
        plan = B.dispatch.align_block(ids, 1, n)
        plan.flat_tokens[0] = t + 3  # outside [0, T): inside `big`, so the read itself is harmless
        experts = [B.Expert(*(torch.from_numpy(rng.normal(0, 0.1, s)).float() for s in ((d, f), (d, f), (f, d))))
                   for _ in range(n)]
        B.dispatch.grouped_execute(big[:t], plan, experts, w, check=False)
        torch.cuda.synchronize()
        print(json.dumps({"build": lib.beam_build_info().decode(), "flag": int(flag.item()), "negative": True}))
        return
    q = bench.Q30
    w = bench.make_layer0()
    cfg = B.MoEBlockConfig(d_h=q["d"], d_ff=q["f"], num_experts=q["n"], top_k=q["k"])
    theta = bench.calibrate_theta(bench.make_tokens(64, 7), w["router"], w["mask"], q["k"], 0.5)
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]),
                                  mask_w=bench.mask_with_theta(w["mask"], theta), dtype=torch.bfloat16, device=dev)
    for t in (1, 2, 8, 64, 300, 8192):
        for dt in (torch.bfloat16, torch.float32):
            x = bench.make_tokens(t, 11).to(dev, dt)
            B.beam_block_forward(x, blk, training=False)
            cases.append(f"q30 T={t} {str(dt)[6:]}")
    B.set_expert_path("tc")
    B.beam_block_forward(bench.make_tokens(64, 3).to(dev), blk, training=False)
    B.set_expert_path("auto")
    cases.append("q30 T=64 tcgen05 forced")
    B.mask_router_backward(bench.make_tokens(64, 5).to(dev), blk, torch.randn(64, q["d"], device=dev), beta=0.1)
    cases.append("mask_router_backward T=64")
    tcfg = B.MoEBlockConfig(d_h=256, d_ff=512, num_experts=8, top_k=2, num_shared=1)
    tb = B.MoEBlock(tcfg, np.random.default_rng(0), dtype=torch.float32, device=dev)
    tb.mask_router = B.MaskRouter(torch.randn(256, 8, device=dev) / 16)
    B.beam_block_forward(torch.randn(1024, 256, device=dev), tb, training=False)
    cases.append("tiny fp32 T=1024 + shared")
    scfg = B.MoEBlockConfig(d_h=2048, d_ff=768, num_experts=128, top_k=8, num_shared=2)
    sb = B.MoEBlock.random(scfg, seed=3, device=dev)
    sb.mask_router = B.MaskRouter(torch.randn(2048, 128, device=dev) / 45)
    for t in (4, 300):
        B.beam_block_forward(torch.randn(t, 2048, device=dev).to(torch.bfloat16), sb, training=False)
        cases.append(f"shared experts T={t}")
    layers = [EPBeamLayer.from_block(blk, rank=r, world=4) for r in range(4)]
    for ts, fixed in (((64, 3, 0, 40), True), ((300, 70, 500, 1), False)):
        virtual_forward(layers, [bench.make_tokens(t, 5 + t).to(dev) for t in ts], fixed=fixed)
        cases.append(f"virtual EP4 {'fixed' if fixed else 'compact'} T={ts}")
    rng = np.random.default_rng(1)
    ids = torch.from_numpy(np.stack([rng.permutation(128)[:8] for _ in range(8192)]).astype(np.int64)).cuda()
    ids[torch.rand(8192, 8, device=dev) < 0.4] = -1
    B.dispatch.align_block(ids, 16, 128)
    cases.append("align_block T=8192 multi-CTA permute")
    torch.cuda.synchronize()
    print(json.dumps({"build": lib.beam_build_info().decode(), "flag": int(flag.item()), "cases": cases}))


if __name__ == "__main__":
    main()
