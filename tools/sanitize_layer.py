"""Layer calls for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Runs the public layer call eagerly (no CUDA graphs) at the Qwen3-30B-A3B shape
for T = 1, 64 (decode kernels: fused gate, weight-streaming experts, combine)
and T = 8192 (prefill: tensor-core router, top-K, multi-CTA permute, pack,
tcgen05 grouped GEMMs, combine), plus the tiny fp32 config, then synchronises.

    compute-sanitizer --tool memcheck python tools/sanitize_layer.py [--quick]
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_14438_b200 as B  # noqa: E402


def main():
    quick = "--quick" in sys.argv
    dev = torch.device("cuda", 0)
    q = bench.Q30
    w = bench.make_layer0()
    cfg = B.MoEBlockConfig(d_h=q["d"], d_ff=q["f"], num_experts=q["n"], top_k=q["k"])
    theta = bench.calibrate_theta(bench.make_tokens(64, 7), w["router"], w["mask"], q["k"], 0.5)
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]),
                                  mask_w=bench.mask_with_theta(w["mask"], theta), dtype=torch.bfloat16, device=dev)
    sizes = (1, 64) if quick else (1, 8, 64, 8192)
    for t in sizes:
        x = bench.make_tokens(t, 11).to(dev)
        out, dec, md = B.beam_block_forward(x, blk, training=False)
        torch.cuda.synchronize()
        print(f"T={t}: ok, masked {(md.mask == 0).float().mean().item():.3f}", flush=True)
    # fp32 tiny config (configs[0]) with shared experts
    tcfg = B.MoEBlockConfig(d_h=256, d_ff=512, num_experts=8, top_k=2, num_shared=1)
    tb = B.MoEBlock(tcfg, __import__("numpy").random.default_rng(0), dtype=torch.float32, device=dev)
    tb.mask_router = B.MaskRouter(torch.randn(256, 8, device=dev) / 16)
    out, _, _ = B.beam_block_forward(torch.randn(1024 if not quick else 64, 256, device=dev), tb, training=False)
    torch.cuda.synchronize()
    print("tiny fp32: ok", flush=True)


if __name__ == "__main__":
    main()
