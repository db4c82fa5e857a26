"""Where does the host-API time go?  Breaks beam_block_forward(pinned host h)
into its pieces at the bench headline workload (Q30, T=64, s=0.5)."""
import time

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2605_14438_b200 as B
from paper_2605_14438_b200.beam import LayerOutputs, layer_forward_into

import bench


def wall(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return float(np.median(ts))


def main():
    dev = torch.device("cuda", 0)
    Q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=Q["d"], d_ff=Q["f"], num_experts=Q["n"], top_k=Q["k"])
    w = bench.make_layer0()
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), norm_w=None,
                                  mask_w=w["mask"], dtype=torch.bfloat16, device=dev)
    hc = bench.make_tokens(64, 7)
    theta = bench.calibrate_theta(hc, w["router"], w["mask"], Q["k"], 0.5)
    blk.mask_router.weight.copy_(bench.mask_with_theta(w["mask"], theta).to(dev))
    h = hc.to(dev)
    h_pin = hc.pin_memory()
    t, d = h.shape
    outs = LayerOutputs(t, d, cfg.num_experts, cfg.top_k, h.dtype, h.device)
    res = {}
    res["desc_us"] = wall(lambda: blk.layer_desc(0.0))
    res["outs_alloc_dev_us"] = wall(lambda: LayerOutputs(t, d, cfg.num_experts, cfg.top_k, h.dtype, h.device))
    res["outs_alloc_pin_us"] = wall(lambda: LayerOutputs(t, d, cfg.num_experts, cfg.top_k, h.dtype, "cpu", pin=True))
    res["h2d_sync_us"] = wall(lambda: (h_pin.to("cuda", non_blocking=True), torch.cuda.synchronize()))
    res["launch_only_us"] = wall(lambda: layer_forward_into(h, blk, outs))
    torch.cuda.synchronize()
    res["layer_sync_us"] = wall(lambda: (layer_forward_into(h, blk, outs), torch.cuda.synchronize()))
    hb = LayerOutputs(t, d, cfg.num_experts, cfg.top_k, h.dtype, "cpu", pin=True)
    res["d2h_sync_us"] = wall(lambda: (hb.copy_from(outs), torch.cuda.synchronize()))
    res["public_api_us"] = wall(lambda: B.beam_block_forward(h_pin, blk, training=False))
    res["public_api_dev_input_us"] = wall(lambda: (B.beam_block_forward(h, blk, training=False), torch.cuda.synchronize()))
    print(res)


if __name__ == "__main__":
    main()
