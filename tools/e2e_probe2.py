"""Host-API breakdown of beam_block_forward(pinned host h) at the bench headline
(Q30, T=64, s=0.5): cumulative host timestamps of each step (median of 50)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_14438_b200 as B  # noqa: E402
from paper_2605_14438_b200.beam import LayerOutputs, layer_forward_into  # noqa: E402


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
    h_pin = hc.pin_memory()
    t, d = hc.shape
    n, k = cfg.num_experts, cfg.top_k
    stamps = []
    for it in range(60):
        torch.cuda.synchronize()
        ts = [time.perf_counter()]
        xd = h_pin.to(dev, non_blocking=True)
        ts.append(time.perf_counter())
        outs = LayerOutputs(t, d, n, k, xd.dtype, dev)
        ts.append(time.perf_counter())
        layer_forward_into(xd, blk, outs, 16)
        ts.append(time.perf_counter())
        hb = LayerOutputs(t, d, n, k, xd.dtype, "cpu", pin=True)
        ts.append(time.perf_counter())
        hb.copy_from(outs)
        ts.append(time.perf_counter())
        torch.cuda.current_stream(dev).synchronize()
        ts.append(time.perf_counter())
        _ = (hb["out"], hb["logits"], hb["topk_ids"], hb["weights"], hb["pre_activation"], hb["raw_mask"], hb["mask"])
        ts.append(time.perf_counter())
        if it >= 10:
            stamps.append(np.diff(ts) * 1e6)
    med = np.median(np.array(stamps), axis=0)
    names = ["h2d_issue", "outs_dev_alloc", "layer_launch", "outs_pin_alloc", "d2h_issue", "sync_wait", "views"]
    print({nm: round(float(v), 1) for nm, v in zip(names, med)}, "total", round(float(med.sum()), 1))
    # GPU-side: events around the pieces
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    gs = []
    for it in range(40):
        torch.cuda.synchronize()
        ev[0].record()
        xd = h_pin.to(dev, non_blocking=True)
        ev[1].record()
        layer_forward_into(xd, blk, outs, 16)
        ev[2].record()
        hb.copy_from(outs)
        ev[3].record()
        torch.cuda.synchronize()
        if it >= 10:
            gs.append([ev[0].elapsed_time(ev[1]) * 1e3, ev[1].elapsed_time(ev[2]) * 1e3, ev[2].elapsed_time(ev[3]) * 1e3])
    print("gpu h2d/layer/d2h us:", np.round(np.median(np.array(gs), axis=0), 1))
    wall = []
    for it in range(40):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        B.beam_block_forward(h_pin, blk, training=False)
        wall.append((time.perf_counter() - t0) * 1e6)
    print("public api us (no flush):", round(float(np.median(wall[10:])), 1))


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def check_direct():
    """Host-output path (out written into mapped pinned memory) == device path."""
    dev = torch.device("cuda", 0)
    Q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=Q["d"], d_ff=Q["f"], num_experts=Q["n"], top_k=Q["k"])
    w = bench.make_layer0()
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), norm_w=None,
                                  mask_w=w["mask"], dtype=torch.bfloat16, device=dev)
    from paper_2605_14438_b200 import _lib
    for t in (1, 64, 8192):
        hc = bench.make_tokens(t, 3).pin_memory()
        o1, d1, m1 = B.beam_block_forward(hc, blk, training=False)
        o2, d2, m2 = B.beam_block_forward(hc.to(dev), blk, training=False)
        torch.cuda.synchronize()
        print("T", t, "mapped", _lib.load().beam_host_mapped(o1.data_ptr()), "out equal", torch.equal(o1, o2.cpu()),
              "ids equal", torch.equal(d1.topk_indices, d2.topk_indices.cpu()),
              "mask equal", torch.equal(m1.mask, m2.mask.cpu()))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "check":
    check_direct()
