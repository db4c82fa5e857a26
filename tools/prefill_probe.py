"""Prefill step timing modes at the bench's Q30 shape (diagnostics): CUDA-graph
replay vs eager launches, with / without the L2 flush between steps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_14438_b200 as B  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    Q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=Q["d"], d_ff=Q["f"], num_experts=Q["n"], top_k=Q["k"])
    w = bench.make_layer0()
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), norm_w=None,
                                  mask_w=w["mask"], dtype=torch.bfloat16, device=dev)
    w["_block"] = blk
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    t = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    s = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    p = bench.run_point(B, w, t, s, 3, 2, flush, dev, seed=11)
    layer = p["layer"]
    for graph in (True, False):
        for fl in (True, False):
            evs = []
            for _ in range(10):
                if fl:
                    flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                layer.replay() if graph else layer.eager()
                b.record()
                evs.append((a, b))
            torch.cuda.synchronize()
            ms = [x.elapsed_time(y) for x, y in evs]
            print(f"T={t} s={s} graph={graph} flush={fl}: median {np.median(ms)*1e3:.1f} us, min {min(ms)*1e3:.1f}")


if __name__ == "__main__":
    main()
