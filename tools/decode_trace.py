"""Phase timeline of the fused decode kernel (beam_trace_decode) at the bench's
Q30 decode shapes, L2 flushed before every call (as in bench.py).

Marks: 0 start, 1 projection done, 2 after barrier 1, 3 top-K done, 4 after
barrier 2, 5 plan built, 6 gate/up done (consumers), 7 after barrier 3,
8 down+combine done, 10 producer done, 11 producer's first ring refill."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_14438_b200 as B  # noqa: E402
from paper_2605_14438_b200 import _lib  # noqa: E402
from paper_2605_14438_b200.beam import LayerOutputs, layer_forward_into  # noqa: E402

NAMES = {0: "start", 1: "proj", 2: "bar1", 3: "topk", 4: "bar2", 5: "plan", 6: "gateup", 7: "bar3",
         8: "down", 10: "prod_done", 11: "prod_refill"}


def main(tokens=(1, 8, 64), sparsities=(0.0, 0.5), flush_l2=True):
    dev = torch.device("cuda", 0)
    Q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=Q["d"], d_ff=Q["f"], num_experts=Q["n"], top_k=Q["k"])
    w = bench.make_layer0()
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), norm_w=None,
                                  mask_w=w["mask"], dtype=torch.bfloat16, device=dev)
    lib = _lib.load()
    G = torch.cuda.get_device_properties(0).multi_processor_count
    tr = torch.zeros(64 + 12 * G, dtype=torch.int64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for t in tokens:
        for sp in sparsities:
            hc = bench.make_tokens(t, 7)
            theta = bench.calibrate_theta(hc, w["router"], w["mask"], Q["k"], sp)
            blk.mask_router.weight.copy_(bench.mask_with_theta(w["mask"], theta).to(dev))
            h = hc.to(dev)
            outs = LayerOutputs(t, Q["d"], Q["n"], Q["k"], h.dtype, dev)
            rows, clk = [], []
            for it in range(10):
                if flush_l2:
                    flush.zero_()
                tr.zero_()
                torch.cuda.synchronize()
                lib.beam_trace_decode(ctypes.c_void_p(tr.data_ptr()))
                layer_forward_into(h, blk, outs)
                torch.cuda.synchronize()
                lib.beam_trace_decode(None)
                v = tr.cpu().numpy().astype(np.float64)
                if it >= 2:
                    marks = v[64:].reshape(12, G)
                    t0 = marks[0].min()
                    rows.append([(marks[m].min() - t0, marks[m].max() - t0) if marks[m].max() > 0 else (0, 0)
                                 for m in NAMES])
                    clk.append(np.concatenate([v[38:40], v[24:28], v[28:31], v[32:34], v[44:45], v[40:44], v[36:38]]))
            med = np.median(np.array(rows), axis=0) / 1e3
            print(f"T={t} s={sp} flush={flush_l2}: " +
                  ", ".join(f"{NAMES[m]}={lo:.1f}/{hi:.1f}" for m, (lo, hi) in zip(NAMES, med)) +
                  " | clk proj stage/compute; topk load/rank/softmax/out; plan stage/scan/place; P4 sum wait/item, item=afrag/mma/release/sync/final; P5 sum wait/compute = " +
                  "/".join(f"{x:.0f}" for x in np.median(np.array(clk), axis=0)), flush=True)


if __name__ == "__main__":
    main(flush_l2=("--no-flush" not in sys.argv))
