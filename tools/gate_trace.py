"""Phase timeline of the fused decode gate (beam_trace_gate) at the bench's Q30
decode shapes (BEAM_GATE_MODE=fused forces it at every T).  Medians over calls,
microseconds from the first CTA's entry; L2 flushed before every call (as in
bench.py) and not.  (Round 2 also traced a thread-block-cluster gate here —
profiles/r02/gate_traces.log — measured slower and removed.)"""
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

FUSED = ["start_skew", "proj_first", "proj_last", "topk_start", "t0_loaded", "t0_selected", "t0_softmax",
         "t0_stored", "topk_done", "permute_start", "permute_done"]


def main(flush_l2=True):
    dev = torch.device("cuda", 0)
    Q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=Q["d"], d_ff=Q["f"], num_experts=Q["n"], top_k=Q["k"])
    w = bench.make_layer0()
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), norm_w=None,
                                  mask_w=w["mask"], dtype=torch.bfloat16, device=dev)
    lib = _lib.load()
    tr = torch.zeros(16, dtype=torch.int64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for t in (1, 8, 64):
        hc = bench.make_tokens(t, 7)
        theta = bench.calibrate_theta(hc, w["router"], w["mask"], Q["k"], 0.5)
        blk.mask_router.weight.copy_(bench.mask_with_theta(w["mask"], theta).to(dev))
        h = hc.to(dev)
        outs = LayerOutputs(t, Q["d"], Q["n"], Q["k"], h.dtype, dev)
        rows = []
        for it in range(12):
            if flush_l2:
                flush.zero_()
            tr.zero_()
            tr[0] = np.iinfo(np.int64).max
            tr[2] = np.iinfo(np.int64).max
            torch.cuda.synchronize()
            lib.beam_trace_gate(ctypes.c_void_p(tr.data_ptr()))
            layer_forward_into(h, blk, outs)
            torch.cuda.synchronize()
            lib.beam_trace_gate(None)
            v = tr.cpu().numpy().astype(np.float64)
            if it >= 2:
                rows.append([v[1] - v[0], v[2] - v[0], v[3] - v[0], v[6] - v[0], v[8] - v[0], v[9] - v[0],
                             v[10] - v[0], v[11] - v[0], v[4] - v[0], v[7] - v[0], v[5] - v[0]])
        med = np.median(np.array(rows), axis=0) / 1e3
        print(f"T={t} flush={flush_l2} fused: " + ", ".join(f"{n}={x:.2f}us" for n, x in zip(FUSED, med)),
              flush=True)


if __name__ == "__main__":
    main(True)
    main(False)
