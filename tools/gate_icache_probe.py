"""Is the fused gate's serial tail (top-K + plan, one CTA) slow after the L2 flush
because its CODE was evicted?  Phase trace of the real T-token gate after the
512 MiB memset, with and without a 'code warm-up': one call of an unrelated
block (same shapes, other weights, other tokens, its own stream and workspace)
between the flush and the traced call — it brings the kernels' instructions back
into L2 but none of the traced call's data.
    python tools/gate_icache_probe.py"""
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
from gate_trace import FUSED  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    Q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=Q["d"], d_ff=Q["f"], num_experts=Q["n"], top_k=Q["k"])
    w = bench.make_layer0()
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), norm_w=None,
                                  mask_w=w["mask"], dtype=torch.bfloat16, device=dev)
    other = B.MoEBlock.from_weights(cfg, w["router"].flip(0).contiguous(), (w["wg"], w["wu"], w["wd"]), norm_w=None,
                                    mask_w=w["mask"].flip(0).contiguous(), dtype=torch.bfloat16, device=dev)
    lib = _lib.load()
    tr = torch.zeros(16, dtype=torch.int64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    side = torch.cuda.Stream(dev)
    for t in (1, 8, 64):
        hc = bench.make_tokens(t, 7)
        theta = bench.calibrate_theta(hc, w["router"], w["mask"], Q["k"], 0.5)
        blk.mask_router.weight.copy_(bench.mask_with_theta(w["mask"], theta).to(dev))
        h = hc.to(dev)
        h2 = bench.make_tokens(t, 99).to(dev)
        outs = LayerOutputs(t, Q["d"], Q["n"], Q["k"], h.dtype, dev)
        outs2 = LayerOutputs(t, Q["d"], Q["n"], Q["k"], h.dtype, dev)
        for warm in (False, True):
            rows = []
            for it in range(12):
                flush.zero_()
                torch.cuda.synchronize()
                if warm:
                    with torch.cuda.stream(side):
                        layer_forward_into(h2, other, outs2)
                    side.synchronize()
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
            print(f"T={t} code_warm={warm}: " + ", ".join(f"{n}={x:.2f}us" for n, x in zip(FUSED, med)), flush=True)


if __name__ == "__main__":
    main()
