"""Save the Q30 layer's outputs (bench weights / tokens, s = 0.5 mask) at the given
T values to an .npz, to compare two library settings bit for bit:
    BEAM_X=0 python tools/layer_outputs.py a.npz 1,64,8192; BEAM_X=1 ... b.npz ...
    python tools/layer_outputs.py --cmp a.npz b.npz"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(path, ts):
    import torch

    import bench
    import paper_2605_14438_b200 as B
    dev = torch.device("cuda", 0)
    q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=q["d"], d_ff=q["f"], num_experts=q["n"], top_k=q["k"])
    w = bench.make_layer0()
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), mask_w=w["mask"],
                                  dtype=torch.bfloat16, device=dev)
    res = {}
    for t in ts:
        hc = bench.make_tokens(t, 7)
        theta = bench.calibrate_theta(hc, w["router"], w["mask"], q["k"], 0.5)
        blk.mask_router.weight.copy_(bench.mask_with_theta(w["mask"], theta).to(dev))
        out, dec, md = B.beam_block_forward(hc.to(dev), blk, training=False, block_size=16)
        res[f"T{t}"] = out.float().cpu().numpy()
        res[f"T{t}_ids"] = dec.topk_indices.cpu().numpy()
    np.savez(path, **res)


def cmp(a, b):
    a, b = np.load(a), np.load(b)
    for k in a.files:
        d = np.abs(a[k].astype(np.float64) - b[k].astype(np.float64))
        print(k, "max abs diff", d.max(), "identical" if d.max() == 0 else "DIFFERENT")


if __name__ == "__main__":
    if sys.argv[1] == "--cmp":
        cmp(sys.argv[2], sys.argv[3])
    else:
        run(sys.argv[1], [int(x) for x in sys.argv[2].split(",")])
