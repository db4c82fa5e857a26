"""Decode points of the Q30 layer (bench.py's workload and timing: CUDA-graph
replay, L2 flushed before every step) with the per-stage breakdown of eager
calls (beam_profile_begin/end).  One JSON line per point.

    python tools/decode_points.py [--T 1,8,64] [--s 0,0.5,0.875] [--steps 50]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_14438_b200 as B  # noqa: E402
from paper_2605_14438_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", default="1,8,64")
    ap.add_argument("--s", default="0,0.5,0.875")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--shape", default="q30", choices=("q30", "olmoe", "q235"))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if args.shape == "q30":
        q = bench.Q30
        cfg = B.MoEBlockConfig(d_h=q["d"], d_ff=q["f"], num_experts=q["n"], top_k=q["k"])
        w = bench.make_layer0()
        w["_block"] = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), mask_w=w["mask"],
                                              dtype=torch.bfloat16, device=dev)
    else:
        w = bench.shape_layer(B, args.shape, dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    lib = _lib.load()
    names = ("gate", "permute", "experts_gateup", "experts_down", "combine")
    for t in (int(x) for x in args.T.split(",")):
        for s in (float(x) for x in args.s.split(",")):
            p = bench.run_point(B, w, t, s, args.steps, 5, flush, dev)
            layer = p["layer"]
            for _ in range(3):
                layer.eager()
            torch.cuda.synchronize()
            lib.beam_profile_begin(args.steps)
            for _ in range(args.steps):
                flush.zero_()
                layer.eager()
            st = (ctypes.c_float * 5)()
            nc = ctypes.c_int()
            lib.beam_profile_end(st, ctypes.byref(nc))
            stages = {nm: round(st[i] * 1e3 / max(nc.value, 1), 2) for i, nm in enumerate(names)}
            print(json.dumps({"shape": args.shape, "T": t, "s": s, "s_real": round(p["s_real"], 4),
                              "E_act": p["e_act"], "us": round(p["ms"] * 1e3, 2), "stages_eager_us": stages,
                              "gate_mode": os.environ.get("BEAM_GATE_MODE", "auto")}), flush=True)
            del p, layer


if __name__ == "__main__":
    main()
