"""Public-API latency with host buffers (bench.py's e2e measure) at the headline
workload, eager launch path vs the cached-CUDA-graph host path
(BEAM_HOST_GRAPH=0 / 1), plus the outputs of both compared bit for bit.
    python tools/e2e_probe.py"""
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run():
    import torch
    sys.path.insert(0, ROOT)
    import bench
    import paper_2605_14438_b200 as B
    dev = torch.device("cuda", 0)
    q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=q["d"], d_ff=q["f"], num_experts=q["n"], top_k=q["k"])
    w = bench.make_layer0()
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]), mask_w=w["mask"],
                                  dtype=torch.bfloat16, device=dev)
    res = {}
    for t in (1, 64):
        h = bench.make_tokens(t, 7)
        theta = bench.calibrate_theta(h, w["router"], w["mask"], q["k"], 0.5)
        blk.mask_router.weight.copy_(bench.mask_with_theta(w["mask"], theta).to(dev))
        hp = h.pin_memory()
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        for _ in range(10):
            B.beam_block_forward(hp, blk, training=False)
        ts = []
        for _ in range(50):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out, dec, md = B.beam_block_forward(hp, blk, training=False)
            ts.append(time.perf_counter() - t0)
        print(f"T={t} graph={os.environ.get('BEAM_HOST_GRAPH', '1')}: e2e mean {np.mean(ts) * 1e6:.1f} us, "
              f"min {np.min(ts) * 1e6:.1f} us -> {t / np.mean(ts):.0f} tok/s", flush=True)
        res[f"T{t}_out"] = out.float().numpy()
        res[f"T{t}_ids"] = dec.topk_indices.numpy()
        res[f"T{t}_mask"] = md.mask.numpy()
        res[f"T{t}_logits"] = dec.logits.numpy()
    np.savez(sys.argv[2], **res)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--run":
        run()
    else:
        os.makedirs("/tmp/e2e", exist_ok=True)
        for g in ("0", "1"):
            subprocess.run([sys.executable, __file__, "--run", f"/tmp/e2e/g{g}.npz"], env={**os.environ, "BEAM_HOST_GRAPH": g},
                           check=True)
        a, b = np.load("/tmp/e2e/g0.npz"), np.load("/tmp/e2e/g1.npz")
        print("outputs identical:", all(np.array_equal(a[k], b[k]) for k in a.files))
