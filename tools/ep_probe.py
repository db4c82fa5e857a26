"""Where the expert-parallel step spends its time (1 rank, NCCL): torch.profiler
summary of one EPBeamLayer.forward at the bench's Q30 decode shape."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_14438_b200 as B  # noqa: E402
from paper_2605_14438_b200.ep import EPBeamLayer  # noqa: E402


def main(t=64):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    q = bench.Q30
    cfg = B.MoEBlockConfig(d_h=q["d"], d_ff=q["f"], num_experts=q["n"], top_k=q["k"])
    w = bench.make_layer0()
    theta = bench.calibrate_theta(bench.make_tokens(t, 7), w["router"], w["mask"], q["k"], 0.5)
    blk = B.MoEBlock.from_weights(cfg, w["router"], (w["wg"], w["wu"], w["wd"]),
                                  mask_w=bench.mask_with_theta(w["mask"], theta), dtype=torch.bfloat16, device=dev)
    layer = EPBeamLayer(blk)
    x = bench.make_tokens(t, 7).to(dev)
    for _ in range(5):
        layer.forward(x)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            layer.forward(x)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 64)
