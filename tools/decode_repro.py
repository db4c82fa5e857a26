"""One fused-decode layer call at the Q30 shape (diagnostics / compute-sanitizer)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_14438_b200 as B  # noqa: E402
from oracle import beam_oracle as O  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from _beamtest import matched_blocks, normwise_rel  # noqa: E402


def main(t=8, mask_std=0.0, seed=108, has_norm=True):
    rng = np.random.default_rng(seed)
    ob = O.make_block(2048, 768, 128, 8, rng, has_norm=has_norm, init_std=0.02)
    ob.mask_w = rng.normal(0, mask_std, (2048, 128)) if mask_std > 0 else np.zeros((2048, 128))
    ob, gb = matched_blocks(ob, "bf16")
    h = torch.from_numpy(rng.normal(size=(t, 2048))).to(torch.bfloat16)
    out, dec, md = B.beam_block_forward(h.cuda(), gb, training=False)
    torch.cuda.synchronize()
    ref = O.beam_block_forward(h.double().numpy(), ob)
    print("rel err", normwise_rel(out.float().cpu().numpy().astype(np.float64), ref.out))


if __name__ == "__main__":
    t = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    ms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    norm = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
    main(t, ms, has_norm=norm)
