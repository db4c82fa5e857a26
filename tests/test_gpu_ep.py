"""Expert-parallel path on the GPU with a single NCCL rank (this run has one
GPU): gating via beam_gate, the exchange through NCCL all_to_all_single, the
local experts via beam_moe_execute; must equal the fused single-GPU layer."""

import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_2605_14438_b200 as B  # noqa: E402
from oracle import beam_oracle as O  # noqa: E402
from _beamtest import mask_margin_ok, matched_blocks, normwise_rel, topk_margin_ok  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("t", [1, 64, 300])
def test_ep_single_rank_matches_layer(nccl_group, t):
    from paper_2605_14438_b200.ep import EPBeamLayer

    rng = np.random.default_rng(40 + t)
    ob = O.make_block(2048, 768, 128, 8, rng, init_std=0.02)
    ob.mask_w = rng.normal(0, 1 / np.sqrt(2048), (2048, 128))
    ob, gb = matched_blocks(ob, "bf16")
    x = torch.from_numpy(rng.normal(size=(t, 2048))).to(torch.bfloat16).cuda()
    ep = EPBeamLayer(gb)
    out_ep = ep.forward(x)
    out, _, _ = B.beam_block_forward(x, gb, training=False)
    # out = h + y is rounded to bf16, so y recovered as out - h carries up to one
    # bf16 ulp of |out| per element on top of the expert-sum differences
    o_ep = out_ep.float().cpu().double().numpy()
    o = out.float().cpu().double().numpy()
    # (for T > 64 the fused layer runs the tcgen05 path: bf16 x_n, act and
    # per-pair rows, vs the fp32 per-pair rows of the EP owner's execute)
    excess = np.abs(o_ep - o) - 2.0 ** -7 * np.abs(o)
    assert excess.max() <= 4e-3, excess.max()
    y_ep, y = o_ep - x.float().cpu().double().numpy(), o - x.float().cpu().double().numpy()
    assert normwise_rel(y_ep, y) <= 6e-2
    ref = O.beam_block_forward(x.double().cpu().numpy(), ob)
    ok = topk_margin_ok(ref.decision.logits, 8, 1e-5) & mask_margin_ok(ref, 1e-5)
    assert normwise_rel(out_ep.float().cpu().double().numpy()[ok], ref.out[ok]) <= 1e-2
