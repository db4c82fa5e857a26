"""CPU tests of the host-side logic: config validation, weight packing layouts,
error behaviour without a GPU."""

import numpy as np
import pytest
import torch

import paper_2605_14438_b200 as B
from paper_2605_14438_b200 import moe as M


def test_config_validation_mirrors_reference():
    with pytest.raises(B.ContractError):
        B.MoEBlockConfig(d_h=4, d_ff=4, num_experts=2, top_k=3)
    with pytest.raises(B.ContractError):
        B.MoEBlockConfig(d_h=0, d_ff=4, num_experts=2, top_k=1)
    with pytest.raises(B.ContractError):
        B.MoEBlockConfig(d_h=4, d_ff=4, num_experts=2, top_k=1, activation="gelu")
    cfg = B.MoEBlockConfig(d_h=37, d_ff=21, num_experts=4, top_k=2)
    assert cfg.d_pad == 40 and cfg.f_pad == 32


@pytest.mark.parametrize("d,f", [(2048, 768), (37, 21), (8, 16)])
def test_pack_gate_up_layout_and_roundtrip(d, f):
    rng = np.random.default_rng(0)
    e = 3
    g = torch.from_numpy(rng.normal(size=(e, d, f))).float()
    u = torch.from_numpy(rng.normal(size=(e, d, f))).float()
    d_pad, f_pad = (d + 7) // 8 * 8, (f + 15) // 16 * 16
    p = M.pack_gate_up(g, u, d_pad, f_pad)
    assert p.shape == (e, 2 * f_pad, d_pad)
    # packed row 32b+i = gate feature 16b+i, 32b+16+i = up feature 16b+i
    for j in (0, f // 2, f - 1):
        b, i = divmod(j, 16)
        assert torch.equal(p[:, 32 * b + i, :d], g[:, :, j])
        assert torch.equal(p[:, 32 * b + 16 + i, :d], u[:, :, j])
    assert torch.all(p[:, :, d:] == 0)
    g2, u2 = M.unpack_gate_up(p, d, f)
    assert torch.equal(g2, g) and torch.equal(u2, u)


def test_pack_down_layout():
    w = torch.arange(2 * 5 * 3, dtype=torch.float32).view(2, 5, 3)  # [E, f, d]
    p = M.pack_down(w, 8, 16)
    assert p.shape == (2, 8, 16)
    assert torch.equal(p[:, :3, :5], w.transpose(1, 2))
    assert torch.all(p[:, 3:] == 0) and torch.all(p[:, :, 5:] == 0)


def test_expert_init_draw_order_matches_reference():
    """moe.py:76-84 draw order (gate, up, down) on the same numpy generator."""
    from oracle import beam_oracle as O

    ob = O.make_block(6, 5, 3, 2, np.random.default_rng(4))
    rng = np.random.default_rng(4)
    rng.normal(0.0, 0.02, (6, 3))  # router first
    e0 = B.Expert.init_random(6, 5, rng)
    assert np.array_equal(e0.w_gate.numpy(), ob.experts[0][0])
    assert np.array_equal(e0.w_down.numpy(), ob.experts[0][2])


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Without a CUDA device every compute entry fails loudly."""
    cfg = B.MoEBlockConfig(d_h=8, d_ff=8, num_experts=4, top_k=2)
    with pytest.raises(B.BeamNativeError):
        B.MoEBlock(cfg, np.random.default_rng(0))
    with pytest.raises(B.BeamNativeError):
        B.dispatch.mask_route(np.zeros((1, 2), np.int64), np.zeros((1, 4)))
    with pytest.raises(B.BeamNativeError):
        B.topk_route(np.zeros((1, 4)), np.eye(4), 2)
