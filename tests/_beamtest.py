"""Shared test helpers: matched (oracle, GPU) blocks on identical values."""

from __future__ import annotations

import numpy as np

from oracle import beam_oracle as O


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bfloat16 (ties to even), as float64."""
    import torch

    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def f32_round(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def matched_blocks(ob: O.OracleBlock, dtype_name: str = "bf16"):
    """Quantise the oracle block's parameters the way the GPU stores them
    (routers/norm fp32, experts bf16 or fp32), write the dequantised values
    back into the oracle block, and build the GPU block from them."""
    import torch

    from paper_2605_14438_b200 import MaskRouter, MoEBlock, MoEBlockConfig

    q = bf16_round if dtype_name == "bf16" else f32_round
    ob.router_w = f32_round(ob.router_w)
    ob.mask_w = f32_round(ob.mask_w)
    if ob.norm_w is not None:
        ob.norm_w = f32_round(ob.norm_w)
    ob.experts = [tuple(q(w) for w in e) for e in ob.experts]
    ob.shared = [tuple(q(w) for w in e) for e in ob.shared]
    cfg = MoEBlockConfig(d_h=ob.d_h, d_ff=ob.d_ff, num_experts=ob.num_experts, top_k=ob.top_k,
                         num_shared=len(ob.shared), has_norm=ob.norm_w is not None,
                         activation=ob.activation)
    dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
    gb = MoEBlock.from_weights(cfg, ob.router_w, ob.experts, ob.shared,
                               norm_w=ob.norm_w, mask_w=ob.mask_w, tau=ob.tau, dtype=dt)
    assert isinstance(gb.mask_router, MaskRouter)
    return ob, gb


def topk_margin_ok(logits: np.ndarray, k: int, tol: float) -> np.ndarray:
    """Per token: True when the K-th/(K+1)-th logit gap exceeds tol (so fp32 vs
    fp64 cannot flip the top-K set or the rank order of ties... within tol)."""
    s = -np.sort(-logits, axis=-1)
    ok = np.ones(logits.shape[0], dtype=bool)
    if k < logits.shape[1]:
        ok &= (s[:, k - 1] - s[:, k]) > tol
    # rank order inside the top-K: adjacent gaps
    for r in range(k - 1):
        ok &= (s[:, r] - s[:, r + 1]) > tol
    return ok


def assert_kept(ok: np.ndarray, floor: float = 0.9) -> None:
    """Tests that exclude near-tie tokens from an exact comparison must still
    compare most of them: a floor on the kept fraction (and at least one token),
    so an all-excluded case cannot pass vacuously."""
    assert ok.size > 0 and ok.any(), "every token excluded as a near tie"
    assert ok.mean() > floor, f"only {ok.mean():.3f} of the tokens kept (floor {floor})"


def normwise_rel(a: np.ndarray, b: np.ndarray) -> float:
    """max |a - b| / max |b| (the 'max rel err' of the north-star tolerance).
    Empty inputs are an error (a comparison of nothing must not pass)."""
    assert b.size > 0, "normwise_rel on an empty selection"
    den = float(np.max(np.abs(b)))
    return float(np.max(np.abs(a - b))) / den if den > 0 else float(np.max(np.abs(a - b), initial=0.0))


def golden_block(g, i):
    """Rebuild the oracle block of golden layer case i (tests/golden/layer.npz)."""
    seed, d, f, n, k, sh, norm, t, bs = (int(v) for v in g[f"c{i}_cfg"])
    p = f"c{i}_"
    experts = [(g[p + "w_gate"][e], g[p + "w_up"][e], g[p + "w_down"][e]) for e in range(n)]
    shared = [(g[p + "s_gate"][s], g[p + "s_up"][s], g[p + "s_down"][s]) for s in range(sh)]
    block = O.OracleBlock(d_h=d, d_ff=f, num_experts=n, top_k=k, router_w=g[p + "router_w"],
                          experts=experts, shared=shared, norm_w=np.ones(d) if norm else None,
                          mask_w=g[p + "mask_w"])
    return block, g[p + "h"], bs


def mask_margin_ok(ref, tol: float) -> np.ndarray:
    """Per token: every candidate's mask pre-activation is either exactly 0 (exact
    in both precisions; inclusive threshold) or farther than tol from it."""
    a = np.take_along_axis(ref.mask.pre_activation, ref.decision.topk_indices, 1)
    return np.all((np.abs(a) > tol) | (a == 0.0), axis=1)


def ste_golden_block(g, i):
    """Oracle block, h, dy, beta of golden mask-router gradient case i (tests/golden/ste.npz)."""
    seed, d, f, n, k, sh, norm, t = (int(v) for v in g[f"c{i}_cfg"])
    p = f"c{i}_"
    experts = [(g[p + "w_gate"][e], g[p + "w_up"][e], g[p + "w_down"][e]) for e in range(n)]
    shared = [(g[p + "s_gate"][s], g[p + "s_up"][s], g[p + "s_down"][s]) for s in range(sh)]
    block = O.OracleBlock(d_h=d, d_ff=f, num_experts=n, top_k=k, router_w=g[p + "router_w"],
                          experts=experts, shared=shared, norm_w=np.ones(d) if norm else None,
                          mask_w=g[p + "mask_w"])
    return block, g[p + "h"], g[p + "dy"], float(g[p + "beta"])
