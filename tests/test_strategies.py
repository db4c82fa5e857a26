"""Routing strategies (baselines.py) through the BEAM kernels.

CPU: the oracle's restatement of baselines.route / block_forward (inference)
reproduces the reference's own outputs (tests/golden/strategies.npz, made by
tests/golden/make_golden.py from the unmodified reference).
GPU: baselines.block_forward on the sm_100a path (beam_layer_forward_routed)
matches the oracle on identical parameters — ids / kept ids bit-exact (away
from fp32-vs-fp64 decision boundaries), outputs within the fp32 tolerance
max|gpu - oracle| / max|oracle| <= 1e-4 (fp32 experts)."""

import os

import numpy as np
import pytest

from oracle import beam_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "strategies.npz")


def _cases():
    g = np.load(GOLD)
    for i in range(int(g["n_cases"])):
        p = f"c{i}_"
        seed, d, f, n, k, sh, norm, t, bsoft = (int(v) for v in g[p + "cfg"])
        kind = str(g[p + "kind"])
        params = {key[len(p + "param_"):]: float(g[key]) for key in g.files if key.startswith(p + "param_")}
        for key in ("k_small", "k_infer", "null_count"):
            if key in params:
                params[key] = int(params[key])
        experts = [(g[p + "w_gate"][e], g[p + "w_up"][e], g[p + "w_down"][e]) for e in range(n)]
        shared = [(g[p + "s_gate"][e], g[p + "s_up"][e], g[p + "s_down"][e]) for e in range(sh)]
        ob = O.OracleBlock(d_h=d, d_ff=f, num_experts=n, top_k=k, router_w=g[p + "router_w"], experts=experts,
                           shared=shared, norm_w=np.ones(d) if norm else None,
                           mask_w=g[p + "mask_w"] if p + "mask_w" in g.files else np.zeros((d, n)),
                           tau=params.get("tau", 0.5))
        yield i, kind, params, bool(bsoft), ob, g[p + "h"], {key[len(p):]: g[key] for key in g.files if key.startswith(p)}


@pytest.mark.parametrize("case", list(range(9)))
def test_oracle_strategies_match_reference(case):
    for i, kind, params, bsoft, ob, h, ref in _cases():
        if i != case:
            continue
        out, rr = O.strategy_block_forward(h, ob, kind, params, bsoft, block_size=4)
        np.testing.assert_array_equal(rr.kept_ids, ref["kept_ids"])
        np.testing.assert_array_equal(rr.candidate_ids, ref["candidate_ids"])
        np.testing.assert_array_equal(rr.active_bits, ref["active_bits"])
        np.testing.assert_array_equal(rr.active_counts, ref["active_counts"])
        np.testing.assert_allclose(rr.weights_hat, ref["weights_hat"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(rr.logits, ref["logits"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(out, ref["out"], rtol=0, atol=1e-10)
        if "raw_mask" in ref:
            np.testing.assert_allclose(rr.raw_mask, ref["raw_mask"], rtol=0, atol=1e-12)


def test_strategy_validation_messages():
    torch = pytest.importorskip("torch")  # noqa: F841
    from paper_2605_14438_b200 import ContractError, MoEBlockConfig
    from paper_2605_14438_b200.baselines import RoutingStrategy, temperature_at

    cfg = MoEBlockConfig(d_h=8, d_ff=4, num_experts=4, top_k=2)
    for kind, params, msg in [("nope", {}, "unknown routing strategy"),
                              ("topk_pruning", {"k_infer": 3}, "k_infer"),
                              ("moe_dynamic", {"phi": 0.0}, "phi"),
                              ("soft_mask", {"tau": 1.0}, "tau"),
                              ("beam", {"k": 1}, "unknown params")]:
        with pytest.raises(ContractError, match=msg):
            RoutingStrategy(kind, params).validate(cfg)
    assert temperature_at(0, 10, 0.1) == 1.0 and temperature_at(10, 10, 0.1) == pytest.approx(0.1)


@pytest.mark.gpu
@pytest.mark.parametrize("case", list(range(9)))
def test_gpu_strategies_match_oracle(case):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2605_14438_b200 as B
    from paper_2605_14438_b200.baselines import RoutingStrategy, block_forward
    from _beamtest import f32_round, normwise_rel, topk_margin_ok

    for i, kind, params, bsoft, ob, h, _ref in _cases():
        if i != case:
            continue
        q = f32_round
        ob.router_w, ob.mask_w = q(ob.router_w), q(ob.mask_w)
        ob.experts = [tuple(q(w) for w in e) for e in ob.experts]
        ob.shared = [tuple(q(w) for w in e) for e in ob.shared]
        h = q(h)
        cfg = B.MoEBlockConfig(d_h=ob.d_h, d_ff=ob.d_ff, num_experts=ob.num_experts, top_k=ob.top_k,
                               num_shared=len(ob.shared), has_norm=ob.norm_w is not None)
        mask_w = ob.mask_w if kind in ("beam", "soft_mask", "soft_mask_tempered") else None
        gb = B.MoEBlock.from_weights(cfg, ob.router_w, ob.experts, ob.shared, norm_w=ob.norm_w, mask_w=mask_w,
                                     tau=ob.tau, dtype=torch.float32)
        out, rr = block_forward(torch.from_numpy(h).float().cuda(), gb, RoutingStrategy(kind, params),
                                training=False, binarize_soft=bsoft, block_size=4)
        ref_out, ref = O.strategy_block_forward(h, ob, kind, params, bsoft, block_size=4)
        kk = rr.candidate_ids.shape[1]
        ok = topk_margin_ok(ref.logits, kk, 1e-5)
        if kind in ("beam", "soft_mask", "soft_mask_tempered"):
            x_n = ob.normalize(h)
            pre = x_n @ ob.mask_w
            temp = params.get("temp_floor", 0.1) if kind == "soft_mask_tempered" else 1.0
            boundary = np.abs(pre / temp - np.log(ob.tau / (1 - ob.tau))) < 1e-5
            ok &= ~boundary.any(axis=1)
        assert ok.mean() > 0.8
        np.testing.assert_array_equal(rr.candidate_ids.cpu().numpy()[ok], ref.candidate_ids[ok])
        np.testing.assert_array_equal(rr.kept_ids.cpu().numpy()[ok], ref.kept_ids[ok])
        o = out.cpu().numpy().astype(np.float64)
        assert normwise_rel(o[ok], ref_out[ok]) <= 1e-4
        assert normwise_rel(rr.weights_hat.cpu().numpy()[ok].astype(np.float64), ref.weights_hat[ok]) <= 1e-5
