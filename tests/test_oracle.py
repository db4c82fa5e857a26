"""Pin the CPU oracle (oracle/beam_oracle.py) against the reference's own
outputs: the committed golden vectors (tests/golden/, generated from the
reference package by tests/golden/make_golden.py) and, where oracle/_ref is
built, live reference runs.  CPU only."""

import numpy as np
import pytest

from oracle import beam_oracle as O
from oracle import ref
from _beamtest import golden_block


def _plan_flat(plan):
    offs = [0]
    for e in range(plan.num_experts):
        offs.append(offs[-1] + plan.padded_count(e))
    toks = np.concatenate(plan.tokens) if plan.num_experts else np.zeros(0, np.int64)
    slots = np.concatenate(plan.slots) if plan.num_experts else np.zeros(0, np.int64)
    return np.asarray(offs), toks, slots


def test_mask_route_golden(golden):
    g = golden("mask_route")
    for i in range(int(g["n_cases"])):
        out = O.mask_route(g[f"ids_{i}"], g[f"a_{i}"])
        assert np.array_equal(out, g[f"out_{i}"]), i


def test_align_block_golden(golden):
    g = golden("align_block")
    for i in range(int(g["n_cases"])):
        plan = O.align_block(g[f"ids_{i}"], int(g[f"bs_{i}"]), int(g[f"n_{i}"]))
        offs, toks, slots = _plan_flat(plan)
        assert np.array_equal(plan.real_counts, g[f"plan_counts_{i}"]), i
        assert np.array_equal(offs, g[f"plan_offsets_{i}"]), i
        assert np.array_equal(toks, g[f"plan_tokens_{i}"]), i
        assert np.array_equal(slots, g[f"plan_slots_{i}"]), i


def test_topk_route_golden(golden):
    g = golden("topk_route")
    for i in range(int(g["n_cases"])):
        dec = O.topk_route(g[f"x_{i}"], g[f"w_{i}"], int(g[f"k_{i}"]))
        assert np.array_equal(dec.topk_indices, g[f"ids_{i}"]), i
        assert np.array_equal(dec.logits, g[f"logits_{i}"]), i
        np.testing.assert_allclose(dec.weights, g[f"weights_{i}"], rtol=0, atol=1e-15)


def test_layer_golden(golden):
    g = golden("layer")
    for i in range(int(g["n_cases"])):
        block, h, bs = golden_block(g, i)
        r = O.beam_block_forward(h, block, block_size=bs)
        p = f"c{i}_"
        assert np.array_equal(r.decision.topk_indices, g[p + "topk_ids"])
        assert np.array_equal(r.masked_ids, g[p + "masked_ids"])
        assert np.array_equal(r.mask.mask, g[p + "mask"])
        offs, toks, slots = _plan_flat(r.plan)
        assert np.array_equal(toks, g[p + "plan_tokens"]) and np.array_equal(slots, g[p + "plan_slots"])
        assert np.array_equal(offs, g[p + "plan_offsets"])
        # identical float64 arithmetic, same op order -> bit-identical
        assert np.array_equal(r.out, g[p + "out"]), i
        assert np.array_equal(r.decision.weights, g[p + "weights"])
        assert np.array_equal(r.mask.raw_mask, g[p + "raw_mask"])


def test_q30_dyadic_golden(golden):
    g = golden("q30route_dyadic")
    h = g["hq"].astype(np.float64) / 8
    router = g["rq"].astype(np.float64) / 256
    mask_w = g["mq"].astype(np.float64) / 256
    dec = O.topk_route(h, router, 8)
    md = O.mask_forward(h, mask_w)
    assert np.array_equal(dec.logits, g["logits"])
    assert np.array_equal(dec.topk_indices, g["topk_ids"])
    assert np.array_equal(md.pre_activation, g["pre_activation"])
    masked = O.mask_route(dec.topk_indices, md.pre_activation)
    assert np.array_equal(masked, g["masked_ids"])
    plan = O.align_block(masked, 16, 128)
    offs, toks, slots = _plan_flat(plan)
    assert np.array_equal(toks, g["plan_tokens"]) and np.array_equal(offs, g["plan_offsets"])
    # fp32 exactness of the dyadic construction: every logit is a
    # multiple of 2^-11 with |value| < 2^9, so float32 holds it exactly
    for arr in (dec.logits, md.pre_activation):
        assert np.array_equal(arr.astype(np.float32).astype(np.float64), arr)
        assert np.array_equal(arr * 2048, np.round(arr * 2048))


def test_grouped_equals_naive_oracle():
    rng = np.random.default_rng(7)
    for _ in range(20):
        t, n, k, d, f = 16, 8, 4, 6, 5
        ids = np.stack([rng.choice(n, size=k, replace=False) for _ in range(t)]).astype(np.int64)
        keep = rng.random((t, k)) >= rng.uniform(0, 1)
        masked = np.where(keep, ids, -1)
        w = np.zeros((t, n))
        for a in range(t):
            for b in range(k):
                if keep[a, b]:
                    w[a, ids[a, b]] = rng.uniform(0.05, 1.0)
        experts = [tuple(rng.normal(0, 0.4, s) for s in ((d, f), (d, f), (f, d))) for _ in range(n)]
        h = rng.normal(size=(t, d))
        plan = O.align_block(masked, int(rng.choice([1, 2, 16])), n)
        assert np.max(np.abs(O.grouped_execute(h, plan, experts, w) - O.naive_execute(h, masked, experts, w))) < 1e-9


def test_contract_errors():
    with pytest.raises(O.ContractError):
        O.align_block(np.zeros((1, 1), np.int64), 0, 1)
    plan = O.align_block(np.array([[0]]), 1, 1)
    e = [(np.ones((1, 1)), np.ones((1, 1)), np.ones((1, 1)))]
    with pytest.raises(O.ContractError):
        O.grouped_execute(np.ones((1, 1)), plan, e, np.zeros((1, 1)))


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_make_block_matches_reference_draw_order():
    beamoe = ref.import_beamoe()
    from beamoe.moe import MoEBlock, MoEBlockConfig

    for sh in (0, 2):
        cfg = MoEBlockConfig(d_h=12, d_ff=7, num_experts=5, top_k=2, num_shared=sh)
        rb = MoEBlock(cfg, np.random.default_rng(3))
        ob = O.make_block(12, 7, 5, 2, np.random.default_rng(3), num_shared=sh)
        assert np.array_equal(rb.router_w.data, ob.router_w)
        for re_, oe in zip(rb.experts + rb.shared, ob.experts + ob.shared):
            assert np.array_equal(re_.w_gate.data, oe[0])
            assert np.array_equal(re_.w_up.data, oe[1])
            assert np.array_equal(re_.w_down.data, oe[2])


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_layer_matches_live_reference():
    beamoe = ref.import_beamoe()
    from beamoe.beam import beam_block_forward
    from beamoe.tensor import Tensor

    rng = np.random.default_rng(21)
    for trial in range(5):
        ob = O.make_block(24, 16, 8, 3, rng, num_shared=trial % 2, init_std=0.3)
        ob.mask_w = rng.normal(0, 1.0, ob.mask_w.shape)
        h = rng.normal(size=(13, 24))
        out, dec, md = beam_block_forward(Tensor(h), ref.to_reference_block(ob, beamoe), training=False)
        r = O.beam_block_forward(h, ob)
        assert np.array_equal(out.data, r.out)
        assert np.array_equal(dec.topk_indices, r.decision.topk_indices)


# ---------------------------------------------------------------------------
# mask-router training (beam.py:87-157) against the reference's autograd tape
# ---------------------------------------------------------------------------


def test_mask_router_backward_matches_reference_tape(golden):
    from _beamtest import ste_golden_block

    g = golden("ste")
    for i in range(int(g["n_cases"])):
        block, h, dy, beta = ste_golden_block(g, i)
        r = O.mask_router_backward(h, block, dy, beta)
        p = f"c{i}_"
        assert np.array_equal(r.decision.topk_indices, g[p + "topk_ids"])
        # training forward == inference forward (test_beam.py:281-292 pins 1e-9)
        assert np.max(np.abs(r.out - g[p + "out"])) < 1e-12
        assert np.max(np.abs(r.grad_pre_activation - g[p + "grad_pre_activation"])) < 1e-10, i
        assert np.max(np.abs(r.grad_weight - g[p + "grad_weight"])) < 1e-10, i
        assert abs(r.loss_reg - float(g[p + "loss_reg"])) < 1e-14
        # non-candidates receive exactly zero (test_beam.py:244-249)
        off = np.ones_like(r.grad_pre_activation, dtype=bool)
        np.put_along_axis(off, r.decision.topk_indices, False, -1)
        assert np.all(g[p + "grad_pre_activation"][off] == 0.0)
        assert np.all(r.grad_pre_activation[off] == 0.0)


def test_ste_backward_kats():
    """test_beam.py:251-257: zero upstream -> candidates strictly positive, rest 0;
    beta < 0 is a ContractError (beam.py:117-118)."""
    rng = np.random.default_rng(77)
    t, n, k = 5, 6, 3
    weights = np.zeros((t, n))
    idx = np.stack([rng.choice(n, size=k, replace=False) for _ in range(t)])
    np.put_along_axis(weights, idx, 1.0 / k, -1)
    a = rng.normal(size=(t, n))
    grad = O.ste_backward(np.zeros((t, n)), weights, a, beta=0.7, k=k)
    assert np.all(grad[weights > 0] > 0.0) and np.all(grad[weights == 0] == 0.0)
    with pytest.raises(O.ContractError):
        O.ste_backward(np.zeros((t, n)), weights, a, beta=-1.0, k=k)


def test_lm_init_matches_reference_draws():
    """paper_2605_14438_b200.lm.TinyMoELM draws its parameters like
    trainer.TinyMoELM (trainer.py:153-176): same seed -> same weights."""
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    ref.import_beamoe()
    import torch
    from beamoe.baselines import RoutingStrategy as RS
    from beamoe.trainer import ModelConfig as MC, TinyMoELM as TM

    from paper_2605_14438_b200 import lm
    from paper_2605_14438_b200.baselines import RoutingStrategy

    kw = dict(vocab_size=40, d_h=32, n_layers=2, n_heads=4, context_length=12, d_ff=48, num_experts=8,
              top_k=4, seed=5)
    r = TM(MC(strategy=RS("beam"), **kw))
    m = lm.TinyMoELM(lm.ModelConfig(strategy=RoutingStrategy("beam"), **kw), device="cpu")
    f32 = lambda a: np.asarray(a, np.float32)  # noqa: E731
    assert np.array_equal(m.wte.numpy(), f32(r.wte.data))
    assert np.array_equal(m.lm_head.numpy(), f32(r.lm_head.data))
    for a, b in zip(m.layers, r.layers):
        for w in ("wq", "wk", "wv", "wo"):
            assert np.array_equal(a[w].numpy(), f32(b[w].data))
        assert np.array_equal(a["block"].router_w.numpy(), f32(b["block"].router_w.data))
    del torch


def test_q30_prefill_dyadic_golden(golden):
    """The oracle's routing half at the prefill size (T=8192, dyadic inputs)
    reproduces the reference's fixture bit for bit (logit / pre-activation
    hashes, ids, mask bits, masked ids, block-16 plan)."""
    import hashlib

    g = golden("q30prefill_dyadic")
    hq = np.random.default_rng(int(g["seed"])).integers(-16, 17, (8192, 2048)).astype(np.int8)
    assert hashlib.sha256(hq.tobytes()).hexdigest() == str(g["hq_sha256"])
    x = hq.astype(np.float64) / 8
    dec = O.topk_route(x, g["rq"].astype(np.float64) / 256, 8)
    md = O.mask_forward(x, g["mq"].astype(np.float64) / 256)
    assert hashlib.sha256(np.ascontiguousarray(dec.logits).tobytes()).hexdigest() == str(g["logits_sha256"])
    assert hashlib.sha256(np.ascontiguousarray(md.pre_activation).tobytes()).hexdigest() == str(
        g["pre_activation_sha256"])
    assert np.array_equal(dec.topk_indices, g["topk_ids"].astype(np.int64))
    assert np.array_equal(np.packbits(md.mask.astype(np.uint8), axis=1), g["mask_bits"])
    masked = O.mask_route(dec.topk_indices, md.pre_activation)
    assert np.array_equal(masked, g["masked_ids"].astype(np.int64))
    offs, toks, slots = _plan_flat(O.align_block(masked, 16, 128))
    assert np.array_equal(offs, g["plan_offsets"].astype(np.int64))
    assert np.array_equal(toks, g["plan_tokens"].astype(np.int64))
    assert np.array_equal(slots, g["plan_slots"].astype(np.int64))
