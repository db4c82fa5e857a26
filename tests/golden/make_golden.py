"""Generate the golden vectors under tests/golden/ FROM THE REFERENCE ITSELF.

Runs the unmodified reference package (``beamoe``, built into ``oracle/_ref``
by ``oracle/build_ref.sh`` from /root/reference/pkg) on seeded inputs and
stores inputs + outputs as compressed ``.npz`` fixtures.  Only needs to run in
the build container (the GPU box has no /root/reference); the fixtures are
committed.

    python tests/golden/make_golden.py

Cases
-----
mask_route_*      — dispatch.mask_route (dispatch/__init__.py:55-62)
align_*           — dispatch.align_block (dispatch/__init__.py:89-126), many block sizes
topk_*            — moe.topk_route incl. ties (moe.py:116-137)
layer_*           — beam.beam_block_forward(training=False) (beam.py:127-165)
                    on small random blocks (norm / shared / non-zero mask router)
strategies        — baselines.block_forward(training=False) (baselines.py:286-323) for every
                    routing strategy (top-k variants, moe_dynamic, ada_moe, beam, soft masks)
ste               — mask-router gradient of beam_block_forward(training=True) through the
                    reference's autograd tape (beam.py:87-157): L = sum(out * dy) + beta *
                    sparsity_loss; pre-activation and mask-weight gradients (the closed form
                    ste_backward, beam.py:100-124, is pinned to this tape by test_beam.py:231-242)
trace             — analysis.SparsityTrace (analysis.py:19-112) CSV text and the Avg-K
                    reductions (avg_k every group key, position_mask_prob, expert_load)
                    over seeded routing cells in both phases
lm                — trainer.TinyMoELM (trainer.py:150-257) with BEAM routing and seeded mask
                    routers: forward logits, sample_greedy tokens across the sliding window
                    (trainer.py:638-673) with its SparsityTrace CSV, evaluate() (:577-636)
q30route_dyadic   — Qwen3-30B-A3B router shape (N=128, K=8, d=2048), dyadic inputs,
                    so logits / pre-activations are exact in fp32 and fp64: top-K ids,
                    mask bits and the plan must match bit-for-bit.
q30prefill_dyadic — the same at the PREFILL size (configs[2], T=8192): bf16-exact
                    dyadic tokens h = hq/8 regenerated from a seed (sha256-checked),
                    router / mask weights j/256 — routes through the tensor-core
                    router, the top-K kernel and the multi-CTA permute; ids, mask
                    bits, masked ids and the block-16 plan are stored (compactly).

    python tests/golden/make_golden.py [name ...]    # default: every fixture
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402


def _plan_arrays(plan):
    offs = np.zeros(plan.num_experts + 1, dtype=np.int64)
    for e in range(plan.num_experts):
        offs[e + 1] = offs[e] + plan.padded_count(e)
    tokens = np.concatenate([np.asarray(t, dtype=np.int64) for t in plan.tokens]) if plan.num_experts else np.zeros(0, np.int64)
    slots = np.concatenate([np.asarray(s, dtype=np.int64) for s in plan.slots]) if plan.num_experts else np.zeros(0, np.int64)
    return dict(plan_counts=np.asarray(plan.real_counts, dtype=np.int64), plan_offsets=offs,
                plan_tokens=tokens, plan_slots=slots, plan_block_size=np.int64(plan.block_size))


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def make_strategies():
    """Every routing strategy of baselines.route through block_forward(training=False)."""
    ref.import_beamoe()
    from beamoe import baselines
    from beamoe.moe import MoEBlockConfig
    from beamoe.tensor import Tensor

    specs = [
        # (seed, kind, params, binarize_soft, d, f, n, k, shared, has_norm, T, mask_std)
        (21, "vanilla_topk", {}, False, 32, 24, 8, 2, 0, True, 29, 0.0),
        (22, "topk_reduced", {"k_small": 1}, False, 32, 24, 8, 3, 0, True, 31, 0.0),
        (23, "topk_pruning", {"k_infer": 2}, False, 32, 24, 8, 4, 1, True, 17, 0.0),
        (24, "moe_dynamic", {"phi": 0.3}, False, 32, 24, 8, 4, 0, True, 40, 0.0),
        (25, "ada_moe", {"null_count": 3}, False, 32, 24, 8, 3, 0, True, 35, 0.0),
        (26, "beam", {"tau": 0.5}, False, 32, 24, 8, 3, 0, True, 33, 1.0),
        (27, "soft_mask", {"tau": 0.5}, False, 32, 24, 8, 3, 0, True, 27, 1.0),
        (28, "soft_mask", {"tau": 0.5}, True, 32, 24, 8, 3, 0, False, 25, 1.0),
        (29, "soft_mask_tempered", {"tau": 0.5, "temp_floor": 0.2}, False, 32, 24, 8, 3, 1, True, 21, 1.0),
    ]
    arrays = {}
    for i, (seed, kind, params, bsoft, d, f, n, k, sh, norm, t, mstd) in enumerate(specs):
        rng = np.random.default_rng(seed)
        cfg = MoEBlockConfig(d_h=d, d_ff=f, num_experts=n, top_k=k, num_shared=sh, has_norm=norm)
        strat = baselines.RoutingStrategy(kind, dict(params))
        block = baselines.build_block(cfg, strat, rng)
        for e in list(block.experts) + list(block.shared):  # larger weights: visible outputs
            for w in (e.w_gate, e.w_up, e.w_down):
                w.data[...] = rng.normal(0, 0.3, w.data.shape)
        if block.mask_router is not None and mstd > 0:
            block.mask_router.weight.data[...] = rng.normal(0, mstd, (d, n))
        h = rng.normal(size=(t, d))
        out, rr = baselines.block_forward(Tensor(h), block, strat, training=False, binarize_soft=bsoft,
                                          block_size=4)
        p = f"c{i}_"
        arrays[p + "cfg"] = np.array([seed, d, f, n, k, sh, int(norm), t, int(bsoft)], np.int64)
        arrays[p + "kind"] = np.array(kind)
        for key, v in params.items():
            arrays[p + "param_" + key] = np.float64(v)
        arrays[p + "h"] = h
        arrays[p + "router_w"] = block.router_w.data
        if block.mask_router is not None:
            arrays[p + "mask_w"] = block.mask_router.weight.data
        arrays[p + "w_gate"] = np.stack([e.w_gate.data for e in block.experts])
        arrays[p + "w_up"] = np.stack([e.w_up.data for e in block.experts])
        arrays[p + "w_down"] = np.stack([e.w_down.data for e in block.experts])
        if sh:
            arrays[p + "s_gate"] = np.stack([e.w_gate.data for e in block.shared])
            arrays[p + "s_up"] = np.stack([e.w_up.data for e in block.shared])
            arrays[p + "s_down"] = np.stack([e.w_down.data for e in block.shared])
        arrays[p + "out"] = out.data
        arrays[p + "weights_hat"] = rr.weights_hat.data
        arrays[p + "logits"] = rr.logits.data
        arrays[p + "candidate_ids"] = rr.candidate_ids
        arrays[p + "active_bits"] = rr.active_bits
        arrays[p + "active_counts"] = rr.active_counts
        arrays[p + "kept_ids"] = rr.kept_ids
        if rr.raw_mask is not None:
            arrays[p + "raw_mask"] = rr.raw_mask.data
    arrays["n_cases"] = np.int64(len(specs))
    save("strategies", **arrays)


def make_ste():
    """Tape gradients of the BEAM training forward w.r.t. the mask router."""
    ref.import_beamoe()
    from beamoe.beam import MaskRouter, beam_block_forward, sparsity_loss
    from beamoe.moe import MoEBlock, MoEBlockConfig
    from beamoe.tensor import Tape, Tensor, add, mul, tsum

    specs = [
        # (seed, d, f, n, k, shared, has_norm, T, mask_std, beta)
        (21, 32, 24, 8, 2, 0, True, 17, 1.0, 0.5),
        (22, 16, 8, 4, 4, 0, False, 9, 0.8, 0.0),
        (23, 32, 24, 16, 3, 1, True, 40, 2.0, 1.3),
        (24, 24, 16, 6, 1, 0, True, 5, 0.5, 2.0),
    ]
    arrays = {}
    for i, (seed, d, f, n, k, sh, norm, t, mstd, beta) in enumerate(specs):
        rng = np.random.default_rng(seed)
        cfg = MoEBlockConfig(d_h=d, d_ff=f, num_experts=n, top_k=k, num_shared=sh, has_norm=norm)
        block = MoEBlock(cfg, rng, init_std=0.3)
        block.mask_router = MaskRouter(Tensor(rng.normal(0, mstd, (d, n)), requires_grad=True))
        h = rng.normal(size=(t, d))
        dy = rng.normal(size=(t, d))
        with Tape() as tape:
            out, dec, mdec = beam_block_forward(Tensor(h), block, training=True)
            task = tsum(mul(out, Tensor(dy)))
            reg = sparsity_loss(mdec.raw_mask, dec.topk_indices)
            tape.backward(add(task, mul(reg, beta)))
        p = f"c{i}_"
        arrays[p + "cfg"] = np.array([seed, d, f, n, k, sh, int(norm), t], np.int64)
        arrays[p + "beta"] = np.float64(beta)
        arrays[p + "h"] = h
        arrays[p + "dy"] = dy
        arrays[p + "router_w"] = block.router_w.data
        arrays[p + "mask_w"] = block.mask_router.weight.data
        arrays[p + "w_gate"] = np.stack([e.w_gate.data for e in block.experts])
        arrays[p + "w_up"] = np.stack([e.w_up.data for e in block.experts])
        arrays[p + "w_down"] = np.stack([e.w_down.data for e in block.experts])
        if sh:
            arrays[p + "s_gate"] = np.stack([e.w_gate.data for e in block.shared])
            arrays[p + "s_up"] = np.stack([e.w_up.data for e in block.shared])
            arrays[p + "s_down"] = np.stack([e.w_down.data for e in block.shared])
        arrays[p + "out"] = out.data
        arrays[p + "topk_ids"] = dec.topk_indices
        arrays[p + "weights"] = dec.weights.data
        arrays[p + "pre_activation"] = mdec.pre_activation.data
        arrays[p + "raw_mask"] = mdec.raw_mask.data
        arrays[p + "loss_reg"] = np.float64(reg.data)
        arrays[p + "grad_pre_activation"] = mdec.pre_activation.grad
        arrays[p + "grad_weight"] = block.mask_router.weight.grad
    arrays["n_cases"] = np.int64(len(specs))
    save("ste", **arrays)


def make_trace():
    """SparsityTrace rows / CSV / Avg-K metrics from the reference."""
    import tempfile

    ref.import_beamoe()
    from beamoe import analysis

    rng = np.random.default_rng(6000)
    tr = analysis.SparsityTrace()
    arrays = {}
    calls = []
    for layer in range(3):
        for phase, seq in (("prefill", 0), ("decode", 1)):
            t, n, k = 9, 16, 4
            ids = np.stack([rng.choice(n, size=k, replace=False) for _ in range(t)]).astype(np.int64)
            ids[rng.random((t, k)) < 0.05] = -1          # null slots (ada_moe)
            bits = (rng.random((t, k)) < 0.6).astype(np.int64)
            bits[ids < 0] = 0
            masked = np.where(bits == 1, ids, -1)
            pos = rng.permutation(40)[:t].astype(np.int64)
            tok = rng.integers(0, 50, t).astype(np.int64)
            for i in range(t):
                tr.record_cell(seq, int(pos[i]), layer, ids[i], bits[i], phase, int(tok[i]))
            calls.append((ids, masked, pos, tok, layer, phase, seq))
    for c, (ids, masked, pos, tok, layer, phase, seq) in enumerate(calls):
        arrays[f"ids_{c}"], arrays[f"masked_{c}"], arrays[f"pos_{c}"], arrays[f"tok_{c}"] = ids, masked, pos, tok
        arrays[f"meta_{c}"] = np.array([layer, analysis.PHASES.index(phase), seq], np.int64)
    arrays["n_calls"] = np.int64(len(calls))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "t.csv")
        tr.to_csv(path)
        arrays["csv"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    import json

    metrics = {g: {repr(k2): v for k2, v in analysis.avg_k(tr, g).items()} for g in analysis.GROUP_KEYS}
    metrics["position_mask_prob"] = {repr(k2): v for k2, v in analysis.position_mask_prob(tr).items()}
    before, after = analysis.expert_load(tr)
    metrics["expert_load_routed"] = {repr(k2): v for k2, v in before.items()}
    metrics["expert_load_kept"] = {repr(k2): v for k2, v in after.items()}
    arrays["metrics_json"] = np.frombuffer(json.dumps(metrics, sort_keys=True).encode(), dtype=np.uint8)
    save("trace", **arrays)


LM_CFG = dict(vocab_size=40, d_h=32, n_layers=2, n_heads=4, context_length=12, d_ff=48, num_experts=8,
              top_k=4, seed=5)


def lm_mask_weights(d, n, layers):
    rng = np.random.default_rng(77)
    return [rng.normal(0.0, 0.5, (d, n)) for _ in range(layers)]


def make_lm():
    """Reference TinyMoELM (BEAM strategy, seeded mask routers) outputs."""
    import tempfile

    ref.import_beamoe()
    from beamoe import analysis
    from beamoe.baselines import RoutingStrategy
    from beamoe.trainer import ModelConfig, TinyMoELM, evaluate, sample_greedy

    cfg = ModelConfig(strategy=RoutingStrategy("beam"), **LM_CFG)
    model = TinyMoELM(cfg)
    for layer, w in zip(model.layers, lm_mask_weights(cfg.d_h, cfg.num_experts, cfg.n_layers)):
        layer["block"].mask_router.weight.data[...] = w
    rng = np.random.default_rng(8)
    ids = rng.integers(0, cfg.vocab_size, (2, cfg.context_length))
    logits, routes = model.forward(ids, training=False)
    prompt = rng.integers(0, cfg.vocab_size, 5)
    trace = analysis.SparsityTrace()
    gen = sample_greedy(model, prompt, 14, trace=trace, sequence_id=3)
    corpus = rng.integers(0, cfg.vocab_size, 101)
    ev = evaluate(model, corpus, batch_size=3)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "t.csv")
        trace.to_csv(path)
        csv_bytes = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    save("lm", ids=ids, logits=logits.data, kept_0=routes[0].kept_ids, kept_1=routes[1].kept_ids,
         prompt=prompt, generated=gen, corpus=corpus, perplexity=np.float64(ev.perplexity),
         avg_k=np.float64(ev.avg_k), token_count=np.int64(ev.token_count), trace_csv=csv_bytes)


Q30_PREFILL_SEED = 8192


def q30prefill_tokens(seed: int = Q30_PREFILL_SEED, t: int = 8192, d: int = 2048) -> np.ndarray:
    """hq (int8, h = hq / 8) of the q30prefill_dyadic fixture (numpy PCG64; the
    fixture stores its sha256 so a changed generator is detected, not trusted)."""
    return np.random.default_rng(seed).integers(-16, 17, (t, d)).astype(np.int8)


def make_q30prefill_dyadic():
    """Routing half of beam_block_forward (moe.py:122-137, beam.py:68-72,
    dispatch/__init__.py:55-62, 89-126) at T = 8192 on dyadic inputs."""
    import hashlib

    ref.import_beamoe()
    from beamoe import dispatch
    from beamoe.beam import MaskRouter, mask_forward
    from beamoe.moe import topk_route
    from beamoe.tensor import Tensor

    d, n, k, t = 2048, 128, 8, 8192
    hq = q30prefill_tokens()
    rng = np.random.default_rng(Q30_PREFILL_SEED + 1)
    rq = rng.integers(-32, 33, (d, n)).astype(np.int8)          # router = rq / 256
    rq[:, 100:104] = rq[:, 96:100]                              # duplicated columns: exact logit ties
    mq = rng.integers(-32, 33, (d, n)).astype(np.int8)          # mask_w = mq / 256
    mq[:, :4] = 0                                               # a == 0 exactly: inclusive boundary
    x = Tensor(hq.astype(np.float64) / 8.0)
    dec = topk_route(x, Tensor(rq.astype(np.float64) / 256.0), k)
    mdec = mask_forward(x, MaskRouter(Tensor(mq.astype(np.float64) / 256.0)))
    masked_ids = dispatch.mask_route(dec.topk_indices, mdec.pre_activation.data)
    plan = dispatch.align_block(masked_ids, 16, num_experts=n)
    pa = _plan_arrays(plan)
    logits = np.ascontiguousarray(dec.logits.data)
    pre = np.ascontiguousarray(mdec.pre_activation.data)
    save("q30prefill_dyadic",
         seed=np.int64(Q30_PREFILL_SEED), hq_sha256=np.array(hashlib.sha256(hq.tobytes()).hexdigest()),
         rq=rq, mq=mq,
         logits_sha256=np.array(hashlib.sha256(logits.tobytes()).hexdigest()),
         pre_activation_sha256=np.array(hashlib.sha256(pre.tobytes()).hexdigest()),
         topk_ids=dec.topk_indices.astype(np.uint8),
         mask_bits=np.packbits(mdec.mask.data.astype(np.uint8), axis=1),
         masked_ids=masked_ids.astype(np.int16),
         weights_topk=np.take_along_axis(dec.weights.data, dec.topk_indices, 1),
         plan_counts=pa["plan_counts"].astype(np.int32), plan_offsets=pa["plan_offsets"].astype(np.int32),
         plan_tokens=pa["plan_tokens"].astype(np.int16), plan_slots=pa["plan_slots"].astype(np.int8))


def main():
    make_lm()
    make_trace()
    make_ste()
    make_strategies()
    beamoe = ref.import_beamoe()
    from beamoe import dispatch
    from beamoe.beam import MaskRouter, beam_block_forward
    from beamoe.moe import MoEBlock, MoEBlockConfig, topk_route
    from beamoe.tensor import Tensor

    # ---------------- mask_route ----------------
    rng = np.random.default_rng(1000)
    cases = []
    # reference KATs (test_dispatch.py:35-53)
    a = np.zeros((1, 8)); a[0, 3] = 0.2; a[0, 5] = -0.1
    cases.append((np.array([[3, 5]], np.int64), a))
    cases.append((np.array([[0, 1], [2, 3]], np.int64), np.zeros((2, 4))))
    cases.append((np.array([[-1, 7, 2]], np.int64), np.zeros((1, 4))))
    # signed zeros + exact boundary
    cases.append((np.array([[0, 1, 2, 3]], np.int64), np.array([[0.0, -0.0, 1e-300, -1e-300]])))
    for _ in range(20):
        t, k, n = int(rng.integers(1, 40)), int(rng.integers(1, 9)), int(rng.integers(2, 130))
        ids = rng.integers(-2, n + 2, (t, k)).astype(np.int64)
        cases.append((ids, rng.normal(size=(t, n))))
    arrays = {}
    for i, (ids, a) in enumerate(cases):
        arrays[f"ids_{i}"] = ids
        arrays[f"a_{i}"] = a
        arrays[f"out_{i}"] = dispatch.mask_route(ids, a)
    arrays["n_cases"] = np.int64(len(cases))
    save("mask_route", **arrays)

    # ---------------- align_block ----------------
    rng = np.random.default_rng(2000)
    arrays = {}
    specs = [(np.array([[0, 1], [1, -1]], np.int64), 2, 2), (np.full((5, 3), -1, np.int64), 16, 4)]
    for bs in (1, 2, 4, 8, 16, 64):
        for _ in range(3):
            n = int(rng.integers(1, 130))
            t, k = int(rng.integers(1, 300)), int(rng.integers(1, 9))
            specs.append((rng.integers(-1, n, (t, k)).astype(np.int64), bs, n))
    for i, (ids, bs, n) in enumerate(specs):
        plan = dispatch.align_block(ids, bs, num_experts=n)
        arrays[f"ids_{i}"] = ids
        arrays[f"bs_{i}"] = np.int64(bs)
        arrays[f"n_{i}"] = np.int64(n)
        for key, v in _plan_arrays(plan).items():
            arrays[f"{key}_{i}"] = v
    arrays["n_cases"] = np.int64(len(specs))
    save("align_block", **arrays)

    # ---------------- topk_route ----------------
    rng = np.random.default_rng(3000)
    arrays = {}
    topk_cases = [
        (np.array([[2.0, 1.0, 0.0, -1.0]]), np.eye(4), 2),      # test_moe.py:64-73
        (np.array([[1.0, 1.0, 1.0, 1.0]]), np.eye(4), 2),       # ties -> lowest index
        (np.array([[5.0, 5.0, 5.0]]), np.eye(3), 2),
        (rng.normal(size=(5, 4)), rng.normal(size=(4, 6)), 6),  # K = N
    ]
    for _ in range(6):
        t, d, n = int(rng.integers(1, 20)), int(rng.integers(1, 40)), int(rng.integers(2, 130))
        k = int(rng.integers(1, min(n, 8) + 1))
        topk_cases.append((rng.normal(size=(t, d)), rng.normal(size=(d, n)), k))
    # many exact ties: small-integer logits
    topk_cases.append((rng.integers(-2, 3, (64, 16)).astype(np.float64), np.eye(16), 8))
    for i, (x, w, k) in enumerate(topk_cases):
        dec = topk_route(Tensor(x), Tensor(w), k)
        arrays[f"x_{i}"] = x
        arrays[f"w_{i}"] = w
        arrays[f"k_{i}"] = np.int64(k)
        arrays[f"logits_{i}"] = dec.logits.data
        arrays[f"ids_{i}"] = dec.topk_indices
        arrays[f"weights_{i}"] = dec.weights.data
    arrays["n_cases"] = np.int64(len(topk_cases))
    save("topk_route", **arrays)

    # ---------------- full layer, inference ----------------
    arrays = {}
    layer_specs = [
        # (seed, d, f, n, k, shared, has_norm, T, mask_std, bs)
        (11, 32, 24, 8, 2, 0, True, 37, 1.0, 16),
        (12, 32, 24, 8, 4, 1, True, 19, 0.5, 4),
        (13, 16, 8, 4, 4, 0, False, 9, 0.0, 1),     # zero-init mask (== vanilla top-k)
        (14, 48, 40, 16, 3, 2, True, 50, 2.0, 8),
        (15, 24, 16, 6, 1, 0, True, 23, 1.0, 2),
    ]
    for i, (seed, d, f, n, k, sh, norm, t, mstd, bs) in enumerate(layer_specs):
        rng = np.random.default_rng(seed)
        cfg = MoEBlockConfig(d_h=d, d_ff=f, num_experts=n, top_k=k, num_shared=sh, has_norm=norm)
        block = MoEBlock(cfg, rng, init_std=0.3)
        block.mask_router = MaskRouter.zero_init(d, n)
        if mstd > 0:
            block.mask_router.weight.data[...] = rng.normal(0, mstd, (d, n))
        h = rng.normal(size=(t, d))
        out, dec, mdec = beam_block_forward(Tensor(h), block, training=False, block_size=bs)
        masked_ids = dispatch.mask_route(dec.topk_indices, mdec.pre_activation.data)
        plan = dispatch.align_block(masked_ids, bs, num_experts=n)
        p = f"c{i}_"
        arrays[p + "cfg"] = np.array([seed, d, f, n, k, sh, int(norm), t, bs], np.int64)
        arrays[p + "h"] = h
        arrays[p + "router_w"] = block.router_w.data
        arrays[p + "mask_w"] = block.mask_router.weight.data
        arrays[p + "w_gate"] = np.stack([e.w_gate.data for e in block.experts])
        arrays[p + "w_up"] = np.stack([e.w_up.data for e in block.experts])
        arrays[p + "w_down"] = np.stack([e.w_down.data for e in block.experts])
        if sh:
            arrays[p + "s_gate"] = np.stack([e.w_gate.data for e in block.shared])
            arrays[p + "s_up"] = np.stack([e.w_up.data for e in block.shared])
            arrays[p + "s_down"] = np.stack([e.w_down.data for e in block.shared])
        arrays[p + "out"] = out.data
        arrays[p + "logits"] = dec.logits.data
        arrays[p + "topk_ids"] = dec.topk_indices
        arrays[p + "weights"] = dec.weights.data
        arrays[p + "pre_activation"] = mdec.pre_activation.data
        arrays[p + "raw_mask"] = mdec.raw_mask.data
        arrays[p + "mask"] = mdec.mask.data
        arrays[p + "masked_ids"] = masked_ids
        for key, v in _plan_arrays(plan).items():
            arrays[p + key] = v
    arrays["n_cases"] = np.int64(len(layer_specs))
    save("layer", **arrays)

    # ---------------- Q30 routing, dyadic (bit-exact suite) ----------------
    rng = np.random.default_rng(4000)
    d, n, k, t = 2048, 128, 8, 64
    hq = rng.integers(-16, 17, (t, d)).astype(np.int8)          # h = hq / 8
    rq = rng.integers(-32, 33, (d, n)).astype(np.int8)          # router = rq / 256
    mq = rng.integers(-32, 33, (d, n)).astype(np.int8)          # mask_w = mq / 256
    mq[:, :4] = 0                                               # a == 0 exactly: inclusive boundary
    h = hq.astype(np.float64) / 8.0
    router = rq.astype(np.float64) / 256.0
    mask_w = mq.astype(np.float64) / 256.0
    cfg = MoEBlockConfig(d_h=d, d_ff=8, num_experts=n, top_k=k, has_norm=False)
    x = Tensor(h)
    dec = topk_route(x, Tensor(router), k)
    from beamoe.beam import mask_forward

    mdec = mask_forward(x, MaskRouter(Tensor(mask_w)))
    masked_ids = dispatch.mask_route(dec.topk_indices, mdec.pre_activation.data)
    plan = dispatch.align_block(masked_ids, 16, num_experts=n)
    arrays = dict(hq=hq, rq=rq, mq=mq, logits=dec.logits.data, topk_ids=dec.topk_indices,
                  weights=dec.weights.data, pre_activation=mdec.pre_activation.data,
                  mask=mdec.mask.data, masked_ids=masked_ids)
    arrays.update(_plan_arrays(plan))
    save("q30route_dyadic", **arrays)
    del cfg


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"make_{name}"]()
    else:
        main()
        make_q30prefill_dyadic()
