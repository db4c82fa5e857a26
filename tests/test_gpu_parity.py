"""Parity of the sm_100a path with the CPU oracle (and the reference's golden
vectors).  Integer / index work must be bit-exact; floating point within the
north-star tolerance written in each test:
  bf16 expert path: max |gpu - oracle| / max |oracle| <= 1e-2
  fp32 expert path: max |gpu - oracle| / max |oracle| <= 1e-4
All calls go through the package API -> C ABI (libbeam_b200.so)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # the gpu marker is deselected on CPU runs
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_14438_b200 as B  # noqa: E402
from paper_2605_14438_b200 import dispatch as D  # noqa: E402
from oracle import beam_oracle as O  # noqa: E402
from _beamtest import assert_kept, golden_block, mask_margin_ok, matched_blocks, normwise_rel, topk_margin_ok  # noqa: E402

TOL_BF16 = 1e-2
TOL_F32 = 1e-4


def _np(t):
    return t.detach().cpu().numpy()


# ---------------------------------------------------------------------------
# golden vectors (generated from the reference itself)
# ---------------------------------------------------------------------------


def test_mask_route_golden(golden):
    g = golden("mask_route")
    for i in range(int(g["n_cases"])):
        ids = torch.from_numpy(g[f"ids_{i}"]).cuda()
        a = torch.from_numpy(g[f"a_{i}"]).cuda()  # float64: compared in fp64
        out = D.mask_route(ids, a)
        assert np.array_equal(_np(out), g[f"out_{i}"]), i


def test_align_block_golden(golden):
    g = golden("align_block")
    for i in range(int(g["n_cases"])):
        ids = torch.from_numpy(g[f"ids_{i}"]).cuda()
        plan = D.align_block(ids, int(g[f"bs_{i}"]), int(g[f"n_{i}"]))
        n = int(g[f"n_{i}"])
        assert np.array_equal(_np(plan.real_counts), g[f"plan_counts_{i}"]), i
        offs = _np(plan.offsets).astype(np.int64)
        assert np.array_equal(offs, g[f"plan_offsets_{i}"]), i
        total = offs[-1]
        assert np.array_equal(_np(plan.flat_tokens[:total]).astype(np.int64), g[f"plan_tokens_{i}"]), i
        assert np.array_equal(_np(plan.flat_slots[:total]).astype(np.int64), g[f"plan_slots_{i}"]), i
        for e in range(n):  # reference-style per-expert views
            a, b = offs[e], offs[e + 1]
            assert np.array_equal(_np(plan.tokens[e]), g[f"plan_tokens_{i}"][a:b])
        assert plan.total_real == int(g[f"plan_counts_{i}"].sum())


def test_topk_route_golden(golden):
    g = golden("topk_route")
    for i in range(int(g["n_cases"])):
        x, w, k = g[f"x_{i}"], g[f"w_{i}"], int(g[f"k_{i}"])
        dec = B.topk_route(torch.from_numpy(x).float().cuda(), torch.from_numpy(w).float().cuda(), k)
        ref_logits = g[f"logits_{i}"]
        ok = topk_margin_ok(ref_logits, k, 1e-4 * (1 + np.abs(ref_logits).max()))
        exact = np.array_equal(x.astype(np.float32).astype(np.float64), x) and np.array_equal(
            w.astype(np.float32).astype(np.float64), w) and np.all(np.abs(x) < 64) and np.all(np.isin(w, (0.0, 1.0)))
        ids = _np(dec.topk_indices)
        if exact:  # small-integer logits: exact in fp32, ties everywhere
            assert np.array_equal(ids, g[f"ids_{i}"]), i
        else:
            assert np.array_equal(ids[ok], g[f"ids_{i}"][ok]), i
        np.testing.assert_allclose(_np(dec.logits), ref_logits, rtol=1e-5, atol=1e-5 * (1 + np.abs(ref_logits).max()))
        wt = _np(dec.weights)
        np.testing.assert_allclose(wt[ok], g[f"weights_{i}"][ok], rtol=0, atol=2e-6)
        assert np.all((wt > 0).sum(-1) == k)


def _golden_oracle_block(g, i):
    return golden_block(g, i)


@pytest.mark.parametrize("dtype_name,tol", [("f32", TOL_F32), ("bf16", TOL_BF16)])
def test_layer_golden(golden, dtype_name, tol):
    g = golden("layer")
    for i in range(int(g["n_cases"])):
        ob, h, bs = _golden_oracle_block(g, i)
        ob, gb = matched_blocks(ob, dtype_name)
        h32 = h.astype(np.float32).astype(np.float64)
        ref = O.beam_block_forward(h32, ob, block_size=bs)
        out, dec, md = B.beam_block_forward(torch.from_numpy(h32).float().cuda(), gb, training=False, block_size=bs)
        ok = topk_margin_ok(ref.decision.logits, ob.top_k, 1e-4)
        ok &= mask_margin_ok(ref, 1e-4)
        assert ok.mean() > 0.8
        assert np.array_equal(_np(dec.topk_indices)[ok], ref.decision.topk_indices[ok]), i
        assert np.array_equal(_np(md.mask)[ok], ref.mask.mask[ok]), i
        o = _np(out).astype(np.float64)
        assert normwise_rel(o[ok], ref.out[ok]) <= tol, (i, normwise_rel(o[ok], ref.out[ok]))
        # MoE update alone (fp32 output path): tighter signal than out = h + y
        y = o - h32
        if dtype_name == "f32":
            assert normwise_rel(y[ok], ref.y[ok]) <= 10 * tol


def test_q30_routing_dyadic_bit_exact(golden):
    """Qwen3-30B-A3B router shape, dyadic inputs: fp32 logits are exact, so the
    top-K ids (tie-heavy), mask bits, masked ids and the plan are bit-exact
    against the reference's own outputs."""
    g = golden("q30route_dyadic")
    h = g["hq"].astype(np.float32) / 8
    router = g["rq"].astype(np.float64) / 256
    mask_w = g["mq"].astype(np.float64) / 256
    d, n, k = 2048, 128, 8
    cfg = B.MoEBlockConfig(d_h=d, d_ff=16, num_experts=n, top_k=k, has_norm=False)
    rng = np.random.default_rng(0)
    experts = [tuple(rng.normal(0, 0.02, s) for s in ((d, 16), (d, 16), (16, d))) for _ in range(n)]
    gb = B.MoEBlock.from_weights(cfg, router, experts, mask_w=mask_w)
    out, dec, md = B.beam_block_forward(torch.from_numpy(h).cuda(), gb, training=False)
    assert np.array_equal(_np(dec.logits).astype(np.float64), g["logits"])
    assert np.array_equal(_np(md.pre_activation).astype(np.float64), g["pre_activation"])
    assert np.array_equal(_np(dec.topk_indices), g["topk_ids"])
    assert np.array_equal(_np(md.mask), g["mask"])
    masked = D.mask_route(dec.topk_indices, md.pre_activation)
    assert np.array_equal(_np(masked), g["masked_ids"])
    plan = D.align_block(masked, 16, n)
    offs = _np(plan.offsets).astype(np.int64)
    assert np.array_equal(offs, g["plan_offsets"])
    assert np.array_equal(_np(plan.flat_tokens[: offs[-1]]).astype(np.int64), g["plan_tokens"])
    assert np.array_equal(_np(plan.flat_slots[: offs[-1]]).astype(np.int64), g["plan_slots"])


def test_q30_prefill_dyadic_bit_exact(golden):
    """configs[2] prefill size, T = 8192, through the AUTO path of the public layer
    call (tensor-core 3-split router, top-K kernel, multi-CTA permute, tcgen05
    grouped GEMMs): on dyadic bf16 tokens the fp32 logits and mask pre-activations
    are exact, so they, the top-K ids (with exact ties from duplicated router
    columns), the mask bits, the masked ids and the block-16 plan must equal the
    REFERENCE's (tests/golden/q30prefill_dyadic.npz, make_golden.py) bit for bit;
    every token's output is checked against the fp64 oracle (1024-token chunks)."""
    import hashlib

    g = golden("q30prefill_dyadic")
    hq = np.random.default_rng(int(g["seed"])).integers(-16, 17, (8192, 2048)).astype(np.int8)
    assert hashlib.sha256(hq.tobytes()).hexdigest() == str(g["hq_sha256"]), "token generator changed"
    d, f, n, k, t = 2048, 768, 128, 8, 8192
    router, mask_w = g["rq"].astype(np.float64) / 256, g["mq"].astype(np.float64) / 256
    gen = torch.Generator().manual_seed(2605)
    wg = torch.empty(n, d, f).normal_(0, 0.02, generator=gen).to(torch.bfloat16)
    wu = torch.empty(n, d, f).normal_(0, 0.02, generator=gen).to(torch.bfloat16)
    wd = torch.empty(n, f, d).normal_(0, 0.02, generator=gen).to(torch.bfloat16)
    cfg = B.MoEBlockConfig(d_h=d, d_ff=f, num_experts=n, top_k=k, has_norm=False)
    gb = B.MoEBlock.from_weights(cfg, router, (wg, wu, wd), mask_w=mask_w)
    x = torch.from_numpy(hq).to(torch.bfloat16).cuda() / 8  # exact in bf16
    out, dec, md = B.beam_block_forward(x, gb, training=False)
    # the in-layer masked ids (same C-ABI call, outputs carved by the wrapper)
    outs = B.beam.LayerOutputs(t, d, n, k, torch.bfloat16, x.device)
    B.beam.layer_forward_into(x, gb, outs)
    torch.cuda.synchronize()
    logits = np.ascontiguousarray(_np(dec.logits).astype(np.float64))
    pre = np.ascontiguousarray(_np(md.pre_activation).astype(np.float64))
    assert hashlib.sha256(logits.tobytes()).hexdigest() == str(g["logits_sha256"])
    assert hashlib.sha256(pre.tobytes()).hexdigest() == str(g["pre_activation_sha256"])
    ids = _np(dec.topk_indices)
    assert np.array_equal(ids, g["topk_ids"].astype(np.int64))
    assert np.array_equal(np.packbits(_np(md.mask).astype(np.uint8), axis=1), g["mask_bits"])
    masked = outs["masked_ids"]
    assert np.array_equal(_np(masked), g["masked_ids"].astype(np.int64))
    assert torch.equal(outs["out"], out)  # deterministic across calls
    np.testing.assert_allclose(np.take_along_axis(_np(dec.weights), ids, 1), g["weights_topk"], rtol=0, atol=1e-6)
    plan = D.align_block(masked, 16, n)  # T*K = 65536 slots: the multi-CTA permute
    offs = _np(plan.offsets).astype(np.int64)
    assert np.array_equal(offs, g["plan_offsets"].astype(np.int64))
    assert np.array_equal(_np(plan.real_counts).astype(np.int64), g["plan_counts"].astype(np.int64))
    assert np.array_equal(_np(plan.flat_tokens[: offs[-1]]).astype(np.int64), g["plan_tokens"].astype(np.int64))
    assert np.array_equal(_np(plan.flat_slots[: offs[-1]]).astype(np.int64), g["plan_slots"].astype(np.int64))
    # outputs: every token vs the oracle on the same (dequantised bf16) weights
    ob = O.OracleBlock(d_h=d, d_ff=f, num_experts=n, top_k=k, router_w=router,
                       experts=[(wg[e].double().numpy(), wu[e].double().numpy(), wd[e].double().numpy())
                                for e in range(n)],
                       shared=[], norm_w=None, mask_w=mask_w)
    o_all = _np(out.float()).astype(np.float64)
    h64 = hq.astype(np.float64) / 8
    worst = 0.0
    for c0 in range(0, t, 1024):
        sub = slice(c0, c0 + 1024)
        ref = O.beam_block_forward(h64[sub], ob)
        assert np.array_equal(ids[sub], ref.decision.topk_indices)
        worst = max(worst, normwise_rel(o_all[sub], ref.out))
    assert worst <= TOL_BF16, worst


# ---------------------------------------------------------------------------
# full layer vs oracle at the north-star shapes
# ---------------------------------------------------------------------------


def _layer_case(d, f, n, k, t, seed, mask_std, dtype_name, shared=0, has_norm=True, h_dtype=torch.float32,
                bs=16, activation="silu"):
    rng = np.random.default_rng(seed)
    ob = O.make_block(d, f, n, k, rng, num_shared=shared, has_norm=has_norm, init_std=0.02, activation=activation)
    ob.mask_w = rng.normal(0, mask_std, (d, n)) if mask_std > 0 else np.zeros((d, n))
    ob, gb = matched_blocks(ob, dtype_name)
    h = rng.normal(size=(t, d))
    h_t = torch.from_numpy(h).to(h_dtype)
    h64 = h_t.to(torch.float64).numpy()
    ref = O.beam_block_forward(h64, ob, block_size=bs)
    out, dec, md = B.beam_block_forward(h_t.cuda(), gb, training=False, block_size=bs)
    return ob, gb, h64, ref, out, dec, md


@pytest.mark.parametrize("t", [1, 8, 64])
@pytest.mark.parametrize("mask_std", [0.0, 1 / np.sqrt(2048)])
def test_layer_q30_decode_bf16(t, mask_std):
    ob, gb, h64, ref, out, dec, md = _layer_case(2048, 768, 128, 8, t, 100 + t, mask_std, "bf16",
                                                 h_dtype=torch.bfloat16)
    ok = topk_margin_ok(ref.decision.logits, 8, 1e-5)
    ok &= mask_margin_ok(ref, 1e-5)
    assert_kept(ok)
    assert np.array_equal(_np(dec.topk_indices)[ok], ref.decision.topk_indices[ok])
    assert np.array_equal(_np(md.mask)[ok], ref.mask.mask[ok])
    o = _np(out.float()).astype(np.float64)
    assert normwise_rel(o[ok], ref.out[ok]) <= TOL_BF16
    y = o - h64
    assert normwise_rel(y[ok], ref.y[ok]) <= 5 * TOL_BF16  # bf16 output rounding of h + y dominates
    if mask_std == 0.0:
        assert np.all(_np(md.mask) == 1.0)


def test_layer_q30_fp32_input_update():
    """fp32 activations in/out: the MoE update y itself within the bf16 tolerance."""
    ob, gb, h64, ref, out, dec, md = _layer_case(2048, 768, 128, 8, 32, 7, 1 / np.sqrt(2048), "bf16")
    ok = topk_margin_ok(ref.decision.logits, 8, 1e-5)
    ok &= mask_margin_ok(ref, 1e-5)
    assert_kept(ok)
    y = _np(out).astype(np.float64) - h64
    assert normwise_rel(y[ok], ref.y[ok]) <= TOL_BF16


def test_layer_tiny_fp32():
    """configs[0]: tiny N=8 K=2 d=256 f=512 T=1024, fp32 -> 1e-4."""
    ob, gb, h64, ref, out, dec, md = _layer_case(256, 512, 8, 2, 1024, 3, 1 / 16, "f32")
    ok = topk_margin_ok(ref.decision.logits, 2, 1e-5)
    ok &= mask_margin_ok(ref, 1e-5)
    assert ok.mean() > 0.95
    assert np.array_equal(_np(dec.topk_indices)[ok], ref.decision.topk_indices[ok])
    o = _np(out).astype(np.float64)
    assert normwise_rel(o[ok], ref.out[ok]) <= TOL_F32
    assert normwise_rel((o - h64)[ok], ref.y[ok]) <= TOL_F32
    np.testing.assert_allclose(_np(dec.weights)[ok], ref.decision.weights[ok], atol=1e-5)
    np.testing.assert_allclose(_np(md.raw_mask), ref.mask.raw_mask, atol=1e-5)


@pytest.mark.parametrize("bs", [1, 2, 4, 8, 16, 64])
def test_layer_shared_and_block_sizes(bs):
    ob, gb, h64, ref, out, dec, md = _layer_case(64, 48, 16, 4, 37, 50 + bs, 0.3, "f32", shared=2, bs=bs)
    ok = topk_margin_ok(ref.decision.logits, 4, 1e-5)
    assert_kept(ok)
    o = _np(out).astype(np.float64)
    assert normwise_rel(o[ok], ref.out[ok]) <= TOL_F32


def test_layer_identity_activation_and_odd_dims():
    ob, gb, h64, ref, out, dec, md = _layer_case(37, 21, 5, 3, 11, 9, 0.5, "f32", activation="identity",
                                                 has_norm=False)
    ok = topk_margin_ok(ref.decision.logits, 3, 1e-5)
    assert_kept(ok)
    assert normwise_rel(_np(out).astype(np.float64)[ok], ref.out[ok]) <= TOL_F32


def test_k_equals_n_and_single_expert():
    for (n, k) in ((6, 6), (1, 1)):
        ob, gb, h64, ref, out, dec, md = _layer_case(32, 16, n, k, 9, 4, 0.5, "f32")
        assert normwise_rel(_np(out).astype(np.float64), ref.out) <= TOL_F32


def test_zero_init_equals_vanilla_topk():
    """P4: zero-init mask router => nothing masked => plain top-K MoE."""
    ob, gb, h64, ref, out, dec, md = _layer_case(64, 32, 8, 2, 20, 11, 0.0, "f32")
    assert np.all(_np(md.mask) == 1.0) and np.all(_np(md.raw_mask) == 0.5)
    assert np.all(_np(md.pre_activation) == 0.0)
    assert normwise_rel(_np(out).astype(np.float64), ref.out) <= TOL_F32


def test_fully_masked_token_passes_through_bit_exactly():
    """P5 / test_beam.py:303-317: every slot masked, no shared experts -> out == h."""
    rng = np.random.default_rng(12)
    cfg = B.MoEBlockConfig(d_h=6, d_ff=5, num_experts=4, top_k=2, has_norm=False)
    gb = B.MoEBlock(cfg, rng, init_std=0.3, dtype=torch.float32)
    gb.mask_router = B.MaskRouter(torch.full((6, 4), -1e3), 0.5)
    h = rng.normal(size=(4, 6))
    h2 = h * np.sign(h.sum(axis=1, keepdims=True))
    x = torch.from_numpy(h2).float().cuda()
    out, dec, md = B.beam_block_forward(x, gb, training=False)
    assert np.all(_np(md.mask) == 0)
    assert torch.equal(out, x)


def test_host_io_matches_device_io():
    ob, gb, h64, ref, out, dec, md = _layer_case(64, 32, 8, 2, 20, 13, 0.2, "f32")
    out_h, dec_h, md_h = B.beam_block_forward(torch.from_numpy(h64).float(), gb, training=False)
    assert not out_h.is_cuda
    assert torch.equal(out_h, out.cpu())
    assert torch.equal(dec_h.topk_indices, dec.topk_indices.cpu())


def test_deterministic_bitwise():
    ob, gb, h64, ref, out, dec, md = _layer_case(2048, 768, 128, 8, 64, 21, 1 / np.sqrt(2048), "bf16",
                                                 h_dtype=torch.bfloat16)
    x = torch.from_numpy(h64).to(torch.bfloat16).cuda()
    for _ in range(3):
        o2, _, _ = B.beam_block_forward(x, gb, training=False)
        assert torch.equal(o2, out)


def test_training_flag_same_forward():
    ob, gb, h64, ref, out, dec, md = _layer_case(32, 16, 4, 2, 9, 14, 0.5, "f32")
    o_t, _, _ = B.beam_block_forward(torch.from_numpy(h64).float().cuda(), gb, training=True)
    assert torch.equal(o_t, out)


def test_tau_other_than_half_rejected():
    cfg = B.MoEBlockConfig(d_h=8, d_ff=8, num_experts=4, top_k=2)
    gb = B.MoEBlock(cfg, np.random.default_rng(0), dtype=torch.float32)
    gb.mask_router = B.MaskRouter.zero_init(8, 4, tau=0.3)
    with pytest.raises(B.ContractError):
        B.beam_block_forward(torch.zeros(2, 8).cuda(), gb, training=False)


def test_mask_forward_kats():
    """test_beam.py:46-65: zero-init opens everything, sigmoid closed form, inclusive boundary."""
    md = B.mask_forward(torch.zeros(4, 5).cuda(), B.MaskRouter.zero_init(5, 3))
    assert torch.all(md.raw_mask == 0.5) and torch.all(md.binary_mask == 1)
    md = B.mask_forward(torch.tensor([[-1.0, 1.0]]).cuda(), B.MaskRouter(torch.eye(2).cuda()))
    np.testing.assert_allclose(_np(md.raw_mask), [[0.26894142, 0.73105858]], atol=1e-6)
    assert _np(md.binary_mask).tolist() == [[0, 1]]
    md = B.mask_forward(torch.tensor([[0.0]]).cuda(), B.MaskRouter(torch.eye(1).cuda()))
    assert float(md.raw_mask[0, 0]) == 0.5 and int(md.binary_mask[0, 0]) == 1


def test_topk_select_numpy_order():
    """moe.topk_select (moe.py:116-119) == np.argsort(-x, stable)[:, :k] in fp32 and
    fp64, with heavy ties, +-0, +-inf and NaN (numpy's sort order: NaN last)."""
    rng = np.random.default_rng(116)
    for dt in (np.float32, np.float64):
        x = rng.integers(-3, 4, (300, 37)).astype(dt)
        x[rng.random(x.shape) < 0.05] = np.nan
        x[rng.random(x.shape) < 0.05] = np.inf
        x[rng.random(x.shape) < 0.05] = -np.inf
        x[rng.random(x.shape) < 0.1] = -0.0
        x[0] = np.nan
        x[1] = -np.inf
        for k in (1, 5, 37):
            ids = B.topk_select(torch.from_numpy(x).cuda(), k)
            assert np.array_equal(_np(ids), np.argsort(-x, axis=-1, kind="stable")[:, :k]), (dt, k)
    y = rng.normal(size=(4, 6, 130))  # leading dims are kept
    assert np.array_equal(_np(B.topk_select(torch.from_numpy(y), 8)), np.argsort(-y, axis=-1, kind="stable")[..., :8])


def test_rms_norm_matches_oracle():
    rng = np.random.default_rng(5)
    h = rng.normal(size=(33, 300)).astype(np.float32)
    w = rng.normal(size=300).astype(np.float32)
    out = B.rms_norm(torch.from_numpy(h).cuda(), torch.from_numpy(w).cuda())
    np.testing.assert_allclose(_np(out), O.rms_norm(h.astype(np.float64), w.astype(np.float64)), rtol=2e-6, atol=2e-6)


# ---------------------------------------------------------------------------
# dispatch stages (test_dispatch.py analogues)
# ---------------------------------------------------------------------------


def _scenario(rng, t=16, n=8, k=4, d=6, f=5, mask_prob=0.4):
    ids = np.stack([rng.choice(n, size=k, replace=False) for _ in range(t)]).astype(np.int64)
    keep = rng.random((t, k)) >= mask_prob
    masked = np.where(keep, ids, np.int64(-1))
    w = np.zeros((t, n))
    for a in range(t):
        for b in range(k):
            if keep[a, b]:
                w[a, ids[a, b]] = rng.uniform(0.05, 1.0)
    h = rng.normal(size=(t, d))
    experts = [tuple(rng.normal(0, 0.4, s) for s in ((d, f), (d, f), (f, d))) for _ in range(n)]
    return h, ids, masked, w, experts


def test_grouped_execute_vs_oracle_and_naive():
    rng = np.random.default_rng(7)
    for trial in range(20):
        h, _, masked, w, experts = _scenario(rng, mask_prob=float(rng.uniform(0, 1)))
        w = w.astype(np.float32).astype(np.float64)
        h = h.astype(np.float32).astype(np.float64)
        experts = [tuple(x.astype(np.float32).astype(np.float64) for x in e) for e in experts]
        bs = int(rng.choice([1, 2, 16]))
        plan = D.align_block(torch.from_numpy(masked).cuda(), bs, 8)
        gexp = [B.Expert(*(torch.from_numpy(x).float() for x in e)) for e in experts]
        y = D.grouped_execute(torch.from_numpy(h).float().cuda(), plan, gexp, torch.from_numpy(w).float().cuda())
        ref = O.grouped_execute(h, O.align_block(masked, bs, 8), experts, w)
        assert normwise_rel(_np(y).astype(np.float64), ref) <= TOL_F32
        yn = D.naive_execute(torch.from_numpy(h).float().cuda(), torch.from_numpy(masked).cuda(), gexp,
                             torch.from_numpy(w).float().cuda())
        assert normwise_rel(_np(yn).astype(np.float64), ref) <= TOL_F32


def test_grouped_execute_contract_errors():
    rng = np.random.default_rng(9)
    h, _, masked, w, experts = _scenario(rng, mask_prob=0.5)
    gexp = [B.Expert(*(torch.from_numpy(x).float() for x in e)) for e in experts]
    plan = D.align_block(torch.from_numpy(masked).cuda(), 16, 8)
    bad = w.copy()
    bad[bad != 0] = 0.0
    with pytest.raises(B.ContractError):
        D.grouped_execute(torch.from_numpy(h).float().cuda(), plan, gexp, torch.from_numpy(bad).float().cuda())
    bad2 = w.copy()
    r, c = np.nonzero(w)
    bad2[r[0], c[0]] = 0.0
    free = [e for e in range(8) if w[r[0], e] == 0.0]
    bad2[r[0], free[0]] = 0.5  # same nnz, but a planned slot now has zero weight
    with pytest.raises(B.ContractError):
        D.grouped_execute(torch.from_numpy(h).float().cuda(), plan, gexp, torch.from_numpy(bad2).float().cuda())


def test_empty_plan_zero_output():
    rng = np.random.default_rng(8)
    h, _, _, _, experts = _scenario(rng)
    gexp = [B.Expert(*(torch.from_numpy(x).float() for x in e)) for e in experts]
    plan = D.align_block(torch.full((16, 4), -1, dtype=torch.int64).cuda(), 16, 8)
    assert plan.total_real == 0 and all(plan.padded_count(e) == 0 for e in range(8))
    y = D.grouped_execute(torch.from_numpy(h).float().cuda(), plan, gexp, torch.zeros(16, 8).cuda())
    assert torch.all(y == 0)


def test_mask_route_kats_and_idempotence():
    a = torch.zeros(1, 8, dtype=torch.float64)
    a[0, 3], a[0, 5] = 0.2, -0.1
    assert D.mask_route(torch.tensor([[3, 5]]), a).tolist() == [[3, -1]]
    assert D.mask_route(torch.tensor([[-1, 7, 2]]), torch.zeros(1, 4)).tolist() == [[-1, -1, 2]]
    rng = np.random.default_rng(1)
    ids = torch.from_numpy(rng.integers(-1, 8, (10, 4))).cuda()
    aa = torch.from_numpy(rng.normal(size=(10, 8))).cuda()
    once = D.mask_route(ids, aa)
    assert torch.equal(D.mask_route(once, aa), once)
    nan = torch.tensor([[float("nan"), -0.0]], dtype=torch.float64)
    assert D.mask_route(torch.tensor([[0, 1]]), nan).tolist() == [[-1, 1]]


def test_align_block_large_prefill_shape():
    """Q30 prefill size (T=8192, K=8, N=128): plan identical to the oracle's."""
    rng = np.random.default_rng(77)
    t, k, n = 8192, 8, 128
    ids = np.stack([rng.permutation(n)[:k] for _ in range(t)]).astype(np.int64)
    ids[rng.random((t, k)) < 0.6] = -1
    for bs in (1, 16, 128):
        plan = D.align_block(torch.from_numpy(ids).cuda(), bs, n)
        ref = O.align_block(ids, bs, n)
        offs = _np(plan.offsets).astype(np.int64)
        ref_offs = np.concatenate([[0], np.cumsum([len(x) for x in ref.tokens])])
        assert np.array_equal(offs, ref_offs)
        assert np.array_equal(_np(plan.flat_tokens[: offs[-1]]).astype(np.int64), np.concatenate(ref.tokens))
        assert np.array_equal(_np(plan.flat_slots[: offs[-1]]).astype(np.int64), np.concatenate(ref.slots))


def test_spec_c9_bench_dispatch_ordering():
    """SPEC criterion 9 (reference tests/test_acceptance.py:299-313, defaults of
    `beamoe bench-dispatch`, cli.py:386-403): T=4096, N=8, K=4, d=256, f=512 —
    executed slots within 2 % of the target and the min time strictly decreasing
    over active fractions 1.0 > 0.5 > 0.25 (masked slots cost nothing)."""
    rows = D.bench_dispatch(num_tokens=4096, num_experts=8, top_k=4, d_h=256, d_ff=512,
                            active_fractions=[1.0, 0.5, 0.25], repetitions=20, seed=0)
    total = 4096 * 4
    for row in rows:
        assert abs(row.slots_executed - row.active_fraction * total) <= 0.02 * total
    assert rows[0].wall_time_ns_min > rows[1].wall_time_ns_min > rows[2].wall_time_ns_min, \
        [r.wall_time_ns_min for r in rows]


def test_bench_dispatch_slot_counts():
    rows = D.bench_dispatch(32, 4, 2, 8, 8, [1.0, 0.5], 2, seed=0)
    assert rows[0].slots_executed == 64
    assert abs(rows[1].slots_executed - 32) <= 2
    with pytest.raises(B.ContractError):
        D.bench_dispatch(8, 4, 2, 4, 4, [0.0], 1)


# ---------------------------------------------------------------------------
# tcgen05 grouped-GEMM expert path (prefill)
# ---------------------------------------------------------------------------


@pytest.fixture
def tc_path():
    B.set_expert_path("tc")
    yield
    B.set_expert_path("auto")


@pytest.mark.parametrize("t,mask_std", [(64, 0.0), (300, 1 / np.sqrt(2048)), (1000, 0.5 / np.sqrt(2048))])
def test_layer_q30_tcgen05_path(tc_path, t, mask_std):
    ob, gb, h64, ref, out, dec, md = _layer_case(2048, 768, 128, 8, t, 500 + t, mask_std, "bf16",
                                                 h_dtype=torch.bfloat16)
    ok = topk_margin_ok(ref.decision.logits, 8, 1e-5) & mask_margin_ok(ref, 1e-5)
    assert_kept(ok)
    assert np.array_equal(_np(dec.topk_indices)[ok], ref.decision.topk_indices[ok])
    o = _np(out.float()).astype(np.float64)
    assert normwise_rel(o[ok], ref.out[ok]) <= TOL_BF16
    y = o - h64
    assert normwise_rel(y[ok], ref.y[ok]) <= 5 * TOL_BF16


def test_tcgen05_matches_weight_streaming(tc_path):
    """Same block, same tokens: the two expert paths agree to bf16 rounding of act."""
    rng = np.random.default_rng(31)
    ob = O.make_block(2048, 768, 128, 8, rng, init_std=0.02)
    ob.mask_w = rng.normal(0, 1 / np.sqrt(2048), (2048, 128))
    ob, gb = matched_blocks(ob, "bf16")
    x = torch.from_numpy(rng.normal(size=(512, 2048))).float().cuda()
    o_tc, _, _ = B.beam_block_forward(x, gb, training=False)
    B.set_expert_path("simt")
    o_s, _, _ = B.beam_block_forward(x, gb, training=False)
    y_tc = _np(o_tc - x).astype(np.float64)
    y_s = _np(o_s - x).astype(np.float64)
    assert normwise_rel(y_tc, y_s) <= 5e-3


def test_prefill_auto_path_q30_8192():
    """Q30 prefill (T=8192) through the auto path (tensor-core router, top-K
    kernel, multi-CTA permute, tcgen05 grouped GEMMs): deterministic, and EVERY
    token checked against the fp64 oracle (in 1024-token chunks) — ids and mask
    bits exact outside near ties, outputs within the bf16 tolerance."""
    rng = np.random.default_rng(8192)
    ob = O.make_block(2048, 768, 128, 8, rng, init_std=0.02)
    ob.mask_w = rng.normal(0, 1 / np.sqrt(2048), (2048, 128))
    ob, gb = matched_blocks(ob, "bf16")
    h = torch.from_numpy(rng.normal(size=(8192, 2048))).to(torch.bfloat16)
    x = h.cuda()
    out, dec, md = B.beam_block_forward(x, gb, training=False)
    out2, _, _ = B.beam_block_forward(x, gb, training=False)
    assert torch.equal(out, out2)
    ids, mask, o_all = _np(dec.topk_indices), _np(md.mask), _np(out.float()).astype(np.float64)
    h64 = h.double().numpy()
    kept, worst = [], 0.0
    for c0 in range(0, 8192, 1024):
        sub = slice(c0, c0 + 1024)
        ref = O.beam_block_forward(h64[sub], ob)
        ok = topk_margin_ok(ref.decision.logits, 8, 1e-5) & mask_margin_ok(ref, 1e-5)
        kept.append(ok)
        assert np.array_equal(ids[sub][ok], ref.decision.topk_indices[ok]), c0
        assert np.array_equal(mask[sub][ok], ref.mask.mask[ok]), c0
        worst = max(worst, normwise_rel(o_all[sub][ok], ref.out[ok]))
    assert_kept(np.concatenate(kept))
    assert worst <= TOL_BF16, worst


def test_tcgen05_pair_matches_single_sm():
    """cta_group::2 (CTA pairs, M = 256) and the 1-SM kernel compute the same GEMMs."""
    rng = np.random.default_rng(77)
    ob = O.make_block(2048, 768, 128, 8, rng, init_std=0.02)
    ob.mask_w = rng.normal(0, 1 / np.sqrt(2048), (2048, 128))
    ob, gb = matched_blocks(ob, "bf16")
    x = torch.from_numpy(rng.normal(size=(700, 2048))).to(torch.bfloat16).cuda()
    try:
        B.set_expert_path("tc")
        o2, _, _ = B.beam_block_forward(x, gb, training=False)
        B.set_expert_path("tc1")
        o1, _, _ = B.beam_block_forward(x, gb, training=False)
    finally:
        B.set_expert_path("auto")
    y2 = _np(o2.float() - x.float()).astype(np.float64)
    y1 = _np(o1.float() - x.float()).astype(np.float64)
    assert normwise_rel(y2, y1) <= 1e-2
    ref = O.beam_block_forward(x.double().cpu().numpy(), ob)
    ok = topk_margin_ok(ref.decision.logits, 8, 1e-5) & mask_margin_ok(ref, 1e-5)
    assert_kept(ok)
    assert normwise_rel(_np(o2.float()).astype(np.float64)[ok], ref.out[ok]) <= TOL_BF16


@pytest.mark.parametrize("t,path", [(8, "auto"), (64, "auto"), (300, "tc")])
def test_shared_experts_bf16_q30(t, path):
    """Shared experts (beam.py:163-164: always-on, weight 1.0, added after the
    routed ones) on the bf16 expert paths at d = 2048: weight streaming (decode)
    and the tcgen05 grouped GEMM (T = 300, forced), against the fp64 oracle."""
    try:
        B.set_expert_path(path)
        ob, gb, h64, ref, out, dec, md = _layer_case(2048, 768, 128, 8, t, 900 + t, 1 / np.sqrt(2048), "bf16",
                                                     shared=2, h_dtype=torch.bfloat16)
    finally:
        B.set_expert_path("auto")
    ok = topk_margin_ok(ref.decision.logits, 8, 1e-5) & mask_margin_ok(ref, 1e-5)
    assert_kept(ok)
    assert np.array_equal(_np(dec.topk_indices)[ok], ref.decision.topk_indices[ok])
    o = _np(out.float()).astype(np.float64)
    assert normwise_rel(o[ok], ref.out[ok]) <= TOL_BF16
    y = o - h64
    assert normwise_rel(y[ok], ref.y[ok]) <= 5 * TOL_BF16
    # a token with every routed slot masked still gets its shared experts
    assert np.abs(ref.y).max() > 0
