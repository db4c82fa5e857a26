"""Mask-router training path on the GPU against the oracle, whose
restatement is pinned to the reference's autograd tape (tests/test_oracle.py,
golden tests/golden/ste.npz).  Tolerances (written per test):
  fp32 experts: max |gpu - oracle| / max |oracle| <= 1e-4 on the gradients
  bf16 experts: <= 2e-2 (the candidate rows are bf16 on the tcgen05 path; the
                gradient is a dot of them with dy, then the STE product)
Off-candidate gradient entries must be exactly 0; routing bit-exact on tokens
away from fp32/fp64 decision boundaries.  All calls go through the C ABI."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_14438_b200 as B  # noqa: E402
from oracle import beam_oracle as O  # noqa: E402
from _beamtest import matched_blocks, normwise_rel, ste_golden_block, topk_margin_ok  # noqa: E402


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def _check(gb, ob, h, dy, beta, tol, min_ok=0.8):
    ref = O.mask_router_backward(h, ob, dy, beta)
    r = B.mask_router_backward(torch.from_numpy(h).float().cuda(), gb, torch.from_numpy(dy).float().cuda(), beta)
    torch.cuda.synchronize()
    ids = r.decision.topk_indices.cpu().numpy()
    ok = topk_margin_ok(ref.decision.logits, ob.top_k, 1e-4)
    assert ok.mean() >= min_ok
    assert np.array_equal(ids[ok], ref.decision.topk_indices[ok])
    ga = _np(r.grad_pre_activation)
    # exact zeros off the candidate set (test_beam.py:244-249)
    off = np.ones_like(ga, dtype=bool)
    np.put_along_axis(off, ids, False, -1)
    assert np.all(ga[off] == 0.0)
    assert normwise_rel(ga[ok], ref.grad_pre_activation[ok]) <= tol, normwise_rel(ga[ok], ref.grad_pre_activation[ok])
    assert normwise_rel(_np(r.dghat)[ok], ref.dghat[ok]) <= tol
    if ok.all():
        assert normwise_rel(_np(r.grad_weight), ref.grad_weight) <= tol
    assert abs(float(r.loss_reg) - ref.loss_reg) <= 1e-5 * max(1.0, abs(ref.loss_reg))
    return r, ref


@pytest.mark.parametrize("dtype_name,tol", [("f32", 1e-4), ("bf16", 2e-2)])
def test_mask_backward_golden(golden, dtype_name, tol):
    g = golden("ste")
    for i in range(int(g["n_cases"])):
        ob, h, dy, beta = ste_golden_block(g, i)
        ob, gb = matched_blocks(ob, dtype_name)
        _check(gb, ob, _f32(h), _f32(dy), beta, tol)


@pytest.mark.parametrize("t,path", [(7, "auto"), (64, "auto"), (512, "auto"), (512, "simt")])
def test_mask_backward_sizes(t, path):
    """Decode- and prefill-sized batches (the latter on the tcgen05 candidate pass)."""
    rng = np.random.default_rng(500 + t)
    d, f, n, k = 256, 128, 32, 4
    ob = O.make_block(d, f, n, k, rng, num_shared=1, init_std=0.05)
    ob.mask_w = rng.normal(0, 1 / 16, (d, n))
    ob, gb = matched_blocks(ob, "bf16")
    h = _f32(rng.normal(size=(t, d)))
    dy = _f32(rng.normal(size=(t, d)))
    B.set_expert_path(path)
    try:
        _check(gb, ob, h, dy, 0.7, 2e-2)
    finally:
        B.set_expert_path("auto")


def test_zero_init_mask_router_gradient():
    """Zero-init W_m: a = 0, sigma'(0) = 1/4 on every candidate (P4)."""
    rng = np.random.default_rng(9)
    d, f, n, k, t = 64, 32, 8, 2, 16
    ob = O.make_block(d, f, n, k, rng, init_std=0.1)
    ob, gb = matched_blocks(ob, "f32")
    h, dy = _f32(rng.normal(size=(t, d))), _f32(rng.normal(size=(t, d)))
    r, ref = _check(gb, ob, h, dy, 0.0, 1e-4)
    assert np.all(_np(r.mask_decision.mask) == 1.0)


def test_ste_backward_dense_and_sparsity_loss():
    rng = np.random.default_rng(3)
    t, n, k = 37, 24, 5
    w = np.zeros((t, n))
    idx = np.stack([rng.choice(n, size=k, replace=False) for _ in range(t)])
    np.put_along_axis(w, idx, rng.dirichlet(np.ones(k), size=t), -1)
    w, a, up = _f32(w), _f32(rng.normal(size=(t, n)) * 3), _f32(rng.normal(size=(t, n)))
    dec = B.MaskDecision(pre_activation=torch.from_numpy(a).float().cuda(),
                         raw_mask=torch.from_numpy(O.sigmoid(a)).float().cuda(),
                         mask=torch.ones(t, n, device="cuda"))
    got = _np(B.ste_backward(torch.from_numpy(up).cuda(), torch.from_numpy(w).cuda(), dec, 0.9, k))
    ref = O.ste_backward(up, w, a, 0.9, k)
    assert np.all(got[w == 0] == 0.0)
    assert normwise_rel(got, ref) <= 1e-5
    loss = float(B.sparsity_loss(dec.raw_mask, torch.from_numpy(idx).cuda()))
    assert abs(loss - O.sparsity_loss(O.sigmoid(a), idx)) <= 1e-6
    with pytest.raises(B.ContractError):
        B.ste_backward(torch.from_numpy(up).cuda(), torch.from_numpy(w).cuda(), dec, -1.0, k)
