"""The host-buffer path of beam_block_forward (beam.py:_HostSession): a cached
CUDA graph of the layer per (block, T, dtype, block size).  It must return
exactly what the eager launch path returns, follow router weights changed in
place between calls, keep one session per T, and match the oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # the gpu marker is deselected on CPU runs
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_14438_b200 as B  # noqa: E402
from paper_2605_14438_b200 import beam as BM  # noqa: E402
from oracle import beam_oracle as O  # noqa: E402
from _beamtest import assert_kept, mask_margin_ok, matched_blocks, normwise_rel, topk_margin_ok  # noqa: E402


def _case(seed=5, d=512, f=256, n=16, k=4):
    rng = np.random.default_rng(seed)
    ob = O.make_block(d, f, n, k, rng, init_std=0.02)
    ob.mask_w = rng.normal(0, 1 / np.sqrt(d), (d, n))
    return rng, matched_blocks(ob, "bf16")


def _call(h, gb, graph: bool, monkeypatch):
    monkeypatch.setenv("BEAM_HOST_GRAPH", "1" if graph else "0")
    out, dec, md = B.beam_block_forward(h, gb, training=False)
    assert not out.is_cuda  # host in -> host out
    return out.float().numpy(), dec.topk_indices.numpy(), dec.logits.numpy(), md.mask.numpy(), md.raw_mask.numpy()


def test_graph_host_path_equals_eager(monkeypatch):
    rng, (ob, gb) = _case()
    for t in (1, 7, 64, 64, 7):  # repeated T reuse their session
        h = torch.from_numpy(rng.normal(size=(t, 512))).to(torch.bfloat16)
        e = _call(h, gb, False, monkeypatch)
        g = _call(h, gb, True, monkeypatch)
        for a, b in zip(e, g):
            assert np.array_equal(a, b)
    keys = [key for key in BM._SESSIONS if key[0] == id(gb)]
    assert sorted(key[1] for key in keys) == [1, 7, 64]


def test_graph_host_path_follows_router_updates(monkeypatch):
    rng, (ob, gb) = _case(seed=9)
    h = torch.from_numpy(rng.normal(size=(16, 512))).to(torch.bfloat16)
    first = _call(h, gb, True, monkeypatch)
    with torch.no_grad():  # in-place update of the mask router (training step)
        gb.mask_router.weight.mul_(-1.0)
    second = _call(h, gb, True, monkeypatch)
    eager = _call(h, gb, False, monkeypatch)
    for a, b in zip(second, eager):
        assert np.array_equal(a, b)
    assert not np.array_equal(first[3], second[3])  # the mask flipped with the weights


def test_graph_host_path_matches_oracle(monkeypatch):
    rng, (ob, gb) = _case(seed=11)
    h = torch.from_numpy(rng.normal(size=(32, 512))).to(torch.bfloat16)
    ref = O.beam_block_forward(h.to(torch.float64).numpy(), ob, block_size=16)
    out, ids, logits, mask, _ = _call(h, gb, True, monkeypatch)
    ok = topk_margin_ok(ref.decision.logits, 4, 1e-5) & mask_margin_ok(ref, 1e-5)
    assert_kept(ok)
    assert np.array_equal(ids[ok], ref.decision.topk_indices[ok])
    assert np.array_equal(mask[ok], ref.mask.mask[ok])
    assert normwise_rel(out[ok].astype(np.float64), ref.out[ok]) <= 1e-2
