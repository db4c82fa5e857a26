"""The tiny MoE LM (trainer.TinyMoELM) on the GPU against the reference's own
outputs (tests/golden/lm.npz): BEAM routing with seeded mask routers, fp32 on
the GPU vs fp64 in the reference.  Tolerances: logits max-rel 1e-4 (fp32 path);
kept ids, greedy tokens (incl. the sliding window) and the sparsity-trace CSV
bit-exact; perplexity rel 1e-5; Avg-K exact."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_14438_b200 import analysis as A  # noqa: E402
from paper_2605_14438_b200 import lm as L  # noqa: E402
from paper_2605_14438_b200.baselines import RoutingStrategy  # noqa: E402
from _beamtest import normwise_rel  # noqa: E402

LM_CFG = dict(vocab_size=40, d_h=32, n_layers=2, n_heads=4, context_length=12, d_ff=48, num_experts=8,
              top_k=4, seed=5)


def _model():
    cfg = L.ModelConfig(strategy=RoutingStrategy("beam"), **LM_CFG)
    m = L.TinyMoELM(cfg, device="cuda")
    rng = np.random.default_rng(77)  # tests/golden/make_golden.py: lm_mask_weights
    for layer in m.layers:
        layer["block"].mask_router.weight.copy_(torch.from_numpy(rng.normal(0.0, 0.5, (cfg.d_h, cfg.num_experts))))
    return m


def test_lm_forward_matches_reference(golden):
    g = golden("lm")
    m = _model()
    logits, routes = m.forward(g["ids"])
    assert normwise_rel(logits.double().cpu().numpy(), g["logits"]) <= 1e-4
    for li in range(2):
        assert np.array_equal(routes[li].kept_ids.cpu().numpy(), g[f"kept_{li}"])


@pytest.mark.parametrize("use_graph", [False, True])
def test_lm_greedy_and_trace_match_reference(golden, tmp_path, use_graph):
    g = golden("lm")
    m = _model()
    tr = A.SparsityTrace("cuda")
    gen = L.sample_greedy(m, g["prompt"], 14, trace=tr, sequence_id=3, use_graph=use_graph)
    assert np.array_equal(gen, g["generated"])
    path = os.path.join(tmp_path, "t.csv")
    tr.to_csv(path)
    assert open(path, "rb").read() == g["trace_csv"].tobytes()


def test_lm_evaluate_matches_reference(golden):
    g = golden("lm")
    ev = L.evaluate(_model(), g["corpus"], batch_size=3)
    assert ev.token_count == int(g["token_count"])
    assert abs(ev.perplexity - float(g["perplexity"])) <= 1e-5 * float(g["perplexity"])
    assert ev.avg_k == float(g["avg_k"])
