"""The reference's tiny MoE language model, inference on the GPU.

Mirrors /root/reference/pkg/src/beamoe/trainer.py: ``ModelConfig`` (:40-84),
``TinyMoELM`` (:150-257: same parameter draws in the same order, so a seed
gives the reference's weights), ``evaluate`` (:577-636) and ``sample_greedy``
(:638-673).  The feed-forward of every layer is the BEAM / routing-strategy MoE
layer through the C ABI (``baselines.block_forward`` ->
``beam_layer_forward_routed``); embeddings, attention and the LM head are plain
fp32 cuBLAS/torch ops around it (not the hot path).

Decoding keeps a KV cache: while the sequence fits the context window the new
token's hidden state is computed from cached keys / values (causal attention
makes it identical to the reference's full re-forward of the window); once the
window slides, positions shift and the reference re-runs the whole window —
so does this implementation.  The cached decode step can be replayed as one
CUDA graph (``use_graph=True``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .baselines import RoutingStrategy, block_forward, build_block
from .moe import MoEBlockConfig, _default_device
from .tensor import ContractError


@dataclass
class ModelConfig:
    """trainer.py:40-84 (same fields, defaults and validation)."""

    vocab_size: int
    d_h: int = 64
    n_layers: int = 2
    n_heads: int = 4
    context_length: int = 64
    d_ff: int = 128
    num_experts: int = 8
    top_k: int = 4
    num_shared: int = 0
    has_norm: bool = True
    activation: str = "silu"
    strategy: RoutingStrategy = field(default_factory=lambda: RoutingStrategy("vanilla_topk"))
    seed: int = 0

    def __post_init__(self):
        if isinstance(self.strategy, dict):
            self.strategy = RoutingStrategy(**self.strategy)
        if self.d_h % self.n_heads != 0:
            raise ContractError("d_h must be divisible by n_heads")
        if self.context_length < 2:
            raise ContractError("context_length must be >= 2")
        self.block_config()

    def block_config(self) -> MoEBlockConfig:
        return MoEBlockConfig(d_h=self.d_h, d_ff=self.d_ff, num_experts=self.num_experts, top_k=self.top_k,
                              num_shared=self.num_shared, has_norm=self.has_norm, activation=self.activation)


def _rms(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    """tensor.py:485-508 forward: x * (mean(x^2) + eps)^-1/2 * w."""
    return x * torch.rsqrt((x * x).mean(dim=-1, keepdim=True) + eps) * w


class TinyMoELM:
    """trainer.py:150-257 on the GPU (fp32 parameters, inference)."""

    def __init__(self, cfg: ModelConfig, device=None):
        self.cfg = cfg
        self.device = torch.device(device) if device is not None else _default_device()
        rng = np.random.default_rng(cfg.seed)
        std = 0.02
        d = cfg.d_h

        def p(shape):  # trainer.py:159-160: same draw order as the reference
            return torch.from_numpy(rng.normal(0.0, std, shape)).to(self.device, torch.float32)

        self.wte = p((cfg.vocab_size, d))
        self.wpe = p((cfg.context_length, d))
        self.layers = []
        for _ in range(cfg.n_layers):
            layer = {"attn_norm": torch.ones(d, device=self.device), "wq": p((d, d)), "wk": p((d, d)),
                     "wv": p((d, d)), "wo": p((d, d))}
            layer["block"] = build_block(cfg.block_config(), cfg.strategy, rng, dtype=torch.float32,
                                         device=self.device)
            self.layers.append(layer)
        self.final_norm = torch.ones(d, device=self.device)
        self.lm_head = p((d, cfg.vocab_size))

    # -- full forward (trainer.py:217-250, training=False) -------------------------
    def _heads(self, z, b, t):
        h = self.cfg.n_heads
        return z.view(b, t, h, self.cfg.d_h // h).transpose(1, 2)

    def _attention(self, layer, x, kv=None):
        b, t, d = x.shape
        xn = _rms(x, layer["attn_norm"])
        q, k, v = (self._heads(xn @ layer[w], b, t) for w in ("wq", "wk", "wv"))
        if kv is not None:
            kv[0][:, :, :t] = k
            kv[1][:, :, :t] = v
        hd = d // self.cfg.n_heads
        scores = (q @ k.transpose(-1, -2)) * (1.0 / np.sqrt(hd))
        causal = torch.ones(t, t, dtype=torch.bool, device=x.device).tril()
        w = torch.softmax(scores.masked_fill(~causal, float("-inf")), dim=-1)  # masked -> exactly 0
        out = (w @ v).transpose(1, 2).reshape(b, t, d)
        return out @ layer["wo"]

    def forward(self, ids, training: bool = False, binarize_soft: bool = False, _kv=None):
        """Logits [B, T, V] (fp32, device) and the per-layer RouteResults."""
        if training:
            raise ContractError("TinyMoELM on the GPU is inference only")
        cfg = self.cfg
        ids = torch.as_tensor(np.asarray(ids, dtype=np.int64) if not isinstance(ids, torch.Tensor) else ids)
        ids = ids.to(self.device, torch.int64)
        if ids.ndim == 1:
            ids = ids[None, :]
        b, t = ids.shape
        if t > cfg.context_length:
            raise ContractError("sequence longer than context_length")
        x = self.wte[ids] + self.wpe[:t]
        routes = []
        for li, layer in enumerate(self.layers):
            x = x + self._attention(layer, x, None if _kv is None else _kv[li])
            out, rr = block_forward(x.reshape(b * t, cfg.d_h), layer["block"], cfg.strategy, False,
                                    binarize_soft=binarize_soft)
            routes.append(rr)
            x = out.view(b, t, cfg.d_h)
        x = _rms(x, self.final_norm)
        return x @ self.lm_head, routes

    # -- cached decode step ----------------------------------------------------------
    def _decode_state(self, binarize_soft: bool):
        """KV cache, step inputs and the captured step graph of batch-1 decoding
        (kept on the model so the graph is captured once)."""
        st = getattr(self, "_dstate", {}).get(binarize_soft)
        if st is None:
            st = {"kv": self._kv_cache(1), "tok": torch.zeros(1, dtype=torch.int64, device=self.device),
                  "pos": torch.zeros((), dtype=torch.int64, device=self.device), "graph": None, "out": None}
            if not hasattr(self, "_dstate"):
                self._dstate = {}
            self._dstate[binarize_soft] = st
        return st

    def _kv_cache(self, b):
        cfg = self.cfg
        hd = cfg.d_h // cfg.n_heads
        shape = (b, cfg.n_heads, cfg.context_length, hd)
        return [(torch.zeros(shape, device=self.device), torch.zeros(shape, device=self.device))
                for _ in self.layers]

    def _decode_step(self, tok, pos, kv, binarize_soft=False):
        """Hidden state of one new token per sequence at position `pos` (device
        int64 scalar tensor) against the cache; returns (logits [B, V], routes)."""
        cfg = self.cfg
        b = tok.shape[0]
        d, h = cfg.d_h, cfg.n_heads
        hd = d // h
        x = self.wte.index_select(0, tok) + self.wpe.index_select(0, pos.view(1))  # [B, d]; no host sync
        ar = torch.arange(cfg.context_length, device=self.device)
        valid = ar <= pos  # cache slots 0..pos
        routes = []
        for li, layer in enumerate(self.layers):
            kc, vc = kv[li]
            xn = _rms(x, layer["attn_norm"])
            q = (xn @ layer["wq"]).view(b, h, 1, hd)
            k = (xn @ layer["wk"]).view(b, h, 1, hd)
            v = (xn @ layer["wv"]).view(b, h, 1, hd)
            kc.index_copy_(2, pos.view(1), k)
            vc.index_copy_(2, pos.view(1), v)
            scores = (q @ kc.transpose(-1, -2)) * (1.0 / np.sqrt(hd))  # [B, H, 1, C]
            w = torch.softmax(scores.masked_fill(~valid, float("-inf")), dim=-1)
            x = x + ((w @ vc).view(b, d) @ layer["wo"])
            out, rr = block_forward(x, layer["block"], cfg.strategy, False, binarize_soft=binarize_soft)
            routes.append(rr)
            x = out
        return _rms(x, self.final_norm) @ self.lm_head, routes


def sample_greedy(model: TinyMoELM, prompt_ids, max_new_tokens: int, trace=None, binarize_soft: bool = False,
                  sequence_id: int = 0, use_graph: bool = False) -> np.ndarray:
    """trainer.py:638-673: greedy decoding; prompt cells traced as prefill,
    generated cells as decode (``analysis.SparsityTrace``)."""
    cfg = model.cfg
    ids = list(np.asarray(prompt_ids, dtype=np.int64)[-cfg.context_length:])
    st = model._decode_state(binarize_soft)  # persistent cache / step tensors / graph
    kv, tok, pos = st["kv"], st["tok"], st["pos"]
    window = np.asarray(ids, dtype=np.int64)[None, :]
    logits, routes = model.forward(window, binarize_soft=binarize_soft, _kv=kv)
    if trace is not None:
        _record(trace, routes, window, sequence_id, "prefill", np.arange(window.shape[1]))
    last = logits[0, -1]
    generated = []
    abs_pos = len(ids)
    for _ in range(max_new_tokens):
        nxt = int(torch.argmax(last))
        generated.append(nxt)
        ids.append(nxt)
        slid = len(ids) > cfg.context_length
        ids = ids[-cfg.context_length:]
        if slid:  # positions shift: the reference re-runs the whole window
            window = np.asarray(ids, dtype=np.int64)[None, :]
            logits, routes = model.forward(window, binarize_soft=binarize_soft, _kv=kv)
            last = logits[0, -1]
            rr_cells = routes
        else:
            tok.fill_(nxt)
            pos.fill_(len(ids) - 1)
            if use_graph:
                if st["graph"] is None:
                    st["graph"], st["out"] = _capture_step(model, tok, pos, kv, binarize_soft)
                st["graph"].replay()
                step_logits, rr_cells = st["out"]
            else:
                step_logits, rr_cells = model._decode_step(tok, pos, kv, binarize_soft)
            last = step_logits[0]
        if trace is not None:
            window = np.asarray(ids, dtype=np.int64)[None, :]
            if slid:
                _record(trace, rr_cells, window, sequence_id, "decode", np.array([abs_pos]),
                        rows=np.array([len(ids) - 1]))
            else:
                _record(trace, rr_cells, window[:, -1:], sequence_id, "decode", np.array([abs_pos]))
        abs_pos += 1
    return np.asarray(generated, dtype=np.int64)


def _capture_step(model, tok, pos, kv, binarize_soft):
    """The cached decode step as one CUDA graph (warmed up on the capture stream
    so the library workspace is not created inside the capture)."""
    dev = model.device
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    snap = [(k.clone(), v.clone()) for k, v in kv]
    with torch.cuda.stream(s):
        model._decode_step(tok, pos, kv, binarize_soft)
    torch.cuda.current_stream(dev).wait_stream(s)
    for (k, v), (k0, v0) in zip(kv, snap):  # the warm-up wrote slot `pos`: restore
        k.copy_(k0)
        v.copy_(v0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        out = model._decode_step(tok, pos, kv, binarize_soft)
    return g, out


def _record(trace, routes, window, sequence_id, phase, positions, rows=None):
    """trainer._record_routes (trainer.py:554-574) through SparsityTrace.record_layer."""
    b, t = window.shape
    sel = slice(None) if rows is None else torch.as_tensor(rows)
    tok = window[0] if rows is None else window[0, rows]
    for li, rr in enumerate(routes):
        cand = rr.candidate_ids[sel]
        kept = torch.where(rr.active_bits[sel] > 0, cand, torch.full_like(cand, -1))
        trace.record_layer(cand, kept, li, phase, sequence_id=np.full(len(positions), sequence_id),
                           position=positions, token_id=tok)


@dataclass
class EvalResult:
    perplexity: float
    avg_k: float
    token_count: int


def evaluate(model: TinyMoELM, corpus_ids, max_windows: int | None = None, batch_size: int = 8,
             binarize_soft: bool = False) -> EvalResult:
    """trainer.py:577-636 (without trace sampling): held-out perplexity over
    non-overlapping windows, inference path, and the mean activated experts."""
    cfg = model.cfg
    t = cfg.context_length
    corpus = np.asarray(corpus_ids, dtype=np.int64)
    n_windows = (len(corpus) - 1) // t
    if max_windows is not None:
        n_windows = min(n_windows, max_windows)
    if n_windows < 1:
        raise ContractError("corpus too small to evaluate")
    total_nll, total_tokens, active_sum, active_cells = 0.0, 0, 0.0, 0
    for start in range(0, n_windows, batch_size):
        count = min(batch_size, n_windows - start)
        xs = np.stack([corpus[i * t: i * t + t] for i in range(start, start + count)])
        ys = torch.from_numpy(np.stack([corpus[i * t + 1: i * t + t + 1] for i in range(start, start + count)]))
        logits, routes = model.forward(xs, binarize_soft=binarize_soft)
        b, tt, v = logits.shape
        nll = torch.nn.functional.cross_entropy(logits.reshape(b * tt, v).double(),
                                                ys.reshape(-1).to(logits.device), reduction="mean")
        total_nll += float(nll) * b * tt
        total_tokens += b * tt
        for rr in routes:
            active_sum += float(rr.active_counts.sum())
            active_cells += rr.active_counts.numel()
    return EvalResult(perplexity=float(np.exp(total_nll / total_tokens)), avg_k=active_sum / active_cells,
                      token_count=total_tokens)
