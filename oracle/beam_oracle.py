"""TEST INFRASTRUCTURE ONLY — float64 numpy restatement of the reference's
BEAM MoE-layer inference path.  Not imported by the product package.

Each function restates one reference function and cites it as
``path:line`` relative to ``/root/reference/pkg/src/beamoe/``.  The semantics
(including tie-breaks, padding, error behaviour and accumulation order) are the
reference's; only the container types differ (plain numpy arrays and a small
``OracleBlock`` instead of the tape ``Tensor``/``MoEBlock`` classes).

Pinned by ``tests/test_oracle.py`` against the golden vectors in
``tests/golden/`` (made by ``tests/golden/make_golden.py`` from the reference
package itself) and, where ``oracle/_ref`` is built, against live reference runs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# tensor.py:21 — most-negative finite float64 used for masked logits
NEG_SENTINEL = np.finfo(np.float64).min


class ContractError(ValueError):
    """tensor.py:32-33 — an input violates a documented precondition."""


class ShapeError(ValueError):
    """tensor.py:24-25."""


# ---------------------------------------------------------------------------
# numerics (tensor.py)
# ---------------------------------------------------------------------------


def sigmoid(x: np.ndarray) -> np.ndarray:
    """tensor.py:406-411 — overflow-free two-tail form."""
    z = np.exp(-np.abs(x))
    t = 1.0 / (1.0 + z)
    return np.where(x >= 0, t, 1.0 - t)


def silu(x: np.ndarray) -> np.ndarray:
    """moe.py:38-39 (``_silu_np``): x * sigmoid(x)."""
    return x * sigmoid(x)


ACTIVATIONS = {"silu": silu, "identity": lambda x: x}  # moe.py:42


def rms_norm(x: np.ndarray, weight: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    """tensor.py:485-487 (``rms_norm_np``); the taped ``rms_norm`` (:490-508)
    computes the same forward values: x * (mean(x^2) + eps)^-1/2 * w."""
    ms = (x * x).mean(axis=-1, keepdims=True) + eps
    return x * (ms**-0.5) * weight


def masked_softmax(x: np.ndarray, masked_value: float) -> np.ndarray:
    """tensor.py:440-451 (``softmax_np`` with a masked value): entries equal to
    the sentinel get exactly 0; a fully masked row is a ContractError."""
    masked = x == masked_value
    if masked.all(axis=-1).any():
        raise ContractError("softmax row with every entry masked")
    finite_max = np.where(masked, -np.inf, x).max(axis=-1, keepdims=True)
    e = np.exp(x - finite_max)
    e[masked] = 0.0
    return e / e.sum(axis=-1, keepdims=True)


# ---------------------------------------------------------------------------
# routing (moe.py) and masking (beam.py)
# ---------------------------------------------------------------------------


def topk_select(logits: np.ndarray, k: int) -> np.ndarray:
    """moe.py:116-119 — k largest per row, descending, ties -> lower index."""
    order = np.argsort(-logits, axis=-1, kind="stable")
    return np.ascontiguousarray(order[..., :k])


@dataclass
class RouterDecision:
    """moe.py:103-113."""

    logits: np.ndarray
    topk_indices: np.ndarray
    weights: np.ndarray


def topk_route(x: np.ndarray, router_w: np.ndarray, k: int) -> RouterDecision:
    """moe.py:122-137 — logits, stable top-k, softmax over the kept logits
    (non-selected entries -> NEG_SENTINEL -> exactly 0 weight)."""
    n = router_w.shape[-1]
    if not 1 <= k <= n:
        raise ContractError("top_k must satisfy 1 <= K <= N")
    logits = x @ router_w
    idx = topk_select(logits, k)
    keep = np.zeros(logits.shape, dtype=bool)
    np.put_along_axis(keep, idx, True, axis=-1)
    masked = np.where(keep, logits, NEG_SENTINEL)  # tensor.py:388-398
    weights = masked_softmax(masked, NEG_SENTINEL)
    return RouterDecision(logits=logits, topk_indices=idx, weights=weights)


@dataclass
class MaskDecision:
    """beam.py:51-65."""

    pre_activation: np.ndarray
    raw_mask: np.ndarray
    mask: np.ndarray

    @property
    def binary_mask(self) -> np.ndarray:
        return self.mask.astype(np.int64)


def mask_forward(x: np.ndarray, mask_w: np.ndarray, tau: float = 0.5) -> MaskDecision:
    """beam.py:68-72 — a = x W_m; raw = sigmoid(a); m = (raw >= tau)
    (``binarize_ste`` forward, tensor.py:469-482, inclusive threshold)."""
    a = x @ mask_w
    raw = sigmoid(a)
    m = (raw >= tau).astype(np.float64)
    return MaskDecision(pre_activation=a, raw_mask=raw, mask=m)


# ---------------------------------------------------------------------------
# dispatch (dispatch/__init__.py, dispatch/_kernels.pyx)
# ---------------------------------------------------------------------------


def mask_route(topk_ids: np.ndarray, mask_pre_activations: np.ndarray) -> np.ndarray:
    """dispatch/__init__.py:55-62 -> _kernels.pyx:17-34: keep id when
    0 <= id < N and a[t, id] >= 0, else -1."""
    ids = np.ascontiguousarray(topk_ids, dtype=np.int64)
    a = np.ascontiguousarray(mask_pre_activations, dtype=np.float64)
    t, k = ids.shape
    n = a.shape[1]
    out = np.empty((t, k), dtype=np.int64)
    for i in range(t):
        for j in range(k):
            e = ids[i, j]
            out[i, j] = -1 if (e < 0 or e >= n or a[i, e] < 0.0) else e
    return out


def group_by_expert(ids: np.ndarray, num_experts: int):
    """_kernels.pyx:37-66 — counting sort: count pass, exclusive scan, stable
    scatter in ascending flat (token, slot) order."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    t, k = ids.shape
    counts = np.zeros(num_experts, dtype=np.int64)
    for e in ids.reshape(-1):
        if e >= 0:
            counts[e] += 1
    cursor = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    total = int(counts.sum())
    token_order = np.empty(total, dtype=np.int64)
    slot_order = np.empty(total, dtype=np.int64)
    for i in range(t):
        for j in range(k):
            e = ids[i, j]
            if e >= 0:
                pos = cursor[e]
                token_order[pos] = i
                slot_order[pos] = j
                cursor[e] = pos + 1
    return counts, token_order, slot_order


@dataclass
class DispatchPlan:
    """dispatch/__init__.py:65-86."""

    block_size: int
    num_experts: int
    tokens: list
    slots: list
    real_counts: np.ndarray

    @property
    def total_real(self) -> int:
        return int(self.real_counts.sum())

    def padded_count(self, expert: int) -> int:
        return len(self.tokens[expert])


def align_block(ids: np.ndarray, block_size: int, num_experts: int | None = None) -> DispatchPlan:
    """dispatch/__init__.py:89-126 — group surviving slots per expert
    (ascending scan order) and pad each group with -1 to a block multiple."""
    if block_size < 1:
        raise ContractError("block_size must be >= 1")
    ids = np.asarray(ids, dtype=np.int64)
    if num_experts is None:
        num_experts = int(ids.max()) + 1 if ids.size and ids.max() >= 0 else 0
    counts, token_order, slot_order = group_by_expert(ids, num_experts)
    tokens, slots = [], []
    offset = 0
    for e in range(num_experts):
        c = int(counts[e])
        padded = ((c + block_size - 1) // block_size) * block_size
        tok = np.full(padded, -1, dtype=np.int64)
        slo = np.full(padded, -1, dtype=np.int64)
        tok[:c] = token_order[offset : offset + c]
        slo[:c] = slot_order[offset : offset + c]
        tokens.append(tok)
        slots.append(slo)
        offset += c
    return DispatchPlan(block_size, num_experts, tokens, slots, counts)


def expert_forward(x: np.ndarray, w_gate, w_up, w_down, activation: str = "silu") -> np.ndarray:
    """moe.py:96-100 — (act(x W_gate) * (x W_up)) W_down."""
    act = ACTIVATIONS[activation]
    return (act(x @ w_gate) * (x @ w_up)) @ w_down


def grouped_execute(h, plan: DispatchPlan, experts, weights_hat, activation="silu"):
    """dispatch/__init__.py:129-157 — per expert ascending, run the expert on
    its real rows and scatter-add ``out * w``; contract checks :143-144, :152-153.
    ``experts`` is a list of (w_gate, w_up, w_down)."""
    if int(np.count_nonzero(weights_hat)) != plan.total_real:
        raise ContractError("weights_hat nonzero count disagrees with plan slots")
    y = np.zeros_like(h)
    for e in range(plan.num_experts):
        c = int(plan.real_counts[e])
        if c == 0:
            continue
        rows = plan.tokens[e][:c]
        w = weights_hat[rows, e]
        if np.any(w == 0.0):
            raise ContractError(f"plan routes a zero-weight slot to expert {e}")
        out = expert_forward(h[rows], *experts[e], activation)
        y[rows] += out * w[:, None]
    return y


def naive_execute(h, masked_ids, experts, weights_hat, activation="silu"):
    """dispatch/__init__.py:160-174 — per-token loop over sorted surviving ids."""
    t, _ = masked_ids.shape
    y = np.zeros_like(h)
    for tok in range(t):
        for e in sorted(int(i) for i in masked_ids[tok] if i >= 0):
            out = expert_forward(h[tok : tok + 1], *experts[e], activation)
            y[tok] += weights_hat[tok, e] * out[0]
    return y


# ---------------------------------------------------------------------------
# block container + layer forward (moe.py:161-220, beam.py:127-165)
# ---------------------------------------------------------------------------


@dataclass
class OracleBlock:
    """Parameters of one BEAM MoE block in the reference's layouts
    (moe.py:177-191, beam.py:46-48): router_w [d, N], experts [(w_gate [d,f],
    w_up [d,f], w_down [f,d])], shared likewise, norm_w [d] or None,
    mask_w [d, N], tau."""

    d_h: int
    d_ff: int
    num_experts: int
    top_k: int
    router_w: np.ndarray
    experts: list
    shared: list = field(default_factory=list)
    norm_w: np.ndarray | None = None
    mask_w: np.ndarray | None = None
    tau: float = 0.5
    activation: str = "silu"

    def normalize(self, h):
        """moe.py:214-215."""
        return rms_norm(h, self.norm_w) if self.norm_w is not None else h


def make_block(d_h, d_ff, num_experts, top_k, rng, num_shared=0, has_norm=True,
               init_std=0.02, activation="silu") -> OracleBlock:
    """moe.py:169-192 — identical draw order to ``MoEBlock.__init__``:
    router (d, N), then per expert (gate, up, down), then shared experts;
    norm weight ones; mask router zero-init (beam.py:46-48)."""
    router_w = rng.normal(0.0, init_std, (d_h, num_experts))
    experts = []
    for _ in range(num_experts):
        experts.append((rng.normal(0.0, init_std, (d_h, d_ff)),
                        rng.normal(0.0, init_std, (d_h, d_ff)),
                        rng.normal(0.0, init_std, (d_ff, d_h))))
    shared = []
    for _ in range(num_shared):
        shared.append((rng.normal(0.0, init_std, (d_h, d_ff)),
                       rng.normal(0.0, init_std, (d_h, d_ff)),
                       rng.normal(0.0, init_std, (d_ff, d_h))))
    return OracleBlock(
        d_h=d_h, d_ff=d_ff, num_experts=num_experts, top_k=top_k,
        router_w=router_w, experts=experts, shared=shared,
        norm_w=np.ones(d_h) if has_norm else None,
        mask_w=np.zeros((d_h, num_experts)), tau=0.5, activation=activation,
    )


@dataclass
class LayerResult:
    out: np.ndarray
    decision: RouterDecision
    mask: MaskDecision
    masked_ids: np.ndarray
    plan: DispatchPlan
    y: np.ndarray  # MoE update before the residual (routed + shared)


def beam_block_forward(h: np.ndarray, block: OracleBlock, block_size: int = 16) -> LayerResult:
    """beam.py:127-165, inference branch (:159-165)."""
    x_n = block.normalize(h)
    decision = topk_route(x_n, block.router_w, block.top_k)
    maskdec = mask_forward(x_n, block.mask_w, block.tau)
    ghat = decision.weights * maskdec.mask  # beam.py:159, no renormalisation
    masked_ids = mask_route(decision.topk_indices, maskdec.pre_activation)
    plan = align_block(masked_ids, block_size, num_experts=block.num_experts)
    y = grouped_execute(x_n, plan, block.experts, ghat, block.activation)
    for e in block.shared:  # beam.py:163-164
        y = y + expert_forward(x_n, *e, block.activation)
    return LayerResult(h + y, decision, maskdec, masked_ids, plan, y)


# ---------------------------------------------------------------------------
# mask-router training (beam.py:87-124, 146-157)
# ---------------------------------------------------------------------------


def sparsity_loss(raw_mask: np.ndarray, topk_indices: np.ndarray) -> float:
    """beam.py:87-97: token-mean L1 of the raw mask over the top-K candidates."""
    t, k = topk_indices.shape
    sel = np.zeros(raw_mask.shape)
    np.put_along_axis(sel, topk_indices, 1.0, axis=-1)
    return float(np.sum(raw_mask * sel) / (t * k))


def ste_backward(upstream: np.ndarray, weights: np.ndarray, pre_activation: np.ndarray,
                 beta: float, k: int) -> np.ndarray:
    """beam.py:100-124: (dL/dghat * g + beta/(K*T) * [g > 0]) * sigma'(a)."""
    if beta < 0:
        raise ContractError("beta must be non-negative")
    t = upstream.shape[0]
    indicator = (weights > 0.0).astype(np.float64)
    s = sigmoid(pre_activation)
    return (upstream * weights + (beta / (k * t)) * indicator) * (s * (1.0 - s))


@dataclass
class MaskGradResult:
    out: np.ndarray            # training forward output (== inference, beam.py:146-157)
    dghat: np.ndarray          # [T, K] dL_task/dghat at the candidate slots (rank order)
    grad_pre_activation: np.ndarray  # [T, N]
    grad_weight: np.ndarray    # [d, N] = x_n^T grad_pre_activation (mask_forward: a = x_n W_m)
    loss_reg: float
    decision: RouterDecision
    mask: MaskDecision


def mask_router_backward(h: np.ndarray, block: OracleBlock, dy: np.ndarray, beta: float) -> MaskGradResult:
    """Mask-router gradient of L = sum(out * dy) + beta * sparsity_loss through
    beam_block_forward(training=True) (beam.py:146-157): every top-K candidate is
    evaluated (moe.py:223-279 compute_ids), dL_task/dghat_i = <dy, E_i(x_n)>,
    then the closed form (beam.py:100-124)."""
    x_n = block.normalize(h)
    decision = topk_route(x_n, block.router_w, block.top_k)
    maskdec = mask_forward(x_n, block.mask_w, block.tau)
    t, k = decision.topk_indices.shape
    ghat = decision.weights * maskdec.mask
    y = np.zeros_like(x_n)
    upstream = np.zeros_like(decision.weights)
    dghat = np.zeros((t, k))
    for row in range(t):
        for r, e in sorted(enumerate(decision.topk_indices[row]), key=lambda p: p[1]):  # ascending expert
            o = expert_forward(x_n[row : row + 1], *block.experts[e], block.activation)[0]
            y[row] += ghat[row, e] * o
            upstream[row, e] = float(dy[row] @ o)
            dghat[row, r] = upstream[row, e]
    for e in block.shared:
        y = y + expert_forward(x_n, *e, block.activation)
    grad = ste_backward(upstream, decision.weights, maskdec.pre_activation, beta, k)
    return MaskGradResult(h + y, dghat, grad, x_n.T @ grad,
                          sparsity_loss(maskdec.raw_mask, decision.topk_indices), decision, maskdec)


# ---------------------------------------------------------------------------
# routing strategies (baselines.py) — inference branch
# ---------------------------------------------------------------------------

STRATEGY_KINDS = ("vanilla_topk", "topk_reduced", "topk_pruning", "moe_dynamic", "ada_moe",
                  "beam", "soft_mask", "soft_mask_tempered")


def softmax(x: np.ndarray) -> np.ndarray:
    """tensor.py softmax over the last axis (max-shifted)."""
    z = x - x.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def dynamic_select(probs: np.ndarray, phi: float) -> np.ndarray:
    """baselines.py:132-143 — smallest descending-probability prefix whose
    cumulative mass reaches phi, at least one expert per token."""
    order = np.argsort(-probs, axis=-1, kind="stable")
    csum = np.take_along_axis(probs, order, axis=-1).cumsum(axis=-1)
    counts = np.minimum((csum < phi).sum(axis=-1) + 1, probs.shape[-1])
    active = np.zeros(probs.shape, dtype=bool)
    ranks = np.arange(probs.shape[-1])[None, :]
    np.put_along_axis(active, order, ranks < counts[:, None], axis=-1)
    return active


@dataclass
class RouteResult:
    """baselines.py:116-129 (the fields the inference path produces)."""

    weights_hat: np.ndarray
    logits: np.ndarray
    candidate_ids: np.ndarray
    active_bits: np.ndarray
    active_counts: np.ndarray
    kept_ids: np.ndarray
    raw_mask: np.ndarray | None = None


def route(block: OracleBlock, x_n: np.ndarray, kind: str, params: dict | None = None,
          binarize_soft: bool = False) -> RouteResult:
    """baselines.py:158-283 with training=False.  ``block.router_w`` may carry
    null columns (ada_moe, baselines.py:212-225)."""
    p = params or {}
    k = block.top_k
    n = block.num_experts
    if kind in ("vanilla_topk", "topk_reduced", "topk_pruning"):  # :173-190
        k_eff = p.get("k_small", k) if kind == "topk_reduced" else (p.get("k_infer", k) if kind == "topk_pruning" else k)
        dec = topk_route(x_n, block.router_w, k_eff)
        ids = dec.topk_indices
        return RouteResult(dec.weights, dec.logits, ids, np.ones(ids.shape, np.int64),
                           np.full(ids.shape[0], k_eff, np.int64), ids)
    if kind == "moe_dynamic":  # :192-210
        logits = x_n @ block.router_w
        probs = softmax(logits)
        active = dynamic_select(probs, p.get("phi", 0.5))
        masked = probs * active.astype(np.float64)
        weights_hat = masked / masked.sum(axis=-1, keepdims=True)
        order = topk_select(probs, k)
        bits = np.take_along_axis(active, order, axis=-1).astype(np.int64)
        counts = active.sum(axis=-1).astype(np.int64)
        kept = np.where(bits == 1, order, np.int64(-1))
        return RouteResult(weights_hat, logits, order, bits, counts, kept)
    if kind == "ada_moe":  # :212-225
        dec = topk_route(x_n, block.router_w, k)
        ids_ext = dec.topk_indices
        real = ids_ext < n
        cand = np.where(real, ids_ext, np.int64(-1))
        return RouteResult(dec.weights[:, :n], dec.logits, cand, real.astype(np.int64),
                           real.sum(axis=-1).astype(np.int64), cand)
    dec = topk_route(x_n, block.router_w, k)
    ids = dec.topk_indices
    tau = block.tau
    if kind == "beam":  # :230-247
        md = mask_forward(x_n, block.mask_w, tau)
        bits = np.take_along_axis(md.mask.astype(np.int64), ids, axis=-1)
        return RouteResult(dec.weights * md.mask, dec.logits, ids, bits, bits.sum(axis=-1),
                           np.where(bits == 1, ids, np.int64(-1)), md.raw_mask)
    # soft variants :250-283
    temp = p.get("temp_floor", 0.1) if kind == "soft_mask_tempered" else 1.0
    a = x_n @ block.mask_w
    soft = sigmoid(a * (1.0 / temp))
    hard = (soft >= tau).astype(np.int64)
    bits_hard = np.take_along_axis(hard, ids, axis=-1)
    if kind == "soft_mask_tempered" or binarize_soft:
        weights_hat = dec.weights * (soft >= tau).astype(np.float64)
        bits = bits_hard
        kept = np.where(bits == 1, ids, np.int64(-1))
    else:
        weights_hat = dec.weights * soft
        bits = np.ones(ids.shape, np.int64)
        kept = ids
    return RouteResult(weights_hat, dec.logits, ids, bits, bits.sum(axis=-1), kept, soft)


def strategy_block_forward(h: np.ndarray, block: OracleBlock, kind: str, params: dict | None = None,
                           binarize_soft: bool = False, block_size: int = 16):
    """baselines.py:286-323, training=False -> (h + y, RouteResult)."""
    x_n = block.normalize(h)
    rr = route(block, x_n, kind, params, binarize_soft)
    plan = align_block(rr.kept_ids, block_size, num_experts=block.num_experts)
    y = grouped_execute(x_n, plan, block.experts, rr.weights_hat, block.activation)
    for e in block.shared:
        y = y + expert_forward(x_n, *e, block.activation)
    return h + y, rr
