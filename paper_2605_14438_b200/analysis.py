"""Sparsity trace of BEAM routing, recorded on the GPU.

Mirrors /root/reference/pkg/src/beamoe/analysis.py: ``TRACE_HEADER`` / ``PHASES``
(:14-16), ``SparsityTrace`` (:19-112: one row per candidate rank, CSV round trip)
and the Avg-K family ``avg_k`` (:127-166), ``position_mask_prob`` (:169-176),
``expert_load`` (:195-212).  The rows of a layer call are produced on the device
by ``beam_trace_rows`` from the gate outputs (rank-ordered top-K ids and the
masked ids), so recording costs one small kernel instead of a Python loop over
cells (trainer._record_routes, trainer.py:554-574); the executed-slot count for
Avg-K is accumulated on the device as a by-product.
"""

from __future__ import annotations

import csv

import numpy as np
import torch

from . import _lib, _runtime
from .moe import _default_device
from .tensor import ContractError, as_torch

PHASES = ("prefill", "decode")
TRACE_HEADER = ["sequence_id", "position", "layer", "rank", "expert_id", "mask_bit", "phase", "token_id"]
GROUP_KEYS = ("overall", "layer", "token_position", "phase", "token_id", "token_layer")
_COLS = ("sequence_id", "position", "layer", "rank", "expert_id", "mask_bit", "phase", "token_id")


def _i64(x, dev, n):
    if x is None:
        return None
    t = as_torch(x).to(dev, torch.int64).reshape(-1).contiguous()
    if t.numel() != n:
        raise ContractError("per-token trace fields must have one entry per token")
    return t


class SparsityTrace:
    """Long-format routing record: rows [n, 8] int64 on the device (phase as
    0 = prefill / 1 = decode), appended per layer call."""

    def __init__(self, device=None):
        self.device = torch.device(device) if device is not None else None
        self._chunks: list[torch.Tensor] = []
        self._active: torch.Tensor | None = None  # u64-as-int64 executed-slot counter

    # -- recording -----------------------------------------------------------------
    def record_layer(self, topk_ids, masked_ids, layer: int, phase: str, sequence_id=None,
                     position=None, token_id=None) -> None:
        """Rows of one layer call: topk_ids / masked_ids [T, K] int64 (the gate
        outputs: RouterDecision.topk_indices and the mask-routed ids, -1 =
        masked); sequence_id / position / token_id [T] (defaults 0, t, 0)."""
        if phase not in PHASES:
            raise ContractError(f"unknown phase {phase!r}")
        ids = as_torch(topk_ids)
        dev = ids.device if ids.is_cuda else (self.device or _default_device())
        self.device = dev
        ids = ids.to(dev, torch.int64).contiguous()
        mids = as_torch(masked_ids).to(dev, torch.int64).contiguous()
        if ids.ndim != 2 or mids.shape != ids.shape:
            raise ContractError("topk_ids and masked_ids must both be [T, K]")
        t, k = ids.shape
        seq, pos, tok = (_i64(v, dev, t) for v in (sequence_id, position, token_id))
        rows = torch.empty(t * k, 8, dtype=torch.int64, device=dev)
        if self._active is None:
            self._active = torch.zeros(1, dtype=torch.int64, device=dev)
        p = lambda v: v.data_ptr() if v is not None else None  # noqa: E731
        _lib.check(_lib.load().beam_trace_rows(ids.data_ptr(), mids.data_ptr(), p(seq), p(pos), p(tok), t, k,
                                               int(layer), PHASES.index(phase), rows.data_ptr(),
                                               self._active.data_ptr(), _runtime.stream_handle(dev)),
                   "beam_trace_rows")
        self._chunks.append(rows)

    def record_decision(self, decision, mask_decision, layer: int, phase: str, sequence_id=None,
                        position=None, token_id=None) -> None:
        """Rows of a beam_block_forward call from its (RouterDecision, MaskDecision)."""
        ids = as_torch(decision.topk_indices).to(torch.int64)
        bits = as_torch(mask_decision.mask).to(ids.device).gather(1, ids.clamp_min(0))
        masked = torch.where((bits > 0) & (ids >= 0), ids, torch.full_like(ids, -1))
        self.record_layer(ids, masked, layer, phase, sequence_id, position, token_id)

    def record_cell(self, sequence_id, position, layer, expert_ids, mask_bits, phase, token_id):
        """analysis.py:41-52 (one cell from host values)."""
        if phase not in PHASES:
            raise ContractError(f"unknown phase {phase!r}")
        e = np.asarray(expert_ids, np.int64)
        b = np.asarray(mask_bits, np.int64)
        dev = self.device or _default_device()
        self.device = dev
        rows = np.stack([np.full(e.size, int(sequence_id)), np.full(e.size, int(position)),
                         np.full(e.size, int(layer)), np.arange(1, e.size + 1), e, b,
                         np.full(e.size, PHASES.index(phase)), np.full(e.size, int(token_id))], axis=1)
        self._chunks.append(torch.from_numpy(rows).to(dev))
        if self._active is None:
            self._active = torch.zeros(1, dtype=torch.int64, device=dev)
        self._active += int(b.sum())

    # -- views -----------------------------------------------------------------------
    def rows(self) -> torch.Tensor:
        if not self._chunks:
            return torch.zeros(0, 8, dtype=torch.int64, device=self.device or "cpu")
        if len(self._chunks) > 1:
            self._chunks = [torch.cat(self._chunks)]
        return self._chunks[0]

    def __len__(self) -> int:
        return sum(c.shape[0] for c in self._chunks)

    @property
    def active_slots(self) -> int:
        """Executed slots recorded so far (device counter)."""
        return int(self._active.item()) if self._active is not None else 0

    @property
    def k(self) -> int:
        r = self.rows()
        return int(r[:, 3].max()) if r.numel() else 0

    def arrays(self) -> dict[str, np.ndarray]:
        r = self.rows().cpu().numpy()
        out = {name: r[:, i].copy() for i, name in enumerate(_COLS)}
        out["phase"] = np.asarray(PHASES)[out["phase"]] if r.size else np.asarray([], dtype="<U7")
        return out

    def to_csv(self, path) -> None:
        """Same bytes as the reference's writer (csv module, \\r\\n rows)."""
        r = self.rows().cpu().numpy()
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(TRACE_HEADER)
            for row in r.tolist():
                row[6] = PHASES[row[6]]
                w.writerow(row)

    @classmethod
    def from_csv(cls, path, device=None) -> "SparsityTrace":
        trace = cls(device)
        with open(path, newline="") as f:
            reader = csv.reader(f)
            if next(reader, None) != TRACE_HEADER:
                raise ContractError(f"unexpected trace header in {path}")
            rows = []
            for lineno, row in enumerate(reader, start=2):
                if len(row) != len(TRACE_HEADER) or row[6] not in PHASES:
                    raise ContractError(f"malformed trace row {lineno} in {path}")
                try:
                    vals = [int(v) for v in row[:6]] + [PHASES.index(row[6]), int(row[7])]
                except ValueError:
                    raise ContractError(f"malformed trace row {lineno} in {path}")
                rows.append(vals)
        if rows:
            trace._chunks.append(torch.tensor(rows, dtype=torch.int64, device=trace.device or _default_device()))
            trace.device = trace._chunks[0].device
            trace._active = trace._chunks[0][:, 5].sum().reshape(1)
        return trace


# ---------------------------------------------------------------------------
# Avg-K and friends, reduced on the device
# ---------------------------------------------------------------------------


def _cells(trace: SparsityTrace):
    r = trace.rows()
    if r.numel() == 0:
        raise ContractError("empty trace")
    keys, inverse = torch.unique(r[:, 0:3], dim=0, return_inverse=True)  # (sequence, position, layer)
    counts = torch.zeros(keys.shape[0], dtype=torch.float64, device=r.device)
    counts.index_add_(0, inverse, r[:, 5].to(torch.float64))
    return r, keys, inverse, counts


def avg_k(trace: SparsityTrace, group_by: str = "overall") -> dict:
    """analysis.py:127-166: mean executed experts per (token, layer) cell."""
    if group_by not in GROUP_KEYS:
        raise ContractError(f"unknown group key {group_by!r}; valid: {GROUP_KEYS}")
    r, keys, inverse, counts = _cells(trace)
    if group_by == "token_layer":
        return {tuple(int(v) for v in kk): float(c) for kk, c in zip(keys.tolist(), counts.tolist())}
    if group_by == "overall":
        return {"overall": float(counts.mean())}
    if group_by in ("layer", "token_position"):
        ck = keys[:, 2 if group_by == "layer" else 1]
    else:  # phase / token_id are constant within a cell: take the cell's first row
        first = torch.full((keys.shape[0],), r.shape[0], dtype=torch.int64, device=r.device)
        first.scatter_reduce_(0, inverse, torch.arange(r.shape[0], device=r.device), reduce="amin")
        ck = r[first, 6 if group_by == "phase" else 7]
    out = {}
    for key in torch.unique(ck).tolist():
        label = PHASES[key] if group_by == "phase" else int(key)
        out[label] = float(counts[ck == key].mean())
    return out


def position_mask_prob(trace: SparsityTrace) -> dict[int, float]:
    """analysis.py:169-176: per rank, the fraction of cells whose slot was masked."""
    r = trace.rows()
    if r.numel() == 0:
        raise ContractError("empty trace")
    out = {}
    for rank in range(1, trace.k + 1):
        sel = r[:, 3] == rank
        out[rank] = float((r[sel, 5] == 0).to(torch.float64).mean())
    return out


def expert_load(trace: SparsityTrace) -> tuple[dict[int, float], dict[int, float]]:
    """analysis.py:195-212: per-expert share of routed slots, before / after masking."""
    r = trace.rows()
    if r.numel() == 0:
        raise ContractError("empty trace")
    routed = r[:, 4] >= 0
    kept = routed & (r[:, 5] == 1)

    def dist(sel):
        ids = r[sel, 4]
        if ids.numel() == 0:
            return {}
        c = torch.bincount(ids)
        return {int(e): float(v) / ids.numel() for e, v in enumerate(c.tolist()) if v}

    return dist(routed), dist(kept)
