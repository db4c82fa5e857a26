"""TEST INFRASTRUCTURE ONLY — host (numpy, float64) restatement of the
expert-parallel data-plane kernels (paper_2605_14438_b200/csrc/ep.cu), used

* by tests/test_ep_gloo.py, injected into ``EPBeamLayer(kernels=...)``, so the
  exchange protocol (protocol agreement, buffer layouts, split sizes, the
  all-to-all sequence, ascending-rank combine) runs with world_size 2 over gloo
  on CPU, and
* by tests/test_gpu_ep.py as the checker of the CUDA pack kernel's layouts.

Per-token semantics are the reference's beam_block_forward (beam.py:127-165;
oracle/beam_oracle.py): gating = topk_route + mask_forward + mask_route, each
surviving slot runs on the rank owning its expert, partial sums in ascending
rank order (dispatch/__init__.py:145-156), then h + y.
"""

from __future__ import annotations

import numpy as np
import torch

from . import beam_oracle as O

TILE = 256  # tokens per tile of the count / pack kernels (ep.cu kEpTile)


def dest_bits(masked: np.ndarray, n: int, n_local: int) -> np.ndarray:
    """[T] destination-rank bitmask (bit p: some surviving slot on rank p)."""
    bits = np.zeros(masked.shape[0], dtype=np.int64)
    for k in range(masked.shape[1]):
        e = masked[:, k]
        ok = (e >= 0) & (e < n)
        bits |= np.where(ok, 1 << np.where(ok, e // n_local, 0), 0)
    return bits


def tile_counts(masked: np.ndarray, n: int, world: int) -> np.ndarray:
    """beam_ep_count: [world, ntiles] rows per (destination, 256-token tile)."""
    t = masked.shape[0]
    bits = dest_bits(masked, n, n // world)
    nt = max((t + TILE - 1) // TILE, 1)
    out = np.zeros((world, nt), dtype=np.int64)
    for p in range(world):
        f = (bits >> p) & 1
        for i in range(nt):
            out[p, i] = int(f[i * TILE:(i + 1) * TILE].sum())
    return out


def pack(h: np.ndarray, masked: np.ndarray, weights: np.ndarray, n: int, world: int, cap: int,
         has_norm: bool, rows: int | None = None):
    """beam_ep_pack: (x [rows, d], meta [rows, 2K+1] int32, send_pos [world, T]).
    Fixed layout (cap > 0): peer p's rows at [p*cap, p*cap + count_p), unused rows
    ids -1; compact (cap == 0): peer blocks back to back.  Rows of a peer are in
    ascending token order; a token goes to a peer once (deduplicated)."""
    t, d = h.shape
    k = masked.shape[1]
    nl = n // world
    bits = dest_bits(masked, n, nl)
    counts = [int(((bits >> p) & 1).sum()) for p in range(world)]
    if cap > 0:
        base = [p * cap for p in range(world)]
        n_rows = world * cap
    else:
        base = list(np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(int))
        n_rows = int(sum(counts)) if rows is None else rows
    x = np.zeros((n_rows, d), dtype=h.dtype)
    meta = np.zeros((n_rows, 2 * k + 1), dtype=np.int32)
    meta[:, :k] = -1
    send_pos = np.full((world, t), -1, dtype=np.int32)
    inv = 1.0 / np.sqrt((h.astype(np.float64) ** 2).mean(axis=1) + 1e-6) if has_norm and t else np.zeros(t)
    for p in range(world):
        r = base[p]
        for tok in range(t):
            if not (bits[tok] >> p) & 1:
                continue
            send_pos[p, tok] = r
            x[r] = h[tok]
            for j in range(k):
                e = int(masked[tok, j])
                mine = 0 <= e < n and e // nl == p
                meta[r, j] = e - p * nl if mine else -1
                meta[r, k + j] = np.float32(weights[tok, e] if mine else 0.0).view(np.int32)
            meta[r, 2 * k] = np.float32(inv[tok] if has_norm else 0.0).view(np.int32)
            r += 1
    return x, meta, send_pos


def execute(x: np.ndarray, meta: np.ndarray, local_experts, norm_w, activation="silu") -> np.ndarray:
    """beam_ep_execute: per received row, its local experts in ascending id,
    ghat-weighted, on x_n = x * inv_rms * norm_w (fp64)."""
    n, d = x.shape
    k = (meta.shape[1] - 1) // 2
    y = np.zeros((n, d))
    for r in range(n):
        inv = float(meta[r, 2 * k:2 * k + 1].view(np.float32)[0])
        xn = x[r].astype(np.float64) * inv * norm_w if norm_w is not None else x[r].astype(np.float64)
        order = sorted((int(e), j) for j, e in enumerate(meta[r, :k]) if e >= 0)
        for e, j in order:
            w = float(meta[r, k + j:k + j + 1].view(np.float32)[0])
            y[r] += w * O.expert_forward(xn[None], *local_experts[e], activation=activation)[0]
    return y


def combine(h: np.ndarray, y_back: np.ndarray, send_pos: np.ndarray) -> np.ndarray:
    """beam_ep_combine: h + partial sums in ascending rank order."""
    y = np.zeros(h.shape)
    for p in range(send_pos.shape[0]):
        for tok in range(h.shape[0]):
            r = send_pos[p, tok]
            if r >= 0:
                y[tok] += y_back[r]
    return h + y


class HostKernels:
    """``EPBeamLayer(kernels=lambda L: HostKernels(L, oracle_block))``: the CPU
    data plane for the protocol tests (gating with the fp64 oracle)."""

    def __init__(self, layer, block: O.OracleBlock):
        self.L = layer
        self.ob = block
        nl = layer.n_local
        self.local_experts = block.experts[layer.rank * nl:(layer.rank + 1) * nl]

    def gate(self, h):
        h64 = h.numpy().astype(np.float64)
        xn = self.ob.normalize(h64)
        dec = O.topk_route(xn, self.ob.router_w, self.ob.top_k)
        md = O.mask_forward(xn, self.ob.mask_w)
        masked = O.mask_route(dec.topk_indices, md.pre_activation)
        return torch.from_numpy(masked), torch.from_numpy(dec.weights)

    def counts(self, masked):
        tiles = tile_counts(masked.numpy(), self.ob.num_experts, self.L.world)
        return torch.from_numpy(tiles.sum(axis=1)), torch.from_numpy(tiles)

    def pack(self, h, masked, weights, cap, tiles=None, rows=None):
        x, meta, pos = pack(h.numpy(), masked.numpy(), weights.numpy(), self.ob.num_experts, self.L.world, cap,
                            self.ob.norm_w is not None, rows)
        return torch.from_numpy(x), torch.from_numpy(meta), torch.from_numpy(pos)

    def local(self, x, meta, mode):
        return torch.from_numpy(execute(x.numpy(), meta.numpy(), self.local_experts, self.ob.norm_w,
                                        self.ob.activation))

    def combine(self, h, y_back, send_pos):
        return torch.from_numpy(combine(h.numpy(), y_back.numpy(), send_pos.numpy()))
