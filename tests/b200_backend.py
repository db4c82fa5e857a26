"""Reference-side binding of the B200 library: a ``beamoe.dispatch`` backend.

This is the file a maintainer of the reference would add as
``src/beamoe/dispatch/_b200.py``: the reference selects a
dispatch backend module from ``_BACKENDS`` (dispatch/__init__.py:21-44) and
calls exactly two functions on it —

    mask_route(topk_ids int64[T,K], mask_logits f64[T,N]) -> int64[T,K]
        (_kernels.pyx:17-34 / _fallback.py:14-26)
    group_by_expert(ids int64[T,K], num_experts) -> (counts int64[N],
        token_order int64[R], slot_order int64[R])
        (_kernels.pyx:37-66 / _fallback.py:29-44)

— here both run on the GPU through the C ABI (``beam_mask_route``,
``beam_group_by_expert`` with block_size 1, i.e. no padding: the reference's
``align_block`` pads on the host).  numpy in, numpy out, like the Cython backend.

It is also a pytest plugin (``python -m pytest -p b200_backend ...``): at
configure time it imports the reference package built in ``oracle/_ref``,
registers itself as backend ``"b200"`` and, with ``BEAM_B200_ACTIVE=1``, makes
it the active backend, so the reference's OWN test suite runs its dispatch
through the sm_100a kernels (tests/test_gpu_integration.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np

BACKEND_NAME = "b200"

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dispatch():
    if _ROOT not in sys.path:
        sys.path.insert(0, _ROOT)
    from paper_2605_14438_b200 import dispatch

    return dispatch


def mask_route(topk_ids: np.ndarray, mask_logits: np.ndarray) -> np.ndarray:
    """_kernels.pyx:17-34: id kept iff 0 <= id < N and mask_logits[t, id] >= 0."""
    import torch

    ids = np.ascontiguousarray(topk_ids, dtype=np.int64)
    a = np.ascontiguousarray(mask_logits, dtype=np.float64)
    if ids.size == 0:
        return ids.copy()
    out = _dispatch().mask_route(torch.from_numpy(ids), torch.from_numpy(a))
    return out.numpy().astype(np.int64, copy=False)


def group_by_expert(ids: np.ndarray, num_experts: int):
    """_kernels.pyx:37-66: per-expert counts and the (token, slot) pairs expert
    by expert, each run in ascending flat (t*K + k) order."""
    import torch

    ids = np.ascontiguousarray(ids, dtype=np.int64)
    if ids.ndim != 2:
        ids = ids.reshape(ids.shape[0], -1)
    plan = _dispatch().align_block(torch.from_numpy(ids), 1, int(num_experts))
    total = int(plan.meta.cpu()[2])
    counts = plan.counts.cpu().numpy().astype(np.int64)
    tokens = plan.flat_tokens[:total].cpu().numpy().astype(np.int64)
    slots = plan.flat_slots[:total].cpu().numpy().astype(np.int64)
    return counts, tokens, slots


# ---------------------------------------------------------------------------
# pytest plugin: register into the reference's backend table
# ---------------------------------------------------------------------------


def register(active: bool = False):
    """Add this module to ``beamoe.dispatch._BACKENDS`` (and make it the active
    backend when ``active``).  Returns the reference's dispatch module."""
    sys.path.insert(0, os.path.join(_ROOT, "oracle", "_ref"))
    from beamoe import dispatch as ref_dispatch

    ref_dispatch._BACKENDS[BACKEND_NAME] = sys.modules[__name__]
    if active:
        ref_dispatch._backend = sys.modules[__name__]
    return ref_dispatch


def pytest_configure(config):
    register(active=os.environ.get("BEAM_B200_ACTIVE") == "1")
    config.addinivalue_line("markers", "slow: long-running trend and benchmark tests")
