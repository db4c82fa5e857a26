"""Device plumbing: current stream handle and cached workspaces (torch memory)."""

from __future__ import annotations

import threading
import warnings

import torch

_lock = threading.Lock()
_workspaces: dict = {}
# Superseded workspaces stay alive: a CUDA graph captured while one of them was
# current still points at it (and at its grid-completion counters), so freeing
# it on growth would make a later replay a use-after-free.  Geometric growth
# bounds what this keeps to ~2x the largest workspace per stream.
_retired: list = []


def stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    """A uint8 scratch buffer of at least ``nbytes`` for the current stream of
    ``device`` (grown geometrically, reused across calls on that stream)."""
    key = (device.index if device.index is not None else torch.cuda.current_device(),
           torch.cuda.current_stream(device).cuda_stream)
    with _lock:
        buf = _workspaces.get(key)
        if buf is None or buf.numel() < nbytes:
            size = max(nbytes, int(buf.numel() * 1.5) if buf is not None else 0, 1 << 20)
            if torch.cuda.is_current_stream_capturing():
                warnings.warn("beam workspace created during CUDA-graph capture: its zero fill "
                              "becomes part of every replay; run one call on the capture stream "
                              "before capturing (torch.cuda.graph(..., stream=that_stream))",
                              RuntimeWarning, stacklevel=3)
            # zero-filled once: the grid-completion counters at its start must
            # begin at 0 (the kernels reset them after every use)
            if buf is not None:
                _retired.append(buf)
            buf = torch.zeros(size, dtype=torch.uint8, device=device)
            _workspaces[key] = buf
        return buf


def release_workspaces() -> None:
    """Drop every cached workspace (only safe once no captured graph that used
    one will be replayed again)."""
    with _lock:
        _workspaces.clear()
        _retired.clear()
