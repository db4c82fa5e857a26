"""Error types of the reference's numerics module, re-exported so callers can
catch the same exceptions (/root/reference/pkg/src/beamoe/tensor.py:24-33).

The reference's fp64 tape ``Tensor`` itself is training machinery and out of
scope; the B200 path works on ``torch.Tensor`` (device memory).  Helpers here
convert reference-style inputs (numpy arrays or objects with a ``.data`` numpy
array, e.g. ``beamoe.tensor.Tensor``) into tensors.
"""

from __future__ import annotations

import numpy as np


class ShapeError(ValueError):
    """Operand shapes do not satisfy an operation's contract (tensor.py:24-25)."""


class NumericError(ArithmeticError):
    """A value that must be finite is NaN or infinite (tensor.py:28-29)."""


class ContractError(ValueError):
    """An input violates a documented precondition (tensor.py:32-33)."""


def as_torch(x, dtype=None):
    """torch.Tensor view/copy of ``x`` (torch tensor, numpy array, or an object
    whose ``.data`` is a numpy array).  float64 host data becomes float32: the
    B200 path computes routing in fp32 and experts in bf16/fp32."""
    import torch

    if isinstance(x, torch.Tensor):
        t = x
    else:
        data = getattr(x, "data", x)
        if isinstance(data, torch.Tensor):
            t = data
        else:
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(data)))
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    elif t.dtype == torch.float64:
        t = t.to(torch.float32)
    return t
