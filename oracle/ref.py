"""TEST INFRASTRUCTURE ONLY — import the unmodified reference package
(``beamoe``) that ``oracle/build_ref.sh`` built into ``oracle/_ref/``.

Used by the parity tests (live reference runs), ``tests/golden/make_golden.py``
and ``bench.py``'s CPU-baseline leg / ``--impl reference`` arm.
"""

from __future__ import annotations

import os
import sys

REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "beamoe"))


def import_beamoe():
    """Return the reference ``beamoe`` package (raises ImportError if absent)."""
    if not available():
        raise ImportError(f"reference not built: run oracle/build_ref.sh (looked in {REF_DIR})")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import beamoe  # noqa: F401
    import beamoe.beam  # noqa: F401
    import beamoe.dispatch  # noqa: F401
    import beamoe.moe  # noqa: F401

    return sys.modules["beamoe"]


def to_reference_block(block, beamoe=None):
    """Build a reference ``MoEBlock`` (with ``MaskRouter``) holding exactly the
    parameters of an ``oracle.beam_oracle.OracleBlock``."""
    import numpy as np

    beamoe = beamoe or import_beamoe()
    from beamoe.beam import MaskRouter
    from beamoe.moe import Expert, MoEBlock, MoEBlockConfig
    from beamoe.tensor import Tensor

    cfg = MoEBlockConfig(d_h=block.d_h, d_ff=block.d_ff, num_experts=block.num_experts,
                         top_k=block.top_k, num_shared=len(block.shared),
                         has_norm=block.norm_w is not None, activation=block.activation)
    rb = MoEBlock.__new__(MoEBlock)
    rb.cfg = cfg
    rb.router_w = Tensor._raw(np.ascontiguousarray(block.router_w, dtype=np.float64))
    rb.experts = [Expert(Tensor._raw(g), Tensor._raw(u), Tensor._raw(d)) for g, u, d in block.experts]
    rb.shared = [Expert(Tensor._raw(g), Tensor._raw(u), Tensor._raw(d)) for g, u, d in block.shared]
    rb.norm_w = Tensor._raw(block.norm_w) if block.norm_w is not None else None
    rb.mask_router = MaskRouter(Tensor._raw(np.ascontiguousarray(block.mask_w, dtype=np.float64)),
                                block.tau)
    return rb
