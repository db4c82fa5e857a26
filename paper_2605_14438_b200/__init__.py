"""B200-native BEAM (Binary Expert Activation Masking) MoE-layer hot path.

A drop-in for the inference path of the reference package ``beamoe``
(arxiv 2605.14438): same public names as ``beamoe.moe`` / ``beamoe.beam`` /
``beamoe.dispatch``, computed by hand-written sm_100a CUDA kernels behind the
C ABI in ``include/beam_b200.h``.  No CPU fallback: without the built library
or a CUDA device every compute entry raises ``BeamNativeError``.
"""

from . import analysis, baselines, dispatch, lm  # noqa: F401
from ._lib import BeamNativeError  # noqa: F401
from .beam import (  # noqa: F401
    MaskDecision,
    MaskGrad,
    MaskRouter,
    beam_block_forward,
    mask_forward,
    mask_router_backward,
    rms_norm,
    set_expert_path,
    sparsity_loss,
    ste_backward,
)
from .moe import (  # noqa: F401
    Expert,
    MoEBlock,
    MoEBlockConfig,
    RouterDecision,
    topk_route,
    topk_select,
)
from .tensor import ContractError, NumericError, ShapeError  # noqa: F401

__all__ = [
    "BeamNativeError", "ContractError", "Expert", "MaskDecision", "MaskRouter", "MoEBlock",
    "MoEBlockConfig", "NumericError", "RouterDecision", "ShapeError", "beam_block_forward",
    "baselines", "dispatch", "mask_forward", "mask_router_backward", "MaskGrad", "rms_norm",
    "sparsity_loss", "ste_backward", "topk_route", "topk_select",
]
