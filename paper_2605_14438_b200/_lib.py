"""ctypes binding of the C ABI in ``include/beam_b200.h`` (``_lib/libbeam_b200.so``).

There is deliberately no fallback: if the library is missing or no CUDA device
is visible, every entry point raises ``BeamNativeError``.
"""

from __future__ import annotations

import ctypes
import os

from .tensor import ContractError, ShapeError

_PKG = os.path.dirname(os.path.abspath(__file__))
# BEAM_LIB=checked loads the device-checked build (bounds assertions, tests
# only); an absolute path loads that file (A/B timing of two builds)
_SEL = os.environ.get("BEAM_LIB", "")
LIB_PATH = (_SEL if os.path.isabs(_SEL) else
            os.path.join(_PKG, "_lib", "libbeam_b200_checked.so" if _SEL == "checked" else "libbeam_b200.so"))

BEAM_OK = 0
BEAM_ERR_ARG = -1
BEAM_ERR_UNSUPPORTED = -2
BEAM_ERR_CUDA = -3
BEAM_ERR_WORKSPACE = -4

BEAM_F32, BEAM_BF16, BEAM_F64 = 0, 1, 2
BEAM_ACT_SILU, BEAM_ACT_IDENTITY = 0, 1
BEAM_ROUTE_BEAM, BEAM_ROUTE_TOPK, BEAM_ROUTE_DYNAMIC, BEAM_ROUTE_ADA, BEAM_ROUTE_SOFT = 0, 1, 2, 3, 4

# every symbol include/beam_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "beam_workspace_bytes",
    "beam_layer_forward",
    "beam_layer_forward_routed",
    "beam_workspace_bytes_routed",
    "beam_gate",
    "beam_moe_execute",
    "beam_mask_route",
    "beam_topk_select",
    "beam_group_by_expert",
    "beam_group_by_expert_workspace_bytes",
    "beam_grouped_execute",
    "beam_rms_norm",
    "beam_ste_backward",
    "beam_sparsity_loss",
    "beam_mask_backward",
    "beam_trace_rows",
    "beam_kernel_launches",
    "beam_set_expert_path",
    "beam_profile_begin",
    "beam_profile_end",
    "beam_trace_gate",
    "beam_last_cuda_error",
    "beam_build_info",
    "beam_host_mapped",
    "beam_router_split",
    "beam_abi_sizeof",
    "beam_debug_checks",
    "beam_ep_tiles",
    "beam_ep_count",
    "beam_ep_pack",
    "beam_ep_workspace_bytes",
    "beam_ep_execute",
    "beam_ep_combine",
)


class BeamNativeError(RuntimeError):
    """The CUDA library is unavailable or a kernel launch failed."""


class LayerDesc(ctypes.Structure):
    """beam_layer_t."""

    _fields_ = [
        ("d_h", ctypes.c_int),
        ("d_ff", ctypes.c_int),
        ("num_experts", ctypes.c_int),
        ("top_k", ctypes.c_int),
        ("num_shared", ctypes.c_int),
        ("has_norm", ctypes.c_int),
        ("activation", ctypes.c_int),
        ("wdtype", ctypes.c_int),
        ("mask_threshold", ctypes.c_float),
        ("norm_w", ctypes.c_void_p),
        ("gate_wT", ctypes.c_void_p),
        ("w_gu", ctypes.c_void_p),
        ("w_down", ctypes.c_void_p),
        ("gate_w3", ctypes.c_void_p),
        ("gate_w3_cols", ctypes.c_int),
    ]


class RouteDesc(ctypes.Structure):
    """beam_route_t."""

    _fields_ = [
        ("kind", ctypes.c_int),
        ("k", ctypes.c_int),
        ("null_count", ctypes.c_int),
        ("phi", ctypes.c_float),
        ("temp", ctypes.c_float),
        ("tau", ctypes.c_float),
        ("binarize", ctypes.c_int),
    ]


class Outputs(ctypes.Structure):
    """beam_outputs_t."""

    _fields_ = [
        ("out", ctypes.c_void_p),
        ("topk_ids", ctypes.c_void_p),
        ("logits", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
        ("pre_activation", ctypes.c_void_p),
        ("raw_mask", ctypes.c_void_p),
        ("mask", ctypes.c_void_p),
        ("masked_ids", ctypes.c_void_p),
        ("decision_event", ctypes.c_void_p),
    ]


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise BeamNativeError(
            f"CUDA library not built: {path} missing (run `python -m paper_2605_14438_b200._build`)")
    lib = ctypes.CDLL(path)
    P, I, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    LP, OP, RP = ctypes.POINTER(LayerDesc), ctypes.POINTER(Outputs), ctypes.POINTER(RouteDesc)
    sig = {
        "beam_workspace_bytes": (S, [LP, I, I, I]),
        "beam_layer_forward": (I, [LP, P, I, I, I, OP, P, S, P]),
        "beam_layer_forward_routed": (I, [LP, RP, P, I, I, I, OP, P, S, P]),
        "beam_workspace_bytes_routed": (S, [LP, RP, I, I]),
        "beam_gate": (I, [LP, P, I, I, OP, P, S, P]),
        "beam_moe_execute": (I, [LP, P, I, I, I, P, P, P, P, S, P]),
        "beam_mask_route": (I, [P, P, I, I, I, I, P, P]),
        "beam_topk_select": (I, [P, I, I, I, I, P, P]),
        "beam_group_by_expert": (I, [P, I, I, I, I, P, P, P, P, P, P, P, S, P]),
        "beam_group_by_expert_workspace_bytes": (S, [I, I, I]),
        "beam_grouped_execute": (I, [LP, P, I, I, I, I, P, P, P, P, P, P, P, P, P, P, S, P]),
        "beam_rms_norm": (I, [P, I, I, I, P, P, P]),
        "beam_ste_backward": (I, [P, P, P, I, I, I, ctypes.c_float, P, P]),
        "beam_sparsity_loss": (I, [P, P, I, I, I, P, P]),
        "beam_mask_backward": (I, [LP, P, I, I, P, ctypes.c_float, I, OP, P, P, P, P, S, P]),
        "beam_trace_rows": (I, [P, P, P, P, P, I, I, I, I, P, P, P]),
        "beam_kernel_launches": (ctypes.c_ulonglong, []),
        "beam_set_expert_path": (I, [I]),
        "beam_profile_begin": (I, [I]),
        "beam_profile_end": (I, [P, P]),
        "beam_trace_gate": (I, [P]),
        "beam_last_cuda_error": (ctypes.c_char_p, []),
        "beam_build_info": (ctypes.c_char_p, []),
        "beam_host_mapped": (I, [P]),
        "beam_router_split": (I, [P, P, I, I, I, P, P]),
        "beam_abi_sizeof": (S, [I]),
        "beam_debug_checks": (I, [P]),
        "beam_ep_tiles": (I, [I]),
        "beam_ep_count": (I, [P, I, I, I, I, P, P]),
        "beam_ep_pack": (I, [P, I, I, I, P, P, I, I, I, I, P, I, P, P, P, P, P]),
        "beam_ep_workspace_bytes": (S, [LP, I, I, I]),
        "beam_ep_execute": (I, [LP, P, I, I, I, P, I, P, P, S, P]),
        "beam_ep_combine": (I, [P, P, I, I, I, P, I, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == BEAM_OK:
        return
    lib = load()
    if rc == BEAM_ERR_ARG:
        raise ContractError(f"{what}: invalid argument")
    if rc == BEAM_ERR_UNSUPPORTED:
        raise ShapeError(f"{what}: shape not supported by the sm_100a kernels")
    if rc == BEAM_ERR_WORKSPACE:
        raise BeamNativeError(f"{what}: workspace too small")
    raise BeamNativeError(f"{what}: CUDA error: {lib.beam_last_cuda_error().decode()}")


def require_device(t) -> None:
    import torch

    if not torch.cuda.is_available():
        raise BeamNativeError("no CUDA device visible: the BEAM B200 kernels have no CPU fallback")
    if not t.is_cuda:
        raise BeamNativeError("expected a CUDA tensor")
