"""CPU checks of the C ABI boundary: the sm_100a library builds, loads, and
exports every entry point include/beam_b200.h declares (no compute calls)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

HEADER = os.path.join(ROOT, "include", "beam_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(beam_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2605_14438_b200 import _build

    return _build.build()


def test_header_declares_expected_entries():
    names = declared_functions()
    for n in ("beam_layer_forward", "beam_mask_route", "beam_group_by_expert", "beam_grouped_execute",
              "beam_gate", "beam_moe_execute", "beam_workspace_bytes", "beam_rms_norm"):
        assert n in names


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (beam_[a-z_0-9]+)$", out, flags=re.M))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header(lib_path):
    from paper_2605_14438_b200 import _lib

    lib = _lib.load(lib_path)
    assert set(_lib.EXPORTS) == set(declared_functions())
    for n in _lib.EXPORTS:
        assert getattr(lib, n) is not None
    assert b"sm_100a" in lib.beam_build_info()


def test_library_is_sm100a_sass(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header(lib_path):
    import ctypes

    from paper_2605_14438_b200 import _lib

    # the ctypes mirrors have the compiled structs' sizes (beam_abi_sizeof)
    lib = _lib.load(lib_path)
    assert ctypes.sizeof(_lib.LayerDesc) == lib.beam_abi_sizeof(0)
    assert ctypes.sizeof(_lib.Outputs) == lib.beam_abi_sizeof(1)
    assert ctypes.sizeof(_lib.RouteDesc) == lib.beam_abi_sizeof(2)
    # 9 x 4-byte fields (8 int + 1 float), 4 pad, 5 pointers, the split's column count (+ pad)
    assert ctypes.sizeof(_lib.LayerDesc) == 9 * 4 + 4 + 5 * 8 + 8
    assert ctypes.sizeof(_lib.Outputs) == 9 * 8  # 8 output pointers + decision_event


def test_workspace_query_is_cpu_only(lib_path):
    """beam_workspace_bytes does arithmetic only (no device needed)."""
    import ctypes

    from paper_2605_14438_b200 import _lib

    lib = _lib.load(lib_path)
    d = _lib.LayerDesc(2048, 768, 128, 8, 0, 1, 0, _lib.BEAM_BF16, 0.0, 1, 1, 1, 1)
    n64 = lib.beam_workspace_bytes(ctypes.byref(d), 64, 0, 16)
    n1 = lib.beam_workspace_bytes(ctypes.byref(d), 1, 0, 16)
    assert n64 > n1 > 0
    bad = _lib.LayerDesc(2048, 768, 128, 129, 0, 1, 0, _lib.BEAM_BF16, 0.0, 1, 1, 1, 1)
    assert lib.beam_workspace_bytes(ctypes.byref(bad), 64, 0, 16) == 0
