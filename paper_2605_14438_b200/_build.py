"""Build the sm_100a CUDA library ``_lib/libbeam_b200.so`` in-tree with nvcc.

Used by ``__graft_entry__.build()`` and runnable directly:
``python -m paper_2605_14438_b200._build``.  The .so is git-ignored but travels
to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import glob
import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libbeam_b200.so")
# device-checked variant (-DBEAM_DEVICE_CHECKS: bounds assertions; tests only)
LIB_CHECKED = os.path.join(LIBDIR, "libbeam_b200_checked.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _digest(extra=()) -> str:
    h = hashlib.sha256()
    files = _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        sorted(glob.glob(os.path.join(CSRC, "*.h"))) + [os.path.join(ROOT, "include", "beam_b200.h")]
    for f in files:
        h.update(f.encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(ARCH + NVCC_FLAGS + list(extra)).encode())
    return h.hexdigest()


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False, jobs: int | None = None, checked: bool = False) -> str:
    """Compile every csrc/*.cu for sm_100a and link the shared library
    (`checked`: the device-checked variant, libbeam_b200_checked.so)."""
    extra = ["-DBEAM_DEVICE_CHECKS"] if checked else []
    lib = LIB_CHECKED if checked else LIB
    stamp = os.path.join(LIBDIR, ".digest_checked" if checked else ".digest")
    digest = _digest(extra)
    if not force and os.path.exists(lib) and os.path.exists(stamp):
        with open(stamp) as fh:
            if fh.read().strip() == digest:
                return lib
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = tempfile.mkdtemp(prefix="beam_b200_build_")
    try:
        objs, procs = [], []
        for src in _sources():
            obj = os.path.join(tmp, os.path.basename(src)[:-3] + ".o")
            cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
            objs.append(obj)
        failed = []
        for src, p in procs:
            out, _ = p.communicate()
            if p.returncode != 0:
                failed.append((src, out))
            elif verbose and out.strip():
                print(out)
        if failed:
            msg = "\n".join(f"--- {s}\n{o}" for s, o in failed)
            raise RuntimeError(f"nvcc failed:\n{msg}")
        tmp_lib = os.path.join(tmp, os.path.basename(lib))
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp_lib, *objs]
        subprocess.run(cmd, check=True, capture_output=not verbose)
        os.replace(tmp_lib, lib)
        with open(stamp, "w") as fh:
            fh.write(digest)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build(force="--force" in sys.argv, verbose=False, checked=True))
