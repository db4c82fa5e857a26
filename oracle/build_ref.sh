#!/usr/bin/env bash
# Test infrastructure only (see oracle/README header in oracle/__init__.py).
#
# Builds the UNMODIFIED reference package `beamoe` (numpy + Cython CPU
# implementation of the BEAM MoE layer, /root/reference/pkg) into
# oracle/_ref/ so that the parity tests, the golden-vector generator and
# bench.py's CPU-baseline leg can run the reference itself.
#
# The build writes into its source tree (Cython generates .c/.so next to the
# .pyx), and /root/reference is read-only, so we build from a scratch copy
# under /tmp.  Outputs land only in oracle/_ref/ (git-ignored, NOT
# gpurun-ignored: the built package travels to the GPU box with the repo).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${BEAM_REFERENCE_PKG:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "build_ref: reference source $SRC not present; keeping existing $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/beamoe_ref_build.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
mkdir -p "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --target "$OUT" "$TMP/pkg" >"$TMP/pip.log" 2>&1 || { cat "$TMP/pip.log" >&2; exit 1; }
# the reference's own test files (not installed by pip) for the reference-side
# backend integration test (tests/test_gpu_integration.py): build output only,
# git-ignored like the rest of oracle/_ref
cp -r "$SRC/tests" "$OUT/reference_tests"
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
from beamoe import dispatch
print("build_ref: beamoe built into", sys.argv[1], "backend =", dispatch.active_backend())
PY
