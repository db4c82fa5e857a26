"""Device-checked build (libbeam_b200_checked.so, -DBEAM_DEVICE_CHECKS) — the
substitute for compute-sanitizer memcheck, which this GPU pool does not run:
every layer path (decode / prefill / tcgen05 / shared experts / EP / permute)
runs with bounds assertions on plan positions, token indices, combine slots and
tensor-core tiles, and must leave the check word at zero; a deliberately
corrupted plan must set it (the checks are live)."""

import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2605_14438_b200", "_lib", "libbeam_b200_checked.so")


def _run(*args):
    if not os.path.exists(CHECKED):
        pytest.fail("libbeam_b200_checked.so not built (__graft_entry__.build())")
    env = dict(os.environ, BEAM_LIB="checked")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_run.py"), *args], capture_output=True,
                       text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_layer_paths_pass_device_checks():
    res = _run()
    assert "device-checked" in res["build"]
    assert res["flag"] == 0, res
    assert len(res["cases"]) >= 16


def test_device_checks_fire_on_a_corrupted_plan():
    res = _run("--negative")
    assert res["flag"] & 4, res  # kChkToken
