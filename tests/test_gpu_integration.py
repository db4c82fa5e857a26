"""The reference-side binding, exercised: the reference package's OWN test files
(copied into oracle/_ref/reference_tests by oracle/build_ref.sh, next to the
reference install) run with the B200 dispatch backend (tests/b200_backend.py)
registered in ``beamoe.dispatch._BACKENDS`` (dispatch/__init__.py:21-44).

* registered only: every ``@pytest.mark.parametrize("backend", BACKENDS)`` case
  of test_dispatch.py runs on "b200", and the two ``test_backends_bit_identical``
  tests (:55-64, :125-135) compare it with the reference's Cython backend;
* registered AND active: the reference's dispatch, BEAM-layer and MoE suites
  (test_dispatch.py, test_beam.py, test_moe.py, non-slow) route every
  ``mask_route`` / ``align_block`` through the sm_100a kernels."""

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "oracle", "_ref", "reference_tests")


def _run_reference_tests(files, active):
    if not os.path.isdir(REF_TESTS):
        pytest.skip("reference tests not built (oracle/build_ref.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, env.get("PYTHONPATH", "")])
    env["BEAM_B200_ACTIVE"] = "1" if active else "0"
    cmd = [sys.executable, "-m", "pytest", "-q", "-rA", "-p", "b200_backend", "-p", "no:cacheprovider",
           "-m", "not slow", "--rootdir", REF_TESTS, *[os.path.join(REF_TESTS, f) for f in files]]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=REF_TESTS, timeout=900)
    return r.returncode, r.stdout + r.stderr


def test_reference_dispatch_suite_with_b200_backend_registered():
    rc, out = _run_reference_tests(["test_dispatch.py"], active=False)
    assert rc == 0, out[-4000:]
    assert "PASSED test_dispatch.py::TestMaskRoute::test_sign_rule[b200]" in out, out[-4000:]
    assert "PASSED test_dispatch.py::TestAlignBlock::test_hand_grouping[b200]" in out, out[-4000:]
    assert "PASSED test_dispatch.py::TestMaskRoute::test_backends_bit_identical" in out, out[-4000:]
    assert "PASSED test_dispatch.py::TestAlignBlock::test_backends_bit_identical" in out, out[-4000:]


def test_reference_suites_with_b200_backend_active():
    rc, out = _run_reference_tests(["test_dispatch.py", "test_beam.py", "test_moe.py"], active=True)
    assert rc == 0, out[-4000:]
    assert " passed" in out and " failed" not in out, out[-4000:]
