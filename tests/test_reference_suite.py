"""The reference's own tests, judging the CUDA kernel through the drop-in
backend (tests/ref_shim.py). Needs oracle/_ref (built by oracle/build_ref.sh
from /root/reference; it travels to the GPU box with the snapshot)."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = ROOT / "oracle" / "_ref"

# reference test files / selections that exercise the kernel boundary
SUITE = [
    "tests/test_backends.py",
    "tests/test_batch.py",
    "tests/test_raycast.py",
    "tests/test_render.py",
    "tests/test_dynamics.py",
]
# test_golden_frames needs pkg/tests/data/golden_frames.npz, absent from the
# reference snapshot; our own golden-frame test covers it.
DESELECT = ["tests/test_render.py::test_golden_frames"]


@pytest.mark.gpu
def test_reference_suite_on_cuda_backend():
    if not (REF / "tests" / "test_backends.py").exists():
        pytest.skip("oracle/_ref/tests not built (run oracle/build_ref.sh here)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT / "tests"), str(ROOT)])
    env["TILECAST_BACKEND"] = "compiled"
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_shim", "-q", "-x", "-p", "no:cacheprovider",
           *SUITE, *[f"--deselect={d}" for d in DESELECT]]
    r = subprocess.run(cmd, cwd=REF, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "passed" in r.stdout
    # the cross-backend parity tests must have run, not been skipped
    assert "skipped" not in r.stdout.splitlines()[-1] or "passed" in r.stdout, tail
