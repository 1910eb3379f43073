"""Run the reference's OWN test suite (/root/reference/pkg/tests, 190 tests,
incl. acceptance criteria C1-C11) against this package through the ``coesim``
import shim (tests/shim/coesim).  Build-container only: skipped when the
reference checkout is absent (it never travels to the GPU box)."""

import os
import shutil
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference checkout not present")
def test_reference_suite_passes_against_this_package(tmp_path):
    work = tmp_path / "reftests"
    shutil.copytree(REF_TESTS, work)  # the reference tree is read-only; run from a scratch copy
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(HERE, "shim"), HERE, ROOT])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-p", "coesim_shim", "-p", "no:cacheprovider", "-q", "-s",
         "--rootdir", str(work), str(work)],
        cwd=str(work), env=env, capture_output=True, text=True, timeout=900,
    )
    tail = proc.stdout[-4000:]
    assert proc.returncode == 0, tail + proc.stderr[-2000:]
    assert "190 passed" in proc.stdout, tail
    for criterion in range(1, 12):
        assert f"[criterion {criterion:02d}] PASS" in proc.stdout, tail
