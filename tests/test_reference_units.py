"""The reference's own doctest units (proj/tests/test_*.cpp, compiled in place
against the in-repo Eigen/doctest shims by oracle/Makefile) — evidence that
the shimmed reference, the source of tests/golden, behaves as the real one."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_unit_suite_passes_under_shim(tmp_path):
    r = subprocess.run([BIN], cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "60 run, 0 failed" in r.stdout
