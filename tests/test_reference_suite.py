"""Regression gate: the reference's own test suite (229 tests, pkg/tests) runs
against the installed moeplan in baseline/_ref — the planner/simulator/cost
model this executor plugs into must be unchanged.  Expected: 228 pass and the
one documented failure, acceptance criterion 8a (mathematically unattainable,
pkg/README.md:55-64, pkg/test_output.txt:241-268).  Skipped where
/root/reference is absent (e.g. the GPU box)."""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference sources not present")
def test_reference_suite_unchanged():
    env = dict(os.environ)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["PYTHONPATH"] = f"{ROOT / 'baseline' / '_ref'}:{REF_TESTS}"
    res = subprocess.run([sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-q", str(REF_TESTS)],
                         capture_output=True, text=True, env=env, cwd="/tmp", timeout=900)
    tail = res.stdout.strip().splitlines()[-1]
    m = re.search(r"(\d+) failed, (\d+) passed", tail)
    assert m, res.stdout[-2000:]
    assert (int(m.group(1)), int(m.group(2))) == (1, 228), tail
    assert "test_criterion_8a_quantization_cosine_all_seeds" in res.stdout
