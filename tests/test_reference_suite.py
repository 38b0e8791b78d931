"""The reference's own test suite (pkg/tests, 174 tests) run against the
drop-in on the B200: tools/reference_suite/run.py rebinds w1flow's stage
functions and types to paper_2110_14734_b200 (INTEGRATION.md Option 2) before
the reference tests are collected.  The tests themselves ship next to the
reference install (baseline/_ref_tests, copied by build())."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_reference_suite_passes_on_the_dropin():
    tests = os.path.join(ROOT, "baseline", "_ref_tests")
    ref = os.path.join(ROOT, "baseline", "_ref", "w1flow")
    if not (os.path.isdir(tests) and os.path.isdir(ref)):
        pytest.skip("reference tests / install not present (run __graft_entry__.build() where the reference exists)")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "reference_suite", "run.py")],
                       capture_output=True, text=True, timeout=1500)
    summary = json.loads(r.stdout.strip().splitlines()[-1])
    tot = summary.get("total", {})
    assert r.returncode == 0, r.stdout[-4000:]
    assert tot.get("passed", 0) == 174 and not tot.get("failure") and not tot.get("error"), tot
