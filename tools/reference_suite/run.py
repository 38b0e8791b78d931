"""Run the reference's own test suite (pkg/tests, 174 tests) against the drop-in.

    python tools/reference_suite/run.py [pytest args...]

The reference tests are not part of this repository: build() copies them from
/root/reference/pkg/tests into baseline/_ref_tests (git-ignored, shipped to
the GPU box with the reference install in baseline/_ref).  The plugin
dropin_plugin.py rebinds the reference's stage functions and types to the
drop-in (Option 2) before the tests are collected, so every
test that reaches zero_condense / rwmd / wcd / delta_condense / the split tree /
WSPD / emit_arcs / assemble / build_network / approx_w1 / nn_search /
exact_w1_dense runs the sm_100a kernels.  The summary (passed / failed /
skipped per file) is written to gpurun_out/reference_suite.json.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main(argv):
    tests = os.path.join(ROOT, "baseline", "_ref_tests")
    if not os.path.isdir(tests):
        tests = "/root/reference/pkg/tests"
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "w1flow")):
        ref = "/root/reference/pkg/src"
    out_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    junit = os.path.join(out_dir, "reference_suite.xml")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([HERE, ROOT, ref, tests, env.get("PYTHONPATH", "")])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", tests, "-p", "dropin_plugin", "-q", "-rfEs",
           "--junitxml", junit, "-o", "cache_dir=/tmp/ref_suite_cache", "--rootdir", tests] + argv
    rc = subprocess.call(cmd, env=env, cwd=tests)
    summary = {"rc": rc}
    try:
        import xml.etree.ElementTree as ET

        per_file = {}
        for case in ET.parse(junit).getroot().iter("testcase"):
            f = case.get("classname", "").split(".")[0]
            st = "passed"
            for tag in ("failure", "error", "skipped"):
                if case.find(tag) is not None:
                    st = tag
            per_file.setdefault(f, {}).setdefault(st, 0)
            per_file[f][st] += 1
        tot = {}
        for d in per_file.values():
            for k, v in d.items():
                tot[k] = tot.get(k, 0) + v
        summary.update(total=tot, per_file=per_file)
    except Exception as exc:  # noqa: BLE001
        summary["parse_error"] = repr(exc)
    with open(os.path.join(out_dir, "reference_suite.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary))
    return rc


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
