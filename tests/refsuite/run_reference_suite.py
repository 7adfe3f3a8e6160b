#!/usr/bin/env python
"""Run the reference's own test suite (panelgwas 0.1.0, /root/reference/pkg/tests: 228 tests)
against the B200 drop-in — TEST INFRASTRUCTURE.

The suite comes from oracle/_ref/reference_tests.zip (built by oracle/make_ref.py where
/root/reference exists; the GPU box has only the archive). It is extracted unmodified into a
temporary directory and run with `panelgwas` resolving to tests/refsuite/shim (an alias of
paper_2604_21095_b200), so every test exercises the drop-in's names, signatures, messages,
exit codes and outputs on the GPU.

Tests excluded by design are listed in EXCLUDED with the reason for each; everything else
must pass. Writes a JSON summary (counts, failures, exclusions) to --json.

  python tests/refsuite/run_reference_suite.py [--json out.json] [-- extra pytest args]
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys
import tempfile
import zipfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
SHIM = Path(__file__).resolve().parent / "shim"
ARCHIVE = ROOT / "oracle" / "_ref" / "reference_tests.zip"

# node id -> why it cannot hold for the drop-in (each justified individually); round 1's one
# exclusion (test_engine.py::...::test_paper_df_matches_simple_ols_without_covariates, |t - OLS t|
# <= 1e-8 in F64 mode) is met since Precision.F64 runs the two-level (~46-bit) panel
EXCLUDED: dict[str, str] = {}


def run(json_out: Path | None, extra: list[str]) -> dict:
    if not ARCHIVE.exists():
        raise SystemExit(f"{ARCHIVE} missing: run oracle/make_ref.py where /root/reference exists")
    with tempfile.TemporaryDirectory(prefix="refsuite_") as tmp:
        tmp = Path(tmp)
        with zipfile.ZipFile(ARCHIVE) as z:
            z.extractall(tmp)
        tests = tmp / "tests"
        env = dict(os.environ)
        env["PYTHONPATH"] = os.pathsep.join([str(SHIM), str(ROOT), env.get("PYTHONPATH", "")]).rstrip(os.pathsep)
        junit = tmp / "junit.xml"
        cmd = [sys.executable, "-m", "pytest", str(tests), "-q", "-p", "no:cacheprovider", "-rfE",
               f"--junitxml={junit}", "--rootdir", str(tmp)]
        for node in EXCLUDED:
            cmd += ["--deselect", f"tests/{node}"]
        proc = subprocess.run(cmd + extra, cwd=tmp, env=env, capture_output=True, text=True)
        out = proc.stdout + proc.stderr
        summary = {"returncode": proc.returncode, "excluded": EXCLUDED}
        tail = out.strip().splitlines()[-1] if out.strip() else ""
        for key in ("passed", "failed", "error", "errors", "skipped", "deselected"):
            m = re.search(rf"(\d+) {key}\b", tail)
            summary[key] = int(m.group(1)) if m else 0
        summary["failures"] = sorted(set(re.findall(r"^(?:FAILED|ERROR) (\S+)", out, re.M)))
        summary["summary_line"] = tail
        summary["log_tail"] = out[-6000:]
    if json_out:
        json_out.parent.mkdir(parents=True, exist_ok=True)
        json_out.write_text(json.dumps(summary, indent=1) + "\n")
    return summary


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", type=Path, default=None)
    ap.add_argument("extra", nargs="*")
    a = ap.parse_args()
    s = run(a.json, a.extra)
    print(s["summary_line"])
    for f in s["failures"]:
        print("FAILED", f)
    return 0 if s["returncode"] == 0 else 1


if __name__ == "__main__":
    raise SystemExit(main())
