"""The reference's own test suite (panelgwas 0.1.0, 228 tests) run unmodified against the
drop-in on the B200 (tests/refsuite/run_reference_suite.py). Every test must pass except the
individually justified exclusions in run_reference_suite.EXCLUDED."""
import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_reference_suite_passes_against_drop_in(tmp_path):
    import sys

    sys.path.insert(0, str(ROOT / "tests" / "refsuite"))
    import run_reference_suite as rs

    if not rs.ARCHIVE.exists():
        pytest.skip("oracle/_ref/reference_tests.zip not built (oracle/make_ref.py needs /root/reference)")
    out = ROOT / "gpurun_out" / "refsuite.json"
    s = rs.run(out, [])
    print(json.dumps({k: s[k] for k in ("passed", "failed", "error", "skipped", "deselected")}))
    assert s["failures"] == [], s["log_tail"]
    assert s["passed"] + len(rs.EXCLUDED) == 228, s["summary_line"]
