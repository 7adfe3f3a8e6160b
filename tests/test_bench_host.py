"""bench.py host-side contract (no GPU): the reference arm runs the reference's own scan loop
from oracle/_ref and prints one JSON line; strong / weak shard shapes."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def test_reference_arm_json_line():
    from oracle import ref_scan_loop

    if not ref_scan_loop.available():
        pytest.skip("oracle/_ref not built (oracle/make_ref.py needs /root/reference)")
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--samples", "400", "--phenotypes", "48",
                          "--steps", "2", "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "tests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["n_markers_total"] == 1_000_000 and d["scaling"] == "strong"


def test_reference_loop_matches_oracle_hits(tmp_path):
    """The reference loop's records == the oracle's threshold scan of the same sample."""
    from oracle import ref_scan_loop, scan_oracle as orc

    if not ref_scan_loop.available():
        pytest.skip("oracle/_ref not built")
    loop = ref_scan_loop.ReferenceScanLoop(300, 16, 600, 0.05, seed=9, batch_size=256, workers=2, workdir=tmp_path)
    out = loop.step()
    raw = loop.source.read_marker_batch(0, 600)
    want = orc.threshold_scan(raw.dosages, loop.prep.ytil, loop.prep.df, 0.05)
    loop.close()
    assert out["records"] == want["rows"].size


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_rank_spans_cover_job(world):
    import bench

    for argv in (["--total-markers", "1000000"], ["--workload", "c4"], ["--markers-per-gpu", "4096"]):
        sys.argv = ["bench.py", *argv]
        a = bench.parse_args()
        spans = [bench.rank_span(a, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == bench.job_markers(a, world)
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        if not a.markers_per_gpu:
            assert all(s % 256 == 0 for s, _ in spans)
    sys.argv = ["bench.py", "--workload", "c4"]
    assert bench.job_markers(bench.parse_args(), 8) == 8_900_000
