"""Recipe: package the reference (panelgwas 0.1.0, pure Python) as the CPU checker under
oracle/_ref/ — TEST / BASELINE INFRASTRUCTURE, not product code.

The reference has no native code to compile; its "build" is an importable
archive. This recipe zips, unmodified,

  /root/reference/pkg/src/panelgwas  ->  oracle/_ref/panelgwas_src.zip   (zipimport: sys.path entry)
  /root/reference/pkg/tests          ->  oracle/_ref/reference_tests.zip (the reference's own suite)

plus a MANIFEST.json of source digests. oracle/_ref/ is git-ignored (no reference source
enters the history) but not gpurun-ignored, so the archives travel to the GPU box, which has
no /root/reference. Users on the box:

  bench.py --impl reference         times the reference's own scan loop (engine._process_batch,
                                    PlinkSource.read_marker_batch, ThresholdWriter) on host cores
  oracle/run_reference_suite.py     runs the reference's test suite against the drop-in

Run: python oracle/make_ref.py   (also called by __graft_entry__.build() when /root/reference exists)
"""

from __future__ import annotations

import hashlib
import json
import sys
import zipfile
from pathlib import Path

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "_ref"
SRC_ZIP = OUT / "panelgwas_src.zip"
TESTS_ZIP = OUT / "reference_tests.zip"
MANIFEST = OUT / "MANIFEST.json"


def _files(root: Path) -> list[Path]:
    return sorted(p for p in root.rglob("*") if p.is_file() and "__pycache__" not in p.parts
                  and p.suffix in (".py", ".txt", ".md", ".toml"))


def _digest(files: list[Path], base: Path) -> str:
    h = hashlib.sha256()
    for p in files:
        h.update(str(p.relative_to(base)).encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def _zip(files: list[Path], base: Path, dest: Path) -> None:
    tmp = dest.with_suffix(".tmp")
    with zipfile.ZipFile(tmp, "w", zipfile.ZIP_DEFLATED) as z:
        for p in files:
            # fixed timestamps: the archive is a pure function of the sources
            info = zipfile.ZipInfo(str(p.relative_to(base)), date_time=(2020, 1, 1, 0, 0, 0))
            info.compress_type = zipfile.ZIP_DEFLATED
            z.writestr(info, p.read_bytes())
    tmp.replace(dest)


def make(force: bool = False) -> bool:
    """Build the archives if /root/reference is present and they are stale. Returns True if present."""
    if not (REF / "src" / "panelgwas").is_dir():
        return SRC_ZIP.exists() and TESTS_ZIP.exists()
    src_files = _files(REF / "src" / "panelgwas")
    test_files = _files(REF / "tests")
    manifest = {"reference": "panelgwas 0.1.0 (/root/reference/pkg)",
                "src_sha256": _digest(src_files, REF / "src"),
                "tests_sha256": _digest(test_files, REF),
                "src_files": len(src_files), "test_files": len(test_files)}
    if not force and MANIFEST.exists() and SRC_ZIP.exists() and TESTS_ZIP.exists():
        if json.loads(MANIFEST.read_text()) == manifest:
            return True
    OUT.mkdir(parents=True, exist_ok=True)
    _zip(src_files, REF / "src", SRC_ZIP)
    _zip(test_files, REF, TESTS_ZIP)
    MANIFEST.write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")
    return True


def import_reference():
    """The reference package from the archive (raises if the recipe has not run)."""
    if not SRC_ZIP.exists():
        raise FileNotFoundError(f"{SRC_ZIP} missing: run oracle/make_ref.py where /root/reference exists")
    if str(SRC_ZIP) not in sys.path:
        sys.path.insert(0, str(SRC_ZIP))
    import panelgwas  # noqa: F401  (the reference, from the zip)

    if not str(getattr(panelgwas, "__file__", "")).startswith(str(SRC_ZIP)):
        raise ImportError(f"panelgwas resolved to {panelgwas.__file__}, not the reference archive")
    return panelgwas


if __name__ == "__main__":
    ok = make(force="--force" in sys.argv)
    print(f"oracle/_ref: {'ready' if ok else 'reference not available'} ({OUT})")
