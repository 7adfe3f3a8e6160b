"""The C-ABI library loads without a GPU and exports every entry point that
include/panelgwas_b200.h declares (no compute calls here)."""
import re
from pathlib import Path

import pytest

from paper_2604_21095_b200 import _native

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols() -> set[str]:
    text = (ROOT / "include" / "panelgwas_b200.h").read_text()
    return set(re.findall(r"^PG_API\s+[\w\s\*]+?\b(pg_\w+)\s*\(", text, flags=re.M))


def test_header_declares_entry_points():
    names = declared_symbols()
    assert {"pg_ctx_create", "pg_scan", "pg_fetch_candidates", "pg_p_from_t"} <= names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    missing = [n for n in sorted(declared_symbols()) if getattr(lib, n, None) is None]
    assert not missing, missing


def test_python_binding_covers_header():
    assert declared_symbols() == set(_native.SIGNATURES)


def test_error_string_and_version_without_gpu():
    lib = _native.load_library()
    assert lib.pg_abi_version() >= 1
    assert isinstance(lib.pg_last_error(), bytes)


def test_status_mapping():
    from paper_2604_21095_b200.errors import ConfigError, FormatError, PanelGwasError

    _native.load_library()
    with pytest.raises(ValueError):
        _native.check(_native.PG_ERR_INVALID)
    with pytest.raises(FormatError):
        _native.check(_native.PG_ERR_FORMAT)
    with pytest.raises(ConfigError):
        _native.check(_native.PG_ERR_CONFIG)
    with pytest.raises(PanelGwasError):
        _native.check(_native.PG_ERR_CUDA)


def test_sm100a_only_binary():
    import subprocess

    so = _native.LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass  # tcgen05.mma kind::i8
    assert "UTMALDG" in sass  # TMA tile loads
    assert "LDTM" in sass     # tcgen05.ld
