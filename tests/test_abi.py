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


def test_native_float_repr_matches_python():
    import ctypes

    import numpy as np

    from paper_2604_21095_b200 import _native

    rng = np.random.default_rng(11)
    vals = np.concatenate([
        rng.standard_normal(2000) * 10.0 ** rng.integers(-30, 30, 2000),
        np.array([0.0, -0.0, 1.0, -1.0, 1e16, 1e17, 9999999999999998.0, 1e-4, 1e-5, 0.0001234, 123456789.0,
                  5e-324, 1.7976931348623157e308, 2.2250738585072014e-308, np.inf, -np.inf, np.nan, 0.1, 1 / 3]),
        rng.random(2000),
    ])
    cap = vals.size * 40
    out = ctypes.create_string_buffer(cap)
    n = ctypes.c_int64(0)
    _native.call("pg_format_float_repr", vals.ctypes.data, vals.size, out, cap, ctypes.byref(n))
    got = out.raw[:n.value].decode().split("\n")[:-1]
    assert got == [repr(float(v)) for v in vals]


def test_native_tsv_lines_match_python_formatting():
    import numpy as np

    import paper_2604_21095_b200 as pg
    from paper_2604_21095_b200 import output

    rng = np.random.default_rng(5)
    markers = [pg.MarkerRecord(str(1 + i % 3), f"rs{i}", 100 * i + 1, "A", "GT", i) for i in range(7)]
    names = ["height", "bmi_z", "phéno"]
    fmt = output._RecordText(812.0, 815, False, names)
    rows = rng.integers(0, 7, 50)
    cols = rng.integers(0, 3, 50)
    r, t, p = rng.standard_normal(50) / 10, rng.standard_normal(50) * 5, rng.random(50) ** 8
    af = rng.random(7)
    miss = rng.integers(0, 9, 7)
    text = output.format_records(markers, af, miss, rows, cols, r, t, p, fmt.pheno_blob, fmt.pheno_off, fmt.mid, False)
    want = "".join(fmt.python_line(markers[i], af[i], int(miss[i]), names[j], r[k], t[k], p[k])
                   for k, (i, j) in enumerate(zip(rows.tolist(), cols.tolist())))
    assert text == want


def test_native_tsv_lines_threaded_equal_serial():
    """Above 32,768 records pg_format_tsv formats chunks on host threads and concatenates them:
    the text equals the serial formatting of the same records (small calls), byte for byte."""
    import numpy as np

    import paper_2604_21095_b200 as pg
    from paper_2604_21095_b200 import output

    rng = np.random.default_rng(8)
    markers = [pg.MarkerRecord(str(1 + i % 22), f"rs{i}", 1000 * i + 1, "A", "GT", i) for i in range(500)]
    names = [f"ph{j}" for j in range(40)]
    fmt = output._RecordText(812.0, 815, True, names)
    n = 70_001
    rows, cols = rng.integers(0, 500, n), rng.integers(0, 40, n)
    r, t, p = rng.standard_normal(n) / 10, rng.standard_normal(n) * 5, rng.random(n) ** 8
    af, miss = rng.random(500), rng.integers(0, 9, 500)
    whole = output.format_records_bytes(markers, af, miss, rows, cols, r, t, p, fmt.pheno_blob, fmt.pheno_off,
                                        fmt.mid, True)
    step = 20_000
    parts = b"".join(output.format_records_bytes(markers, af, miss, rows[a:a + step], cols[a:a + step], r[a:a + step],
                                                 t[a:a + step], p[a:a + step], fmt.pheno_blob, fmt.pheno_off, fmt.mid,
                                                 True) for a in range(0, n, step))
    assert whole == parts and whole.count(b"\n") == n


def test_full_writer_marker_sidecar_matches_python_formatting(tmp_path, monkeypatch):
    """FullMatrixWriter renders <out>.markers.tsv natively (pg_format_marker_lines); the lines
    equal the reference's per-marker f-string with repr() floats, skipped markers omitted."""
    import numpy as np

    import paper_2604_21095_b200 as pg
    from paper_2604_21095_b200 import output

    monkeypatch.setattr(output, "_WRITE_CHUNK", 20)  # exercise the parallel pwrite split
    rng = np.random.default_rng(11)
    m, p = 9, 3
    markers = tuple(pg.MarkerRecord(str(1 + i % 2), f"rs{i}", 10 * i + 7, "AC", "T", 100 + i) for i in range(m))
    af = np.r_[rng.random(m - 2), 0.5, 1.0 / 3.0]
    miss = rng.integers(0, 5, m)
    skip = np.zeros(m, np.int8)
    skip[[2, 5]] = 1
    t_rows = rng.standard_normal((m - 2, p)).astype(np.float32)
    w = output.FullMatrixWriter(tmp_path / "f.bin", np.float32, 10.0, 12, False, ["a", "b", "c"])
    w.emit(output.BatchStats(markers=markers, allele_frequency=af, missing_count=miss, skip_reason=skip,
                             clamp_count=0, t_rows=t_rows))
    w.finalize()
    t, lines, names = output.read_full_matrix(tmp_path / "f.bin")
    want = [f"{mk.source_index}\t{mk.chrom}\t{mk.id}\t{mk.pos}\t{mk.allele2}\t{mk.allele1}\t{repr(float(af[i]))}\t"
            f"{int(miss[i])}" for i, mk in enumerate(markers) if not skip[i]]
    assert lines == want
    assert names == ["a", "b", "c"]
    assert np.array_equal(t, t_rows)


def test_topk_merge_matches_lexsort():
    """pg_topk_merge (threaded above 65,536 records) against a lexsort of held ++ fresh by
    (phenotype, p, source index) cut to k per phenotype — with p ties, k = 1, empty sides and
    phenotypes that have no records."""
    import ctypes

    import numpy as np

    from paper_2604_21095_b200 import _native

    rng = np.random.default_rng(3)
    for n_pheno, k, n_held_raw, n_fresh in ((5, 1, 0, 40), (300, 7, 1500, 90_000), (64, 3, 400, 0), (1, 4, 9, 9)):
        def draw(n, src0):
            col = rng.integers(0, max(1, n_pheno - 1), n)  # the last phenotype stays empty
            p = np.where(rng.random(n) < 0.3, 0.5, rng.random(n))  # ties
            return col.astype(np.int64), p, (src0 + rng.permutation(n)).astype(np.int64)

        hc, hp, hs = draw(n_held_raw, 0)
        order = np.lexsort((hs, hp, hc))
        hc, hp, hs = hc[order], hp[order], hs[order]
        rank = np.arange(hc.size) - np.searchsorted(hc, hc, side="left")
        keep = rank < k  # a valid held state: at most k per phenotype
        hc, hp, hs = hc[keep], hp[keep], hs[keep]
        fc, fp, fs = draw(n_fresh, 10**9)  # every candidate after every held record
        allc, allp, alls = np.concatenate([hc, fc]), np.concatenate([hp, fp]), np.concatenate([hs, fs])
        order = np.lexsort((alls, allp, allc))
        r = np.arange(order.size) - np.searchsorted(allc[order], allc[order], side="left")
        want = order[r < k]
        out = np.empty(n_pheno * k, dtype=np.int64)
        n_out = ctypes.c_int64(0)
        arrs = [np.ascontiguousarray(a) for a in (hc, hp, hs, fc, fp, fs)]
        _native.call("pg_topk_merge", n_pheno, k, arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data,
                     hc.size, arrs[3].ctypes.data, arrs[4].ctypes.data, arrs[5].ctypes.data, fc.size,
                     out.ctypes.data, ctypes.byref(n_out))
        assert np.array_equal(out[:n_out.value], want), (n_pheno, k)
