"""Native table parser (pg_table_parse, csrc/table_parse.cu) == the csv-module path ==
the reference loader (phenotypes.load_table, /root/reference/pkg/src/panelgwas/phenotypes.py:67-138)."""
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2604_21095_b200 import phenotypes
from paper_2604_21095_b200.errors import PanelGwasError

REF = Path("/root/reference/pkg/src")

TRICKY = ["1.5", " 2.25 ", "+3", "-0", "NA", "NaN", "nan", "-9", "-9.0", "-9e0", "", "  ", "1e-400", "4.9e-324",
          "1e400", "inf", "-Infinity", "NAN", "abc", "1.", ".5", "0x10", "1e", "--5", "+-5", "1e5", "007",
          "2.2250738585072014e-308", "1.7976931348623157e308", "1.7976931348623159e308", "0.1", "3.14159265358979323846"]


def _write(path: Path, text: str) -> Path:
    path.write_bytes(text.encode())
    return path


def _tables(path, **kw):
    native = phenotypes._load_table_native(path, kw.get("id_column", "IID"), kw.get("delimiter", "\t"))
    csvp = phenotypes._load_table_csv(path, kw.get("id_column", "IID"), kw.get("delimiter", "\t"))
    return native, csvp


def _same(a, b):
    assert a[0] == b[0] and a[1] == b[1]
    assert np.array_equal(a[2], b[2], equal_nan=True)
    assert np.array_equal(np.signbit(a[2]), np.signbit(b[2]))
    assert np.array_equal(a[3], b[3])


def test_tricky_cells_native_equals_csv(tmp_path):
    rows = ["FID\tIID\ty1\ty2"]
    for i, tok in enumerate(TRICKY):
        rows.append(f"f{i}\ts{i}\t{tok}\t{TRICKY[-1 - i]}")
    p = _write(tmp_path / "t.tsv", "\n".join(rows) + "\n")
    native, csvp = _tables(p)
    assert native is not None
    _same(native, csvp)
    t = phenotypes.load_table(p)
    assert t.unparseable_count.tolist() == csvp[3].tolist()
    assert t.values[TRICKY.index("-9.0"), 1] == -9.0 and np.isnan(t.values[TRICKY.index("-9"), 1])
    assert t.values[TRICKY.index("1e-400"), 1] == 0.0 and t.values[TRICKY.index("4.9e-324"), 1] == 5e-324


def test_crlf_blank_lines_and_no_trailing_newline(tmp_path):
    p = _write(tmp_path / "t.tsv", "IID\ta\tb\r\n\r\ns1\t1\t2\r\n\ns2\t3\tNA\r\ns3\t5\t6")
    native, csvp = _tables(p)
    assert native is not None
    _same(native, csvp)
    assert native[0] == ["s1", "s2", "s3"]


def test_ragged_row_line_number(tmp_path):
    p = _write(tmp_path / "t.tsv", "IID\ta\tb\ns1\t1\t2\n\ns2\t3\n")
    with pytest.raises(PanelGwasError, match=r":4: ragged row with 2 cells, header has 3"):
        phenotypes.load_table(p)
    with pytest.raises(PanelGwasError, match=r":4: ragged row with 2 cells, header has 3"):
        phenotypes._load_table_csv(p, "IID", "\t")


@pytest.mark.parametrize("text", ['IID\ta\n"s1"\t1\n', "IID\ta\nsé1\t1\n", "IID\ta\ns1\t1_000\n",
                                  "IID\ta\ns1\t1\rs2\t2\n"])
def test_generic_inputs_fall_back(tmp_path, text):
    p = _write(tmp_path / "t.tsv", text)
    assert phenotypes._load_table_native(p, "IID", "\t") is None
    t = phenotypes.load_table(p)
    assert t.n_rows >= 1


def test_other_delimiter_and_id_column(tmp_path):
    p = _write(tmp_path / "t.csv", "sample,x,y\nA,1,2\nB,,3\n")
    native, csvp = _tables(p, id_column="sample", delimiter=",")
    _same(native, csvp)


def test_random_table_matches_csv(tmp_path):
    rng = np.random.default_rng(4)
    n, p = 300, 57
    vals = rng.standard_normal((n, p)) * 10.0 ** rng.integers(-8, 8, (n, p))
    cells = np.array([[repr(float(v)) for v in row] for row in vals], dtype=object)
    cells[rng.random((n, p)) < 0.05] = "NA"
    lines = ["IID\t" + "\t".join(f"ph{j}" for j in range(p))]
    lines += [f"id{i}\t" + "\t".join(cells[i]) for i in range(n)]
    path = _write(tmp_path / "r.tsv", "\n".join(lines) + "\n")
    native, csvp = _tables(path)
    _same(native, csvp)


@pytest.mark.skipif(not REF.exists(), reason="reference tree not present")
def test_matches_reference_loader(tmp_path):
    rows = ["FID\tIID\ty1\ty2"]
    for i, tok in enumerate(TRICKY):
        rows.append(f"f{i}\ts{i}\t{tok}\t{TRICKY[-1 - i]}")
    p = _write(tmp_path / "t.tsv", "\n".join(rows) + "\n")
    sys.path.insert(0, str(REF))
    try:
        from panelgwas import phenotypes as ref
    finally:
        sys.path.remove(str(REF))
    want = ref.load_table(p)
    got = phenotypes.load_table(p)
    assert got.ids == want.ids and got.column_names == want.column_names
    assert np.array_equal(got.values, want.values, equal_nan=True)
    assert got.missing_count.tolist() == want.missing_count.tolist()
    assert got.unparseable_count.tolist() == want.unparseable_count.tolist()


def test_multithreaded_line_scan_native_equals_csv(tmp_path):
    """A body over 8 MB takes the threaded newline scan: chunk edges fall inside lines, CRLF
    and LF endings are mixed, blank lines keep the physical line numbers of a ragged row."""
    rng = np.random.default_rng(8)
    n, p = 2300, 400
    vals = rng.standard_normal((n, p))
    lines = ["IID\t" + "\t".join(f"p{j}" for j in range(p))]
    for i in range(n):
        end = "\r" if i % 3 == 0 else ""
        lines.append(f"S{i}\t" + "\t".join(repr(float(v)) for v in vals[i]) + end)
        if i % 97 == 0:
            lines.append("")
    text = "\n".join(lines) + "\n"
    assert len(text) > 9 << 20
    path = _write(tmp_path / "big.tsv", text)
    native, csvp = _tables(path)
    assert native is not None
    _same(native, csvp)
    assert np.array_equal(native[2], vals)
    # a ragged row deep in the file is reported with its physical line number by both readers
    lines[2000] = lines[2000] + "\t1.0"
    path = _write(tmp_path / "ragged.tsv", "\n".join(lines) + "\n")
    with pytest.raises(PanelGwasError, match=":2001: ragged row") as e1:
        phenotypes._load_table_native(path, "IID", "\t")
    with pytest.raises(PanelGwasError, match=":2001: ragged row") as e2:
        phenotypes._load_table_csv(path, "IID", "\t")
    assert str(e1.value) == str(e2.value)
