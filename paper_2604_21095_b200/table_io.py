"""Delimited-table readers behind `phenotypes.load_table`.

Two readers with identical results (tests/test_table_parse.py checks them against each other):

* `read_native` — mmap the file and hand the body to the multi-threaded native parser
  (pg_table_parse, csrc/table_parse.cu). It accepts the plain byte grammar (ASCII, no quotes,
  LF / CRLF line ends) and answers PG_TABLE_GENERIC for anything else;
* `read_generic` — the csv module, for quoted cells, bare CR, non-ASCII text and the remaining
  corners of float() syntax.

Cell rules follow the reference loader (/root/reference/pkg/src/panelgwas/phenotypes.py:52-120):
cells are stripped; "", NA, NaN, nan and -9 are missing; anything float() rejects, and any
non-finite value, is missing and counted per column as unparseable; blank lines are skipped;
a row whose cell count differs from the header's is an error.
"""

from __future__ import annotations

import csv
import mmap
import os
from ctypes import byref, c_int64
from pathlib import Path

import numpy as np

from .errors import PanelGwasError

MISSING_TOKENS = frozenset({"", "NA", "NaN", "nan", "-9"})

# (ids, value column names, values [rows, cols], unparseable per column, missing per column or None)
Parsed = tuple


def _id_position(path: Path, header: list[str], id_column: str) -> tuple[list[str], int]:
    cols = [h.strip() for h in header]
    try:
        return cols, cols.index(id_column)
    except ValueError:
        raise PanelGwasError(f"{path}: header has no {id_column!r} column (columns: {', '.join(cols)})") from None


def _ragged(path: Path, lineno: int, cells: int, width: int) -> PanelGwasError:
    return PanelGwasError(f"{path}:{lineno}: ragged row with {cells} cells, header has {width}")


# --- native reader -----------------------------------------------------------------------------


def read_native(path: Path, id_column: str, delimiter: str) -> Parsed | None:
    """Parse with pg_table_parse; None when the file needs the generic reader."""
    if len(delimiter) != 1 or not delimiter.isascii() or delimiter in "\"\r\n":
        return None
    size = path.stat().st_size
    if size == 0:
        raise PanelGwasError(f"{path}: empty file, expected a header row")
    with open(path, "rb") as fh, mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ) as mm:
        eol = mm.find(b"\n")
        first = mm[: size if eol < 0 else eol].removesuffix(b"\r")
        if not first or not first.isascii() or any(c in first for c in (b'"', b"\r", b"\x00")):
            return None
        header, at = _id_position(path, first.decode().split(delimiter), id_column)
        view = np.frombuffer(mm, dtype=np.uint8)
        try:
            body = _native_body(path, mm, view.ctypes.data, size, size if eol < 0 else eol + 1, len(header), at,
                                delimiter)
        finally:
            del view  # drop the buffer export before the mmap closes
    if body is None:
        return None
    ids, values, bad, missing = body
    return ids, header[:at] + header[at + 1:], values, bad, missing


def _native_body(path: Path, mm, addr: int, size: int, body_at: int, width: int, at: int, delimiter: str):
    """Two calls of pg_table_parse: count rows, then fill (values, ID spans, per-column counts)."""
    from . import _native

    lib = _native.load_library()
    rows, err_line, err_cells = c_int64(0), c_int64(0), c_int64(0)
    # leave two cores to the CUDA context creation that runs concurrently (engine.run_scan)
    threads = max(1, (os.cpu_count() or 4) - 2)
    fixed = (addr, size, body_at, delimiter.encode(), width, at, threads, 2)

    def run(*outputs) -> bool:
        status = lib.pg_table_parse(*fixed, byref(rows), *outputs, byref(err_line), byref(err_cells))
        if status == _native.PG_TABLE_GENERIC:
            return False
        if status == _native.PG_ERR_FORMAT and err_line.value:
            raise _ragged(path, err_line.value, err_cells.value, width)
        _native.check(status)
        return True

    if not run(None, None, None, None, None):
        return None
    n, k = rows.value, width - 1
    values = np.empty((n, k))
    starts, lengths = np.empty(n, np.int64), np.empty(n, np.int64)
    missing, bad = np.zeros(k, np.int64), np.zeros(k, np.int64)
    if not run(values.ctypes.data, starts.ctypes.data, lengths.ctypes.data, missing.ctypes.data, bad.ctypes.data):
        return None
    ids = [mm[s:s + ln].decode() for s, ln in zip(starts.tolist(), lengths.tolist())]
    return ids, values, bad, missing


# --- generic reader ----------------------------------------------------------------------------


def _cell_value(text: str) -> tuple[float, int]:
    """(value, 1 if the cell counts as unparseable) of a stripped cell."""
    if text in MISSING_TOKENS:
        return np.nan, 0
    try:
        v = float(text)
    except ValueError:
        return np.nan, 1
    return (v, 0) if np.isfinite(v) else (np.nan, 1)


def read_generic(path: Path, id_column: str, delimiter: str) -> Parsed:
    """csv-module reader (missing counts are left to the caller: last tuple entry None)."""
    with open(path, newline="") as fh:
        reader = csv.reader(fh, delimiter=delimiter)
        header_row = next(reader, None)
        if header_row is None:
            raise PanelGwasError(f"{path}: empty file, expected a header row")
        header, at = _id_position(path, header_row, id_column)
        width = len(header)
        ids: list[str] = []
        body: list[list[str]] = []
        for lineno, row in enumerate(reader, start=2):
            if not row:
                continue
            if len(row) != width:
                raise _ragged(path, lineno, len(row), width)
            ids.append(row.pop(at).strip())
            body.append(row)
    names = header[:at] + header[at + 1:]
    values = np.empty((len(body), len(names)))
    bad = np.zeros(len(names), dtype=np.int64)
    for i, row in enumerate(body):
        for j, cell in enumerate(row):
            values[i, j], flag = _cell_value(cell.strip())
            bad[j] += flag
    return ids, names, values, bad, None
