"""Native BGEN index + inflate (csrc/bgen_io.cu) on CPU: rows == Python-zlib inflate,
mixed 8/16-bit widening is exact, every validation error raises the reference's class and
message, and (when the reference tree is present) catalog + dosages equal
panelgwas.genotypes.bgen.BgenSource (/root/reference/pkg/src/panelgwas/genotypes/bgen.py)."""
import struct
import sys
import zlib
from pathlib import Path

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from oracle import scan_oracle as orc
from paper_2604_21095_b200.errors import FormatError, UnsupportedFeatureError

REF = Path("/root/reference/pkg/src")


def _cohort(m=40, n=37, seed=0):
    rng = np.random.default_rng(seed)
    d = rng.uniform(0, 2, (m, n))
    d[rng.random((m, n)) < 0.1] = np.nan
    d[::3] = np.round(d[::3])
    return d, [f"s{i}" for i in range(n)]


def _python_rows(path: Path, src) -> list[bytes]:
    """Inflate every block with Python's zlib (the reference's library call)."""
    blob = path.read_bytes()
    out = []
    for off, size in zip(src._offsets.tolist(), src._sizes.tolist()):
        data = zlib.decompress(blob[off + 4:off + size])
        n = struct.unpack("<I", data[:4])[0]
        bits = data[8 + n + 1]
        out.append((bits, data[10 + n:], data[8:8 + n]))
    return out


@pytest.mark.parametrize("bits", [8, 16])
def test_rows_equal_python_inflate(tmp_path, bits):
    from bgen_fixture import write_bgen

    d, ids = _cohort()
    p = write_bgen(tmp_path / "a.bgen", d, ids, bits=bits)
    with pg.BgenSource(p) as src:
        kind, rows, rb = src.read_raw_block(0, src.n_markers)
        want = _python_rows(p, src)
    n = len(ids)
    assert rb == n * (2 * bits // 8 + 1)
    for i, (b, probs, ploidy) in enumerate(want):
        assert b == bits
        assert rows[i, :len(probs)].tobytes() == probs and rows[i, len(probs):].tobytes() == ploidy


def test_mixed_precision_widens_exactly(tmp_path):
    from bgen_fixture import write_bgen

    d, ids = _cohort(m=6, n=11, seed=3)
    a = write_bgen(tmp_path / "a8.bgen", d, ids, bits=8).read_bytes()
    b = write_bgen(tmp_path / "b16.bgen", d, ids, bits=16).read_bytes()
    # splice: header + samples from a, then variants 0-2 of the 8-bit file and 3-5 of the 16-bit file
    with pg.BgenSource(tmp_path / "a8.bgen") as sa, pg.BgenSource(tmp_path / "b16.bgen") as sb:
        head = a[:sa._first_variant]
        ends_a = [o + s for o, s in zip(sa._offsets.tolist(), sa._sizes.tolist())]
        ends_b = [o + s for o, s in zip(sb._offsets.tolist(), sb._sizes.tolist())]
        starts_b = [sb._first_variant] + ends_b[:-1]
        mixed = head + a[sa._first_variant:ends_a[2]] + b[starts_b[3]:ends_b[5]]
    (tmp_path / "mix.bgen").write_bytes(mixed)
    with pg.BgenSource(tmp_path / "mix.bgen") as src:
        kind, rows, rb = src.read_raw_block(0, 6)
    assert kind == pg._native.PG_GENO_BGEN16 and rb == 5 * 11
    for i in range(6):
        probs = rows[i, :4 * 11].view("<u2")
        ploidy = rows[i, 4 * 11:]
        got = orc.decode_bgen(probs, ploidy, 16)
        with pg.BgenSource(tmp_path / ("a8.bgen" if i < 3 else "b16.bgen")) as one:
            _, r1, rb1 = one.read_raw_block(i, 1)
            bits1 = 8 if i < 3 else 16
            w = 2 * 11 * bits1 // 8
            ref = orc.decode_bgen(r1[0, :w].view("u1" if bits1 == 8 else "<u2"), r1[0, w:], bits1)
        assert np.array_equal(got, ref, equal_nan=True)  # bit-identical dosages


def _patch_block(tmp_path, mutate, name):
    """Re-compress variant 0's block after `mutate(data: bytearray) -> bytes`."""
    from bgen_fixture import write_bgen

    d, ids = _cohort(m=2, n=5, seed=1)
    p = write_bgen(tmp_path / f"{name}.bgen", d, ids)
    with pg.BgenSource(p) as src:
        off, size = int(src._offsets[0]), int(src._sizes[0])
    blob = bytearray(p.read_bytes())
    data = bytearray(zlib.decompress(bytes(blob[off + 4:off + size])))
    new = mutate(data)
    comp = struct.pack("<I", len(new)) + zlib.compress(bytes(new))
    out = bytes(blob[:off - 4]) + struct.pack("<I", len(comp)) + comp + bytes(blob[off + size:])
    q = tmp_path / f"{name}_x.bgen"
    q.write_bytes(out)
    return q


@pytest.mark.parametrize("name,mutate,exc,msg", [
    ("samples", lambda d: bytes(struct.pack("<I", 6) + d[4:]), FormatError, "sample count 6 != header 5"),
    ("alleles", lambda d: bytes(d[:4] + struct.pack("<H", 3) + d[6:]), UnsupportedFeatureError, "3 alleles in genotype"),
    ("ploidy", lambda d: bytes(d[:6] + bytes([1, 2]) + d[8:]), UnsupportedFeatureError, "ploidy range 1..2"),
    ("haploid", lambda d: bytes(d[:8] + bytes([1]) + d[9:]), UnsupportedFeatureError, "non-diploid"),
    ("size", lambda d: bytes(d + b"\x00"), FormatError, "genotype block is 26 bytes, expected 25"),
])
def test_validation_errors(tmp_path, name, mutate, exc, msg):
    q = _patch_block(tmp_path, mutate, name)
    with pg.BgenSource(q) as src:
        with pytest.raises(exc, match=msg):
            src.read_raw_block(0, 2)


def test_inflated_size_mismatch_and_short_block(tmp_path):
    from bgen_fixture import write_bgen

    d, ids = _cohort(m=2, n=5, seed=2)
    p = write_bgen(tmp_path / "s.bgen", d, ids)
    with pg.BgenSource(p) as src:
        off = int(src._offsets[0])
    blob = bytearray(p.read_bytes())
    blob[off:off + 4] = struct.pack("<I", 999)  # declared uncompressed length
    (tmp_path / "s2.bgen").write_bytes(bytes(blob))
    with pg.BgenSource(tmp_path / "s2.bgen") as src:
        with pytest.raises(FormatError, match="inflated to 25 bytes, expected 999"):
            src.read_raw_block(0, 1)


@pytest.mark.skipif(not REF.exists(), reason="reference tree not present")
def test_matches_reference_reader(tmp_path):
    from bgen_fixture import write_bgen

    sys.path.insert(0, str(REF))
    try:
        from panelgwas.genotypes.bgen import BgenSource as RefBgen
    finally:
        sys.path.remove(str(REF))
    for bits in (8, 16):
        d, ids = _cohort(m=25, n=33, seed=bits)
        p = write_bgen(tmp_path / f"r{bits}.bgen", d, ids, bits=bits)
        ref = RefBgen(p)
        with pg.BgenSource(p) as src:
            assert [vars(m) if hasattr(m, "__dict__") else m for m in src.marker_catalog] == \
                [vars(m) if hasattr(m, "__dict__") else m for m in ref.marker_catalog]
            kind, rows, rb = src.read_raw_block(0, 25)
        w = 2 * 33 * bits // 8
        want = ref.read_marker_batch(0, 25).dosages
        for i in range(25):
            got = orc.decode_bgen(rows[i, :w].view("u1" if bits == 8 else "<u2"), rows[i, w:], bits)
            assert np.array_equal(got, want[i], equal_nan=True)
        ref.close()


def test_bgen_catalog_ids_and_utf8(tmp_path):
    """The byte-backed BGEN catalog: id = rsid, else the variant id; UTF-8 identifiers and
    alleles survive into records and record prefixes."""
    import struct
    import zlib

    from paper_2604_21095_b200.genotypes.bgen import BgenSource

    n = 3

    def variant(vid, rsid, chrom, pos, a1, a2):
        data = struct.pack("<IHBB", n, 2, 2, 2) + bytes([2] * n) + bytes([0, 8]) + bytes([255, 0] * n)
        comp = zlib.compress(data)
        return (struct.pack("<H", len(vid)) + vid + struct.pack("<H", len(rsid)) + rsid + struct.pack("<H", len(chrom))
                + chrom + struct.pack("<IH", pos, 2) + struct.pack("<I", len(a1)) + a1 + struct.pack("<I", len(a2)) + a2
                + struct.pack("<II", len(comp) + 4, len(data)) + comp)

    body = [variant(b"v1", b"", b"1", 10, b"A", b"G"), variant(b"v2", b"rs2", "Xé".encode(), 20, b"AT", "α".encode()),
            variant(b"", b"", b"2", 30, b"C", b"T")]
    path = tmp_path / "u.bgen"
    path.write_bytes(struct.pack("<I", 20) + struct.pack("<III", 20, 3, n) + b"bgen" + struct.pack("<I", 1 | 2 << 2)
                     + b"".join(body))
    src = BgenSource(path, sample_ids=["a", "b", "c"])
    assert [(m.chrom, m.id, m.pos, m.allele1, m.allele2) for m in src.marker_catalog] == [
        ("1", "v1", 10, "A", "G"), ("Xé", "rs2", 20, "AT", "α"), ("2", "", 30, "C", "T")]
    assert src.marker_catalog[1:2].prefixes(False) == ["Xé\trs2\t20\tα\tAT\t"]
