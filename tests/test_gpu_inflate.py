"""GPU zlib inflate (csrc/inflate.cu) and compressed BGEN staging (pg_stage_bgen):
byte-identical to zlib.decompress over every DEFLATE block type / strategy, corrupt streams
rejected, and scans through the GPU-inflate path == the host-inflate path (bitwise) with
the reference reader's exceptions on bad blocks."""
import zlib

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from paper_2604_21095_b200 import _native
from paper_2604_21095_b200.errors import FormatError

pytestmark = pytest.mark.gpu


def _gpu_inflate(streams, out_stride=None, skip=0):
    blob = b"".join(streams)
    off = np.cumsum([0] + [len(s) for s in streams[:-1]]).astype(np.int64)
    size = np.array([len(s) for s in streams], dtype=np.int64)
    stride = out_stride or (max(1 << 16, 4 * max(len(s) for s in streams) * 16))
    out = np.zeros(len(streams) * stride, dtype=np.uint8)
    out_len = np.zeros(len(streams), dtype=np.int64)
    status = np.zeros(len(streams), dtype=np.int32)
    b = np.frombuffer(blob, dtype=np.uint8).copy()
    _native.call("pg_debug_inflate", b.ctypes.data, b.size, off.ctypes.data, size.ctypes.data, len(streams), skip,
                 out.ctypes.data, stride, out_len.ctypes.data, status.ctypes.data)
    return [(int(st), out[i * stride:i * stride + int(n)].tobytes()) for i, (st, n) in enumerate(zip(status, out_len))]


def _decoder_env(decoder, monkeypatch):
    """warp: a warp per stream (default); lanesN: N lanes per stream (32 / N streams per warp);
    tokens: the two-phase decoder."""
    if decoder == "tokens":
        monkeypatch.setenv("PG_INFLATE_MODE", "tokens")
    elif decoder.startswith("lanes"):
        monkeypatch.setenv("PG_INFLATE_LANES", decoder[5:])


def _payloads(rng):
    n = 23000
    g = rng.binomial(2, 0.3, n)
    hard = np.stack([np.where(g == 0, 255, 0), np.where(g == 1, 255, 0)], 1).astype(np.uint8).tobytes()
    frac = rng.integers(0, 256, 2 * n, dtype=np.uint8).tobytes()
    return [b"", b"a", b"abc" * 1000, bytes(range(256)) * 300, hard, frac, rng.bytes(70000),
            b"\x00" * 100000, (b"xy" * 7 + b"z") * 5000]


@pytest.mark.parametrize("level,strategy", [(0, zlib.Z_DEFAULT_STRATEGY), (1, zlib.Z_DEFAULT_STRATEGY),
                                            (6, zlib.Z_DEFAULT_STRATEGY), (9, zlib.Z_DEFAULT_STRATEGY),
                                            (6, zlib.Z_FIXED), (6, zlib.Z_RLE), (6, zlib.Z_HUFFMAN_ONLY),
                                            (6, zlib.Z_FILTERED)])
@pytest.mark.parametrize("decoder", ["warp", "lanes8", "lanes4", "tokens"])
def test_matches_zlib(level, strategy, decoder, monkeypatch):
    """Both GPU decoders (warp per stream; two-phase tokens, PG_INFLATE_MODE=tokens) == zlib."""
    _decoder_env(decoder, monkeypatch)
    rng = np.random.default_rng(level * 10 + strategy)
    data = _payloads(rng)
    streams = []
    for d in data:
        c = zlib.compressobj(level, zlib.DEFLATED, 15, 9, strategy)
        streams.append(c.compress(d) + c.flush())
    got = _gpu_inflate(streams, out_stride=1 << 17)
    for (st, out), d in zip(got, data):
        assert st == 0 and out == d


@pytest.mark.parametrize("decoder", ["warp", "lanes8", "lanes4", "tokens"])
def test_many_streams_and_multiple_blocks(decoder, monkeypatch):
    _decoder_env(decoder, monkeypatch)
    rng = np.random.default_rng(7)
    data = [rng.integers(0, 3, rng.integers(1, 200000), dtype=np.uint8).tobytes() for _ in range(200)]
    streams = []
    for i, d in enumerate(data):
        c = zlib.compressobj(6)
        # flushes inside the stream force several blocks, incl. empty stored ones (Z_SYNC_FLUSH)
        mid = len(d) // 3
        streams.append(c.compress(d[:mid]) + c.flush(zlib.Z_SYNC_FLUSH) + c.compress(d[mid:]) + c.flush())
    got = _gpu_inflate(streams, out_stride=200000)
    for (st, out), d in zip(got, data):
        assert st == 0 and out == d


@pytest.mark.parametrize("decoder", ["warp", "lanes8", "lanes4", "tokens"])
def test_corrupt_streams_rejected(decoder, monkeypatch):
    _decoder_env(decoder, monkeypatch)
    good = zlib.compress(b"hello world " * 500)
    bad_header = b"\x78\x9d" + good[2:]                            # FCHECK wrong
    bad_sum = good[:-1] + bytes([good[-1] ^ 1])                     # Adler-32 mismatch
    truncated = good[: len(good) // 2]
    bad_type = b"\x78\x9c" + bytes([0x07]) + good[3:]               # BTYPE = 3
    got = _gpu_inflate([good, bad_header, bad_sum, truncated, bad_type], out_stride=1 << 14)
    assert got[0] == (0, b"hello world " * 500)
    for st, _ in got[1:]:
        assert st != 0
    # output larger than the stride
    assert _gpu_inflate([good], out_stride=100)[0][0] != 0


def _bgen_dataset(tmp_path, bits, m=300, n=160, seed=0, missing=0.05):
    from bgen_fixture import write_bgen
    from conftest_helpers import write_tsv

    rng = np.random.default_rng(seed)
    d = rng.uniform(0, 2, (m, n))
    d[::4] = np.round(d[::4])
    d[rng.random((m, n)) < missing] = np.nan
    d[7] = 1.0  # monomorphic
    ids = [f"S{i + 1}" for i in range(n)]
    p = write_bgen(tmp_path / f"g{bits}.bgen", d, ids, bits=bits)
    y = rng.standard_normal((n, 5))
    y[:, 1] += 0.5 * np.nan_to_num(d[11], nan=1.0)
    pheno = write_tsv(tmp_path / "pheno.tsv", ids, [f"ph{j}" for j in range(5)], y)
    return pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=p), pheno


def _scan(spec, pheno, out, **kw):
    return pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, out_path=out, p_threshold=1.0,
                                     summary_to_stderr=False, precision=pg.Precision.F64, device_batch=64, **kw))


@pytest.mark.parametrize("bits", [8, 16])
def test_scan_gpu_inflate_equals_host_inflate(tmp_path, bits, monkeypatch):
    spec, pheno = _bgen_dataset(tmp_path, bits)
    _scan(spec, pheno, tmp_path / "gpu.tsv")
    monkeypatch.setenv("PANELGWAS_HOST_INFLATE", "1")
    _scan(spec, pheno, tmp_path / "host.tsv")
    assert (tmp_path / "gpu.tsv").read_bytes() == (tmp_path / "host.tsv").read_bytes()


def test_stage_bgen_errors_match_host(tmp_path):
    import struct

    spec, pheno = _bgen_dataset(tmp_path, 8, m=20, n=40)
    with pg.BgenSource(spec.bgen_path) as src:
        off = int(src._offsets[5])
    blob = bytearray(spec.bgen_path.read_bytes())
    bad = bytearray(blob)
    bad[off:off + 4] = struct.pack("<I", 77)  # declared uncompressed length
    (tmp_path / "len.bgen").write_bytes(bytes(bad))
    bad = bytearray(blob)
    bad[off + 10] ^= 0xFF  # inside the deflate stream
    (tmp_path / "z.bgen").write_bytes(bytes(bad))
    for name, exc, msg in (("len.bgen", FormatError, "expected 77"), ("z.bgen", FormatError, "zlib|inflated")):
        s = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=tmp_path / name)
        with pytest.raises(exc, match=msg):
            _scan(s, pheno, tmp_path / f"{name}.tsv")


def test_stage_bgen_mixed_precision(tmp_path, monkeypatch):
    """8-bit and 16-bit blocks in one batch: widened on the device, same output as the host path."""
    from bgen_fixture import write_bgen
    from conftest_helpers import write_tsv

    rng = np.random.default_rng(5)
    n = 50
    d = rng.uniform(0, 2, (12, n))
    ids = [f"S{i + 1}" for i in range(n)]
    a = write_bgen(tmp_path / "a.bgen", d, ids, bits=8).read_bytes()
    b = write_bgen(tmp_path / "b.bgen", d, ids, bits=16).read_bytes()
    with pg.BgenSource(tmp_path / "a.bgen") as sa, pg.BgenSource(tmp_path / "b.bgen") as sb:
        ends_a = [o + s for o, s in zip(sa._offsets.tolist(), sa._sizes.tolist())]
        ends_b = [o + s for o, s in zip(sb._offsets.tolist(), sb._sizes.tolist())]
        mixed = a[:ends_a[5]] + b[ends_b[5]:]
    (tmp_path / "mix.bgen").write_bytes(mixed)
    pheno = write_tsv(tmp_path / "p.tsv", ids, ["q1", "q2"], rng.standard_normal((n, 2)))
    spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=tmp_path / "mix.bgen")
    _scan(spec, pheno, tmp_path / "gpu.tsv")
    monkeypatch.setenv("PANELGWAS_HOST_INFLATE", "1")
    _scan(spec, pheno, tmp_path / "host.tsv")
    assert (tmp_path / "gpu.tsv").read_bytes() == (tmp_path / "host.tsv").read_bytes()


def test_bgen_keep_subset_and_odd_sizes(tmp_path, monkeypatch):
    """GPU-inflate path with excluded samples (keep list), an odd sample count, a single
    phenotype and a batch size that does not divide M: identical to the host-inflate path
    and to the oracle-level reference goldens' invariants (AF / missing bit-exact)."""
    from bgen_fixture import write_bgen
    from conftest_helpers import write_tsv

    rng = np.random.default_rng(13)
    n, m = 77, 53
    ids = [f"S{i + 1}" for i in range(n)]
    d = rng.uniform(0, 2, (m, n))
    d[rng.random(d.shape) < 0.08] = np.nan
    spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=write_bgen(tmp_path / "g.bgen", d, ids, bits=16))
    pheno = write_tsv(tmp_path / "p.tsv", ids, ["only"], rng.standard_normal((n, 1)))
    keep = tmp_path / "keep.txt"
    keep.write_text("\n".join(ids[::2] + ids[5:9]) + "\n")
    kw = dict(source=spec, pheno_path=pheno, p_threshold=1.0, precision=pg.Precision.F64, summary_to_stderr=False,
              device_batch=17, keep_path=keep)
    s1 = pg.run_scan(pg.ScanConfig(out_path=tmp_path / "gpu.tsv", **kw))
    monkeypatch.setenv("PANELGWAS_HOST_INFLATE", "1")
    s2 = pg.run_scan(pg.ScanConfig(out_path=tmp_path / "host.tsv", **kw))
    assert (tmp_path / "gpu.tsv").read_bytes() == (tmp_path / "host.tsv").read_bytes()
    assert s1.markers_scanned == s2.markers_scanned == m
    recs = pg.load_association_records(tmp_path / "gpu.tsv")
    kept = sorted(set(range(0, n, 2)) | set(range(5, 9)))
    for r in recs[:10]:
        i = int(r.id[2:]) - 1
        row = d[i, kept]
        assert r.missing_count == int(np.isnan(row).sum())
