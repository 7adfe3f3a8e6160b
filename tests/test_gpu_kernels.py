"""Device kernels behind the library API vs golden reference outputs and the oracle.

Bit-exact: genotype decode (PLINK / BGEN), missing counts, skip flags.
Tolerance (fp64 libm differences only): p-values, t, prepare, correlate."""
from pathlib import Path

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from oracle import scan_oracle as orc

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def nan_eq(a, b):
    return np.array_equal(np.nan_to_num(a, nan=-7.0), np.nan_to_num(b, nan=-7.0))


def test_decode_bed_codes_bit_exact():
    g = np.load(GOLD / "decode.npz")
    for i in range(6):
        got = pg.decode_bed_codes(g[f"fixed{i}_bytes"].tobytes(), int(g[f"fixed{i}_n"]))
        assert nan_eq(got, g[f"fixed{i}_dosage"])
    n = int(g["rand_n"])
    for i in range(g["rand_packed"].shape[0]):
        assert nan_eq(pg.decode_bed_codes(g["rand_packed"][i].tobytes(), n), g["rand_dosage"][i])
    with pytest.raises(pg.FormatError):
        pg.decode_bed_codes(b"\x00\x00", 4)


def test_plink_reader_round_trip(tmp_path):
    rng = np.random.default_rng(77)
    for case in range(20):
        m, n = int(rng.integers(1, 17)), int(rng.integers(1, 26))
        d = rng.integers(0, 3, size=(m, n)).astype(np.float64)
        d[rng.random((m, n)) < 0.15] = np.nan
        pg.write_bed_trio(tmp_path / f"rt{case}", d, [f"I{j}" for j in range(n)])
        src = pg.PlinkSource(tmp_path / f"rt{case}.bed", tmp_path / f"rt{case}.bim", tmp_path / f"rt{case}.fam")
        b = src.read_marker_batch(0, m)
        b32 = src.read_marker_batch(0, m, dtype=np.float32)
        src.close()
        assert nan_eq(b.dosages, d)
        assert b32.dosages.dtype == np.float32 and nan_eq(b32.dosages, d.astype(np.float32))
        assert np.array_equal(b.missing_count, np.isnan(d).sum(axis=1))


def test_bgen_decode_bit_exact():
    g = np.load(GOLD / "bgen.npz")
    for bits in (8, 16):
        src = pg.BgenSource(GOLD / f"bgen{bits}.bgen")
        raw = src.read_marker_batch(0, src.n_markers)
        src.close()
        assert nan_eq(raw.dosages, g[f"b{bits}_dosage"])
        assert np.array_equal(raw.missing_count, g[f"b{bits}_missing"])


def test_p_from_t_matches_reference():
    g = np.load(GOLD / "pvalues.npz")
    # the log-prefactor lgamma(a+b) - lgamma(a) - lgamma(b) cancels ~log10(a) digits at large df;
    # device and host libm lgamma differ by a few ulps there (reference itself is only that accurate)
    for i, df in enumerate(g["dfs"]):
        rtol = 1e-12 if df <= 100 else (2e-9 if df <= 1e5 else 5e-8)
        got = pg.p_from_t(g["t"], df)
        bad = ~np.isclose(got, g["p"][i], rtol=rtol, atol=0)
        assert not bad.any(), (df, g["t"][bad][:5], got[bad][:5], g["p"][i][bad][:5])
    assert pg.p_from_t(0.0, 7.0) == 1.0
    assert pg.p_from_t(np.inf, 7.0) == pg.P_FLOOR
    with pytest.raises(ValueError):
        pg.p_from_t(1.0, 0.5)


def test_closed_forms():
    t = np.array([0.1, 0.7, 1.3, 2.5, 10.0])
    np.testing.assert_allclose(pg.p_from_t(t, 1.0), (2 / np.pi) * np.arctan(1 / t), rtol=1e-12)
    np.testing.assert_allclose(pg.p_from_t(t, 2.0), 1.0 - t / np.sqrt(2.0 + t * t), rtol=1e-12)


def test_reg_inc_beta_and_threshold():
    g = np.load(GOLD / "pvalues.npz")
    np.testing.assert_allclose(pg.reg_inc_beta(g["ib_a"], g["ib_b"], g["ib_x"]), g["ib"], rtol=1e-11, atol=1e-300)
    for k, (pt, df) in enumerate(g["crit_cases"]):
        assert pg.t_threshold_for_p(pt, df) == pytest.approx(g["crit"][k], rel=1e-12)
    assert pg.t_threshold_for_p(1e-4, 22998.0) == pytest.approx(3.8912744581499874, rel=1e-11)
    with pytest.raises(ValueError):
        pg.reg_inc_beta(0.0, 1.0, 0.5)


def test_t_from_r():
    g = np.load(GOLD / "pvalues.npz")
    for i, df in enumerate((2.0, 11.0, 22998.0)):
        got = pg.t_from_r(g["r"], df)
        np.testing.assert_allclose(got, g["t_from_r"][i], rtol=1e-14)
    assert pg.t_from_r(1.0, 10.0) == np.inf and pg.t_from_r(-1.0, 10.0) == -np.inf
    assert pg.t_from_r(0.5, 2.0) == pytest.approx(np.sqrt(2.0 / 3.0), rel=1e-15)


def test_prepare_matches_reference():
    g = np.load(GOLD / "prepare.npz")
    d = g["dosages"]
    raw = pg.RawBatch(tuple(pg.MarkerRecord("1", f"m{i}", i, "A", "B", i) for i in range(d.shape[0])), d,
                      np.isnan(d).sum(axis=1))
    std = pg.prepare_genotype_batch(raw)
    np.testing.assert_allclose(std.matrix, g["matrix"], atol=1e-12)
    assert nan_eq(std.allele_frequency, g["af"])
    assert np.array_equal(std.missing_count, g["missing"]) and np.array_equal(std.skip_reason, g["skip"])
    s32 = pg.prepare_genotype_batch(raw, dtype=np.float32)
    assert s32.matrix.dtype == np.float32


def test_correlate_handworked_and_row_stable():
    g, _, _ = pg.standardize_columns(np.array([0.0, 1.0, 2.0, 1.0])[:, None])
    y, _, _ = pg.standardize_columns(np.array([0.0, 1.0, 1.0, 2.0])[:, None])
    r, clamped = pg.correlate(g.T, y)
    assert r[0, 0] == pytest.approx(0.5, abs=1e-15) and clamped == 0
    rng = np.random.default_rng(21)
    gt, _, _ = pg.standardize_columns(rng.standard_normal((100, 777)))
    yt, _, _ = pg.standardize_columns(rng.standard_normal((100, 9)))
    gt = np.ascontiguousarray(gt.T)
    full, _ = pg.correlate(gt, yt)
    ref, _ = orc.correlate(gt, yt)
    np.testing.assert_allclose(full, ref, atol=1e-14)
    for split in (1, 7, 64, 300, 777):
        parts = np.vstack([pg.correlate(gt[s:s + split], yt)[0] for s in range(0, 777, split)])
        assert np.array_equal(parts, full)
    r, clamped = pg.correlate(np.array([[2.0, -2.0]]), np.array([[1.0], [-1.0]]))
    assert r[0, 0] == 1.0 and clamped == 1
    with pytest.raises(ValueError):
        pg.correlate(np.zeros((2, 3)), np.zeros((4, 1)))


def test_compute_stats_block():
    """compute_stats (reference kernel.py:493-504; tests/test_kernel.py:297, :305-320):
    r/t/p of a whole block on the device == oracle correlate -> t_from_r -> p_from_t, with
    the StatBlock invariants, the clamp count and the hand-worked pair r 0.5 -> t(df 2) = sqrt(2/3), p 0.5."""
    g, _, _ = pg.standardize_columns(np.array([0.0, 1.0, 2.0, 1.0])[:, None])
    y, _, _ = pg.standardize_columns(np.array([0.0, 1.0, 1.0, 2.0])[:, None])
    s = pg.compute_stats(np.ascontiguousarray(g.T), y, df=2.0)
    assert s.r[0, 0] == pytest.approx(0.5, abs=1e-15) and s.t[0, 0] == pytest.approx(np.sqrt(2 / 3), rel=1e-14)
    assert s.p[0, 0] == pytest.approx(0.5, rel=1e-13) and s.clamp_count == 0 and s.df == 2.0
    rng = np.random.default_rng(30)
    gt, _, _ = pg.standardize_columns(rng.standard_normal((60, 40)))
    yt, _, _ = pg.standardize_columns(rng.standard_normal((60, 7)))
    gt = np.ascontiguousarray(gt.T)
    s = pg.compute_stats(gt, yt, df=58.0)
    r, _ = orc.correlate(gt, yt)
    np.testing.assert_allclose(s.r, r, atol=1e-14)
    np.testing.assert_allclose(s.t, orc.t_from_r(r, 58.0), rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(s.p, orc.p_from_t(orc.t_from_r(r, 58.0), 58.0), rtol=1e-11)
    assert s.r.shape == s.t.shape == s.p.shape == (40, 7)
    assert np.all(np.abs(s.r) <= 1.0) and np.all(np.sign(s.t) == np.sign(s.r))
    assert np.all((s.p > 0.0) & (s.p <= 1.0)) and s.p_underflow_count == 0
    s2 = pg.compute_stats(gt, yt, df=58.0, with_p=False)
    assert s2.p is None and np.array_equal(s2.t, s.t)
    # a clamped pair and an underflowing p
    s3 = pg.compute_stats(np.array([[2.0, -2.0]]), np.array([[1.0], [-1.0]]), df=1e6)
    assert s3.clamp_count == 1 and s3.t[0, 0] == np.inf and s3.p_underflow_count == 1


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,n_cov", [(300, 12, 3), (2000, 64, 10), (5000, 700, 20), (1100, 33, 0),
                                       (12000, 1601, 5)])  # 154 MB: chunked pinned upload
def test_device_panel_prep_matches_host(n, p, n_cov):
    """pg_ctx_prepare_panel == kernel.residualize + standardize_columns (reference
    kernel.py:310-347) to 1e-12 relative, flags identical; commit == set_panel on the
    host-prepared matrix (quantized limbs + scales bitwise, barring rint ties)."""
    import torch

    from paper_2604_21095_b200 import kernel
    from paper_2604_21095_b200._device import DeviceContext

    rng = np.random.default_rng(n + p)
    c = rng.standard_normal((n, n_cov))
    y = c @ rng.standard_normal((n_cov, p)) * 0.3 + rng.standard_normal((n, p)) * rng.uniform(0.5, 50, p) + 7.0
    y[:, 3] = 5.0  # constant -> zero variance after centring
    if n_cov:
        y[:, 5] = 2.0 * c[:, 0] - 1.0  # lies in span(Q) -> zero variance after residualization
    basis = kernel.build_covariate_basis(c, True)
    want, want_sd, want_flat = kernel.standardize_columns(kernel.residualize(y, basis))
    with DeviceContext(0) as ctx:
        flat, sd = ctx.prepare_panel(y, basis.q)
        got = ctx.fetch_prepared_panel()
        assert np.array_equal(flat, want_flat)
        ok = ~want_flat
        np.testing.assert_allclose(sd[ok], want_sd[ok], rtol=1e-12)
        np.testing.assert_allclose(got[:, ok], want[:, ok], rtol=1e-10, atol=1e-12)
        assert np.all(got[:, ~ok] == 0.0)
        kept = np.nonzero(ok)[0]
        gidx = np.arange(n, dtype=np.int64)
        ctx.commit_panel(kept, gidx, n)
        nb = ctx.panel_bytes()
        a = torch.empty(nb, dtype=torch.uint8, device="cuda")
        ctx.export_panel(a.data_ptr())
        ctx.set_panel(np.ascontiguousarray(want[:, kept]), gidx, n)
        b = torch.empty(nb, dtype=torch.uint8, device="cuda")
        ctx.export_panel(b.data_ptr())
        p_pad, k_pad = -(-kept.size // 256) * 256, -(-n // 64) * 64
        plane = p_pad * k_pad

        def unpack(buf):
            raw = buf.cpu().numpy()
            lim = raw[:3 * plane].view(np.int8).astype(np.int64).reshape(3, p_pad, k_pad)
            q = 32385 * lim[0] + 127 * lim[1] + lim[2]
            return q, raw[3 * plane:3 * plane + 8 * p_pad].view(np.float64)

        qa, sa = unpack(a)
        qb, sb = unpack(b)
        np.testing.assert_allclose(sa, sb, rtol=1e-14)
        assert np.abs(qa - qb).max() <= 1  # quantized to the same 23-bit grid up to rint ties


@pytest.mark.gpu
def test_device_panel_prep_rejects_non_finite():
    from paper_2604_21095_b200._device import DeviceContext

    y = np.ones((10, 3))
    y[4, 1] = np.inf
    with DeviceContext(0) as ctx:
        with pytest.raises(ValueError, match="finite"):
            ctx.prepare_panel(y, None)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["plink", "plink_missing", "dense_real"])
def test_k_sliced_contraction_matches_oracle(case):
    """Cohorts above 131,072 samples (one int32-exact slice) run the contraction in K slices
    summed in int64: statistics equal the oracle's float64 path (PLINK fused, PLINK with
    missing calls, real-valued dosages through the wide-digit GEMM)."""
    from paper_2604_21095_b200 import _native
    from paper_2604_21095_b200._device import DeviceContext

    rng = np.random.default_rng(140)
    n, m, p = 140_000, 64, 8
    y = rng.standard_normal((n, p))
    y -= y.mean(axis=0)
    y /= np.sqrt((y * y).mean(axis=0))
    y[:, 1] += 0.05 * rng.standard_normal(n)
    af = rng.uniform(0.1, 0.9, (m, 1))
    g = rng.binomial(2, af, size=(m, n)).astype(np.float64)
    y[:, 2] += 0.02 * (g[7] - g[7].mean())  # a planted association
    if case == "plink_missing":
        g[rng.random(g.shape) < 0.02] = np.nan
    with DeviceContext(0) as ctx:
        ytil = y / np.sqrt((y * y).mean(axis=0))
        ytil -= ytil.mean(axis=0)
        ytil /= np.sqrt((ytil * ytil).mean(axis=0))
        ctx.set_panel(ytil, np.arange(n, dtype=np.int64), n)
        ctx.set_scan(float(n - 2), _native.PG_MODE_FULL, None)
        if case == "dense_real":
            d = np.clip(g + rng.normal(0, 0.2, g.shape), 0, 2)
            res = ctx.scan(_native.PG_GENO_DENSE_F64, np.ascontiguousarray(d).view(np.uint8), 8 * n)
        else:
            d = g
            bpm = (n + 3) // 4
            codes = np.where(np.isnan(g), 1, np.array([3, 2, 0], np.uint8)[np.nan_to_num(g).astype(int)])
            codes = np.pad(codes.astype(np.uint8), ((0, 0), (0, bpm * 4 - n))).reshape(m, bpm, 4)
            packed = (codes[:, :, 0] | (codes[:, :, 1] << 2) | (codes[:, :, 2] << 4)
                      | (codes[:, :, 3] << 6)).astype(np.uint8)
            res = ctx.scan(_native.PG_GENO_BED, packed, bpm)
    ref = orc.threshold_scan(d, ytil, float(n - 2), 1.0)
    t_ref = np.zeros((m, p))
    t_ref[ref["rows"], ref["cols"]] = ref["t"]
    rel = np.abs(res.t_rows - t_ref) / np.maximum(1.0, np.abs(t_ref))
    assert rel.max() <= 1e-4
    assert abs(t_ref[7, 2]) > 4 and np.sign(res.t_rows[7, 2]) == np.sign(t_ref[7, 2])


@pytest.mark.gpu
def test_c_abi_misuse_fails_loudly():
    """State and argument errors come back as the mapped exceptions, never a crash or a
    silently empty result."""
    from paper_2604_21095_b200 import _native
    from paper_2604_21095_b200._device import DeviceContext
    from paper_2604_21095_b200.errors import FormatError, PanelGwasError

    rows = np.zeros((4, 3), np.uint8)
    with DeviceContext(0) as ctx:
        with pytest.raises(PanelGwasError, match="no panel"):
            ctx.scan(_native.PG_GENO_BED, rows, 3)
        ctx.set_panel(np.random.default_rng(0).standard_normal((10, 2)), np.arange(10, dtype=np.int64), 10)
        ctx.set_scan(8.0, _native.PG_MODE_THRESHOLD, np.full(2, 0.5))
        with pytest.raises(FormatError, match="expected 3"):
            ctx.scan(_native.PG_GENO_BED, np.zeros((4, 5), np.uint8), 5)
        with pytest.raises(ValueError, match="slot"):
            ctx.stage(2, _native.PG_GENO_BED, rows, 3)
        with pytest.raises(PanelGwasError, match="no batch in flight"):
            ctx.stage_bgen_end(0)
        with pytest.raises(PanelGwasError, match="holds no staged batch"):
            ctx.scan_staged(1)
        with pytest.raises(ValueError, match="r_bar required"):
            ctx.set_scan(8.0, _native.PG_MODE_THRESHOLD, None)
        res = ctx.scan(_native.PG_GENO_BED, rows, 3)  # still usable after the errors
        assert res.n_markers == 4
