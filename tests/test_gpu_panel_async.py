"""Pipelined panel upload (pg_ctx_set_panel_async): the raw phenotype matrix is uploaded in
phenotype chunks, each residualized, standardized and quantized as it lands, and the first
batch's GEMM runs one chunk at a time. Against the synchronous pg_ctx_prepare_panel +
pg_ctx_commit_panel of every column: the exported panel is bit-identical, and THRESHOLD and
FULL scans (fused two-limb, three-limb, missing-call side GEMM, F64 two-level panel) return
identical results."""
import numpy as np
import pytest
import torch

from oracle import scan_oracle as orc
from paper_2604_21095_b200 import _native
from paper_2604_21095_b200._device import DeviceContext
from paper_2604_21095_b200.kernel import build_covariate_basis

pytestmark = pytest.mark.gpu


def _pinned(a: np.ndarray) -> np.ndarray:
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def _packed(d):
    m, n = d.shape
    codes = np.where(np.isnan(d), 1, np.select([d == 2, d == 1, d == 0], [0, 2, 3])).astype(np.uint8)
    bpm = (n + 3) // 4
    codes = np.pad(codes, ((0, 0), (0, 4 * bpm - n)))
    q = codes.reshape(m, bpm, 4)
    return (q[:, :, 0] | (q[:, :, 1] << 2) | (q[:, :, 2] << 4) | (q[:, :, 3] << 6)).astype(np.uint8), bpm


def _panel_bytes(ctx):
    buf = torch.empty(ctx.panel_bytes(), dtype=torch.uint8, device="cuda")
    ctx.export_panel(buf.data_ptr())
    torch.cuda.synchronize()
    return buf.cpu().numpy()


def _case(seed, n_src=613, n_kept=590, p=700, cov=3):
    rng = np.random.default_rng(seed)
    y = rng.standard_normal((n_kept, p)) * rng.uniform(0.5, 3.0, p) + rng.uniform(-2, 2, p)
    c = rng.standard_normal((n_kept, cov))
    gidx = np.sort(rng.choice(n_src, n_kept, replace=False)).astype(np.int64)
    return y, build_covariate_basis(c, True).q, gidx, n_src


@pytest.mark.parametrize("f64,p", [(False, 700), (True, 700), (False, 100), (True, 1)])
def test_async_panel_bitwise_equals_sync(f64, p):
    y, q, gidx, n_src = _case(1, p=p)
    with DeviceContext(0) as a, DeviceContext(0) as b:
        a.set_f64_panel(f64)
        b.set_f64_panel(f64)
        flat, sd = a.prepare_panel(y, q)
        a.commit_panel(np.arange(y.shape[1]), gidx, n_src)
        b.set_panel_async(_pinned(y), q, gidx, n_src, chunk_cols=256)  # 3 chunks, the last padded
        flat_b, sd_b = b.panel_async_wait()
        assert not flat.any() and np.array_equal(flat, flat_b) and np.array_equal(sd, sd_b)
        assert np.array_equal(_panel_bytes(a), _panel_bytes(b))


def _scan_pair(a, b, kind, block, bpm, mode, rbar, df):
    out = []
    for ctx in (a, b):
        ctx.set_scan(df, mode, rbar)
        out.append(ctx.scan(kind, block, bpm))
    return out


@pytest.mark.parametrize("missing", [0.0, 0.3])
@pytest.mark.parametrize("mode", ["thr", "full", "thr3", "f64"])
def test_async_first_batch_scans_equal_sync(missing, mode):
    """The first scan after set_panel_async runs its GEMM per phenotype chunk (or, for the
    side GEMM / three-limb / F64 paths, waits for the whole panel): identical results."""
    y, q, gidx, n_src = _case(7, p=900)
    rng = np.random.default_rng(3)
    m = 700
    d = rng.binomial(2, rng.uniform(0.05, 0.95, m)[:, None], size=(m, n_src)).astype(np.float64)
    rows = rng.random(m) < missing
    d[rows] = np.where(rng.random((rows.sum(), n_src)) < 0.05, np.nan, d[rows])
    packed, bpm = _packed(d)
    df = float(len(gidx) - 1 - q.shape[1])
    kmode = _native.PG_MODE_FULL if mode == "full" else _native.PG_MODE_THRESHOLD
    rbar = None if mode == "full" else np.full(y.shape[1], orc.premask_abs_r(1e-2, df))
    with DeviceContext(0) as a, DeviceContext(0) as b:
        if mode == "thr3":
            a.set_two_limb_premask(False)
            b.set_two_limb_premask(False)
        if mode == "f64":
            a.set_f64_panel(True)
            b.set_f64_panel(True)
        a.prepare_panel(y, q)
        a.commit_panel(np.arange(y.shape[1]), gidx, n_src)
        yp = _pinned(y)
        b.set_panel_async(yp, q, gidx, n_src, chunk_cols=256)
        for batch in (packed[:400], packed[400:]):  # the second batch runs on the completed panel
            ra, rb = _scan_pair(a, b, _native.PG_GENO_BED, batch, bpm, kmode, rbar, df)
            if kmode == _native.PG_MODE_FULL:
                assert np.array_equal(ra.t_rows, rb.t_rows)
            else:
                for f in ("cand_rows", "cand_cols", "cand_r", "cand_t", "cand_p"):
                    assert np.array_equal(getattr(ra, f), getattr(rb, f)), f
                assert ra.n_candidates > 0
            assert np.array_equal(ra.af, rb.af) and np.array_equal(ra.skip, rb.skip)
        b.panel_async_wait()


def test_async_panel_zero_variance_and_errors():
    y, q, gidx, n_src = _case(11, p=300)
    y[:, 5] = 4.0  # constant: zero variance after the intercept
    with DeviceContext(0) as ctx:
        ctx.set_panel_async(_pinned(y), q, gidx, n_src, chunk_cols=256)
        flat, sd = ctx.panel_async_wait()
        assert flat[5] and flat.sum() == 1
        # the zero-variance column stays in the panel with r = 0
        ctx.set_scan(float(len(gidx) - 4), _native.PG_MODE_FULL, None)
        d = np.random.default_rng(2).binomial(2, 0.4, size=(50, n_src)).astype(float)
        packed, bpm = _packed(d)
        res = ctx.scan(_native.PG_GENO_BED, packed, bpm)
        assert np.all(res.t_rows[:, 5] == 0.0) and np.all(res.t_rows[:, 4] != 0.0)
        y2 = y.copy()
        y2[17, 200] = np.nan
        ctx.set_panel_async(_pinned(y2), q, gidx, n_src, chunk_cols=256)
        with pytest.raises(ValueError, match="finite"):
            ctx.panel_async_wait()
        with pytest.raises(ValueError, match="page-locked"):
            ctx.set_panel_async(np.ascontiguousarray(y), q, gidx, n_src)


@pytest.mark.parametrize("f64", [False, True])
def test_panel_shares_assemble_the_sync_panel(f64):
    """Multi-GPU panel preparation on one GPU: two contexts each prepare their share of the
    phenotype columns (pg_ctx_set_panel_async_cols), exchange rows (export / import_panel_rows)
    and both end up with the synchronous path's panel, bit for bit (incl. the last share's
    padding rows and the F64 lo level)."""
    y, q, gidx, n_src = _case(13, p=700)  # shares [0, 512) and [512, 700) (+ padding to 768)
    cut = 512
    with DeviceContext(0) as ref, DeviceContext(0) as a, DeviceContext(0) as b:
        for cx in (ref, a, b):
            cx.set_f64_panel(f64)
        ref.prepare_panel(y, q)
        ref.commit_panel(np.arange(y.shape[1]), gidx, n_src)
        shares = [(a, 0, cut), (b, cut, y.shape[1])]
        for cx, c0, c1 in shares:
            cx.set_panel_async_cols(_pinned(np.ascontiguousarray(y[:, c0:c1])), y.shape[1], c0, q, gidx, n_src,
                                    chunk_cols=256)
        for cx, c0, c1 in shares:
            flat, _ = cx.panel_async_wait()
            assert flat.shape == (c1 - c0,) and not flat.any()
        p_pad = (y.shape[1] + 255) // 256 * 256
        rows = {}
        for cx, c0, c1 in shares:
            r1 = p_pad if c1 == y.shape[1] else c1
            buf = torch.empty(cx.panel_rows_bytes(r1 - c0), dtype=torch.uint8, device="cuda")
            cx.export_panel_rows(buf.data_ptr(), c0, r1)
            rows[cx] = (buf, c0, r1)
        torch.cuda.synchronize()
        a.import_panel_rows(rows[b][0].data_ptr(), rows[b][1], rows[b][2])
        b.import_panel_rows(rows[a][0].data_ptr(), rows[a][1], rows[a][2])
        want = _panel_bytes(ref)
        assert np.array_equal(_panel_bytes(a), want) and np.array_equal(_panel_bytes(b), want)


@pytest.mark.parametrize("f64", [False, True])
def test_follower_context_scans_equal_leader(f64):
    """pg_ctx_follow_panel: a second context takes the pipelined panel chunk by chunk. Its
    first scan (run before the leader has scanned, so it drives the chunk issuing itself)
    equals the leader's and the synchronous context's, bit for bit; a second pipelined panel
    on the leader releases the follower, which can follow again."""
    y, q, gidx, n_src = _case(21, p=900)
    rng = np.random.default_rng(6)
    m = 600
    d = rng.binomial(2, rng.uniform(0.05, 0.95, m)[:, None], size=(m, n_src)).astype(np.float64)
    packed, bpm = _packed(d)
    df = float(len(gidx) - 1 - q.shape[1])
    rbar = np.full(y.shape[1], orc.premask_abs_r(1e-2, df))
    with DeviceContext(0) as ref, DeviceContext(0) as lead, DeviceContext(0) as fol:
        for cx in (ref, lead, fol):
            cx.set_f64_panel(f64)
        ref.prepare_panel(y, q)
        ref.commit_panel(np.arange(y.shape[1]), gidx, n_src)
        ref.set_scan(df, _native.PG_MODE_THRESHOLD, rbar)
        want = ref.scan(_native.PG_GENO_BED, packed, bpm)
        for rep in range(2):
            yp = _pinned(y)
            lead.set_panel_async(yp, q, gidx, n_src, chunk_cols=256)
            fol.follow_panel(lead)
            for cx in (fol, lead):  # the follower first
                cx.set_scan(df, _native.PG_MODE_THRESHOLD, rbar)
                got = cx.scan(_native.PG_GENO_BED, packed, bpm)
                for f in ("cand_rows", "cand_cols", "cand_r", "cand_t", "cand_p"):
                    assert np.array_equal(getattr(got, f), getattr(want, f)), (rep, f)
            lead.panel_async_wait()
        assert np.array_equal(_panel_bytes(fol), _panel_bytes(ref))
