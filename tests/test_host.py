"""Host-side logic (no GPU): table parsing and alignment, reader metadata
validation and error messages, writers and file formats, configuration,
simulator determinism. Mirrors the reference test strategy."""
import json
import logging

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from paper_2604_21095_b200 import engine, output
from paper_2604_21095_b200.errors import ConfigError, FormatError, PanelGwasError, UnsupportedFeatureError


def write(path, text):
    path.write_text(text)
    return path


# ----------------------------------------------------------------------------- tables
class TestTables:
    def test_missing_tokens_and_unparseable(self, tmp_path, caplog):
        p = write(tmp_path / "t.tsv", "IID\ta\tb\nS1\tNA\t1.5\nS2\t-9\tfoo\nS3\tnan\tinf\nS4\t2\t\n")
        with caplog.at_level(logging.WARNING):
            t = pg.load_table(p)
        assert t.ids == ["S1", "S2", "S3", "S4"] and t.column_names == ["a", "b"]
        assert np.isnan(t.values[:3, 0]).all() and t.values[3, 0] == 2.0
        assert list(t.missing_count) == [3, 3]
        assert list(t.unparseable_count) == [0, 2]
        assert any("unparseable" in r.message for r in caplog.records)

    def test_fast_path_and_id_column_anywhere(self, tmp_path):
        p = write(tmp_path / "t.csv", "x,IID,y\n1.0,A,2.0\n3.0,B,4.0\n")
        t = pg.load_table(p, delimiter=",")
        assert t.column_names == ["x", "y"] and t.values.tolist() == [[1.0, 2.0], [3.0, 4.0]]

    @pytest.mark.parametrize("body,msg", [
        ("", "empty file"),
        ("ID\ta\nS1\t1\n", "no 'IID' column"),
        ("IID\ta\nS1\t1\t2\n", "ragged"),
        ("IID\ta\nS1\t1\nS1\t2\n", "duplicate sample ID"),
    ])
    def test_errors(self, tmp_path, body, msg):
        with pytest.raises(PanelGwasError, match=msg):
            pg.load_table(write(tmp_path / "t.tsv", body))

    def test_alignment_order_and_log(self, tmp_path):
        ph = pg.load_table(write(tmp_path / "p.tsv", "IID\ty\nS3\t1\nS1\t2\nS2\t3\nS9\t4\nS4\t5\n"))
        cv = pg.load_table(write(tmp_path / "c.tsv", "IID\tc\nS1\t0\nS2\t1\nS3\t2\nS5\t3\n"))
        al = pg.align_samples(["S1", "S2", "S3", "S4", "S5", "S6"], ph, cv, keep_list=None, remove_list={"S6"})
        assert al.kept_sample_ids == ["S1", "S2", "S3"]
        assert al.genotype_row_index.tolist() == [0, 1, 2]
        assert al.phenotype_row_index.tolist() == [1, 2, 0]
        assert al.exclusion_log["remove-listed"] == 1
        assert al.exclusion_log["not-in-covariates"] == 1 and al.exclusion_log["not-in-phenotypes"] == 1
        assert al.table_ids_not_in_genotypes == 1
        with pytest.raises(PanelGwasError, match="at least 3"):
            pg.align_samples(["S1", "S2"], ph)

    def test_keep_then_remove_wins(self, tmp_path):
        ph = pg.load_table(write(tmp_path / "p.tsv", "IID\ty\n" + "".join(f"S{i}\t{i}\n" for i in range(6))))
        al = pg.align_samples([f"S{i}" for i in range(6)], ph, keep_list={"S0", "S1", "S2", "S3"},
                              remove_list={"S0"})
        assert al.kept_sample_ids == ["S1", "S2", "S3"]
        assert al.exclusion_log["not-keep-listed"] == 2

    def test_build_panel_impute_and_fail(self, tmp_path):
        ph = pg.load_table(write(tmp_path / "p.tsv", "IID\ty\tz\nA\t1\t5\nB\tNA\t6\nC\t3\t7\n"))
        al = pg.align_samples(["A", "B", "C"], ph)
        panel = pg.build_panel(ph, al)
        assert panel.y[:, 0].tolist() == [1.0, 2.0, 3.0]
        assert panel.missing_count.tolist() == [1, 0]
        with pytest.raises(PanelGwasError, match="missing"):
            pg.build_panel(ph, al, pg.MissingPolicy.FAIL)
        bad = pg.load_table(write(tmp_path / "q.tsv", "IID\ty\nA\tNA\nB\tNA\nC\tNA\n"))
        with pytest.raises(PanelGwasError, match="entirely missing"):
            pg.build_panel(bad, pg.align_samples(["A", "B", "C"], bad))

    def test_covariates_never_imputed(self, tmp_path):
        ph = pg.load_table(write(tmp_path / "p.tsv", "IID\ty\nA\t1\nB\t2\nC\t3\n"))
        cv = pg.load_table(write(tmp_path / "c.tsv", "IID\tc\nA\t1\nB\tNA\nC\t3\n"))
        al = pg.align_samples(["A", "B", "C"], ph, cv)
        with pytest.raises(PanelGwasError, match="never imputed"):
            pg.covariate_matrix(cv, al)


# ----------------------------------------------------------------------------- panel math (host, once per scan)
class TestPanelPrep:
    def test_basis_intercept_and_rank(self):
        b = pg.build_covariate_basis(np.zeros((4, 0)))
        assert b.rank == 1 and np.allclose(b.q[:, 0], 0.5)
        a = np.random.default_rng(0).standard_normal(30)
        b = pg.build_covariate_basis(np.column_stack([a, 2 * a]), column_names=["a", "a2"])
        assert b.rank == 2 and b.dropped_columns == ("a2",)
        with pytest.raises(PanelGwasError, match="degrees of freedom"):
            pg.build_covariate_basis(np.random.default_rng(1).random((3, 2)))

    def test_residualize_hand_example(self):
        x = np.array([1.0, 2.0, 3.0, 4.0])
        out = pg.residualize(np.array([1.0, 3.0, 2.0, 4.0])[:, None], pg.build_covariate_basis(x[:, None]))
        np.testing.assert_allclose(out[:, 0], [-0.3, 0.9, -0.9, 0.3], atol=1e-12)

    def test_standardize(self):
        out, sd, zero = pg.standardize_columns(np.array([[-1.0, 3.25], [0.0, 3.25], [1.0, 3.25]]))
        assert zero.tolist() == [False, True] and np.all(out[:, 1] == 0)
        assert np.mean(out[:, 0] ** 2) == pytest.approx(1.0)


# ----------------------------------------------------------------------------- readers (metadata only)
def trio(tmp_path, d, ids=None):
    ids = ids or [f"I{j}" for j in range(d.shape[1])]
    return pg.write_bed_trio(tmp_path / "g", d, ids)


class TestPlinkMetadata:
    def valid(self, tmp_path):
        return trio(tmp_path, np.array([[0.0, 1.0, 2.0, np.nan]]), ["a", "b", "c", "d"])

    def test_open(self, tmp_path):
        bed, bim, fam = self.valid(tmp_path)
        src = pg.open_genotype_source(pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=bed, bim_path=bim,
                                                    fam_path=fam))
        assert (src.n_samples, src.n_markers, src.counts_allele1) == (4, 1, True)
        kind, rows, rb = src.read_raw_block(0, 5)
        assert rows.shape == (1, 1) and rb == 1
        src.close()

    @pytest.mark.parametrize("mutate,msg", [
        (lambda b: b.__setitem__(2, 0), "sample-major"),
        (lambda b: b.__setitem__(0, 0), "magic"),
        (lambda b: b.__setitem__(2, 7), "mode byte"),
    ])
    def test_header_errors(self, tmp_path, mutate, msg):
        bed, bim, fam = self.valid(tmp_path)
        blob = bytearray(bed.read_bytes())
        mutate(blob)
        bed.write_bytes(bytes(blob))
        with pytest.raises(FormatError, match=msg):
            pg.PlinkSource(bed, bim, fam)

    def test_size_and_text_errors(self, tmp_path, caplog):
        bed, bim, fam = self.valid(tmp_path)
        bed.write_bytes(bed.read_bytes() + b"\x00")
        with pytest.raises(FormatError, match="imply"):
            pg.PlinkSource(bed, bim, fam)
        bed, bim, fam = self.valid(tmp_path)
        fam.write_text("a a 0 0 0 -9\na a 0 0 0 -9\nc c 0 0 0 -9\nd d 0 0 0 -9\n")
        with pytest.raises(FormatError, match="duplicate sample ID"):
            pg.PlinkSource(bed, bim, fam)
        bed, bim, fam = self.valid(tmp_path)
        bim.write_text("1 snp1 0 5\n")
        with pytest.raises(FormatError, match="6 columns"):
            pg.PlinkSource(bed, bim, fam)
        bim.write_text("1 snp1 0 -5 A B\n")
        with pytest.raises(FormatError, match="negative position"):
            pg.PlinkSource(bed, bim, fam)
        bim.write_text("1 snp1 0 5 A A\n")
        with caplog.at_level("WARNING"):
            pg.PlinkSource(bed, bim, fam).close()
        assert any("identical alleles" in r.message for r in caplog.records)
        bim.unlink()
        with pytest.raises(FormatError, match="missing file"):
            pg.PlinkSource(bed, bim, fam)

    def test_batch_bounds(self, tmp_path):
        src = pg.PlinkSource(*trio(tmp_path, np.zeros((3, 5))))
        with pytest.raises(ValueError):
            src.read_raw_block(99, 1)
        with pytest.raises(ValueError):
            src.read_raw_block(0, 0)
        assert src.read_raw_block(1, 10)[1].shape[0] == 2
        src.close()


class TestBgenMetadata:
    def test_features_and_errors(self, tmp_path):
        from bgen_fixture import write_bgen

        d = np.array([[0.0, 1.0, 2.0], [0.5, np.nan, 1.5]])
        ids = ["a", "b", "c"]
        p = write_bgen(tmp_path / "ok.bgen", d, ids)
        src = pg.BgenSource(p)
        assert src.n_samples == 3 and src.n_markers == 2 and not src.counts_allele1
        assert src.sample_ids == ids and src.marker_catalog[1].id == "rs2"
        kind, rows, rb = src.read_raw_block(0, 2)
        assert rb == 3 * 3 and rows[1, 6 + 1] & 0x80  # ploidy byte of the missing call
        src.close()
        with pytest.raises(UnsupportedFeatureError, match="layout"):
            pg.BgenSource(write_bgen(tmp_path / "l1.bgen", d, ids, layout=1))
        with pytest.raises(UnsupportedFeatureError, match="zstd"):
            pg.BgenSource(write_bgen(tmp_path / "z.bgen", d, ids, compression=2))
        with pytest.raises(UnsupportedFeatureError, match="3 alleles"):
            pg.BgenSource(write_bgen(tmp_path / "k3.bgen", d, ids, n_alleles=3))
        with pytest.raises(FormatError, match="sample identifiers"):
            pg.BgenSource(write_bgen(tmp_path / "noid.bgen", d, ids, include_sample_ids=False))
        src = pg.BgenSource(write_bgen(tmp_path / "ph.bgen", d, ids, phased=1))
        with pytest.raises(UnsupportedFeatureError, match="phased"):
            src.read_raw_block(0, 1)
        src.close()
        src = pg.BgenSource(write_bgen(tmp_path / "b4.bgen", d, ids, bits=4))
        with pytest.raises(UnsupportedFeatureError, match="4-bit"):
            src.read_raw_block(0, 1)
        src.close()
        blob = p.read_bytes()
        (tmp_path / "trunc.bgen").write_bytes(blob[:-5])
        with pytest.raises(FormatError, match="truncated"):
            pg.BgenSource(tmp_path / "trunc.bgen")

    def test_corrupt_zlib(self, tmp_path):
        from bgen_fixture import write_bgen

        p = write_bgen(tmp_path / "c.bgen", np.array([[0.0, 1.0, 2.0]]), ["a", "b", "c"])
        blob = bytearray(p.read_bytes())
        blob[-4] ^= 0xFF
        blob[-6] ^= 0xFF
        p.write_bytes(bytes(blob))
        src = pg.BgenSource(p)
        with pytest.raises(FormatError, match="zlib|inflated"):
            src.read_raw_block(0, 1)
        src.close()

    def test_expected_dosage(self):
        assert pg.bgen_expected_dosage(1, 0, 0) == 0 and pg.bgen_expected_dosage(0, 0, 1) == 2
        assert pg.bgen_expected_dosage(0.25, 0.5, 0.25) == 1


class TestDense:
    def test_orientation_range_and_dtype(self, tmp_path):
        d = np.array([[0.0, 1.0, 2.0], [np.nan, 2.0, 0.0]])
        np.save(tmp_path / "g.npy", d.T)
        (tmp_path / "s.txt").write_text("a\nb\nc\n")
        spec = pg.SourceSpec(pg.GenotypeFormat.DENSE, dense_path=tmp_path / "g.npy",
                             sample_id_path=tmp_path / "s.txt",
                             dense_orientation=pg.DenseOrientation.SAMPLES_BY_MARKERS)
        src = pg.open_genotype_source(spec)
        b = src.read_marker_batch(0, 2)
        assert np.array_equal(np.nan_to_num(b.dosages, nan=-1), np.nan_to_num(d, nan=-1))
        assert b.missing_count.tolist() == [0, 1]
        np.save(tmp_path / "bad.npy", np.array([[0.0, 2.5, 1.0]]))
        bad = pg.DenseSource(tmp_path / "bad.npy", ["a", "b", "c"])
        with pytest.raises(FormatError, match="outside"):
            bad.read_marker_batch(0, 1)
        np.save(tmp_path / "i.npy", np.zeros((2, 3), dtype=np.int32))
        with pytest.raises(FormatError, match="float32/float64"):
            pg.DenseSource(tmp_path / "i.npy", ["a", "b", "c"])
        with pytest.raises(FormatError, match="sidecar"):
            pg.DenseSource(tmp_path / "g.npy", ["a"], pg.DenseOrientation.SAMPLES_BY_MARKERS)


# ----------------------------------------------------------------------------- writers
def _batch(markers, cand):
    rows, cols, r, t, p = (np.array(x) for x in zip(*cand)) if cand else (np.empty(0, int),) * 5
    return output.BatchStats(
        markers=tuple(markers), allele_frequency=np.full(len(markers), 0.25), missing_count=np.zeros(len(markers), int),
        skip_reason=np.zeros(len(markers), np.int8), clamp_count=0, cand_rows=rows.astype(np.int64),
        cand_cols=cols.astype(np.int64), cand_r=r.astype(float), cand_t=t.astype(float), cand_p=p.astype(float))


class TestWriters:
    def test_fmt_float_round_trip(self):
        for x in (123.0, 3.1e-05, 0.1, 1e16, -2.5e-300, 1.0 / 3.0):
            assert float(output.fmt_float(x)) == x
        assert output.fmt_float(123.0) == "123.0" and output.fmt_float(3.1e-05) == "3.1e-05"

    def test_threshold_writer(self, tmp_path):
        mk = [pg.MarkerRecord("1", f"snp{i + 1}", i + 1, "A", "B", i) for i in range(3)]
        w = output.ThresholdWriter(tmp_path / "o.tsv", 0.01, 18.0, 20, True, ["ph1", "ph2"])
        w.emit(_batch(mk, [(0, 1, 0.5, 2.5, 0.02), (2, 0, -0.7, -4.1, 0.001), (2, 1, 0.9, 8.0, 2.2250738585072014e-308)]))
        assert w.finalize() == 2 and w.p_underflow_count == 1
        recs = pg.load_association_records(tmp_path / "o.tsv")
        assert [(r.id, r.phenotype, r.n, r.df, r.counted_allele) for r in recs] == [
            ("snp3", "ph1", 20, 18, "A"), ("snp3", "ph2", 20, 18, "A")]

    def test_topk_ties_by_source_index(self, tmp_path):
        mk = [pg.MarkerRecord("1", f"snp{i + 1}", i + 1, "A", "B", i) for i in range(4)]
        w = output.TopKWriter(tmp_path / "t.tsv", 2, 10.0, 12, False, ["ph1"])
        w.emit(_batch(mk[:2], [(0, 0, 0.1, 0.3, 0.5), (1, 0, 0.9, 5.0, 1e-4)]))
        assert np.isfinite(w.worst_abs_t[0]) and w.worst_abs_t[0] == pytest.approx(0.3)
        w.emit(_batch(mk[2:], [(0, 0, 0.9, 5.0, 1e-4), (1, 0, 0.2, 0.9, 0.4)]))
        assert w.finalize() == 2
        recs = pg.load_association_records(tmp_path / "t.tsv")
        assert [r.id for r in recs] == ["snp2", "snp3"]  # equal p: earlier source index first
        assert recs[0].counted_allele == "B"  # counts_allele1=False swaps labels

    def test_topk_writer_matches_brute_force(self, tmp_path):
        """The native per-phenotype merge (pg_topk_merge) over many batches — candidates in
        (marker, phenotype) order, p ties within and across batches, phenotypes that never
        fill k — keeps exactly the k smallest (p, source index) records of each phenotype."""
        rng = np.random.default_rng(12)
        n_pheno, k, n_batches, per = 7, 5, 9, 40
        names = [f"ph{j + 1}" for j in range(n_pheno)]
        w = output.TopKWriter(tmp_path / "t.tsv", k, 30.0, 40, True, names)
        allrec = []
        for b in range(n_batches):
            mk = [pg.MarkerRecord("1", f"snp{b * per + i + 1}", b * per + i + 1, "A", "B", b * per + i)
                  for i in range(per)]
            cand = []
            for i in range(per):
                for j in range(n_pheno - 1):  # the last phenotype never gets a record
                    if rng.random() < 0.4:
                        p = float(rng.choice([0.5, 0.25, 0.125, 1e-3])) if rng.random() < 0.5 else float(rng.random())
                        cand.append((i, j, 0.1, 2.0 - p, p))
                        allrec.append((j, p, b * per + i))
            w.emit(_batch(mk, cand))
        assert w.finalize() > 0
        recs = pg.load_association_records(tmp_path / "t.tsv")
        got = [(int(r.phenotype[2:]) - 1, r.p, int(r.id[3:]) - 1) for r in recs]
        want = []
        for j in range(n_pheno):
            want += sorted((x for x in allrec if x[0] == j), key=lambda x: (x[1], x[2]))[:k]
        assert got == want

    def test_full_matrix_round_trip(self, tmp_path):
        mk = [pg.MarkerRecord("1", f"snp{i + 1}", i + 1, "A", "B", i) for i in range(3)]
        w = output.FullMatrixWriter(tmp_path / "f.bin", np.float32, 5.0, 7, True, ["p1", "p2"])
        b = _batch(mk, [])
        b.skip_reason = np.array([0, 1, 0], np.int8)
        b.t_rows = np.array([[1.0, 2.0], [3.0, 4.0]])
        w.emit(b)
        assert w.finalize() == 4
        t, lines, phenos = pg.read_full_matrix(tmp_path / "f.bin")
        assert t.dtype == np.dtype("<f4") and t.tolist() == [[1.0, 2.0], [3.0, 4.0]]
        assert [ln.split("\t")[2] for ln in lines] == ["snp1", "snp3"] and phenos == ["p1", "p2"]
        blob = bytearray((tmp_path / "f.bin").read_bytes())
        blob[0] = 0
        (tmp_path / "g.bin").write_bytes(bytes(blob))
        for s in ("markers.tsv", "phenotypes.txt"):
            (tmp_path / f"g.bin.{s}").write_bytes((tmp_path / f"f.bin.{s}").read_bytes())
        with pytest.raises(PanelGwasError, match="magic"):
            pg.read_full_matrix(tmp_path / "g.bin")
        with pytest.raises(PanelGwasError, match="float32/float64"):
            output.FullMatrixWriter(tmp_path / "h.bin", np.int32, 5.0, 7, True, ["p1"])

    def test_bad_tsv_header(self, tmp_path):
        with pytest.raises(PanelGwasError, match="unexpected header"):
            pg.load_association_records(write(tmp_path / "x.tsv", "A\tB\n"))


# ----------------------------------------------------------------------------- engine configuration
class TestEngineConfig:
    def test_plan_batches(self):
        assert pg.plan_batches(10, 4) == [(0, 4), (4, 4), (8, 2)]
        assert pg.plan_batches(4, 10) == [(0, 4)]
        with pytest.raises(ValueError):
            pg.plan_batches(0, 4)
        with pytest.raises(ValueError):
            pg.plan_batches(5, 0)

    @pytest.mark.parametrize("kw", [dict(p_threshold=0.0), dict(batch_size=0), dict(top_k=0), dict(worker_count=0)])
    def test_validation_before_any_device_work(self, tmp_path, kw):
        spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=tmp_path / "x.bed", bim_path=tmp_path / "x.bim",
                             fam_path=tmp_path / "x.fam")
        with pytest.raises(ConfigError):
            pg.run_scan(pg.ScanConfig(source=spec, pheno_path=tmp_path / "p", out_path=tmp_path / "o", **kw))

    def test_premask_helpers(self):
        r = engine.abs_t_to_abs_r(np.array([0.0, 3.0, np.inf]), 10.0)
        assert r[0] == 0 and r[1] == pytest.approx(3 / np.sqrt(19)) and r[2] == 1.0
        bar = engine.topk_premask(np.array([-np.inf, 3.0, 50.0]), 40.0, 10.0)
        assert bar[0] == -1.0 and 0 < bar[1] < bar[2] < 1

    def test_summary_keys(self):
        s = engine.ScanSummary(*([1] * 18), exclusion_log={"remove-listed": 2})
        d = s.to_dict()
        assert d["excluded_remove-listed"] == 2 and "tests" not in d and len(d) == 19
        json.dumps(d)


# ----------------------------------------------------------------------------- simulator
class TestSimulate:
    def test_determinism_and_packing(self, tmp_path):
        spec = pg.SimSpec(seed=5, n_samples=30, n_markers=40, n_phenotypes=3, n_covariates=2, causal_fraction=0.1)
        a = pg.simulate_cohort(spec, tmp_path / "a")
        b = pg.simulate_cohort(spec, tmp_path / "b")
        for k in ("bed_path", "pheno_path", "covar_path", "truth_path"):
            assert getattr(a, k).read_bytes() == getattr(b, k).read_bytes()
        from paper_2604_21095_b200.simulate import pack_bed_codes

        assert pack_bed_codes(np.array([[2.0, 1.0, np.nan, 0.0]])).tolist() == [[0b11011000]]
        with pytest.raises(PanelGwasError, match="hard call"):
            pack_bed_codes(np.array([[0.5]]))
        with pytest.raises(ConfigError):
            pg.SimSpec(seed=1, n_samples=0, n_markers=1, n_phenotypes=1)


def test_bim_native_path_equals_line_reader(tmp_path):
    from paper_2604_21095_b200.genotypes import plink

    lines = [f"{1 + i % 22}\trs{i}\t0.{i}\t{100 * i + 7}\t{'ACGT'[i % 4]}\t{'TGCA'[i % 4]}" for i in range(500)]
    lines.insert(10, "")  # blank lines are skipped by both
    lines[20] = "  " + lines[20].replace("\t", "   ") + "  "  # any whitespace between fields
    p = tmp_path / "a.bim"
    p.write_text("\n".join(lines) + "\n")
    fast = plink._parse_bim_native(p)
    assert fast is not None and fast == plink._parse_bim_lines(p)
    assert [r.source_index for r in fast] == list(range(500))
    bad = tmp_path / "b.bim"
    bad.write_text("1 rs1 0 5 A G\n1 rs2 0 6 A\n")
    assert plink._parse_bim_native(bad) is None
    with pytest.raises(FormatError, match="expected 6 columns"):
        plink._parse_bim(bad)
    neg = tmp_path / "c.bim"
    neg.write_text("1 rs1 0 -5 A G\n")
    with pytest.raises(FormatError, match="negative position"):
        plink._parse_bim(neg)


def test_marker_catalog_behaves_like_the_reference_list():
    """Sources expose marker_catalog as a lazy column catalog; it must read like the
    reference's list[MarkerRecord] (indexing, slicing, iteration, equality, len)."""
    from paper_2604_21095_b200.genotypes.types import MarkerCatalog, MarkerRecord

    cols = (["1", "2", "X"], ["rs1", "rs2", "rs3"], [10, 20, 30], ["A", "C", "G"], ["T", "G", "A"])
    want = [MarkerRecord(c, i, p, a, b, k) for k, (c, i, p, a, b) in enumerate(zip(*cols))]
    cat = MarkerCatalog(*cols)
    assert len(cat) == 3 and list(cat) == want and cat == want
    assert cat[0] == want[0] and cat[-1] == want[2]
    assert cat[1:] == want[1:] and cat[1:][0].source_index == 1
    assert cat[::2] == want[::2]
    assert [m.id for m in cat[1:3]] == ["rs2", "rs3"]
    assert cat[1:].prefixes(True) == ["2\trs2\t20\tC\tG\t", "X\trs3\t30\tG\tA\t"]
    assert cat.prefixes(False)[0] == "1\trs1\t10\tT\tA\t"
    assert cat[1:].source_indices().tolist() == [1, 2]
    with pytest.raises(IndexError):
        cat[3]


@pytest.mark.parametrize("text", [
    "1\trs1\t0\t10\tA\tG\n2 rs2 0.5 +20 C T\r\n\n  X\trs3\t0\t007\tG\tG  \n",  # plain, CRLF, blank, '+', '007'
    "1\trs1\t0\t10\tA\tG",                        # no final newline
    "1\trs1\t0\t1_000\tA\tG\n",                   # Python int() digit groups: generic reader
    "1\trs1\t0\t-5\tA\tG\n",                      # negative position: the reference's error
    "1\trs1\t0\t10\tA\n",                         # 5 fields
    "1\trs1\t0\t10\tA\tG\tx\n",                   # 7 fields
    "1\trs1\t0\t10\tA\tG\r2\trs2\t0\t5\tA\tG\n",   # bare CR: a line break for Python
    "1\trsé\t0\t10\tA\tG\n",                      # non-ASCII
    "1\trs1\t0\tten\tA\tG\n",                     # bad position
])
def test_native_bim_index_equals_line_reader(tmp_path, text):
    """pg_bim_index + ByteCatalog give the line-by-line reader's catalog, or defer to it."""
    from paper_2604_21095_b200.errors import FormatError
    from paper_2604_21095_b200.genotypes import plink

    path = tmp_path / "g.bim"
    path.write_bytes(text.encode())
    try:
        want = plink._parse_bim_lines(path)
    except FormatError as exc:
        want = exc
    native = plink._parse_bim_native(path)
    if isinstance(want, FormatError):
        assert native is None
        with pytest.raises(FormatError, match=str(want).split(": ", 1)[1][:20]):
            plink._parse_bim(path)
        return
    got = plink._parse_bim(path)
    assert list(got) == want and len(got) == len(want)
    if native is not None:
        assert got[1:].prefixes(False) == [f"{m.chrom}\t{m.id}\t{m.pos}\t{m.allele2}\t{m.allele1}\t" for m in want[1:]]


def test_device_batch_sizes(monkeypatch):
    """Markers per device launch: PLINK 65,536; dosage sources 8,192 by default and up to
    32,768 through --batch-size with wide digits (8,192 with the ternary planes); FULL and
    K-sliced runs shrink it to their memory bounds; never more markers than the scan has."""
    from pathlib import Path

    import paper_2604_21095_b200 as pg
    from paper_2604_21095_b200.engine import device_batch_size

    def cfg(fmt, **kw):
        spec = pg.SourceSpec(fmt, bed_path=Path("a.bed"), bim_path=Path("a.bim"), fam_path=Path("a.fam"),
                             bgen_path=Path("a.bgen"))
        return pg.ScanConfig(source=spec, pheno_path=Path("p.tsv"), out_path=Path("o.tsv"), **kw)

    plink, bgen = pg.GenotypeFormat.PLINK_BED, pg.GenotypeFormat.BGEN
    assert device_batch_size(cfg(plink), 10**6, 20480, 23000) == 65536
    assert device_batch_size(cfg(plink), 1000, 20480, 23000) == 1000
    assert device_batch_size(cfg(bgen), 10**6, 4096, 23000) == 8192
    assert device_batch_size(cfg(bgen, batch_size=32768), 10**6, 4096, 23000) == 32768
    assert device_batch_size(cfg(bgen, batch_size=10**6), 10**6, 4096, 23000) == 32768
    monkeypatch.setenv("PANELGWAS_WIDE_DIGITS", "0")
    assert device_batch_size(cfg(bgen, batch_size=32768), 10**6, 4096, 23000) == 8192
    monkeypatch.delenv("PANELGWAS_WIDE_DIGITS")
    full = device_batch_size(cfg(plink, output_mode=pg.OutputMode.FULL), 10**6, 20480, 23000)
    assert 256 <= full < 65536
    sliced = device_batch_size(cfg(plink), 10**6, 20480, 500_000)
    assert 256 <= sliced < 65536


def test_device_batch_bounds_candidates(tmp_path):
    """THRESHOLD / TOPK device batches keep the expected candidate pairs under the budget:
    at p = 1 (every pair a candidate) a C3-sized scan shrinks its 65,536-marker launches so
    markers x phenotypes stays far below 2^31 (the round-1 int32 counter overflowed here)."""
    from paper_2604_21095_b200 import engine

    spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=tmp_path / "g.bed")
    P = 20480
    for kw in ({"p_threshold": 1.0}, {"p_threshold": 0.3}, {"output_mode": pg.OutputMode.TOPK, "top_k": 16384}):
        cfg = pg.ScanConfig(source=spec, pheno_path=tmp_path / "p", out_path=tmp_path / "o", batch_size=131072,
                            **kw)
        b = engine.device_batch_size(cfg, 1_000_000, P, 23000)
        assert b * P <= engine._CAND_BUDGET * 1.01 and b * P < 2**31, (kw, b)
    cfg = pg.ScanConfig(source=spec, pheno_path=tmp_path / "p", out_path=tmp_path / "o", p_threshold=1e-4)
    assert engine.device_batch_size(cfg, 1_000_000, P, 23000) == 65536  # the C3 default is unchanged
