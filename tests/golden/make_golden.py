"""Generate the golden fixtures by running the REFERENCE implementation.

Run here (the reference is importable only in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything written to tests/golden/ is data produced by /root/reference/pkg
(panelgwas 0.1.0) on seeded inputs; the GPU box never reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import panelgwas as ref  # noqa: E402
from panelgwas import kernel as rk  # noqa: E402
from bgen_writer import write_bgen  # noqa: E402  (reference test helper)

OUT = Path(__file__).resolve().parent


def sha(path: Path) -> str:
    return hashlib.sha256(Path(path).read_bytes()).hexdigest()


def records_arrays(path: Path, markers_index: dict, pheno_index: dict) -> dict:
    recs = ref.load_association_records(path)
    return {
        "rows": np.array([markers_index[r.id] for r in recs], dtype=np.int64),
        "cols": np.array([pheno_index[r.phenotype] for r in recs], dtype=np.int64),
        "r": np.array([r.r for r in recs]),
        "t": np.array([r.t for r in recs]),
        "p": np.array([r.p for r in recs]),
        "af": np.array([r.af for r in recs]),
        "n_miss": np.array([r.missing_count for r in recs], dtype=np.int64),
    }


def make_decode() -> None:
    rng = np.random.default_rng(606)
    fixed = [(bytes([0b11011000]), 4), (b"\x00", 4), (b"\xff", 4), (bytes([0b01010101]), 4),
             (bytes([0b11100000]), 3), (bytes([0b00011011, 0b11100100]), 8)]
    out = {}
    for i, (b, n) in enumerate(fixed):
        out[f"fixed{i}_bytes"] = np.frombuffer(b, dtype=np.uint8)
        out[f"fixed{i}_n"] = np.int64(n)
        out[f"fixed{i}_dosage"] = ref.decode_bed_codes(b, n)
    n = 37
    bpm = (n + 3) // 4
    packed = rng.integers(0, 256, size=(64, bpm), dtype=np.uint8)
    out["rand_packed"] = packed
    out["rand_n"] = np.int64(n)
    out["rand_dosage"] = np.stack([ref.decode_bed_codes(packed[i].tobytes(), n) for i in range(64)])
    np.savez_compressed(OUT / "decode.npz", **out)


def make_pvalues() -> None:
    rng = np.random.default_rng(7)
    t = np.concatenate([[0.0, 1e-8, 0.5, 1.0, 1.96, 3.0, 3.8912744581499874, 10.0, 38.0, 40.0, 60.0,
                         np.inf, -np.inf, -2.5], rng.standard_normal(200) * 6])
    dfs = np.array([1.0, 2.0, 3.0, 10.0, 58.0, 298.0, 1998.0, 22998.0, 1e6])
    p = np.stack([ref.p_from_t(t, df) for df in dfs])
    crit_cases = [(1e-4, 22998.0), (1e-4, 1998.0), (0.05, 10.0), (1e-8, 100.0), (1.0, 5.0), (0.2, 40.0),
                  (1e-300, 22998.0), (2.2250738585072014e-308, 22998.0), (1e-6, 198.0)]
    crit = np.array([ref.t_threshold_for_p(a, b) for a, b in crit_cases])
    a = rng.uniform(0.1, 50.0, 300)
    b = rng.uniform(0.1, 50.0, 300)
    x = rng.uniform(0.0, 1.0, 300)
    ib = ref.reg_inc_beta(a, b, x)
    r = np.concatenate([[0.0, 0.5, -0.5, 1.0, -1.0, 0.999999999, 1e-12], rng.uniform(-1, 1, 100)])
    tr = np.stack([ref.t_from_r(r, df) for df in (2.0, 11.0, 22998.0)])
    np.savez_compressed(OUT / "pvalues.npz", t=t, dfs=dfs, p=p, crit_cases=np.array(crit_cases), crit=crit,
                        ib_a=a, ib_b=b, ib_x=x, ib=ib, r=r, t_from_r=tr)


def make_prepare() -> None:
    rng = np.random.default_rng(12)
    d = rng.integers(0, 3, size=(40, 57)).astype(np.float64)
    d[rng.random(d.shape) < 0.08] = np.nan
    d[3] = 2.0
    d[7] = np.nan
    d[11] = 1.0
    d[11, 5] = np.nan
    d[20, :] = np.nan
    d[20, 9] = 0.0
    d[0] = [0.0, 1.0, 2.0, 1.0] * 14 + [0.0]
    raw = ref.RawBatch(tuple(ref.MarkerRecord("1", f"m{i}", i, "A", "B", i) for i in range(40)), d,
                       np.isnan(d).sum(axis=1))
    std = ref.prepare_genotype_batch(raw)
    np.savez_compressed(OUT / "prepare.npz", dosages=d, matrix=std.matrix, af=std.allele_frequency,
                        missing=std.missing_count, variance=std.variance_before_scaling, skip=std.skip_reason)


def scan_fixture(name: str, spec_kw: dict, runs: dict) -> None:
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        spec = ref.SimSpec(**spec_kw)
        cohort = ref.simulate_cohort(spec, tmp / "data")
        files = {k: sha(getattr(cohort, k)) for k in ("bed_path", "bim_path", "fam_path", "pheno_path", "truth_path")}
        if cohort.covar_path:
            files["covar_path"] = sha(cohort.covar_path)
        src = ref.SourceSpec(ref.GenotypeFormat.PLINK_BED, bed_path=cohort.bed_path, bim_path=cohort.bim_path,
                             fam_path=cohort.fam_path)
        mindex = {f"snp{i + 1}": i for i in range(spec.n_markers)}
        pindex = {f"ph{j + 1}": j for j in range(spec.n_phenotypes)}
        arrays = {}
        meta = {"spec": spec_kw, "sha256": files, "runs": {}}
        for run_name, kw in runs.items():
            out = tmp / f"{run_name}.out"
            cfg = ref.ScanConfig(source=src, pheno_path=cohort.pheno_path, out_path=out,
                                 covar_path=cohort.covar_path, summary_to_stderr=False, **kw["config"])
            summary = ref.run_scan(cfg)
            meta["runs"][run_name] = {"config": {k: (v.value if hasattr(v, "value") else v)
                                                 for k, v in kw["config"].items()},
                                      "summary": {k: v for k, v in summary.to_dict().items()
                                                  if not k.startswith("time_") and k != "wall_s"}}
            if kw["config"].get("output_mode") is ref.OutputMode.FULL:
                tmat, lines, phenos = ref.read_full_matrix(out)
                keep = np.array([int(ln.split("\t")[0]) for ln in lines], dtype=np.int64)
                sub = kw.get("row_stride", 1)
                arrays[f"{run_name}_t"] = tmat[::sub]
                arrays[f"{run_name}_rows"] = keep[::sub]
                if kw.get("keep_bytes"):
                    (OUT / f"{name}_{run_name}.bin").write_bytes(out.read_bytes())
            else:
                for k, v in records_arrays(out, mindex, pindex).items():
                    arrays[f"{run_name}_{k}"] = v
                if kw.get("keep_bytes"):
                    (OUT / f"{name}_{run_name}.tsv").write_bytes(out.read_bytes())
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")


def make_bgen() -> None:
    rng = np.random.default_rng(23)
    m, n = 30, 45
    d = np.round(rng.uniform(0, 2, size=(m, n)) * 20) / 20
    d[rng.random(d.shape) < 0.06] = np.nan
    d[4] = 1.0
    ids = [f"S{i + 1}" for i in range(n)]
    y = rng.standard_normal((n, 3))
    out = {"dosage_in": d, "y": y}
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        for bits in (8, 16):
            path = write_bgen(tmp / f"g{bits}.bgen", d, ids, bits=bits)
            (OUT / f"bgen{bits}.bgen").write_bytes(path.read_bytes())
            src = ref.BgenSource(path)
            raw = src.read_marker_batch(0, m)
            src.close()
            out[f"b{bits}_dosage"] = raw.dosages
            out[f"b{bits}_missing"] = raw.missing_count
            pheno = tmp / "pheno.tsv"
            with open(pheno, "w") as fh:
                fh.write("IID\tph1\tph2\tph3\n")
                for i, sid in enumerate(ids):
                    fh.write(sid + "\t" + "\t".join(repr(float(v)) for v in y[i]) + "\n")
            (OUT / "bgen_pheno.tsv").write_bytes(pheno.read_bytes())
            cfg = ref.ScanConfig(source=ref.SourceSpec(ref.GenotypeFormat.BGEN, bgen_path=path), pheno_path=pheno,
                                 out_path=tmp / "o.tsv", p_threshold=1.0, precision=ref.Precision.F64,
                                 summary_to_stderr=False)
            ref.run_scan(cfg)
            recs = ref.load_association_records(tmp / "o.tsv")
            out[f"b{bits}_rows"] = np.array([int(r.id[2:]) - 1 for r in recs])
            out[f"b{bits}_cols"] = np.array([int(r.phenotype[2:]) - 1 for r in recs])
            out[f"b{bits}_t"] = np.array([r.t for r in recs])
            out[f"b{bits}_p"] = np.array([r.p for r in recs])
            out[f"b{bits}_af"] = np.array([r.af for r in recs])
    np.savez_compressed(OUT / "bgen.npz", **out)


def make_ols() -> None:
    """Effect sizes from the reference's own per-pair OLS (oracle.ols_single, oracle.py:35-90)
    on the s1 and c1 cohorts: y ~ 1 + C + g (the extension-mode / adjusted-df target) and the
    marginal slope of the covariate-residualized phenotype y_res ~ 1 + g (the paper-mode
    target), g mean-imputed as prepare_genotype_batch does (kernel.py:392-408)."""
    rng = np.random.default_rng(2024)
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        for name, kw, n_pairs in (("s1", S1_SPEC, 1200), ("c1", C1_SPEC, 400)):
            spec = ref.SimSpec(**kw)
            cohort = ref.simulate_cohort(spec, tmp / name)
            n, m = spec.n_samples, spec.n_markers
            ids = [f"S{i + 1}" for i in range(n)]
            src = ref.PlinkSource(cohort.bed_path, cohort.bim_path, cohort.fam_path)
            dos = src.read_marker_batch(0, m).dosages
            src.close()
            ptab = ref.load_table(cohort.pheno_path)
            ctab = ref.load_table(cohort.covar_path)
            align = ref.align_samples(ids, ptab, ctab)
            y = ref.build_panel(ptab, align).y
            c = ref.covariate_matrix(ctab, align)
            basis = rk.build_covariate_basis(c, True)
            y_res = rk.residualize(y, basis)
            rows = rng.integers(0, m, n_pairs)
            cols = rng.integers(0, spec.n_phenotypes, n_pairs)
            res = {"beta_adj": [], "se_adj": [], "t_adj": [], "beta_paper": [], "se_paper": [], "t_paper": []}
            for i, j in zip(rows.tolist(), cols.tolist()):
                g = dos[i].copy()
                miss = np.isnan(g)
                g[miss] = g[~miss].mean()
                a = ref.ols_single(y[:, j], g, c)
                b = ref.ols_single(y_res[:, j], g)
                for key, o in (("adj", a), ("paper", b)):
                    res[f"beta_{key}"].append(o.beta)
                    res[f"se_{key}"].append(o.se)
                    res[f"t_{key}"].append(o.t)
            out[f"{name}_rows"] = rows
            out[f"{name}_cols"] = cols
            for k, v in res.items():
                out[f"{name}_{k}"] = np.array(v)
    np.savez_compressed(OUT / "ols.npz", **out)


S1_SPEC = dict(seed=11, n_samples=300, n_markers=600, n_phenotypes=12, n_covariates=3, causal_fraction=0.03,
               effect_sd=0.3, genotype_missing_rate=0.02, phenotype_missing_rate=0.01)
C1_SPEC = dict(seed=1, n_samples=2000, n_markers=10000, n_phenotypes=64, n_covariates=10, causal_fraction=0.01,
               effect_sd=0.15)


def main() -> None:
    if sys.argv[1:] == ["ols"]:
        make_ols()
        print("ols fixture written to", OUT)
        return
    make_decode()
    make_pvalues()
    make_prepare()
    F64 = ref.Precision.F64
    scan_fixture(
        "s1",
        S1_SPEC,
        {
            "all_f64": {"config": dict(p_threshold=1.0, precision=F64)},
            "thr_f64": {"config": dict(p_threshold=1e-3, precision=F64), "keep_bytes": True},
            "thr_f32": {"config": dict(p_threshold=1e-3)},
            "topk_f64": {"config": dict(output_mode=ref.OutputMode.TOPK, top_k=5, precision=F64), "keep_bytes": True},
            "full_f64": {"config": dict(output_mode=ref.OutputMode.FULL, precision=F64)},
            "adj_f64": {"config": dict(p_threshold=1.0, precision=F64, df_mode=ref.DfMode.ADJUSTED,
                                       residualize_genotypes=True)},
        },
    )
    scan_fixture(
        "c1",
        C1_SPEC,
        {
            "thr_f64": {"config": dict(p_threshold=1e-4, precision=F64)},
            "thr_f32": {"config": dict(p_threshold=1e-4)},
            "full_f64": {"config": dict(output_mode=ref.OutputMode.FULL, precision=F64), "row_stride": 13},
        },
    )
    make_bgen()
    make_ols()
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
