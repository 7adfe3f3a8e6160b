"""Shared helpers: regenerate the golden cohorts locally and build oracle inputs."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLD = Path(__file__).parent / "golden"


def spec_of(name: str) -> dict:
    return json.loads((GOLD / f"{name}.json").read_text())["spec"]


def regenerate(name: str, out_dir: Path) -> dict:
    """Write the cohort with this package's simulator (byte-identical to the reference's)."""
    from paper_2604_21095_b200.simulate import SimSpec, simulate_cohort

    kw = dict(spec_of(name))
    if "af_range" in kw:
        kw["af_range"] = tuple(kw["af_range"])
    c = simulate_cohort(SimSpec(**kw), Path(out_dir) / name)
    return {"bed_path": c.bed_path, "bim_path": c.bim_path, "fam_path": c.fam_path,
            "pheno_path": c.pheno_path, "covar_path": c.covar_path, "truth_path": c.truth_path}


def oracle_inputs(name: str, out_dir: Path):
    """(dosages [M, N], ytil [N, P], df, paths) for the oracle, from regenerated files."""
    from oracle import scan_oracle as orc
    from paper_2604_21095_b200 import phenotypes

    paths = regenerate(name, out_dir)
    spec = spec_of(name)
    n, m = spec["n_samples"], spec["n_markers"]
    bpm = (n + 3) // 4
    blob = np.frombuffer(Path(paths["bed_path"]).read_bytes()[3:], dtype=np.uint8).reshape(m, bpm)
    dos = orc.decode_bed(blob, n)
    ids = [f"S{i + 1}" for i in range(n)]
    ptab = phenotypes.load_table(paths["pheno_path"])
    ctab = phenotypes.load_table(paths["covar_path"]) if paths["covar_path"] else None
    align = phenotypes.align_samples(ids, ptab, ctab)
    panel = phenotypes.build_panel(ptab, align)
    c = phenotypes.covariate_matrix(ctab, align) if ctab is not None else np.zeros((n, 0))
    q = orc.covariate_basis(c)
    ytil, zero = orc.standardized_panel(panel.y, q)
    assert not zero.any()
    return dos, ytil, float(n - 2), paths


def panel_inputs(name: str, out_dir: Path):
    """(dosages [M, N], imputed panel y [N, P], covariates C [N, c], basis Q, paths) of a golden
    cohort, regenerated locally, with the package's host table logic (reference behaviour)."""
    from oracle import scan_oracle as orc
    from paper_2604_21095_b200 import phenotypes

    paths = regenerate(name, out_dir)
    spec = spec_of(name)
    n, m = spec["n_samples"], spec["n_markers"]
    bpm = (n + 3) // 4
    blob = np.frombuffer(Path(paths["bed_path"]).read_bytes()[3:], dtype=np.uint8).reshape(m, bpm)
    dos = orc.decode_bed(blob, n)
    ids = [f"S{i + 1}" for i in range(n)]
    ptab = phenotypes.load_table(paths["pheno_path"])
    ctab = phenotypes.load_table(paths["covar_path"])
    align = phenotypes.align_samples(ids, ptab, ctab)
    y = phenotypes.build_panel(ptab, align).y
    c = phenotypes.covariate_matrix(ctab, align)
    return dos, y, c, orc.covariate_basis(c), paths


def load_cohort(name: str):
    return np.load(GOLD / f"{name}.npz")
