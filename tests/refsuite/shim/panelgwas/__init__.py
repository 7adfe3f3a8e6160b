"""Alias package `panelgwas` -> the B200 drop-in `paper_2604_21095_b200` (TEST INFRASTRUCTURE).

Lets the reference's own test suite (/root/reference/pkg/tests, shipped as
oracle/_ref/reference_tests.zip) run unmodified against the drop-in: `import panelgwas`,
`from panelgwas.cli import main`, `python -m panelgwas.cli` all resolve to this package's
modules (registered once in sys.modules, so exception classes and module state are shared).
The reference's `panelgwas.oracle` (per-pair OLS) maps to the drop-in's `validation`.
`panelgwas.cli` is a real file (cli.py) so that `python -m panelgwas.cli` runs; on import it
replaces itself with the drop-in's cli module.
"""
import importlib
import sys

import paper_2604_21095_b200 as _impl
from paper_2604_21095_b200 import *  # noqa: F401,F403

__version__ = _impl.__version__
__all__ = list(getattr(_impl, "__all__", []))

_ALIASES = {
    "engine": "engine", "errors": "errors", "kernel": "kernel", "output": "output",
    "phenotypes": "phenotypes", "simulate": "simulate", "oracle": "validation", "genotypes": "genotypes",
    "genotypes.types": "genotypes.types", "genotypes.plink": "genotypes.plink", "genotypes.bgen": "genotypes.bgen",
    "genotypes.dense": "genotypes.dense",
}
for _alias, _target in _ALIASES.items():
    _mod = importlib.import_module(f"paper_2604_21095_b200.{_target}")
    sys.modules[f"{__name__}.{_alias}"] = _mod
    if "." not in _alias:
        globals()[_alias] = _mod
