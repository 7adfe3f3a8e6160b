"""`panelgwas.cli` -> `paper_2604_21095_b200.cli` (TEST INFRASTRUCTURE). A file rather than a
sys.modules alias so `python -m panelgwas.cli` (reference tests/test_cli.py:274-279) can run it."""
import sys

from paper_2604_21095_b200 import cli as _cli

if __name__ == "__main__":
    raise SystemExit(_cli.main())
sys.modules[__name__] = _cli
