"""`python -m paper_2604_21095_b200 ...` — the panelgwas CLI.

Every output file is closed by the time main() returns, so the process leaves with os._exit
after flushing stdio: interpreter teardown (collecting millions of marker records, unmapping
the phenotype table) and CUDA context destruction would otherwise add about a second to a
C3-sized run without changing any result."""
import os
import sys

from .cli import main

code = main()
sys.stdout.flush()
sys.stderr.flush()
os._exit(code if isinstance(code, int) else 1)
