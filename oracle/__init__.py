"""TEST INFRASTRUCTURE ONLY — never imported by the product package.

CPU restatement (numpy) of the reference `panelgwas` scan path, used as the
parity checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg. Pinned against golden vectors produced by running the
reference itself (tests/golden/make_golden.py); see oracle/scan_oracle.py.
"""
