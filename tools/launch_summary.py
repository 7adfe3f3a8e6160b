#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: this library's
kernels (namespace pg::) by total time, with their share of the library's device time."""
import csv
import sys
from collections import defaultdict


def main(path: str, title: str) -> None:
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    k, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    other = 0.0
    for r in rows[1:]:
        ns = float(r[v].replace(",", ""))
        if "pg::" in r[k] or "cub::" in r[k]:
            tot[r[k]] += ns
            cnt[r[k]] += 1
        else:
            other += ns
    total = sum(tot.values())
    print(title)
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised; compare shares)")
    print(f"# this library's kernels only; torch launches of the synthetic-data generator excluded ({other / 1e6:.1f} ms)")
    print(f"{'total_ms':>10} {'share':>6} {'calls':>5}  kernel")
    for name, ns in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{ns / 1e6:10.3f} {100 * ns / total:5.1f}% {cnt[name]:5d}  {name[:130]}")
    print(f"{total / 1e6:10.3f} 100.0% {sum(cnt.values()):5d}  (library total)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "# launch list")
