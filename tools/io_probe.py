#!/usr/bin/env python
"""Host write-path probe for FULL output: GB/s of writing a 1 GiB block to a file in the page
cache (single write vs N-thread pwrite at disjoint offsets; pageable vs pinned source)."""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def run(path, buf, threads, reps=4):
    mv = memoryview(buf).cast("B")
    n = mv.nbytes
    fd = os.open(path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
    pool = ThreadPoolExecutor(threads) if threads > 1 else None
    best = 1e9
    for r in range(reps):
        base = r * n
        t0 = time.perf_counter()
        if pool is None:
            done = 0
            while done < n:
                done += os.pwrite(fd, mv[done:], base + done)
        else:
            cuts = [n * k // threads for k in range(threads + 1)]
            list(pool.map(lambda k: os.pwrite(fd, mv[cuts[k]:cuts[k + 1]], base + cuts[k]), range(threads)))
        best = min(best, time.perf_counter() - t0)
    os.close(fd)
    os.unlink(path)
    return n / best / 1e9


def main():
    from paper_2604_21095_b200 import _native

    n = 1 << 30
    page = np.ones(n, np.uint8)
    pin = _native.PinnedBuffer(n)
    pin.array[:] = 1
    out = {}
    for name, buf in (("pageable", page), ("pinned", pin.array)):
        for th in (1, 2, 4, 8):
            out[f"{name}_t{th}_GBps"] = round(run("/tmp/io_probe.bin", buf, th), 2)
    t0 = time.perf_counter()
    b2 = _native.PinnedBuffer(n)
    out["pin_alloc_1GiB_s"] = round(time.perf_counter() - t0, 3)
    b2.close()
    pin.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
