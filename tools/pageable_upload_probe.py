#!/usr/bin/env python
"""Wall time of pg_ctx_prepare_panel on a pageable C3-size phenotype matrix (the CLI path:
threaded copies into pinned bounce buffers, H2D, device preparation) vs a pinned one."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_21095_b200._device import DeviceContext  # noqa: E402


def main():
    n, p = 23000, 20480
    y = np.random.default_rng(1).standard_normal((n, p))
    yp = torch.empty((n, p), dtype=torch.float64).pin_memory()
    yp.numpy()[...] = y
    with DeviceContext(0) as ctx:
        for name, arr in (("pageable", y), ("pinned", yp.numpy()), ("pageable", y), ("pinned", yp.numpy())):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.prepare_panel(arr, None)
            print(f"prepare_panel {name:8s} {1e3 * (time.perf_counter() - t0):7.1f} ms")


if __name__ == "__main__":
    main()
