#!/usr/bin/env python
"""Do host-to-device copies on different streams overtake each other? Issues a C3-size
pipelined panel upload (pg_ctx_set_panel_async), then a 47 MB pinned copy on another stream,
and prints when that copy completes vs when the panel is done (wall clock, diagnostics).
With every chunk copy issued at once (before lazy issuing) the 47 MB copy completed at
59-69 ms, together with the 3.77 GB panel: copies run in submission order."""
import sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2604_21095_b200._device import DeviceContext
from paper_2604_21095_b200.kernel import build_covariate_basis
n, p = 23000, 20480
dev = torch.device("cuda:0")
yh = torch.randn(n, p, dtype=torch.float64).pin_memory()
c = np.random.default_rng(1).standard_normal((n, 10))
basis = build_covariate_basis(c, True)
gidx = np.arange(n, dtype=np.int64)
src = torch.empty(47_000_000, dtype=torch.uint8).pin_memory()
dst = torch.empty(47_000_000, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream()
with DeviceContext(0) as ctx:
    for rep in range(3):
        ctx.set_panel_async(yh.numpy(), basis.q, gidx, n, chunk_cols=2560)
        t0 = time.perf_counter()
        with torch.cuda.stream(st):
            dst.copy_(src, non_blocking=True)
        st.synchronize()
        t1 = time.perf_counter()
        ctx.panel_async_wait()
        t2 = time.perf_counter()
        print(f"47 MB H2D issued after the panel chunks: {1e3*(t1-t0):.1f} ms; panel done at {1e3*(t2-t0):.1f} ms")
