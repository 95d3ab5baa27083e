"""Smoothing step / kernel timings at larger sizes of the paper's circle (Q2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

for nlev in (10, 11, 12):
    w = workloads.Workload(f"paper-circle-Q2-{2 << (nlev - 1)}", -1.105, -1.105, 2.21, 2, nlev, 0.0, 0.0, 1.0, 2)
    g = cutfem.Problem.from_workload(w)
    L = nlev - 1
    info = g.level_info(L)
    x = g.to_device(np.random.default_rng(1).standard_normal(info.nl * info.nl))
    b = g.to_device(np.random.default_rng(2).standard_normal(info.nl * info.nl))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def t(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.fill_(1.0)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); fn(); e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return float(np.median(ts))
    ms = t(lambda: g.smooth(L, x, b))
    cart = t(lambda: g.colour_step(L, 2, 0, x, b))
    cut = t(lambda: g.colour_step(L, 3, 0, x, b)) / (4 * w.n_c)   # one cut step of the ping-pong sweeps
    z = g.zeros()
    vc = t(lambda: (z.zero_(), g.vcycle(z, b)), 5)
    cart_bytes = 24.0 * 4 * info.n_inside
    cut_bytes = sum(info.cut_step_bytes[:4]) / 4.0
    print(f"n={info.n} dofs={info.n_dofs} step={ms*1e3:.1f}us ({info.n_dofs/ms/1e6:.3g} DoF/s) "
          f"cart_sweep={cart*1e3:.1f}us ({cart_bytes/cart/1e6:.0f} GB/s) cut_step={cut*1e3:.1f}us "
          f"({cut_bytes/cut/1e6:.0f} GB/s) vcycle={vc:.2f}ms cut patches/colour={list(info.n_cutp)[:4]}", flush=True)
    g.close()
