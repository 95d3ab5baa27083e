"""Per-level timing of the V-cycle building blocks on config1 (events, no
profiler): smoothing step, cut sweeps (kind 3), fused Cartesian sweep
(kind 2), operator apply, restriction, prolongation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

w = workloads.CONFIG1
g = cutfem.Problem.from_workload(w)


def timed(fn, n=50):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


for l in range(1, w.n_levels):
    info = g.level_info(l)
    x = g.to_device(workloads.lattice_vector(w, 1, l), l)
    b = g.to_device(workloads.lattice_vector(w, 2, l), l)
    y = g.zeros(l)
    c = g.zeros(l - 1)
    t_s = timed(lambda: g.smooth(l, x, b))
    t_cut = timed(lambda: g.colour_step(l, 3, 0, x, b))
    t_cart = timed(lambda: g.colour_step(l, 2, 0, x, b))
    t_a = timed(lambda: g.apply_operator(l, x, y))
    t_r = timed(lambda: g.restrict(l, x, c))
    t_p = timed(lambda: g.prolongate_add(l, c, x))
    print(f"level {l} n={info.n} cutp={list(info.n_cutp)[:4]} smooth {t_s:.1f} us  cut sweeps {t_cut:.1f}  "
          f"cart {t_cart:.1f}  apply {t_a:.1f}  restrict {t_r:.1f}  prolong {t_p:.1f}", flush=True)
