"""Per level of config1: the cut sweep (colour_step kind 3) as one launch
(k_cut_sweep) vs the launch-per-colour-step chain (CUTFEM_SWEEP=0), and the
Cartesian sweep, warm (no L2 flush: the V-cycle regime), median of 50."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

w = getattr(workloads, os.environ.get("WL", "CONFIG1"))


def timed(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    return float(np.median(out))


probs = {}
for tag, env in (("sweep", {}), ("chain", {"CUTFEM_SWEEP": "0"})):
    os.environ.update(env)
    probs[tag] = cutfem.Problem.from_workload(w)
    for k in env:
        os.environ.pop(k)
for l in range(w.n_levels):
    row = []
    for tag in ("sweep", "chain"):
        g = probs[tag]
        x = g.to_device(workloads.lattice_vector(w, 1, l), l)
        b = g.to_device(workloads.lattice_vector(w, 2, l), l)
        row.append(timed(lambda: g.colour_step(l, 3, 0, x, b)))
        if tag == "sweep":
            cart = timed(lambda: g.colour_step(l, 2, 0, x, b))
            info = g.level_info(l)
    print(f"level {l} n={info.n:4d}: cut sweep one-launch {row[0]:6.1f} us ({info.sweep_ctas[0]} CTAs, x{info.sweep_redundancy[0]:.1f})"
          f"  chain {row[1]:6.1f} us   cartesian {cart:6.1f} us", flush=True)
for tag, g in probs.items():
    bb = g.to_device(workloads.lattice_vector(w, 2))
    z = g.zeros()
    print(tag, "vcycle", round(timed(lambda: (z.zero_(), g.vcycle(z, bb)), 20), 1), "us")
