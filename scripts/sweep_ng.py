"""Time the one-launch cut sweep of config1's finest level (and of the whole
V-cycle) for several CTA counts (CUTFEM_SWEEP_NG), L2 flushed before each
launch.  python scripts/sweep_ng.py [ng ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

w = getattr(workloads, os.environ.get("WL", "CONFIG1"))
L = w.n_levels - 1
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def timed(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(n):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    return float(np.median(out))


for ng in sys.argv[1:] or ["0"]:
    if ng != "0":
        os.environ["CUTFEM_SWEEP_NG"] = ng
    else:
        os.environ.pop("CUTFEM_SWEEP_NG", None)
    g = cutfem.Problem.from_workload(w)
    info = g.level_info(L)
    x = g.to_device(workloads.lattice_vector(w, 1))
    b = g.to_device(workloads.lattice_vector(w, 2))
    tf = timed(lambda: g.colour_step(L, 3, 0, x, b))
    tr = timed(lambda: g.colour_step(L, 3, 1, x, b)) if False else float("nan")
    ts = timed(lambda: g.smooth(L, x, b))
    z = g.zeros()
    tv = timed(lambda: (z.zero_(), g.vcycle(z, b)))
    print(f"ng={ng:>4s} ctas={info.sweep_ctas[0]:4d} red={info.sweep_redundancy[0]:.2f} "
          f"map={info.sweep_map_bytes[0] / 1e6:.1f}MB  cut sweep {tf:7.2f} us  step {ts:7.2f} us  vcycle {tv:7.1f} us",
          flush=True)
    g.close()
