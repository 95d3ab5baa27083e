"""Per-level timing of the cut sweeps (colour_step kind 3) and smoothing step,
dataflow kernel (default) vs one launch per cut step (CUTFEM_DF=0), config1.
Warm (back to back) and with the L2 flushed before every call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

w = getattr(workloads, sys.argv[1]) if len(sys.argv) > 1 else workloads.CONFIG1
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def mk(env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return cutfem.Problem.from_workload(w)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v


def timed(fn, n=50, fl=False):
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    if not fl:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / n * 1e3
    for _ in range(n):
        flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / n * 1e3


envs = [("df", {}), ("step", {"CUTFEM_DF": "0"})] + [(f"df-{k}={v}", {k: v}) for k, v in
                                                        (a.split("=") for a in sys.argv[2:])]
gs = [(n, mk(e)) for n, e in envs]
for l in range(1, w.n_levels):
    row = []
    for name, g in gs:
        x = g.to_device(workloads.lattice_vector(w, 1, l), l)
        b = g.to_device(workloads.lattice_vector(w, 2, l), l)
        row.append(f"{name}: cut {timed(lambda: g.colour_step(l, 3, 0, x, b)):.1f}/"
                   f"{timed(lambda: g.colour_step(l, 3, 0, x, b), 20, True):.1f}fl "
                   f"smooth {timed(lambda: g.smooth(l, x, b)):.1f}")
    print(f"level {l} n={g.level_info(l).n}: " + " | ".join(row), flush=True)
for name, g in gs:
    z = g.zeros()
    b = g.to_device(workloads.lattice_vector(w, 2))
    print(name, "vcycle us", timed(lambda: (z.zero_(), g.vcycle(z, b)), 20))
