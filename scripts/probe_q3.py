"""3D Q3 (configs[3]'s degree) at growing sizes: setup time, device memory,
smoothing step / V-cycle / CG times (CUDA events), cut-patch statistics."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

for nlev in [int(a) for a in sys.argv[1:]] or [5, 6]:
    w = workloads.sphere(f"sphere-Q3-{2 ** nlev}", 2, nlev, 3)
    torch.cuda.synchronize()
    t = time.time()
    g = cutfem.Problem.from_workload(w)
    torch.cuda.synchronize()
    ts = time.time() - t
    L = w.n_levels - 1
    info = g.level_info(L)
    x = g.to_device(workloads.lattice_vector(w, 1))
    b = g.to_device(workloads.lattice_vector(w, 2))

    def tm(fn, n):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / n

    ms = tm(lambda: g.smooth(L, x, b), 3)
    z = g.zeros()
    vc = tm(lambda: (z.zero_(), g.vcycle(z, b)), 2)
    xs = g.zeros()
    torch.cuda.synchronize()
    t = time.time()
    it, rel = g.solve_cg_mg(xs, b, tol=1e-8, max_it=100)
    torch.cuda.synchronize()
    print(f"{w.name}: {info.n_dofs} DoFs, setup {ts:.1f} s, mem {torch.cuda.mem_get_info()}, "
          f"cut patches {sum(info.n_cutp[:8])}, method bytes/sweep {sum(info.cut_method_bytes[:8]) / 1e9:.2f} GB, "
          f"smooth {ms:.2f} ms = {info.n_dofs / ms * 1e3:.3e} DoF/s, vcycle {vc:.1f} ms, CG {it} it {time.time() - t:.2f} s",
          flush=True)
    g.close()
