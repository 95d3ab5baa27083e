"""Setup + timing of the 3D path on BASELINE configs[2] (sphere, Q2, 128^3)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

nlev = int(sys.argv[1]) if len(sys.argv) > 1 else 7
w = workloads.Workload(workloads.CONFIG2.name, *[getattr(workloads.CONFIG2, f) for f in
                       ("x0", "y0", "length", "n_coarse")], nlev,
                       *[getattr(workloads.CONFIG2, f) for f in ("cx", "cy", "r", "p", "n_c", "tol", "dim", "z0", "cz")])
t0 = time.time()
g = cutfem.Problem.from_workload(w)
torch.cuda.synchronize()
print(f"setup {time.time() - t0:.1f}s", flush=True)
L = nlev - 1
info = g.level_info(L)
print("n", info.n, "dofs", info.n_dofs, "cut cells", info.n_cut, "ghost", info.n_ghost_faces,
      "cart", list(info.n_cart), "cutp", list(info.n_cutp), flush=True)
x = g.to_device(workloads.lattice_vector(w, 1))
b = g.to_device(workloads.lattice_vector(w, 2))
def timed(fn, n=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
ms = timed(lambda: g.smooth(L, x, b))
print(f"smoothing step {ms:.3f} ms = {info.n_dofs / ms / 1e6:.3g} GDoF/s", flush=True)
cart = timed(lambda: g.colour_step(L, 0, 0, x, b))
cut = timed(lambda: g.colour_step(L, 1, 0, x, b))
print(f"cart colour {cart*1e3:.1f} us, cut colour {cut*1e3:.1f} us", flush=True)
z = g.zeros()
vms = timed(lambda: (z.zero_(), g.vcycle(z, b)), 3)
print(f"vcycle {vms:.2f} ms", flush=True)
xs = g.zeros()
t = time.time()
it, rel = g.solve_cg_mg(xs, b, tol=w.tol)
torch.cuda.synchronize()
print(f"cg {it} it rel {rel:.2e} in {(time.time()-t)*1e3:.1f} ms (incl. graph capture)", flush=True)
t = time.time()
it, rel = g.solve_cg_mg(xs, b, tol=w.tol)
torch.cuda.synchronize()
print(f"cg {it} it rel {rel:.2e} in {(time.time()-t)*1e3:.1f} ms", flush=True)
