"""Full-size parity goldens of the benchmarked calls, computed by the ORACLE only.

Writes tests/golden/fullsize_<name>.npz for
  * config1 (BASELINE.json configs[1]: circle, Q2, 512^2, 680 065 DoFs) and
  * a 3D sphere at 64^3 cells, Q2 (the multi-wave 3D level of configs[2]'s
    hierarchy; 128^3 is out of reach of the oracle's per-patch Python loops),
with, from the seeded inputs x0 = lattice_vector(w, 31), b = lattice_vector(w, 32)
(each side masks them with its own DoF mask):
  y_fwd = S(x0, b)            one forward smoothing step on the finest level
                              (P eq. smoother-split, l.196-210)
  y_rev = S^T(x0, b)          the reverse (post-)smoothing step (reading R9)
  v     = V(b)                one V-cycle from x = 0 (P l.124, l.217)
  cg_it, cg_rel               CG + V-cycle to ||r|| <= 1e-8 ||b|| (north_star)
as float64 values in the oracle's DoF order.  config1's GPU test builds the
oracle live instead (~2 min); the 3D file stores the outputs on a fixed
subset to stay small: every DoF whose node lies within 3 h of the sphere
(where the cut patches act) and every 11th other DoF (`idx`).  No value comes
from the CUDA path.  The GPU tests (tests/test_gpu_fullsize.py,
tests/test_gpu_3d.py) compare against these.

    python scripts/make_fullsize_goldens.py [config1] [sphere64]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from oracle.solver import from_workload  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
CASES = {
    "config1": workloads.CONFIG1,
    "sphere64": workloads.sphere("sphere-Q2-64^3", 2, 6, 2),
}


def make(name):
    w = CASES[name]
    t = time.time()
    h = from_workload(w)
    lv = h.fine.lv
    print(f"{name}: oracle hierarchy {time.time() - t:.0f} s, {lv.n_dofs} DoFs", flush=True)
    x0 = workloads.lattice_vector(w, 31)[lv.dof_nodes]
    b = workloads.lattice_vector(w, 32)[lv.dof_nodes]
    y_fwd = h.fine.smooth(x0.copy(), b, w.n_c)
    y_rev = h.fine.smooth(x0.copy(), b, w.n_c, reverse=True)
    v = h.precondition(b)
    _, it, hist = h.solve_cg(b, w.tol)
    out = os.path.join(GOLD, f"fullsize_{name}.npz")
    if w.dim == 3:
        nl = lv.nl
        c, bb, a = np.unravel_index(lv.dof_nodes, (nl, nl, nl))
        # approximate node positions (uniform sub-grid; only selects the subset)
        pos = lambda k, o: o + k * lv.h / w.p
        rad = np.sqrt((pos(a, w.x0) - w.cx) ** 2 + (pos(bb, w.y0) - w.cy) ** 2 + (pos(c, w.z0) - w.cz) ** 2)
        idx = np.flatnonzero((np.abs(rad - w.r) < 3 * lv.h) | (np.arange(lv.n_dofs) % 11 == 0)).astype(np.int32)
        np.savez_compressed(out, idx=idx, y_fwd=y_fwd[idx], y_rev=y_rev[idx], v=v[idx], cg_it=it,
                            cg_rel=hist[-1] / hist[0], n_dofs=lv.n_dofs, workload=w.name, seeds=np.array([31, 32]),
                            tol=w.tol)
    else:
        np.savez_compressed(out, y_fwd=y_fwd, y_rev=y_rev, v=v, cg_it=it, cg_rel=hist[-1] / hist[0],
                            n_dofs=lv.n_dofs, workload=w.name, seeds=np.array([31, 32]), tol=w.tol)
    print(f"{name}: wrote {out} ({os.path.getsize(out) / 1e6:.1f} MB), CG {it} iterations, "
          f"{time.time() - t:.0f} s total", flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or list(CASES):
        make(n)
