import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
from oracle.solver import from_workload
from oracle.dim3 import cell_matrix3, cut_cell_rules3, CUT
from oracle.assemble import Params
from paper_2508_11608_b200 import cutfem
w = workloads.sphere("dbg", 2, 3, 1)
o = from_workload(w)
g = cutfem.Problem.from_workload(w)
l = 2
ld = o.levels[l]; lv = ld.lv
nd = lv.n_dofs
Ag = np.zeros((nd, nd))
for j in range(nd):
    e = np.zeros(lv.nl ** 3); e[lv.dof_nodes[j]] = 1.0
    y = g.zeros(l); g.apply_operator(l, g.to_device(e, l), y)
    Ag[:, j] = g.to_host(y, l)[lv.dof_nodes]
Ao = ld.A.toarray()
D = np.abs(Ag - Ao)
print("max diff", D.max(), "at", np.unravel_index(D.argmax(), D.shape), "max |A|", np.abs(Ao).max())
bad = np.argwhere(D > 1e-8 * np.abs(Ao).max())
print("n bad entries", len(bad))
# map dofs to lattice coords
def coord(i):
    node = lv.dof_nodes[i]; c, r = divmod(node, lv.nl * lv.nl); b, a = divmod(r, lv.nl); return (a, b, c)
for i, j in bad[:10]:
    print(coord(i), coord(j), Ag[i, j], Ao[i, j])
# cells that are cut: count quadrature points per cut cell from oracle
info = g.level_info(l)
print("gpu n_cut", info.n_cut, "vq", info.n_vol_qp, "sq", info.n_surf_qp)
nv = ns = 0
for k, j, i in zip(*np.nonzero(lv.cell_type == CUT)):
    lo = lv.lo(i, j, k)
    vp, vw, sp, sw, sn = cut_cell_rules3(lo, lo + lv.h, lv.sphere, 2)
    nv += len(vw); ns += len(sw)
print("oracle n_cut", (lv.cell_type == CUT).sum(), "vq", nv, "sq", ns)
