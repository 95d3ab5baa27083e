import sys, numpy as np
sys.path.insert(0,'.')
import workloads
from oracle.solver import from_workload
from paper_2508_11608_b200 import cutfem
w = workloads.sphere("sphere-Q3-8", 2, 3, 3)
g = cutfem.Problem.from_workload(w)
o = from_workload(w)
for l, ld in enumerate(o.levels):
    xl = workloads.lattice_vector(w, 30 + l, l)
    y = g.zeros(l); g.apply_operator(l, g.to_device(xl, l), y)
    yg = g.to_host(y, l)[ld.lv.dof_nodes]; yo = ld.A @ xl[ld.lv.dof_nodes]
    bad = ~np.isfinite(yg)
    print(l, 'n', ld.lv.n, 'nan', bad.sum(), 'of', yg.size, 'err(finite)', np.abs(yg[~bad]-yo[~bad]).max()/np.abs(yo).max(), 'ncut', int((ld.lv.cell_type==2).sum()))
    # unit vector probes at level 0
    if l == 0:
        for k in range(0, ld.lv.n_dofs, 37):
            e = np.zeros(ld.lv.nl**3); e[ld.lv.dof_nodes[k]] = 1.0
            y = g.zeros(l); g.apply_operator(l, g.to_device(e, l), y)
            yy = g.to_host(y, l)[ld.lv.dof_nodes]
            print('  col', k, 'nan', int((~np.isfinite(yy)).sum()), 'err', np.nanmax(np.abs(yy - ld.A[:, k].toarray().ravel())))
