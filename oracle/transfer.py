"""Intergrid transfer.

Prolongation: the embedding, I_l u_{l-1}(x) = u_{l-1}(x) for x in Omega_l
(l.130-133); as a matrix, P[j, i] = phi^{l-1}_i(x_j) at the fine nodes x_j.
Restriction: the transpose of the prolongation (l.137).

Test infrastructure only (see oracle/__init__.py).
"""
import numpy as np
import scipy.sparse as sp

from .fe import basis_1d, gauss_lobatto_nodes


def prolongation_matrix(coarse, fine):
    """Sparse P (n_fine x n_coarse), P[j, i] = phi^c_i(x_j).

    For each fine DoF node x_j, an active fine cell containing it is chosen;
    its parent coarse cell is active (Omega_l ⊆ Omega_{l-1}, l.128) and
    contains x_j; the coarse basis functions that do not vanish at x_j are
    the (p+1)^2 Lagrange functions of that coarse cell (continuity makes the
    choice of cell irrelevant)."""
    p = fine.p
    xi = gauss_lobatto_nodes(p)
    rows, cols, vals = [], [], []
    for jf, node in enumerate(fine.dof_nodes):
        b, a = divmod(int(node), fine.nl)
        cells = fine.node_support(a, b)
        i_f, j_f = cells[0]
        kx, ky = a - i_f * p, b - j_f * p
        I, J = i_f // 2, j_f // 2
        if coarse.cell_type[J, I] == 0:
            raise RuntimeError("fine active cell with inactive parent violates Omega_l ⊆ Omega_{l-1}")
        xc = ((i_f % 2) + xi[kx]) / 2.0
        yc = ((j_f % 2) + xi[ky]) / 2.0
        bx = basis_1d(p, [xc])[:, 0]
        by = basis_1d(p, [yc])[:, 0]
        for n in range(p + 1):
            for m in range(p + 1):
                wgt = bx[m] * by[n]
                ic = coarse.dof_index[(J * p + n) * coarse.nl + (I * p + m)]
                if wgt != 0.0 and ic >= 0:   # (ic < 0: fitted boundary node, coefficient 0)
                    rows.append(jf); cols.append(int(ic)); vals.append(wgt)
    return sp.csr_matrix((vals, (rows, cols)), shape=(fine.n_dofs, coarse.n_dofs))
