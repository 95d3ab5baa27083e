"""Oracle pins for transfer, patch smoother, V-cycle, CG/GMRES (PAPER.md
l.123-212, Tables 1-3)."""
import os

import numpy as np
import pytest

import workloads
from oracle.assemble import Params
from oracle.fe import gauss_lobatto_nodes
from oracle.geometry import CARTESIAN, CUTPATCH, Circle, Level
from oracle.solver import Hierarchy, LevelData, fractional_iterations, from_workload
from oracle.transfer import prolongation_matrix

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def interp(lv, fn):
    xi = gauss_lobatto_nodes(lv.p)
    b, a = np.divmod(lv.dof_nodes, lv.nl)
    def pos(k, o):
        c = np.minimum(k // lv.p, lv.n - 1)
        return o + (c + xi[k - c * lv.p]) * lv.h
    return fn(pos(a, lv.x0), pos(b, lv.y0))


@pytest.mark.parametrize("p", [1, 2, 3])
def test_prolongation_reproduces_polynomials(p):
    # I_l u_{l-1} = u_{l-1} on Omega_l: for u in Q_p the
    # prolongated coarse interpolant is the fine interpolant
    C = Circle(0.0, 0.0, 1.0)
    c, f = Level(-1.105, -1.105, 2.21, 8, C, p), Level(-1.105, -1.105, 2.21, 16, C, p)
    P = prolongation_matrix(c, f)
    q = lambda x, y: (x ** p) * (y ** p) - 0.5 * x * y + 2.0 * y ** p + 1.0
    assert np.allclose(P @ interp(c, q), interp(f, q), atol=1e-12)
    assert np.allclose(P @ np.ones(c.n_dofs), 1.0, atol=1e-13)  # partition of unity


def test_smoother_fixed_point_and_local_exactness():
    h = from_workload(workloads.CONFIG0)
    ld = h.fine
    x = np.random.default_rng(0).standard_normal(ld.lv.n_dofs)
    b = ld.A @ x
    y = x.copy()
    ld.smooth(y, b, 2)
    assert np.allclose(y, x, atol=1e-12)
    # a single patch correction annihilates the residual on its interior set
    b = np.random.default_rng(1).standard_normal(ld.lv.n_dofs)
    for idx in (0, len(ld.patches) // 2, len(ld.patches) - 1):
        x = np.zeros_like(b)
        I = ld.patches[idx].interior
        x[I] += ld.inv[idx] @ (b - ld.A @ x)[I]
        assert np.abs((b - ld.A @ x)[I]).max() < 1e-12 * np.abs(b).max()


def test_colour_parallel_equals_sequential_without_ghost_coupling():
    # With no cut cells there are no ghost faces, so same-colour patches do not
    # couple and the coloured smoother equals the sequential multiplicative
    # sweep of eq. (smoother).
    lv = Level(0.0, 0.0, 1.0, 8, Circle(0.5, 0.5, 10.0), 2)
    ld = LevelData(lv, Params())
    rng = np.random.default_rng(3)
    b = rng.standard_normal(lv.n_dofs)
    x0 = rng.standard_normal(lv.n_dofs)
    x1 = x0.copy()
    for c in range(4):
        ld.colour_step(x1, b, CARTESIAN, c)
    x2 = x0.copy()
    for c in range(4):
        for idx in ld.groups[(CARTESIAN, c)]:
            I = ld.patches[idx].interior
            x2[I] += np.linalg.solve(ld.A[I][:, I].toarray(), (b - ld.A @ x2)[I])
    assert np.allclose(x1, x2, atol=1e-11)


def test_sequential_sweep_reduces_energy():
    h = from_workload(workloads.CONFIG0)
    ld = h.fine
    A = ld.A
    rng = np.random.default_rng(4)
    xs = rng.standard_normal(ld.lv.n_dofs)
    b = A @ xs
    x = np.zeros_like(b)
    en = lambda x: (x - xs) @ (A @ (x - xs))
    e_prev = en(x)
    for idx, pt in enumerate(ld.patches):
        I = pt.interior
        if I.size:
            x[I] += ld.inv[idx] @ (b - A @ x)[I]
            e = en(x)
            assert e <= e_prev * (1 + 1e-12)
            e_prev = e


def test_vcycle_linear_and_symmetric():
    h = from_workload(workloads.CONFIG0)
    rng = np.random.default_rng(5)
    v, w = rng.standard_normal((2, h.fine.lv.n_dofs))
    Vv, Vw = h.precondition(v), h.precondition(w)
    assert np.allclose(h.precondition(2.5 * v), 2.5 * Vv, rtol=1e-12, atol=1e-12)
    assert abs(v @ Vw - w @ Vv) < 1e-10 * abs(v @ Vw)
    assert v @ Vv > 0 and w @ Vw > 0


def test_cg_config0_converges():
    h = from_workload(workloads.CONFIG0)
    b = np.random.default_rng(6).standard_normal(h.fine.lv.n_dofs)
    x, it, hist = h.solve_cg(b, 1e-8)
    assert hist[-1] <= 1e-8 * hist[0]
    assert np.linalg.norm(b - h.fine.A @ x) <= 1.01e-8 * np.linalg.norm(b)
    assert it < 20


def test_fractional_iterations_closed_form():
    assert fractional_iterations(5, 1e-10, 1.0) == pytest.approx(4.0)
    assert fractional_iterations(8, 1e-8, 1.0) == pytest.approx(8.0)


def tables():
    rows = []
    for line in open(os.path.join(GOLD, "paper_tables.txt")):
        t = line.split("#")[0].split()
        if t:
            rows.append((t[0], int(t[1]), int(t[2]), int(t[3]), int(t[4])))
    return rows


def run(table, L, p, nc):
    w = workloads.paper_level(p, L, n_c=nc)
    h = from_workload(w, symmetric=False)
    b = np.random.default_rng(7).standard_normal(h.fine.lv.n_dofs)
    if table == "T2":
        return h.solve_gmres(b, 1e-9, 300)[1]
    it = h.solve_vcycle(b, 1e-9, 300)[1]
    return -1 if it is None else it


@pytest.mark.parametrize("row", [r for r in tables() if r[2] == 1 and r[0] == "T2"], ids=lambda r: "%s-L%d-Q%d-nc%d" % r[:4])
def test_q1_gmres_counts_match_paper(row):
    # Q1 GMRES counts of Table 2 within +-2 (gamma_D, gamma_1 and the
    # patch-set reading R3 are not fixed by the paper)
    table, L, p, nc, paper = row
    got = run(table, L, p, nc)
    assert abs(got - paper) <= 2, (got, paper)


@pytest.mark.parametrize("L", [6, 7])
def test_q1_vcycle_counts_band(L):
    # Table 3 (stationary V-cycle, Q1, l.271-290): two-sided band
    # paper/2 <= oracle <= paper; more iterations than GMRES; n_c = 2 beats
    # n_c = 1 (l.269-270)
    paper = {(r[1], r[2], r[3]): r[4] for r in tables() if r[0] == "T3"}
    it1, it2 = run("T3", L, 1, 1), run("T3", L, 1, 2)
    assert paper[(L, 1, 1)] // 2 <= it1 <= paper[(L, 1, 1)]
    assert paper[(L, 1, 2)] // 2 <= it2 <= paper[(L, 1, 2)]
    assert it2 < it1
    assert it2 >= run("T2", L, 1, 2)


@pytest.mark.parametrize("L", [6, 7])
def test_q2_q3_gmres_band_nc2_and_nc_helps_q3(L):
    # Table 2, n_c = 2 columns (= Table 1 circle block): two-sided band
    # paper/3 <= oracle <= paper for Q2 and Q3 (the oracle's smoother is
    # stronger than the paper's at Q2/Q3; DESIGN.md "Q2/Q3 iteration counts:
    # sensitivity study" lists the readings tried), and a second cut sweep
    # helps Q3 ("a second smoothing step on the cut cells is crucial", l.268)
    paper = {(r[1], r[2], r[3]): r[4] for r in tables() if r[0] == "T2"}
    for p in (2, 3):
        got = run("T2", L, p, 2)
        assert paper[(L, p, 2)] / 3.0 <= got <= paper[(L, p, 2)], (p, got)
    assert run("T2", L, 3, 2) < run("T2", L, 3, 1)
    assert run("T2", L, 2, 1) <= paper[(L, 2, 1)]


@pytest.mark.xfail(strict=True, reason="known gap, DESIGN.md 'Q2/Q3 iteration counts: sensitivity study': no reading "
                   "tried reproduces Table 2's Q3 n_c=1 blow-up (132 GMRES iterations at L=6)")
def test_q3_nc1_gmres_blowup_table2():
    paper = {(r[1], r[2], r[3]): r[4] for r in tables() if r[0] == "T2"}
    assert run("T2", 6, 3, 1) >= paper[(6, 3, 1)] / 2


@pytest.mark.xfail(strict=True, reason="known gap, DESIGN.md 'Q2/Q3 iteration counts: sensitivity study': the oracle's "
                   "stationary V-cycle converges for Q3 n_c=1 where Table 3 prints divergence")
def test_q3_nc1_vcycle_divergence_table3():
    assert run("T3", 6, 3, 1) == -1


@pytest.mark.parametrize("L,paper_row", [(6, (5.4, 5.7, 5.8)), (7, (5.0, 5.3, 5.5))])
def test_table4_fractional_iterations_band(L, paper_row):
    # Table 4 (l.295-313): Q1 GMRES fractional iteration counts
    # n_frac = n_it (-8) / log10(||r_n|| / ||r_0||) (l.350-353) at
    # gamma_1 = 0.05, 0.10, 0.15 (n_c = 2 as in Table 1): within 1.0 of the
    # printed values and non-decreasing in gamma_1 over that window, as printed
    got = []
    for g1 in (0.05, 0.10, 0.15):
        w = workloads.paper_level(1, L, n_c=2)
        h = from_workload(w, prm=Params(gamma_k=[g1]), symmetric=False)
        b = np.random.default_rng(7).standard_normal(h.fine.lv.n_dofs)
        _, it, hist = h.solve_gmres(b, 1e-9, 300)
        got.append(fractional_iterations(it, hist[-1], hist[0]))
    for g, p in zip(got, paper_row):
        assert abs(g - p) <= 1.0, (got, paper_row)
    assert got[0] <= got[1] + 0.02 and got[1] <= got[2] + 0.02, got
