"""Sensitivity study of the oracle's iteration counts against PAPER.md
Tables 2-3 (l.247-290): which reading of the paper's unstated choices moves
the Q2/Q3 counts towards the printed ones?

Calls only `oracle/` and `workloads` (test infrastructure).  Prints one row
per (variant, L): GMRES (right-preconditioned, tol 1e-9) and stationary
V-cycle counts for Q1-Q3 with n_c = 1, 2 (forward post-smoother, as the
paper's GMRES/V-cycle runs; "div" = divergence).  The table in DESIGN.md
("Q2/Q3 iteration counts: sensitivity study") is this script's output.

    python scripts/oracle_sensitivity.py [L ...] [--variants a,b,...]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import workloads  # noqa: E402
from oracle.assemble import Params, assemble_rhs  # noqa: E402
from oracle.solver import from_workload  # noqa: E402

PAPER_T2 = {(6, 1): (8, 6), (6, 2): (11, 9), (6, 3): (132, 17), (7, 1): (8, 6), (7, 2): (9, 8), (7, 3): (193, 14),
            (8, 1): (7, 6), (8, 2): (8, 7), (8, 3): (217, 13)}
PAPER_T3 = {(6, 1): (14, 10), (6, 2): (33, 24), (6, 3): ("div", 121), (7, 1): (14, 9), (7, 2): (22, 18),
            (7, 3): ("div", 75), (8, 1): (12, 8), (8, 2): (18, 13), (8, 3): ("div", 47)}

# variant name -> (Params kwargs, Hierarchy kwargs, solver kwargs)
VARIANTS = {
    "base (R3 active, R5 sigma=-1, R7, R9/R10 principal)": ({}, {}, {}),
    "left-preconditioned GMRES": ({}, {}, {"left": True}),
    "rhs f=1 (instead of random)": ({}, {}, {"rhs": "f1"}),
    "sigma=+1 (h^(2k+1) as printed)": ({"sigma": 1}, {}, {}),
    "gamma_D=2.5p(p+1)": ({"gamma_D": "half"}, {}, {}),
    "gamma_D=20p(p+1)": ({"gamma_D": "x4"}, {}, {}),
    "gamma_k=0.05 (Tables 4-6 low end)": ({"gamma_k": 0.05}, {}, {}),
    "gamma_k=0.15 (Tables 4-6 high end)": ({"gamma_k": 0.15}, {}, {}),
    "patches at vertices in Omega (l.143 literal)": ({}, {"vertices": "inside"}, {}),
    "A_j patch-local (no boundary ghost faces)": ({}, {"local": "patch_matrix"}, {}),
    "A_j and residual patch-local": ({}, {"local": "patch"}, {}),
    "A_j without ghost penalty": ({}, {"local": "no_ghost"}, {}),
    "vertices in Omega + A_j,residual patch-local": ({}, {"vertices": "inside", "local": "patch"}, {}),
    "vertices in Omega + A_j patch-local": ({}, {"vertices": "inside", "local": "patch_matrix"}, {}),
    "sigma=+1 + A_j patch-local": ({"sigma": 1}, {"local": "patch_matrix"}, {}),
}


def params(p, kw):
    kw = dict(kw)
    if kw.get("gamma_D") == "half":
        kw["gamma_D"] = 2.5 * p * (p + 1)
    elif kw.get("gamma_D") == "x4":
        kw["gamma_D"] = 20.0 * p * (p + 1)
    if "gamma_k" in kw:
        kw["gamma_k"] = [kw["gamma_k"]] * p
    return Params(**kw)


def counts(L, p, nc, pkw, hkw, skw):
    w = workloads.paper_level(p, L, n_c=nc)
    h = from_workload(w, prm=params(p, pkw), symmetric=False, **hkw)
    lv = h.fine.lv
    if skw.get("rhs") == "f1":
        b = assemble_rhs(lv, params(p, pkw), lambda x, y: np.ones_like(x), lambda x, y: np.zeros_like(x))
    else:
        b = np.random.default_rng(7).standard_normal(lv.n_dofs)
    g = h.solve_gmres(b, 1e-9, 400, left=skw.get("left", False))[1]
    v = h.solve_vcycle(b, 1e-9, 400)[1]
    return g, ("div" if v is None else v)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    Ls = [int(a) for a in args] or [6]
    names = list(VARIANTS)
    for a in sys.argv[1:]:
        if a.startswith("--variants="):
            keys = a.split("=", 1)[1].split(",")
            names = [n for n in names if any(n.startswith(k) for k in keys)]
    print("| variant | L | GMRES Q1 nc1/nc2 | GMRES Q2 | GMRES Q3 | V-cycle Q1 | V-cycle Q2 | V-cycle Q3 |")
    print("|---|---|---|---|---|---|---|---|")
    for L in Ls:
        pg = " | ".join("%s/%s" % PAPER_T2[(L, p)] for p in (1, 2, 3))
        pv = " | ".join("%s/%s" % PAPER_T3[(L, p)] for p in (1, 2, 3))
        print(f"| **paper (Tables 2, 3)** | {L} | {pg} | {pv} |")
        for name in names:
            pkw, hkw, skw = VARIANTS[name]
            t = time.time()
            g, v = {}, {}
            for p in (1, 2, 3):
                for nc in (1, 2):
                    g[(p, nc)], v[(p, nc)] = counts(L, p, nc, pkw, hkw, skw)
            gs = " | ".join(f"{g[(p, 1)]}/{g[(p, 2)]}" for p in (1, 2, 3))
            vs = " | ".join(f"{v[(p, 1)]}/{v[(p, 2)]}" for p in (1, 2, 3))
            print(f"| {name} | {L} | {gs} | {vs} |", flush=True)
            sys.stderr.write(f"  {name}: {time.time() - t:.1f}s\n")


if __name__ == "__main__":
    main()
