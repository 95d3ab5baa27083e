"""CPU oracle for the CutFEM vertex-patch multigrid hot path (arxiv 2508.11608).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path
(`paper_2508_11608_b200/`) may import, call or link anything under `oracle/`.
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs use it.

The oracle is a plain, slow, obviously-correct fp64 implementation written from
PAPER.md.  It assembles the global sparse matrix A_l of eq. (cutfem-ghost)
 and runs the coloured multiplicative vertex-patch smoother
of eq. (smoother)/(smoother-split) inside the V-cycle
 and CG / GMRES.  Each function cites the passage it
follows.  Where PAPER.md is silent or ambiguous the reading taken is listed in
DESIGN.md section "Readings" and cited as R<n> here.

Modules
  fe          Q_p Gauss-Lobatto Lagrange basis
  geometry    mesh hierarchy, cell classification, vertex patches, colouring
              
  quadrature  Gauss rules, cut-cell volume/surface rules
  assemble    DoFs, sparse A_l, rhs
  transfer    prolongation / restriction
  solver      patch smoother, V-cycle, CG, GMRES

Parity pins: every function here is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py against values the paper prints (tests/golden/) or
mathematical facts (closed forms, invariants, brute force).
"Oracle pins" for the list.
"""
