"""Seeded synthetic workloads shared by the oracle-side tests and the CUDA path.

This module holds NO arithmetic of the method: only the problem descriptions
(box, circle, degree, levels, parameters) of the BASELINE.json configs and
seeded random lattice vectors.  Each side applies its own DoF mask to the
lattice vectors (the mask itself is pinned bit-exactly by the parity tests).

Lattice layout: a level with n cells per side and
degree p has NL = n p + 1 lattice nodes per side; vectors are NL*NL fp64 values
indexed b*NL + a (b = y index, a = x index).
"""
from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    x0: float          # box lower-left corner (square box)
    y0: float
    length: float      # box side
    n_coarse: int      # cells per side on level 0
    n_levels: int      # levels 0..n_levels-1, n_l = n_coarse 2^l
    cx: float          # circle centre and radius (analytic level set)
    cy: float
    r: float
    p: int             # Q_p degree
    n_c: int = 2       # cut-patch sweeps per smoothing step
    tol: float = 1e-8  # CG relative residual tolerance
    dim: int = 2       # 3: sphere (cx, cy, cz, r) in the cube [x0, x0+length]^3
    z0: float = 0.0
    cz: float = 0.0
    domain: str = "cut"  # "cut": circle / sphere level set; "fitted": the box itself, Dirichlet on its boundary

    @property
    def n_fine(self):
        return self.n_coarse * 2 ** (self.n_levels - 1)


# BASELINE.json configs[0]: "2D circle r=0.3 on [-0.5,0.5]^2, Q1, 16x16
# background mesh, 3-level V(1,1)-CG to 1e-8".
CONFIG0 = Workload("config0-circle-r0.3-Q1-16x16", -0.5, -0.5, 1.0, 4, 3, 0.0, 0.0, 0.3, 1)

# BASELINE.json configs[1]: "2D circle, Q2, 512x512 background mesh, 1 GPU,
# fp64".  The circle is the paper's section-4 setup (unit circle, 2x2 coarse
# mesh, box [-1.105,1.105]^2 -- reading R1 in DESIGN.md).
CONFIG1 = Workload("config1-circle-Q2-512x512", -1.105, -1.105, 2.21, 2, 9, 0.0, 0.0, 1.0, 2)


# BASELINE.json configs[2]: "3D sphere, Q2, 128^3 background mesh, 1 GPU,
# fp64" -- the 3D analogue of the section-4 setup (unit sphere in
# [-1.105,1.105]^3, 2^3 coarse cells, levels up to 128^3).
CONFIG2 = Workload("config2-sphere-Q2-128^3", -1.105, -1.105, 2.21, 2, 7, 0.0, 0.0, 1.0, 2, dim=3, z0=-1.105, cz=0.0)


def sphere(name, n_coarse, n_levels, p, x0=-1.105, length=2.21, c=(0.0, 0.0, 0.0), r=1.0):
    return Workload(name, x0, x0, length, n_coarse, n_levels, c[0], c[1], r, p, dim=3, z0=x0, cz=c[2])


# BASELINE.json configs[3]: "3D sphere, Q3/Q4 higher order, 256^3 background
# mesh, slab-partitioned over 2/4/8 B200": Q3 at 256^3 (180 M DoFs; the
# 641 k cut-patch inverses are stored packed symmetric, ~55 GB, and the whole
# problem takes ~125 GB of one B200; under --gpus N the z-slab partition runs
# it with the setup replicated on every rank).  3D Q4 is not supported.
CONFIG3 = Workload("config3-sphere-Q3-256^3", -1.105, -1.105, 2.21, 2, 8, 0.0, 0.0, 1.0, 3, dim=3, z0=-1.105, cz=0.0)


def fitted(name, n_coarse, n_levels, p, dim=2, x0=-1.105, length=2.21, tol=1e-8):
    """Fitted box (BASELINE.json configs[4]; the paper's "Square" baseline,
    P Table 1 / Fig. 2): Omega = the open box [x0, x0 + length]^dim, strong
    homogeneous Dirichlet condition on its boundary, no cut cells."""
    return Workload(name, x0, x0, length, n_coarse, n_levels, 0.0, 0.0, 0.0, p, 2, tol, dim=dim, z0=x0,
                    domain="fitted")


# BASELINE.json configs[4]: "3D sphere vs fitted cube at equal DoF, Q2": the
# fitted cube with 96^3 cells has 191^3 = 6 967 871 DoFs, config2's sphere
# (128^3 cells) 6 896 585 (+1 %); and the 2D analogue of config1: the fitted
# square with 384^2 cells has 767^2 = 588 289 DoFs vs config1's 680 065 (the
# closest n = n_0 2^k whose coarse level fits the exact coarse solve, n_0 <= 6).
CONFIG4_CUBE = fitted("config4-fitted-cube-Q2-96^3", 3, 6, 2, dim=3)
CONFIG4_SQUARE = fitted("config4-fitted-square-Q2-384^2", 3, 8, 2, dim=2)


def paper_level(p, L, n_c=2, tol=1e-9):
    """PAPER.md section 4 setup at table level L (reading R1): the unit circle
    in [-1.105,1.105]^2 with a 2x2 coarsest mesh; Q1 uses 2^(L-1) cells per
    side, Q2/Q3 use 2^(L-2) (the numbering of Fig. 2's data and Table 1)."""
    n_fine = 2 ** (L - 1) if p == 1 else 2 ** (L - 2)
    n_levels = int(np.log2(n_fine))  # 2, 4, ..., n_fine
    return Workload(f"paper-L{L}-Q{p}", -1.105, -1.105, 2.21, 2, n_levels, 0.0, 0.0, 1.0, p, n_c, tol)


def lattice_nodes(w, level=None):
    lvl = w.n_levels - 1 if level is None else level
    return w.n_coarse * 2 ** lvl * w.p + 1


def lattice_vector(w, seed, level=None):
    """Seeded N(0,1) values on every lattice node of a level (unmasked)."""
    nl = lattice_nodes(w, level)
    return np.random.default_rng(seed).standard_normal(nl ** w.dim)


def with_degree(w, p):
    return replace(w, p=p, name=f"{w.name}-Q{p}")
