"""Helpers shared by the GPU parity tests (CUDA path vs oracle)."""
import functools

import numpy as np

import workloads
from oracle.geometry import CARTESIAN, CUTPATCH
from oracle.solver import from_workload as oracle_from_workload

KIND = {0: CARTESIAN, 1: CUTPATCH}


@functools.lru_cache(maxsize=8)
def oracle(w, symmetric=True):
    return oracle_from_workload(w, symmetric=symmetric)


def gpu(w, **kw):
    from paper_2508_11608_b200 import cutfem
    return cutfem.Problem.from_workload(w, **kw)


def lattice_random(w, seed, level):
    return workloads.lattice_vector(w, seed, level)


def compact(lv, lattice):
    """oracle DoF vector from a (NL*NL,) lattice vector"""
    return np.asarray(lattice)[lv.dof_nodes]


def expand(lv, vec):
    out = np.zeros(lv.nl * lv.nl)
    out[lv.dof_nodes] = vec
    return out


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
