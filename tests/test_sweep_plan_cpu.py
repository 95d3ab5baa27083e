"""Host logic of the one-launch cut sweep (csrc/sweep.cuh, `build_sweep`), on
CPU through the host-only C-ABI entry `cutfem_sweep_plan` -- no GPU.

The sweep lets every CTA compute the final values of the nodes it owns alone,
by replaying the backward dependency cone of those nodes (P eq.
smoother-split l.196-210; R9: every patch of a colour step reads the state
the step starts from).  The planner is checked against a direct simulation:
the cut patches of a real level (oracle geometry and sparsity: interior
nodes, coupled exterior nodes) carry a random affine toy map each; the full
sequential colour sweep is run once, and every CTA's cone is run alone from
the initial state -- its owned nodes must end with exactly the full sweep's
values.  The owned sets must partition the interior nodes."""
import numpy as np
import pytest

from oracle.assemble import Params, assemble_matrix
from oracle.geometry import CUTPATCH, Circle, Level, build_patches


def level_patches(n, p, cx=0.0, cy=0.0, r=1.0):
    """cut patches with interiors, as (I, J, colour), interior and coupled
    exterior lattice nodes in the library's numbering b * ld + a"""
    lv = Level(-1.105, -1.105, 2.21, n, Circle(cx, cy, r), p)
    A = assemble_matrix(lv, Params()).tocsr()
    nl = lv.nl
    ld = (nl + 1) & ~1
    node = lv.dof_nodes                       # dof -> b * nl + a
    lat = (node // nl) * ld + node % nl       # dof -> b * ld + a
    ijc, ins, exs = [], [], []
    for pt in build_patches(lv):
        if pt.kind != CUTPATCH or not pt.interior.size:
            continue
        I = pt.interior
        E = np.setdiff1d(np.unique(A[I].indices), I)
        ijc.append((pt.I, pt.J, pt.colour))
        ins.append(lat[I])
        exs.append(lat[E])
    ca = (cx - (-1.105)) / (2.21 / n) * p
    return lv, ld, np.array(ijc), ins, exs, ca, (cy - (-1.105)) / (2.21 / n) * p


def toy_maps(ins, exs, seed):
    rng = np.random.default_rng(seed)
    return [(rng.uniform(-0.3, 0.3, (len(i), len(e))), rng.uniform(-1, 1, len(i))) for i, e in zip(ins, exs)]


def run_steps(state, steps, ijc, ins, exs, maps, S, reverse, only=None):
    """colour steps s = 0..S-1 (colour s mod 4, or 3 - s mod 4 reversed); all
    patches of a step read the state the step starts from.  only[s]: the
    patches to run at step s (a cone), else every patch of the colour"""
    for s in range(S):
        c = (3 - s % 4) if reverse else s % 4
        ks = only[s] if only is not None else [k for k in range(len(ins)) if ijc[k][2] == c]
        snap = dict(state)
        for k in ks:
            assert ijc[k][2] == c, "a cone holds a patch of the wrong colour"
            W, c0 = maps[k]
            xe = np.array([snap[e] for e in exs[k]])
            out = W @ xe + c0
            for i, nd in enumerate(ins[k]):
                state[nd] = out[i]
    return state


@pytest.mark.parametrize("n,p,ng,reverse,S", [(64, 2, 148, 0, 8), (64, 2, 148, 1, 8), (64, 1, 148, 0, 8),
                                              (32, 3, 148, 0, 8), (64, 2, 148, 0, 4), (32, 2, 148, 1, 16),
                                              (32, 2, 7, 1, 8), (32, 2, 0, 0, 8), (16, 2, 1, 0, 8)])
def test_cones_reproduce_the_sweep(n, p, ng, reverse, S):
    from paper_2508_11608_b200 import cutfem
    lv, ld, ijc, ins, exs, ca, cb = level_patches(n, p)
    owned, cones = cutfem.sweep_plan(n, p, ld, S, reverse, 148, ng, ijc, ins, exs, ca, cb)
    if ng:
        assert len(owned) <= ng
    dyn = set(int(v) for i in ins for v in i)
    allown = [v for o in owned for v in o]
    assert len(allown) == len(set(allown)) and set(allown) == dyn   # a partition of the interior nodes
    maps = toy_maps(ins, exs, 1 + n + p)
    rng = np.random.default_rng(7)
    nodes = sorted(dyn | set(int(v) for e in exs for v in e))
    init = dict(zip(nodes, rng.standard_normal(len(nodes))))
    full = run_steps(dict(init), range(S), ijc, ins, exs, maps, S, reverse)
    for g, own in enumerate(owned):
        local = run_steps(dict(init), range(S), ijc, ins, exs, maps, S, reverse, only=cones[g])
        for nd in own:
            assert local[nd] == full[nd], (g, nd)
    # a cone never runs a patch twice in one step, and with several CTAs some
    # patches are recomputed (redundancy >= 1)
    tasks = sum(len(set(c)) for cg in cones for c in cg)
    assert all(len(c) == len(set(c)) for cg in cones for c in cg)
    once = sum(1 for s in range(S) for k in range(len(ins)) if ijc[k][2] == ((3 - s % 4) if reverse else s % 4))
    assert tasks <= len(owned) * once


def test_off_centre_circle_and_bad_arguments():
    from paper_2508_11608_b200 import cutfem
    lv, ld, ijc, ins, exs, ca, cb = level_patches(32, 2, cx=0.0137, cy=-0.0211, r=0.9071)
    owned, cones = cutfem.sweep_plan(32, 2, ld, 8, 0, 148, 148, ijc, ins, exs, ca, cb)
    maps = toy_maps(ins, exs, 3)
    nodes = sorted(set(int(v) for i in ins for v in i) | set(int(v) for e in exs for v in e))
    init = dict(zip(nodes, np.random.default_rng(9).standard_normal(len(nodes))))
    full = run_steps(dict(init), range(8), ijc, ins, exs, maps, 8, 0)
    for g, own in enumerate(owned):
        local = run_steps(dict(init), range(8), ijc, ins, exs, maps, 8, 0, only=cones[g])
        assert all(local[nd] == full[nd] for nd in own)
    with pytest.raises(cutfem.CutfemError):
        cutfem.sweep_plan(32, 2, ld, 6, 0, 148, 0, ijc, ins, exs, ca, cb)   # S not a multiple of 4
