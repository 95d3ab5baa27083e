"""Dependency-cone study for a one-launch cut sweep (design aid, host only).

The cut sweep of one smoothing step is S = 4 n_c colour steps over the cut
patches (P eq. smoother-split l.196-210, R9).  A CTA that owns the dynamic
nodes of a T x T cell tile can produce their final values without talking to
any other CTA if it recomputes, at every step s, the backward dependency cone:
the step-s patches whose interior meets the nodes it needs after step s, which
in turn need the coupled window nodes (nonzero columns of A) after step s-1.
This script measures, on the oracle's patches and sparsity pattern, how much
redundant work and map data that costs per tile size.

    python scripts/cone_study.py [n] [p]
"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from oracle.geometry import Circle, Level, build_patches, CUTPATCH  # noqa: E402
from oracle.assemble import assemble_matrix  # noqa: E402
from oracle.solver import Params  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    n_c = 2
    t0 = time.time()
    lv = Level(-1.105, -1.105, 2.21, n, Circle(0.0, 0.0, 1.0), p)
    A = assemble_matrix(lv, Params()).tocsr()
    pts = [pt for pt in build_patches(lv) if pt.kind == CUTPATCH and pt.interior.size]
    print(f"n={n} p={p}: {len(pts)} cut patches, setup {time.time() - t0:.1f} s")
    # per patch: interior dofs, exterior coupled dofs (nonzero columns of A_IE)
    ext, mapd = [], []
    for pt in pts:
        I = pt.interior
        cols = np.unique(A[I].indices)
        E = np.setdiff1d(cols, I)
        ext.append(E)
        mapd.append(I.size * (I.size + E.size))
    mapd = np.array(mapd)
    dyn = np.zeros(lv.n_dofs, bool)
    for pt in pts:
        dyn[pt.interior] = True
    # node -> cell tile; patch interiors by dof
    node = lv.dof_nodes
    na, nb = node % lv.nl, node // lv.nl
    col = np.array([pt.colour for pt in pts])
    S = 4 * n_c
    # patches containing a given dof in their interior, per colour
    owner = {}
    for k, pt in enumerate(pts):
        for d in pt.interior:
            owner.setdefault(int(d), []).append(k)
    tot_map = mapd.sum() * n_c   # non-redundant map doubles per sweep
    for T in (8, 12, 16, 24, 32, 48, 64):
        ti = np.minimum(na // p, n - 1) // T
        tj = np.minimum(nb // p, n - 1) // T
        ntx = (n + T - 1) // T
        tile = tj * ntx + ti
        tiles = np.unique(tile[dyn])
        red_map, max_step_map, max_slots, max_tasks = 0, 0, 0, 0
        per_tile = []
        for t in tiles:
            need = set(np.flatnonzero(dyn & (tile == t)).tolist())
            slots = set(need)
            tmap, tasks = 0, 0
            for s in range(S - 1, -1, -1):
                c = s % 4
                Ts = set()
                for d in need:
                    for k in owner.get(d, ()):
                        if col[k] == c:
                            Ts.add(k)
                step_map = sum(int(mapd[k]) for k in Ts)
                max_step_map = max(max_step_map, step_map)
                tmap += step_map
                tasks += len(Ts)
                for k in Ts:
                    need.update(int(e) for e in ext[k] if dyn[e])
                    slots.update(int(e) for e in ext[k])
                    slots.update(int(e) for e in pts[k].interior)
            red_map += tmap
            per_tile.append(tmap)
            max_slots = max(max_slots, len(slots))
            max_tasks = max(max_tasks, tasks)
        per_tile = np.array(per_tile)
        print(f"T={T:3d}: tiles {tiles.size:4d}  redundancy {red_map / tot_map:5.2f}  map MB/sweep "
              f"{8 * red_map / 1e6:6.1f} (min {8 * tot_map / 1e6:.1f})  max/tile {8 * per_tile.max() / 1e3:6.0f} KB "
              f"mean {8 * per_tile.mean() / 1e3:6.0f} KB  max step map {8 * max_step_map / 1e3:5.0f} KB  "
              f"max slots {max_slots}  max tasks {max_tasks}")


if __name__ == "__main__":
    main()


def segments_study(n=512, p=2, ngs=(74, 100, 139, 148)):
    """Redundancy of equal-work ownership segments ordered by angle around the
    circle centre (the tightest 1D split of the cut band) -- cones exact."""
    n_c = 2
    S = 4 * n_c
    lv = Level(-1.105, -1.105, 2.21, n, Circle(0.0, 0.0, 1.0), p)
    A = assemble_matrix(lv, Params()).tocsr()
    pts = [pt for pt in build_patches(lv) if pt.kind == CUTPATCH and pt.interior.size]
    ext = [np.setdiff1d(np.unique(A[pt.interior].indices), pt.interior) for pt in pts]
    mapd = np.array([pt.interior.size * (pt.interior.size + e.size) for pt, e in zip(pts, ext)])
    dyn = np.zeros(lv.n_dofs, bool)
    owner = {}
    for k, pt in enumerate(pts):
        dyn[pt.interior] = True
        for d in pt.interior:
            owner.setdefault(int(d), []).append(k)
    col = np.array([pt.colour for pt in pts])
    node = lv.dof_nodes
    ang = np.arctan2(node // lv.nl - lv.nl / 2, node % lv.nl - lv.nl / 2)
    dn = np.flatnonzero(dyn)
    # work per dynamic node: map doubles of its patches / their interior sizes
    w = np.zeros(lv.n_dofs)
    for k, pt in enumerate(pts):
        w[pt.interior] += mapd[k] / pt.interior.size
    order = dn[np.argsort(ang[dn])]
    tot_map = mapd.sum() * n_c
    for ng in ngs:
        cw = np.cumsum(w[order])
        grp = np.minimum((cw / cw[-1] * ng).astype(int), ng - 1)
        cone_b = []
        for g in range(ng):
            need = set(order[grp == g].tolist())
            b = 0
            for s in range(S - 1, -1, -1):
                c = s % 4
                Ts = {k for d in need for k in owner.get(d, ()) if col[k] == c}
                b += sum(int(mapd[k]) for k in Ts)
                for k in Ts:
                    need.difference_update(pts[k].interior.tolist())
                for k in Ts:
                    need.update(int(e) for e in ext[k] if dyn[e])
            cone_b.append(8 * b)
        cone_b = np.array(cone_b)
        print(f"angular ng={ng}: redundancy {cone_b.sum() / 8 / tot_map:.2f}, max cone {cone_b.max() / 1e3:.0f} KB, "
              f"median {np.median(cone_b) / 1e3:.0f} KB")
