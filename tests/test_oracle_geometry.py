"""Oracle pins for classification, DoFs, ghost faces, patches, colouring."""
import os

import numpy as np
import pytest

from oracle.geometry import (CARTESIAN, CUT, CUTPATCH, INSIDE, OUTSIDE, Circle, Level, build_patches,
                             ghost_faces, hierarchy)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def read_golden(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.split("#")[0].split()
        if line:
            rows.append(line)
    return rows


@pytest.mark.parametrize("row", read_golden("paper_fig2_dofs.txt"), ids=lambda r: "Q%s-n%s" % (r[0], r[1]))
def test_dof_counts_match_paper_fig2(row):
    # DoF counts of the circle domain printed in Fig. 2
    p, n, dofs = map(int, row)
    lv = Level(-1.105, -1.105, 2.21, n, Circle(0.0, 0.0, 1.0), p)
    assert lv.n_dofs == dofs


def test_classification_by_sampling():
    # Inside cells: every sample point in the closed disk; Outside: none in the
    # open disk; Cut: samples on both sides (dense 65x65 sampling per cell).
    C = Circle(0.0, 0.0, 1.0)
    lv = Level(-1.105, -1.105, 2.21, 16, C, 1)
    s = np.linspace(0, 1, 65)
    for j in range(lv.n):
        for i in range(lv.n):
            xl, xh, yl, yh = lv.cell_bounds(i, j)
            X, Y = np.meshgrid(xl + (xh - xl) * s, yl + (yh - yl) * s)
            d2 = X * X + Y * Y
            t = lv.cell_type[j, i]
            if t == INSIDE:
                assert d2.max() <= 1.0
            elif t == OUTSIDE:
                assert d2.min() >= 1.0 - 1e-12
            else:
                assert d2.min() < 1.0 < d2.max()


def test_fine_active_implies_parent_active():
    # Omega_l ⊆ Omega_{l-1}
    levels = hierarchy(-1.105, -1.105, 2.21, 2, 7, Circle(0.0, 0.0, 1.0), 1)
    for c, f in zip(levels[:-1], levels[1:]):
        act_f = f.cell_type != OUTSIDE
        act_parent = np.repeat(np.repeat(c.cell_type != OUTSIDE, 2, axis=0), 2, axis=1)
        assert not np.any(act_f & ~act_parent)


def test_ghost_faces_brute_force():
    # F_G by a quadratic scan over all cell pairs
    lv = Level(-0.5, -0.5, 1.0, 12, Circle(0.02, -0.01, 0.3), 2)
    cells = [(i, j) for j in range(lv.n) for i in range(lv.n)]
    ref = set()
    for a in cells:
        for b in cells:
            if abs(a[0] - b[0]) + abs(a[1] - b[1]) != 1 or a > b:
                continue
            ta, tb = lv.cell_type[a[1], a[0]], lv.cell_type[b[1], b[0]]
            if ta != OUTSIDE and tb != OUTSIDE and (ta == CUT or tb == CUT):
                lo = min(a, b, key=lambda c: (c[0] + c[1]))
                ref.add((0 if a[1] == b[1] else 1, lo[0], lo[1]))
    assert set(ghost_faces(lv)) == ref
    assert len(ghost_faces(lv)) == len(ref)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_patches_cover_colour_and_shape(p):
    lv = Level(-1.105, -1.105, 2.21, 16, Circle(0.0, 0.0, 1.0), p)
    pts = build_patches(lv)
    covered = np.zeros(lv.n_dofs, dtype=int)
    for pt in pts:
        covered[pt.interior] += 1
        if pt.kind == CARTESIAN:
            assert pt.interior.size == (2 * p - 1) ** 2
            assert len(pt.cells) == 4
        # vertices inside Omega have all four cells active
        X, Y = lv.x0 + pt.I * lv.h, lv.y0 + pt.J * lv.h
        if X * X + Y * Y < 1.0:
            assert len(pt.cells) == 4
    assert covered.min() >= 1        # the patches cover every DoF (reading R3)
    # same-colour patches of one kind are cell-disjoint with disjoint interior sets
    for kind in (CARTESIAN, CUTPATCH):
        for c in range(4):
            grp = [pt for pt in pts if pt.kind == kind and pt.colour == c]
            cells = [cl for pt in grp for cl in pt.cells]
            assert len(cells) == len(set(cells))
            dofs = np.concatenate([pt.interior for pt in grp]) if grp else np.zeros(0)
            assert dofs.size == np.unique(dofs).size


def test_all_inside_patches_count():
    # a circle containing the whole box: every interior vertex patch is Cartesian,
    # 4 colours of sizes {16,12,12,9} on 8x8 cells (7x7 interior vertices)
    lv = Level(0.0, 0.0, 1.0, 8, Circle(0.5, 0.5, 10.0), 2)
    pts = [pt for pt in build_patches(lv) if pt.kind == CARTESIAN]
    sizes = sorted(sum(1 for pt in pts if pt.colour == c) for c in range(4))
    assert sizes == [9, 12, 12, 16]
