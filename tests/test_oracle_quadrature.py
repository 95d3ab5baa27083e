"""Oracle pins for the quadrature module against closed forms."""
import math

import numpy as np
import pytest

from oracle.geometry import CUT, INSIDE, Circle, Level
from oracle.quadrature import cut_cell_rules, tensor_gauss


def test_tensor_gauss_exactness():
    pts, w = tensor_gauss(0.0, 1.0, 0.0, 1.0, 3)
    assert abs(w @ (pts[:, 0] ** 5 * pts[:, 1] ** 5) - 1.0 / 36.0) < 1e-15
    pts, w = tensor_gauss(-1.0, 2.0, 0.5, 0.75, 2)
    assert abs(w.sum() - 0.75) < 1e-15


def segment_area():
    # T = [0.5,1.5]x[-0.5,0.5] ∩ unit disk = {0.5<=x<=1, |y|<=min(sqrt(1-x^2), 0.5)}
    F = lambda x: 0.5 * (x * math.sqrt(1 - x * x) + math.asin(x))   # ∫ sqrt(1-x^2)
    x1 = math.sqrt(0.75)
    return (x1 - 0.5) * 1.0 + 2 * (F(1.0) - F(x1))


def test_single_cut_cell_closed_forms():
    C = Circle(0.0, 0.0, 1.0)
    vp, vw, sp, sw, sn = cut_cell_rules(0.5, 1.5, -0.5, 0.5, C, 10)
    assert abs(vw.sum() - segment_area()) < 1e-12
    # arc inside the cell: |y| <= 0.5 on the unit circle -> angle in [-pi/6, pi/6]
    assert abs(sw.sum() - math.pi / 3) < 1e-12
    # points on Gamma, outward unit normals
    assert np.allclose(np.hypot(sp[:, 0], sp[:, 1]), 1.0, atol=1e-14)
    assert np.allclose(np.hypot(sn[:, 0], sn[:, 1]), 1.0, atol=1e-14)
    assert np.all((sn * sp).sum(axis=1) > 0)
    # first moment ∫ x dA over the segment piece: ∫_{0.5}^{1} x * 2 min(sqrt(1-x^2),.5) dx
    x1 = math.sqrt(0.75)
    m1 = 0.5 * (x1 ** 2 - 0.25) + (2.0 / 3.0) * (1 - x1 ** 2) ** 1.5
    assert abs(vw @ vp[:, 0] - m1) < 1e-12


def test_quarter_disk_converges():
    # cell with the circle centre at a corner: quarter disk, area pi/4, arc pi/2,
    # ∫ x^2 dA = pi/16.  The arc has a vertical tangent at a cell corner, so the
    # rule converges algebraically; check the error decreases with n.
    C = Circle(0.0, 0.0, 1.0)
    errs = []
    for n in (4, 8, 16, 32):
        vp, vw, sp, sw, sn = cut_cell_rules(0.0, 1.0, 0.0, 1.0, C, n)
        errs.append((abs(vw.sum() - math.pi / 4), abs(sw.sum() - math.pi / 2),
                     abs(vw @ vp[:, 0] ** 2 - math.pi / 16)))
    errs = np.array(errs)
    assert np.all(np.diff(errs, axis=0) < 0)
    assert errs[-1][0] < 1e-5 and errs[-1][2] < 1e-5 and errs[-1][1] < 0.02


@pytest.mark.parametrize("n,tol_area,tol_arc", [(32, 1e-7, 1e-7), (128, 1e-10, 1e-10)])
def test_global_area_and_perimeter(n, tol_area, tol_arc):
    # sum over all active cells of the volume weights = |Omega| = pi, of the
    # surface weights = |Gamma| = 2 pi (closed forms)
    lv = Level(-1.105, -1.105, 2.21, n, Circle(0.0, 0.0, 1.0), 2)
    area = float((lv.cell_type == INSIDE).sum()) * lv.h ** 2
    arc = 0.0
    for j, i in zip(*np.nonzero(lv.cell_type == CUT)):
        xl, xh, yl, yh = lv.cell_bounds(i, j)
        vp, vw, sp, sw, sn = cut_cell_rules(xl, xh, yl, yh, lv.circle, 3)
        area += vw.sum()
        arc += sw.sum()
    assert abs(area - math.pi) < tol_area
    assert abs(arc - 2 * math.pi) < tol_arc


def test_off_centre_circle_area():
    C = Circle(0.013, -0.021, 0.3)
    lv = Level(-0.5, -0.5, 1.0, 64, C, 1)
    area = float((lv.cell_type == INSIDE).sum()) * lv.h ** 2
    for j, i in zip(*np.nonzero(lv.cell_type == CUT)):
        vp, vw, *_ = cut_cell_rules(*lv.cell_bounds(i, j), C, 4)
        area += vw.sum()
    assert abs(area - math.pi * 0.09) < 1e-9
