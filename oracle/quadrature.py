"""Quadrature on cut cells ("we have to use a substitute
quadrature of sufficient accuracy ... We employ the algorithm from [Saye2015]
to generate these quadrature rules on the intersected cells").

Reading R6: Saye's height-function algorithm specialised to one
analytic circle in 2D, where the roots of phi along a line are known in closed
form.  For a cut cell:
  1. height direction d = y if |y_c - c_y| >= |x_c - c_x| (cell centre vs
     circle centre, i.e. the larger normal component), else x; the other axis
     is the base axis t.
  2. the base interval [t_lo, t_hi] is split at the points where Gamma crosses
     the two faces normal to d and at c_t +- r, where they lie strictly inside.
  3. on each base sub-interval an n-point Gauss rule in t; at each base node
     the inside part of the height line is the single interval
     [max(s_lo, c_s - S), min(s_hi, c_s + S)], S = sqrt(r^2 - (t - c_t)^2)
     (the disk is convex), integrated with an n-point Gauss rule.
  4. surface rule: at each base node the points c_s +- S strictly inside
     (s_lo, s_hi) are points of Gamma, weight = w_t * r / S (arc length),
     normal = (x - c) / r (outward).
Test infrastructure only (see oracle/__init__.py).
"""
import math

import numpy as np

from .fe import gauss_legendre


def tensor_gauss(xl, xh, yl, yh, n):
    """n x n tensor Gauss rule on a box (points (m,2), weights (m,))."""
    g, w = gauss_legendre(n)
    X, Y = np.meshgrid(xl + (xh - xl) * g, yl + (yh - yl) * g, indexing="ij")
    W = np.outer(w * (xh - xl), w * (yh - yl))
    return np.stack([X.ravel(), Y.ravel()], axis=1), W.ravel()


def cut_cell_rules(xl, xh, yl, yh, circle, n):
    """Volume rule on T ∩ Omega and surface rule on Gamma ∩ T for one cell.

    Returns (vol_pts (m,2), vol_w (m,), surf_pts (k,2), surf_w (k,),
    surf_normals (k,2)), all in physical coordinates."""
    cx, cy, r = circle.cx, circle.cy, circle.r
    xc = 0.5 * (xl + xh)
    yc = 0.5 * (yl + yh)
    if abs(yc - cy) >= abs(xc - cx):
        # height direction y, base axis x
        t_lo, t_hi, s_lo, s_hi, ct, cs, swap = xl, xh, yl, yh, cx, cy, False
    else:
        t_lo, t_hi, s_lo, s_hi, ct, cs, swap = yl, yh, xl, xh, cy, cx, True
    r2 = r * r
    brk = [t_lo, t_hi]
    for s_face in (s_lo, s_hi):
        D = r2 - (s_face - cs) * (s_face - cs)
        if D > 0.0:
            q = math.sqrt(D)
            brk += [ct - q, ct + q]
    brk += [ct - r, ct + r]
    brk = sorted(set(b for b in brk if t_lo <= b <= t_hi))
    g, w = gauss_legendre(n)
    vp, vw, sp, sw, sn = [], [], [], [], []
    for ta, tb in zip(brk[:-1], brk[1:]):
        if not tb > ta:
            continue
        for gk, wk in zip(g, w):
            t = ta + (tb - ta) * gk
            wt = wk * (tb - ta)
            D = r2 - (t - ct) * (t - ct)
            if not D > 0.0:
                continue
            S = math.sqrt(D)
            lo = max(s_lo, cs - S)
            hi = min(s_hi, cs + S)
            if hi > lo:
                for gm, wm in zip(g, w):
                    s = lo + (hi - lo) * gm
                    vp.append((s, t) if swap else (t, s))
                    vw.append(wt * wm * (hi - lo))
            for s in (cs - S, cs + S):
                if s_lo < s < s_hi:
                    x, y = (s, t) if swap else (t, s)
                    sp.append((x, y))
                    sw.append(wt * r / S)
                    sn.append(((x - cx) / r, (y - cy) / r))
    as2 = lambda a: np.array(a, dtype=np.float64).reshape(-1, 2)
    return as2(vp), np.array(vw, dtype=np.float64), as2(sp), np.array(sw, dtype=np.float64), as2(sn)
