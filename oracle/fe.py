"""Q_p nodal basis by interpolation in Gauss-Lobatto points (PAPER.md l.79:
"Q_p(T) is the space of tensor product polynomials of degree up to p with a
nodal basis defined by interpolation in Gauss-Lobatto points").

Test infrastructure only (see oracle/__init__.py).
"""
from functools import lru_cache
from math import factorial

import numpy as np
from numpy.polynomial import Polynomial, legendre


@lru_cache(maxsize=None)
def gauss_lobatto_nodes(p):
    """The p+1 Gauss-Lobatto points on [0,1]: 0, 1 and the roots of P_p'."""
    if p < 1:
        raise ValueError("degree must be >= 1")
    if p == 1:
        return np.array([0.0, 1.0])
    c = np.zeros(p + 1)
    c[p] = 1.0
    inner = np.sort(legendre.legroots(legendre.legder(c)).real)
    x = np.concatenate([[-1.0], inner, [1.0]])
    return 0.5 * (x + 1.0)


@lru_cache(maxsize=None)
def lagrange_polys(p):
    """Lagrange polynomials L_0..L_p on the Gauss-Lobatto nodes of [0,1]."""
    nodes = gauss_lobatto_nodes(p)
    polys = []
    for i in range(p + 1):
        others = np.delete(nodes, i)
        num = Polynomial.fromroots(others)
        polys.append(num / float(np.prod(nodes[i] - others)))
    return tuple(polys)


@lru_cache(maxsize=None)
def lagrange_derivs(p, k):
    """d^k L_i / dxi^k, i = 0..p, as polynomials (cached)."""
    return tuple(L.deriv(k) if k > 0 else L for L in lagrange_polys(p))


def basis_1d(p, x, k=0):
    """Matrix [i, q] = d^k L_i / dxi^k (x_q) on the reference interval [0,1]."""
    x = np.asarray(x, dtype=np.float64)
    return np.array([D(x) for D in lagrange_derivs(p, k)])


def gauss_legendre(n):
    """n-point Gauss-Legendre rule on [0,1] (points, weights)."""
    x, w = legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def ghost_weight(k, h, gamma_k, sigma):
    """Coefficient gamma_k h^(2k+sigma) / (k!)^2 of the ghost penalty
    (sigma is reading R5 in DESIGN.md)."""
    return gamma_k * h ** (2 * k + sigma) / float(factorial(k)) ** 2
