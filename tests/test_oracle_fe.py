"""Oracle pins for the Q_p basis against closed forms."""
import math

import numpy as np
import pytest

from oracle.fe import basis_1d, gauss_legendre, gauss_lobatto_nodes




def test_gauss_lobatto_closed_forms():
    # closed forms of the Gauss-Lobatto points on [0,1]
    assert np.allclose(gauss_lobatto_nodes(1), [0, 1], atol=0, rtol=0)
    assert np.allclose(gauss_lobatto_nodes(2), [0, 0.5, 1], atol=1e-15)
    s5 = 1 / math.sqrt(5)
    assert np.allclose(gauss_lobatto_nodes(3), [0, (1 - s5) / 2, (1 + s5) / 2, 1], atol=1e-15)
    s37 = math.sqrt(3 / 7)
    assert np.allclose(gauss_lobatto_nodes(4), [0, (1 - s37) / 2, 0.5, (1 + s37) / 2, 1], atol=1e-15)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_nodal_partition_and_reproduction(p):
    nodes = gauss_lobatto_nodes(p)
    assert np.allclose(basis_1d(p, nodes), np.eye(p + 1), atol=1e-13)
    x = np.linspace(-0.3, 1.3, 23)
    assert np.allclose(basis_1d(p, x).sum(axis=0), 1.0, atol=1e-13)
    # k-th derivative of the interpolant of x^m equals the exact derivative (m <= p)
    for m in range(p + 1):
        for k in range(p + 1):
            exact = (math.factorial(m) / math.factorial(m - k) * x ** (m - k)) if k <= m else 0 * x
            got = nodes ** m @ basis_1d(p, x, k)
            assert np.allclose(got, exact, atol=1e-11)


def test_q1_hat_functions():
    x = np.array([0.0, 0.25, 1.0])
    assert np.allclose(basis_1d(1, x), [[1, 0.75, 0], [0, 0.25, 1]])
    assert np.allclose(basis_1d(1, x, 1), [[-1, -1, -1], [1, 1, 1]])


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_gauss_legendre_exactness(n):
    g, w = gauss_legendre(n)
    for m in range(2 * n):
        assert abs(w @ g ** m - 1.0 / (m + 1)) < 1e-14
