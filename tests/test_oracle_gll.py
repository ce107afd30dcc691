"""Pins for oracle C-1 (GLL basis): closed forms, quadrature exactness, D exactness.

SURVEY.md §8(c) C-1; north star "GLL weights sum to 2 and D
differentiates degree <= p polynomials exactly".
"""
import math

import numpy as np
import pytest

import oracle
from tests.dense_ref import lagrange_deriv_matrix


def test_closed_form_p1_p2():
    z, w, D = oracle.gll(1)
    assert np.array_equal(z, [-1.0, 1.0]) and np.array_equal(w, [1.0, 1.0])
    z, w, D = oracle.gll(2)
    np.testing.assert_allclose(z, [-1.0, 0.0, 1.0], atol=1e-16)
    np.testing.assert_allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=1e-15)
    # textbook 3-point GLL derivative matrix
    np.testing.assert_allclose(D, [[-1.5, 2.0, -0.5], [-0.5, 0.0, 0.5], [0.5, -2.0, 1.5]], atol=1e-15)


def test_closed_form_p3_p4():
    # p=3: +-1, +-1/sqrt(5); weights 1/6, 5/6.  p=4: 0, +-sqrt(3/7); weights 1/10, 49/90, 32/45
    z, w, _ = oracle.gll(3)
    np.testing.assert_allclose(z, [-1, -1 / np.sqrt(5), 1 / np.sqrt(5), 1], atol=2e-16)
    np.testing.assert_allclose(w, [1 / 6, 5 / 6, 5 / 6, 1 / 6], rtol=2e-15)
    z, w, _ = oracle.gll(4)
    s = np.sqrt(3 / 7)
    np.testing.assert_allclose(z, [-1, -s, 0, s, 1], atol=2e-16)
    np.testing.assert_allclose(w, [0.1, 49 / 90, 32 / 45, 49 / 90, 0.1], rtol=2e-15)


@pytest.mark.parametrize("p", list(range(1, 16)))
def test_weights_quadrature_and_symmetry(p):
    z, w, D = oracle.gll(p)
    # north star: |sum w - 2| <= 4e-16, read as 2 ulp(1) = 4.44e-16 (DESIGN.md §3 R-1):
    # the exact sum (fsum) of the stored weights, for every p up to the configs' 11;
    # beyond p = 11 the weights carry a few ulps more.
    assert abs(math.fsum(w) - 2.0) <= (4.5e-16 if p <= 11 else 1.0e-15)
    assert np.all(np.diff(z) > 0)
    np.testing.assert_allclose(z, -z[::-1], atol=1e-15)
    # exact for x^k, k <= 2p-1: int_{-1}^{1} x^k = 2/(k+1) for even k, 0 for odd
    for k in range(2 * p):
        exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
        assert abs(np.dot(w, z ** k) - exact) <= 1.2e-15, (p, k)


@pytest.mark.parametrize("p", list(range(1, 16)))
def test_D_differentiates_polynomials(p):
    z, w, D = oracle.gll(p)
    assert np.max(np.abs(D @ np.ones(p + 1))) <= 1e-15 * (p + 1) ** 2
    for k in range(1, p + 1):
        err = np.max(np.abs(D @ z ** k - k * z ** (k - 1)))
        assert err <= 1e-12, (p, k, err)
    # end diagonal entries -/+ p(p+1)/4, interior 0 (exact-arithmetic values)
    assert abs(D[0, 0] + p * (p + 1) / 4) <= 1e-12
    assert abs(D[p, p] - p * (p + 1) / 4) <= 1e-12
    if p > 1:
        assert np.max(np.abs(np.diag(D)[1:-1])) <= 1e-12


@pytest.mark.parametrize("p", [2, 3, 5, 7])
def test_D_matches_lagrange_polynomials(p):
    z, _, D = oracle.gll(p)
    np.testing.assert_allclose(D, lagrange_deriv_matrix(z), atol=1e-11)


def test_local_grad3_r_coordinate():
    """u = r on the reference element gives ur = 1, us = ut = 0."""
    for p in (2, 5, 7, 11):
        z, _, D = oracle.gll(p)
        n = p + 1
        u = np.tile(z, n * n)            # u[i + n j + n^2 k] = z_i
        ur, us, ut = oracle.local_grad3(p, D, u)
        assert np.max(np.abs(ur - 1)) < 1e-12
        assert np.max(np.abs(us)) < 1e-12 and np.max(np.abs(ut)) < 1e-12
        # t-coordinate: ut = 1
        u = np.repeat(z, n * n)
        ur, us, ut = oracle.local_grad3(p, D, u)
        assert np.max(np.abs(ut - 1)) < 1e-12 and np.max(np.abs(ur)) < 1e-12
