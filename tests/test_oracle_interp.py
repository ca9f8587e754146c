"""Pins of the interpolation-baseline oracle (oracle/interp.py; Eq. (2.2)).

Each pin checks the oracle against mathematics that does not depend on how it is written: the
Kronecker property and partition of unity of the Lagrange basis, exact reproduction of polynomials
(the monomial expansion written out, not the oracle's product formula), the textbook Chebyshev
interpolation error bound, the nestedness identity U_c R_c = L^(parent)(X_c) (exact because
L^(parent) has degree p - 1 per variable), and the convergence of the H^2 matvec to dense K x.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from oracle import interp


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8, 12])
def test_lagrange_kronecker_and_partition_of_unity(p):
    z = interp.cheb_ref(p)
    assert np.all(np.diff(z) < 0) and np.all(np.abs(z) < 1.0)  # distinct, inside (-1, 1)
    np.testing.assert_allclose(interp.lagrange_1d(z, z), np.eye(p), atol=1e-14)
    u = np.linspace(-1.0, 1.0, 101)
    np.testing.assert_allclose(interp.lagrange_1d(z, u).sum(axis=1), 1.0, atol=1e-12)


@pytest.mark.parametrize("p,d", [(2, 1), (4, 2), (5, 3), (3, 4)])
def test_tensor_interpolation_reproduces_polynomials(p, d):
    """sum_alpha f(q_alpha) L_alpha(x) = f(x) for f of degree <= p - 1 in each variable."""
    rng = np.random.default_rng(11 + p + d)
    coef = rng.standard_normal((p,) * d)

    def f(X):  # sum_a coef[a] prod_c x_c^{a_c}, the monomial expansion written out
        out = np.zeros(len(X))
        for a in np.ndindex(*coef.shape):
            out += coef[a] * np.prod([X[:, c] ** a[c] for c in range(d)], axis=0)
        return out

    center, half = rng.standard_normal(d), 0.3 + rng.random()
    z = interp.cheb_ref(p)
    Q = interp.cheb_points(center, half, z)
    X = center + half * (2.0 * rng.random((50, d)) - 1.0)
    U = interp.lagrange_nd(X, center, half, z)
    np.testing.assert_allclose(U @ f(Q), f(X), rtol=1e-10, atol=1e-10 * np.abs(coef).sum())


@pytest.mark.parametrize("p", range(2, 11))
def test_chebyshev_error_bound_exp(p):
    """|e^u - I_p e^u| <= max|f^(p)| / (2^(p-1) p!) on [-1, 1] (first-kind nodes), max|f^(p)| = e."""
    z = interp.cheb_ref(p)
    u = np.linspace(-1.0, 1.0, 2001)
    err = np.max(np.abs(interp.lagrange_1d(z, u) @ np.exp(z) - np.exp(u)))
    assert err <= math.e / (2 ** (p - 1) * math.factorial(p)) * (1 + 1e-9) + 1e-15


@pytest.fixture(scope="module")
def sphere_tree():
    oracle.build()
    pts = synth.three_spheres(1500, 5)
    return pts, oracle.OracleH2(pts, 24, 0.5)


@pytest.mark.parametrize("p", [2, 4])
def test_nested_transfers(sphere_tree, p):
    """For a leaf c with parent P: L^(P)(X_c) = U_c R_c exactly (L^(P) has degree p - 1 per variable,
    reproduced by the child's interpolation), and every node's box contains its points."""
    pts, o = sphere_tree
    m = interp.InterpH2(o, p, 2, 1.0)
    checked = 0
    for c in range(m.nn):
        if m.k[c] == 0:
            continue
        Xc = m.X[m.begin[c]:m.end[c]]
        assert np.all(np.abs(Xc - m.center[c]) <= m.half[c] * (1 + 1e-12))
        P = m.parent[c]
        if not m.is_leaf[c] or P < 0 or m.k[P] == 0:
            continue
        direct = interp.lagrange_nd(Xc, m.center[P], m.half[P], m.z)
        np.testing.assert_allclose(m.U[c] @ m.transfer(c), direct, atol=1e-11)
        checked += 1
    assert checked > 10


def test_bases_exist_exactly_where_a_farfield_does(sphere_tree):
    pts, o = sphere_tree
    m = interp.InterpH2(o, 2, 2, 1.0)
    ilo, ili = o.il()
    for i in range(m.nn):
        anc, far = i, False
        while anc >= 0:
            far = far or ilo[anc + 1] > ilo[anc]
            anc = m.parent[anc]
        assert (m.k[i] > 0) == far


def test_matvec_converges_to_dense(sphere_tree):
    """The interpolation H^2 matvec error against dense K x falls with p (Gaussian, smooth: geometric)."""
    pts, o = sphere_tree
    n = len(pts)
    x = synth._rng(9).standard_normal(n)
    yd = oracle.dense_rows(pts, 2, 1.0, x, np.arange(n))
    errs = []
    for p in (2, 3, 4, 5):
        y = interp.InterpH2(o, p, 2, 1.0).matvec(x)
        errs.append(np.linalg.norm(y - yd) / np.linalg.norm(yd))
    assert all(b < 0.5 * a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-4


def test_memory_counts(sphere_tree):
    pts, o = sphere_tree
    m = interp.InterpH2(o, 3, 2, 1.0)
    mem = m.memory_entries()
    ilo, ili = o.il()
    pairs = sum(1 for i in range(m.nn) for j in ili[ilo[i]:ilo[i + 1]] if j > i)
    assert mem["coupling"] == pairs * m.r ** 2
    assert mem["u"] == sum(((m.end[i] - m.begin[i]) if m.is_leaf[i] else m.nchild[i] * m.r) * m.r
                           for i in range(m.nn) if m.k[i] > 0)
    assert mem["total"] == mem["u"] + mem["coupling"] + mem["nearfield"]
