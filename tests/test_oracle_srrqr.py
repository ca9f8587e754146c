"""Pins for the oracle's SRRQR refinement of getBasis (PAPER Eq.(4.1): "P [I; G] ...
||G||_max is bounded by a prescribed constant"; Gu & Eisenstat's strong rank-revealing swaps at
fixed rank).

  * the Kahan matrix (the textbook case where column pivoting takes no pivots and leaves G huge):
    CPQR's max|G| is far above f, SRRQR's is <= f and its smallest R11 diagonal grows;
  * whenever CPQR already has max|G| <= f, SRRQR changes nothing (same skeleton, same U bitwise);
  * on generic and kernel matrices: max|G| <= f, U restricted to the skeleton = I, the rank is the
    CPQR rank, and the residual obeys the strong-RRQR bound ||A - U A_S||_2 <= sqrt(1 + f^2 k (n-k))
    sigma_{k+1}(A) (Gu-Eisenstat Thm. 3.2);
  * through the whole H^2 build: every U_i entry is bounded by f and the matvec error stays at the
    CPQR build's.
"""
import numpy as np
import pytest

import synth


def kahan(n, theta=1.2, pert=1e-10):
    c, s = np.cos(theta), np.sin(theta)
    R = np.triu(-c * np.ones((n, n)), 1) + np.eye(n)
    R = np.diag(s ** np.arange(n)) @ R
    return R @ np.diag((1 - pert) ** np.arange(n))  # column norms decrease: CPQR keeps the order


def test_kahan_cpqr_fails_srrqr_bounds_g(orc):
    n = 40
    R = kahan(n)
    A = R.T                                           # orc_id factors A^T = R
    # every residual column norm of the Kahan matrix at step t is s^t: tol = s^(n - 1.5) stops at n - 1
    tol = np.sin(1.2) ** (n - 1.5)
    sk0, U0 = orc.interp_decomp(A, tol)
    sk1, U1, sw = orc.interp_decomp_srrqr(A, tol, 2.0)
    k = len(sk0)
    assert len(sk1) == k == n - 1
    rest0 = np.setdiff1d(np.arange(n), sk0)
    rest1 = np.setdiff1d(np.arange(n), sk1)
    g0, g1 = np.abs(U0[rest0]).max(), np.abs(U1[rest1]).max()
    assert g0 > 1e3 and g1 <= 2.0 * (1 + 1e-12) and sw >= 1, (g0, g1, sw)
    s_min = lambda sk: np.linalg.svd(A[sk], compute_uv=False)[-1]  # noqa: E731
    assert s_min(sk1) > 10 * s_min(sk0)


def test_srrqr_is_cpqr_when_g_is_small(orc):
    rng = np.random.default_rng(7)
    A = rng.standard_normal((60, 40)) @ rng.standard_normal((40, 80)) * 1e-3 + rng.standard_normal((60, 80)) * 1e-12
    sk0, U0 = orc.interp_decomp(A, 1e-8)
    rest = np.setdiff1d(np.arange(60), sk0)
    f = 1.0001 * np.abs(U0[rest]).max()
    sk1, U1, sw = orc.interp_decomp_srrqr(A, 1e-8, f)
    assert sw == 0 and np.array_equal(sk0, sk1) and np.array_equal(U0, U1)


@pytest.mark.parametrize("f", [1.05, 1.5, 2.0])
@pytest.mark.parametrize("kind", ["lowrank", "coulomb"])
def test_srrqr_invariants_and_residual_bound(orc, f, kind):
    rng = np.random.default_rng(11)
    if kind == "lowrank":
        A = rng.standard_normal((120, 30)) @ np.diag(np.logspace(0, -12, 30)) @ rng.standard_normal((30, 90))
    else:
        X = rng.random((150, 3))
        Y = rng.random((100, 3)) + np.array([2.0, 0.0, 0.0])
        A = 1.0 / np.linalg.norm(X[:, None] - Y[None], axis=2)
    tol = 1e-9
    sk0, _ = orc.interp_decomp(A, tol)
    sk, U, sw = orc.interp_decomp_srrqr(A, tol, f)
    k, n = len(sk), A.shape[0]
    assert k == len(sk0)
    np.testing.assert_array_equal(U[sk], np.eye(k))
    rest = np.setdiff1d(np.arange(n), sk)
    assert np.abs(U[rest]).max() <= f * (1 + 1e-10)
    sig = np.linalg.svd(A, compute_uv=False)
    res = np.linalg.norm(A - U @ A[sk], 2)
    assert res <= np.sqrt(1 + f * f * k * (n - k)) * sig[k] * (1 + 1e-6) + 1e-14 * sig[0], (res, sig[k])


def test_h2_build_with_srrqr(orc):
    pts = synth.uniform_cube(5000, 3, seed=9)
    a = orc.OracleH2(pts, 32, 0.5)
    a.build(1, 0.0, 1e-7)
    b = orc.OracleH2(pts, 32, 0.5, srrqr_f=1.2)
    b.build(1, 0.0, 1e-7)
    assert np.array_equal(a.export(orc.K), b.export(orc.K))
    assert np.abs(b.export(orc.U)).max() <= 1.2 * (1 + 1e-10)
    assert b.srrqr_swaps() > 0
    x = np.random.default_rng(1).standard_normal(5000)
    yd = orc.dense_rows(pts, 1, 0.0, x, np.arange(5000))
    ea = np.linalg.norm(a.matvec(x) - yd) / np.linalg.norm(yd)
    eb = np.linalg.norm(b.matvec(x) - yd) / np.linalg.norm(yd)
    assert eb <= 3 * ea, (ea, eb)
