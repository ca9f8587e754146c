"""Pins for the oracle's non-symmetric path: Algorithm 2 with separate row and column sets
(lines 4-12): getBasis(K_{Xbar^(row) Y*}) -> U_i, X^_i^(row) and getBasis(K_{Y* Xbar^(col)}^T)
-> V_i, X^_i^(col); coupling blocks B_ij = K(X^_i^(row), X^_j^(col)) for every ordered admissible pair
and nearfield blocks for every ordered nearfield pair; the H^2 product with V on the way
up and U on the way down.  Kernel: the shifted multiquadric sqrt(1 + c |x - y + a|^2) of P:711-716
(kappa(x, y) != kappa(y, x)).

Pinned by: the kernel's closed form and its non-symmetry; a symmetric kernel run through the
non-symmetric path reproduces the symmetric build bit for bit (V = U, X^(col) = X^(row), the same
product); a single leaf is the dense matrix exactly; the column bases satisfy their interpolative
identity; the matvec error against brute-force dense K x falls as id_tol falls; the calibration's
two orientations (reading E7).
"""
import numpy as np
import pytest

import synth

C_MQ, A_MQ = 100.0, np.array([0.0, 0.3])


def _mq_np(A, B, c=C_MQ, a=A_MQ):
    return np.sqrt(1.0 + c * (((A[:, None, :] - B[None, :, :]) + a) ** 2).sum(-1))


def test_mq_kernel_closed_form_and_nonsymmetry(orc):
    orc.set_kernel_shift(A_MQ)
    rng = np.random.default_rng(0)
    X = rng.random((20, 2))
    Y = rng.random((20, 2))
    K = np.array([[orc.kernel(7, C_MQ, x, y) for y in Y] for x in X])
    np.testing.assert_allclose(K, _mq_np(X, Y), rtol=1e-15)
    Kt = np.array([[orc.kernel(7, C_MQ, y, x) for y in Y] for x in X])
    assert np.abs(K - Kt).max() > 1.0                          # not symmetric
    assert orc.kernel(7, C_MQ, np.array([0.0, 0.0]), A_MQ) == 1.0    # x - y + a = 0


@pytest.mark.parametrize("kid,param", [(1, 0.0), (2, 0.3), (3, 0.2)])
def test_symmetric_kernel_through_nonsym_path_is_bitwise_the_symmetric_build(orc, kid, param):
    pts = synth.clustered(3000, 3, seed=31, k=3, sigma=0.1)
    a = orc.OracleH2(pts, 32, 0.5)
    r = a.build(kid, param, 1e-6)
    b = orc.OracleH2(pts, 32, 0.5, nonsym=True)
    rb = b.build(kid, param, 1e-6)
    assert r == rb
    assert np.array_equal(b.export(orc.K_COL), b.export(orc.K))
    assert np.array_equal(b.export(orc.SKC_IDX), b.export(orc.SK_IDX))
    assert np.array_equal(b.export(orc.V), b.export(orc.U))
    assert np.array_equal(b.export(orc.U), a.export(orc.U))
    x = np.random.default_rng(1).standard_normal(3000)
    assert np.array_equal(a.matvec(x), b.matvec(x))
    # every ordered block: twice the off-diagonal entries of the symmetric-once store
    na, _ = a.fill()
    nb, _ = b.fill()
    nd = b.nodes()
    off, idx = b.nf()
    diag = sum((nd["end"][i] - nd["begin"][i]) ** 2 for i in range(len(nd["level"])) if off[i + 1] > off[i])
    assert nb == 2 * na - diag


def test_nonsym_single_leaf_is_dense_exact(orc):
    orc.set_kernel_shift(A_MQ)
    pts = synth.uniform_cube(60, 2, seed=2)
    o = orc.OracleH2(pts, 64, 0.5, nonsym=True)
    o.build(7, C_MQ, 1e-6)
    x = np.random.default_rng(2).standard_normal(60)
    y = o.matvec(x)
    np.testing.assert_allclose(y, _mq_np(pts, pts) @ x, rtol=1e-13)


def test_nonsym_column_bases_interpolate(orc):
    """K(Y_i^*, Xbar_i^(col)) = K(Y_i^*, X^_i^(col)) V_i^T up to ~id_tol (Eq.(4.1) transposed)."""
    orc.set_kernel_shift(A_MQ)
    pts = synth.uniform_cube(4000, 2, seed=3)
    o = orc.OracleH2(pts, 32, 0.5, nonsym=True)
    tol = 1e-7
    o.build(7, C_MQ, tol)
    X = o.tree_points()
    nd = o.nodes()
    kc = o.export(orc.K_COL)
    so, si = o.skeletons_col()
    vo, V = o.export(orc.V_OFF), o.export(orc.V)
    yo, yi = o.ystar()
    checked = 0
    for i in range(1, len(kc)):
        if kc[i] == 0:
            continue
        if nd["is_leaf"][i]:
            xb = np.arange(nd["begin"][i], nd["end"][i])
        else:
            ch = range(nd["first_child"][i], nd["first_child"][i] + nd["nchild"][i])
            xb = np.concatenate([si[so[c]:so[c + 1]] for c in ch])
        Y = X[yi[yo[i]:yo[i + 1]]]
        A = _mq_np(Y, X[xb])                                   # K(Y*, Xbar^(col))
        Vi = V[vo[i]:vo[i + 1]].reshape(kc[i], len(xb)).T      # |Xbar| x k
        sk = si[so[i]:so[i + 1]]
        rec = _mq_np(Y, X[sk]) @ Vi.T
        assert np.linalg.norm(A - rec) <= 50 * tol * np.linalg.norm(A), i
        checked += 1
    assert checked > 20


def test_nonsym_matvec_error_falls_with_tol(orc):
    orc.set_kernel_shift(A_MQ)
    pts = synth.uniform_cube(4096, 2, seed=4)
    x = np.random.default_rng(4).standard_normal(4096)
    yd = _mq_np(pts, pts) @ x
    errs, rows_cols = [], []
    for tol in (1e-2, 1e-4, 1e-6, 1e-8):
        o = orc.OracleH2(pts, 32, 0.5, nonsym=True)
        o.build(7, C_MQ, tol)
        y = o.matvec(x)
        errs.append(np.linalg.norm(y - yd) / np.linalg.norm(yd))
        yo = orc.dense_rows(pts, 7, C_MQ, x, np.arange(4096))
        np.testing.assert_allclose(yo, yd, rtol=1e-12)          # the oracle's dense rows = numpy
        rows_cols.append(int(o.export(orc.K).sum() != o.export(orc.K_COL).sum()))
    assert errs[0] > errs[1] > errs[2] > errs[3], errs
    assert errs[3] < 1e-4, errs                                 # (the method error is >> id_tol)
    assert any(rows_cols)                                       # row and column ranks differ somewhere


def test_nonsym_calibration_takes_both_orientations(orc):
    orc.set_kernel_shift(np.array([0.0, 0.6]))
    pts = synth.uniform_cube(4000, 2, seed=5)
    o = orc.OracleH2(pts, 32, 0.5, nonsym=True)
    r = o.calibrate(7, C_MQ, 1e-6)
    rl = o.calib_levels()
    W = float(np.max(pts.max(0) - pts.min(0)))
    for l in range(len(rl)):
        if rl[l]:
            r0 = orc.calib_level(2, 7, C_MQ, 1e-6, 0.5, W * 2.0 ** -l, l, 0)
            r1 = orc.calib_level(2, 7, C_MQ, 1e-6, 0.5, W * 2.0 ** -l, l, 1)
            assert rl[l] == max(r0, r1)
    assert r == max(1, rl.max())
