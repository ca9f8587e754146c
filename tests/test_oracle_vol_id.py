"""Pins for oracle steps C (volume DataReduct) and F (pivoted-QR ID).

C is pinned by SPEC's hand-derived examples, by a KD-tree nearest-neighbour library
routine (scipy.spatial.cKDTree) at every grid node, and by the subset / budget / equivariance
invariants.  F is pinned by LAPACK dgeqp3 (scipy.linalg.qr(pivoting=True)) pivots and
|R| diagonals on generic matrices, an exact diagonal case for the stop rule (reading F2), exact
reconstruction at full rank, rank-1 input, the interpolative identity, the
rank bound of Eq.(4.4), and a truncated-SVD error bound.
"""
import numpy as np
import pytest
import scipy.linalg
from scipy.spatial import cKDTree


# ---------------------------------------------------------------- C. Vol

def test_vol_passthrough(orc):
    X = np.random.default_rng(0).random((10, 2))
    assert list(orc.vol(X, [7, 3, 5], 4)) == [3, 5, 7]          # |S| <= k -> S sorted (C5)
    assert list(orc.vol(X, [9, 1, 2, 4], 4)) == [1, 2, 4, 9]


def test_vol_four_corners(orc):
    X = np.array([[0, 0], [1, 0], [0, 1], [1, 1], [0.5, 0.5]], float)   # S:140 plus a centre point
    assert list(orc.vol(X, [0, 1, 2, 3, 4], 4)) == [0, 1, 2, 3]        # m=2: each cell centre's corner


def test_vol_m1_box_centre(orc):
    X = np.array([[0.0, 0.0], [0.9, 0.1], [0.45, 0.52], [1.0, 1.0]])   # m=1 -> nearest to centre
    assert list(orc.vol(X, [0, 1, 2, 3], 3)) == [2]                    # 3 < 2^2 -> m = 1


def test_vol_grid_100_points_2x2(orc):
    # 100 grid points (i/9, j/9); cell centres (.25|.75)^2 -> nearest grid values 2/9, 7/9
    g = np.arange(10) / 9
    X = np.stack(np.meshgrid(g, g, indexing="ij"), -1).reshape(-1, 2)
    got = orc.vol(X, np.arange(100), 4)
    expect = sorted(int(i * 10 + j) for i in (2, 7) for j in (2, 7))
    assert list(got) == expect


def test_vol_tie_lowest_index(orc):
    # two points equidistant from the single grid node (m=1 box centre) -> the lower index
    X = np.array([[0.0], [1.0], [0.25], [0.75]])
    assert list(orc.vol(X, [0, 1, 2, 3], 1)) == [2]
    assert list(orc.vol(X, [3, 2, 1, 0], 1)) == [2]


@pytest.mark.parametrize("d,ns,k", [(1, 200, 7), (2, 500, 36), (3, 1000, 64), (3, 300, 343), (5, 800, 243)])
def test_vol_nearest_against_kdtree(orc, d, ns, k):
    rng = np.random.default_rng(d * 100 + k)
    X = rng.random((ns + 50, d)) * rng.random(d) * 3 - 1
    S = np.sort(rng.choice(ns + 50, ns, replace=False)).astype(np.int32)
    got = orc.vol(X, S, k)
    m = int(np.floor(k ** (1 / d) + 1e-9))
    while (m + 1) ** d <= k:
        m += 1
    while m ** d > k:
        m -= 1
    assert len(got) <= m ** d <= k
    assert len(set(got.tolist())) == len(got) and list(got) == sorted(got)
    assert set(got.tolist()) <= set(S.tolist())
    P = X[S]
    lo, hi = P.min(0), P.max(0)
    axes = [lo[c] + (np.arange(m) + 0.5) * ((hi[c] - lo[c]) / m) for c in range(d)]
    Q = np.stack(np.meshgrid(*axes, indexing="ij"), -1).reshape(-1, d)
    dist, nn = cKDTree(P).query(Q)
    # every KD-tree nearest neighbour is matched by a selected point at the same distance
    for q, dq in zip(Q, dist):
        dsel = np.sqrt(((X[got] - q) ** 2).sum(1)).min()
        assert dsel <= dq * (1 + 1e-12) + 1e-300


def test_vol_scale_translate_equivariance(orc):
    rng = np.random.default_rng(3)
    X = rng.random((400, 3))
    S = np.arange(400)
    base = orc.vol(X, S, 27)
    assert list(orc.vol(X * 4.0 + 2.0, S, 27)) == list(base)      # dyadic scale + shift: exact
    assert list(orc.vol(X * 0.5 - 8.0, S, 27)) == list(base)


# ---------------------------------------------------------------- F. CPQR / ID

@pytest.mark.parametrize("shape", [(8, 8), (20, 12), (12, 30), (64, 100), (57, 256)])
def test_cpqr_pivots_match_lapack_dgeqp3(orc, shape):
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    M = rng.standard_normal(shape)
    k, piv, Mo = orc.cpqr(M, 1e-300)
    Q, R, P = scipy.linalg.qr(M, pivoting=True, mode="economic")
    kk = min(shape)
    assert k == kk
    assert list(piv[:kk]) == list(P[:kk])
    np.testing.assert_allclose(np.abs(np.diag(Mo)[:kk]), np.abs(np.diag(R)), rtol=1e-10)


def test_cpqr_pivots_match_lapack_on_kernel_block(orc):
    rng = np.random.default_rng(5)
    X = rng.random((256, 3))
    Y = rng.random((64, 3)) + 3.0
    A = 1.0 / np.sqrt(((X[:, None, :] - Y[None]) ** 2).sum(-1))
    M = A.T.copy()
    tol = 1e-8
    k, piv, Mo = orc.cpqr(M, tol)
    Q, R, P = scipy.linalg.qr(M, pivoting=True, mode="economic")
    dR = np.abs(np.diag(R))
    k_lapack = int(np.sum(dR >= tol * dR[0]))
    assert k == k_lapack
    assert list(piv[:k]) == list(P[:k])


def test_cpqr_stop_rule_exact_diagonal(orc):
    # diag(1, 1/2, ..., 2^-9) in scrambled column order: R_tt = 2^-t exactly; stop at tol boundary
    d = 2.0 ** -np.arange(10)
    order = np.array([3, 7, 0, 9, 1, 5, 2, 8, 4, 6])
    M = np.zeros((10, 10))
    for c, j in enumerate(order):
        M[j, c] = d[j]
    k, piv, _ = orc.cpqr(M, 2.0 ** -4)           # boundary |R_55| = tol * |R_11| is kept (F2)
    assert k == 5
    assert [order[p] for p in piv[:k]] == [0, 1, 2, 3, 4]
    k2, _, _ = orc.cpqr(M, 2.0 ** -4 * 1.0000001)
    assert k2 == 4
    assert orc.cpqr(np.zeros((4, 6)), 1e-6)[0] == 0   # R11 = 0 -> k = 0


def test_id_full_rank_reconstructs_exactly(orc):
    rng = np.random.default_rng(9)
    A = rng.standard_normal((30, 12))
    skel, U = orc.interp_decomp(A, 1e-300)
    assert len(skel) == 12
    np.testing.assert_allclose(U @ A[skel], A, atol=1e-12 * np.abs(A).max())
    np.testing.assert_array_equal(U[skel], np.eye(12))             # interpolative identity


def test_id_rank_one(orc):
    rng = np.random.default_rng(10)
    u, v = rng.standard_normal(40), rng.standard_normal(25)
    A = np.outer(u, v)
    skel, U = orc.interp_decomp(A, 1e-10)
    assert len(skel) == 1
    assert np.abs(U @ A[skel] - A).max() <= 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("seed", range(4))
def test_id_svd_bound(orc, seed):
    rng = np.random.default_rng(seed)
    m, n = 60, 40
    Ua, _ = np.linalg.qr(rng.standard_normal((m, m)))
    Va, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = 2.0 ** -np.arange(n)
    A = (Ua[:, :n] * s) @ Va.T
    tol = 1e-6
    skel, U = orc.interp_decomp(A, tol)
    k = len(skel)
    assert k <= n                                                   # Eq.(4.4)
    err = np.linalg.norm(A - U @ A[skel], 2)
    sk1 = s[k] if k < n else 0.0
    assert err <= 10 * np.sqrt(k * (m - k) + 1) * (k + 1) * sk1 + 1e-14   # S:265 (loose)
    assert err <= 1e3 * tol * s[0]
    np.testing.assert_array_equal(U[skel], np.eye(k))
