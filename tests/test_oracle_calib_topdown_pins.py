"""Pins for the two oracle parts round 1 left "parity unpinned": the r calibration (step E) and the
composition of HiDR's top-down sweep (step D, Algorithm 1 lines 14-21).

E (Alg. 2 line 2; "r1 = r2 = r ... increasing ... until the error on O(1) random
well-separated points is below the tolerance"; readings E1-E6 in DESIGN.md):
  * the point sets follow E4/E6: an independent Python SplitMix64 regenerates Z1 and Z2 bit for
    bit (pins the generator, the level seed, the box width and the w/tau shift);
  * Eckart-Young: the ID approximant U K(Z1[skel], Z2) has rank k, so e >= the best rank-k
    relative Frobenius error sqrt(sum_{i>k} s_i^2) / ||K||_F (numpy SVD of K(Z1, Z2));
  * the CPQR ID coefficients are the least-squares ones on the columns the ID saw (A^T P = QR:
    the skeleton rows span Q1 and T = R11^-1 R12 is the projection), so e equals the error of
    the lstsq fit on K(Z1, Z2*) applied to the FULL K(Z1, Z2), and is >= the lstsq fit on the
    full K (pins "error against K(Z1,Z2), not K(Z1,Z2*)" and the Frobenius norm);
  * pass-through at m^d >= 256: every residual column norm < 1e-3 eps |R11| at the stop and
    |R11| <= ||K||_F, so e <= sqrt(256 - k) 1e-3 eps;
  * composition: the per-level r equals calib_level at w = W 2^-l for exactly the levels holding
    an admissible pair (W from the points, reading A1), r = their max, and calib_level is the
    first m whose trial passes (e < 1e-2 eps, E2);
  * special cases: a near-constant Gaussian (h = 1e6) and a vanishing one (h = 0.01) give r = 1.
D top-down: Y_i^* = Vol(T_i, r) with T_i = Y_p^* U (U_{j in IL(i)} X_j^*) checked
  against a hand-derived golden (tests/golden/hidr_1d_16_r2.txt) and, on random data, against a
  KD-tree (scipy cKDTree) nearest-point selection over the union built from the exports.
"""
import os

import numpy as np
import pytest
from scipy.spatial import cKDTree

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hidr_1d_16_r2.txt")
MASK = (1 << 64) - 1


def _splitmix64(state):
    """DESIGN.md E6, written from its text: state += golden gamma, then the two xor-shift
    multiplies and the final xor-shift."""
    state = (state + 0x9E3779B97F4A7C15) & MASK
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return state, z ^ (z >> 31)


def _kernel_np(kid, p, A, B):
    """Closed forms (BASELINE configs) in numpy, independent of the oracle's C code."""
    r = np.sqrt(((A[:, None, :] - B[None, :, :]) ** 2).sum(-1))
    if kid == synth.KERNEL_COULOMB:
        with np.errstate(divide="ignore"):
            return np.where(r > 0, 1.0 / np.where(r > 0, r, 1.0), 0.0)
    if kid == synth.KERNEL_GAUSSIAN:
        return np.exp(-(r / p) ** 2)
    if kid == synth.KERNEL_MATERN32:
        t = np.sqrt(3.0) * r / p
        return (1 + t) * np.exp(-t)
    raise ValueError(kid)


CASES = [  # (d, kernel, param, eps, w, level)
    (3, synth.KERNEL_COULOMB, 0.0, 1e-6, 0.25, 2),
    (3, synth.KERNEL_COULOMB, 0.0, 1e-8, 0.125, 3),
    (3, synth.KERNEL_GAUSSIAN, 0.5, 1e-6, 0.5, 1),
    (2, synth.KERNEL_MATERN32, 0.1, 1e-6, 0.25, 2),
    (2, synth.KERNEL_MATERN32, 0.1, 1e-6, 0.0625, 4),
    (5, synth.KERNEL_GAUSSIAN, 1.0, 1e-4, 1.1, 1),
]


@pytest.mark.parametrize("d,tau,w,level", [(3, 0.5, 0.25, 2), (2, 0.5, 0.0625, 4), (5, 0.5, 1.1, 1),
                                           (3, 0.7, 0.3, 0)])
def test_calib_points_follow_e6(orc, d, tau, w, level):
    Z1, Z2 = orc.calib_points(d, tau, w, level)
    st = 2206018850 + level
    draws = []
    for _ in range(2 * 256 * d):
        st, z = _splitmix64(st)
        draws.append((z >> 11) * 2.0 ** -53)
    u = np.array(draws).reshape(2, 256, d)
    assert np.array_equal(Z1, u[0] * w)
    assert np.array_equal(Z2, u[1] * w + w / tau)              # shifted by w / tau per coordinate
    assert Z1.min() >= 0 and Z1.max() < w and (Z2 - w / tau).min() >= 0


def _trials(orc, d, kid, p, eps, w, level, mmax):
    out = []
    for m in range(1, mmax + 1):
        t = orc.calib_trial_ex(d, kid, p, eps, 0.5, w, level, m)
        out.append((m, t))
        if t["G"] >= 256:
            break
    return out


@pytest.mark.parametrize("d,kid,p,eps,w,level", CASES)
def test_calib_trial_error_bounds_and_lstsq_identity(orc, d, kid, p, eps, w, level):
    Z1, Z2 = orc.calib_points(d, 0.5, w, level)
    K = _kernel_np(kid, p, Z1, Z2)
    nK = np.linalg.norm(K)
    s = np.linalg.svd(K, compute_uv=False)
    mmax = {2: 16, 3: 7, 5: 4}[d]
    for m, t in _trials(orc, d, kid, p, eps, w, level, mmax):
        e, k, skel, sel = t["e"], t["k"], t["skel"], t["sel"]
        assert t["G"] == m ** d
        assert len(sel) == min(256, m ** d) if t["G"] >= 256 else len(sel) <= m ** d
        assert 1 <= k <= len(sel) and len(set(skel.tolist())) == k
        ey = np.sqrt((s[k:] ** 2).sum()) / nK                  # Eckart-Young (Frobenius)
        assert e >= ey * (1 - 1e-6) - 1e-15, (m, e, ey)
        # the ID coefficients are the lstsq coefficients on the columns Z2* ...
        Ks = K[skel]
        Ut = np.linalg.lstsq(Ks[:, sel].T, K[:, sel].T, rcond=None)[0]
        e_fit = np.linalg.norm(K - Ut.T @ Ks) / nK             # ... applied to the full K(Z1, Z2)
        assert abs(e - e_fit) <= 1e-4 * e_fit + 1e-12, (m, e, e_fit)
        Uf = np.linalg.lstsq(Ks.T, K.T, rcond=None)[0]         # best fit on the full block
        e_best = np.linalg.norm(K - Uf.T @ Ks) / nK
        assert e >= e_best * (1 - 1e-6) - 1e-13, (m, e, e_best)
        if t["G"] >= 256:                                      # pass-through bound
            assert np.array_equal(sel, np.arange(256))
            assert e <= np.sqrt(256 - k) * 1e-3 * eps * (1 + 1e-6) + 1e-14, (e, k)


@pytest.mark.parametrize("d,kid,p,eps,w,level", CASES[:4])
def test_calib_level_is_first_passing_m(orc, d, kid, p, eps, w, level):
    r = orc.calib_level(d, kid, p, eps, 0.5, w, level)
    for m, t in _trials(orc, d, kid, p, eps, w, level, 16):
        if t["e"] < 1e-2 * eps or t["G"] >= 256:
            assert r == t["G"], (r, m, t["e"])
            return
        assert r > t["G"]
    pytest.fail("no passing trial")


@pytest.mark.parametrize("pts_fn,kid,p,eps,q", [
    (lambda: synth.uniform_cube(6000, 3, seed=11), synth.KERNEL_COULOMB, 0.0, 1e-6, 32),
    (lambda: synth.clustered(5000, 2, seed=12, k=3, sigma=0.08), synth.KERNEL_MATERN32, 0.1, 1e-6, 24),
    (lambda: synth.uniform_cube(3000, 3, seed=13) * 2.0 + 1.0, synth.KERNEL_GAUSSIAN, 0.5, 1e-6, 16),
])
def test_calibrate_composes_levels(orc, pts_fn, kid, p, eps, q):
    pts = pts_fn()
    h = orc.OracleH2(pts, q, 0.5)
    r = h.calibrate(kid, p, eps)
    rl = h.calib_levels()
    nd = h.nodes()
    off, _ = h.il()
    W = float(np.max(pts.max(0) - pts.min(0)))                 # reading A1: cube of the max extent
    has = np.zeros(len(rl), bool)
    for i in range(len(nd["level"])):
        if off[i + 1] > off[i]:
            has[nd["level"][i]] = True
    assert has.any()
    for l in range(len(rl)):
        if has[l]:
            assert rl[l] == orc.calib_level(pts.shape[1], kid, p, eps, 0.5, W * 2.0 ** -l, l), l
        else:
            assert rl[l] == 0
    assert r == max(1, rl.max())


def test_calibration_near_constant_gaussian_gives_r1(orc):
    h = orc.OracleH2(synth.uniform_cube(4096, 3, seed=14), 32, 0.5)
    assert h.calibrate(synth.KERNEL_GAUSSIAN, 1e6, 1e-6) == 1  # K ~ 1: rank 1 to ~1e-11


# ---------------------------------------------------------------- D. HiDR top-down composition

def test_hidr_golden_1d_16(orc):
    pts = (np.arange(16) / 16.0).reshape(16, 1)
    h = orc.OracleH2(pts, 2, 0.5)
    h.hidr(2)
    xo, xi = h.xstar()
    yo, yi = h.ystar()
    seen = 0
    with open(GOLDEN) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            node, rest = line.split(":")
            xs, ys = rest.split("|")
            i = int(node)
            assert xi[xo[i]:xo[i + 1]].tolist() == [int(t) for t in xs.split()], i
            assert yi[yo[i]:yo[i + 1]].tolist() == [int(t) for t in ys.split()], i
            seen += 1
    assert seen == 15


def _vol_kdtree(P, k):
    """Vol(S, k) with the nearest-point step done by scipy's KD-tree (grid as readings C2-C3)."""
    if len(P) <= k:
        return None
    d = P.shape[1]
    m = int(np.floor(k ** (1.0 / d) + 1e-9))
    while (m + 1) ** d <= k:
        m += 1
    while m ** d > k:
        m -= 1
    lo, hi = P.min(0), P.max(0)
    axes = [lo[c] + (np.arange(m) + 0.5) * ((hi[c] - lo[c]) / m) for c in range(d)]
    Q = np.stack(np.meshgrid(*axes, indexing="ij"), -1).reshape(-1, d)
    return np.unique(cKDTree(P).query(Q)[1])


@pytest.mark.parametrize("d,n,q,r,seed", [(2, 1500, 12, 9, 21), (3, 2500, 20, 27, 22), (3, 1200, 8, 8, 23)])
def test_hidr_topdown_is_vol_of_parent_and_il_union(orc, d, n, q, r, seed):
    pts = synth.clustered(n, d, seed=seed, k=3, sigma=0.12)
    h = orc.OracleH2(pts, q, 0.5)
    h.hidr(r)
    nd = h.nodes()
    X = h.tree_points()
    xo, xi = h.xstar()
    yo, yi = h.ystar()
    off, idx = h.il()
    checked = 0
    for i in range(1, len(nd["level"])):
        p = nd["parent"][i]
        T = set(yi[yo[p]:yo[p + 1]].tolist())
        for j in idx[off[i]:off[i + 1]]:
            T.update(xi[xo[j]:xo[j + 1]].tolist())
        T = np.array(sorted(T), np.int64)
        ys = yi[yo[i]:yo[i + 1]]
        assert set(ys.tolist()) <= set(T.tolist())
        if len(T) <= r:
            assert ys.tolist() == T.tolist()
            continue
        sel = _vol_kdtree(X[T], r)
        assert ys.tolist() == T[sel].tolist(), i
        checked += 1
    assert checked > 20
