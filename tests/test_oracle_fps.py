"""Pins of the oracle's farthest point sampling (PAPER §3.3; reading C6: the first point
is the one nearest the centre of the tight bounding box -- the m = 1 case of Vol --, then the point
of largest distance to the selected set, ties to the lowest index; distances as in C4)."""
import numpy as np
import pytest

import oracle
import synth


def _c4(x, y):
    s = 0.0
    for a, b in zip(x, y):
        s = s + (a - b) * (a - b)
    return s


def _fps_brute(X, S, k):
    """Plain-Python FPS on tiny inputs, written from the paper's description."""
    S = list(S)
    if len(S) <= k:
        return sorted(set(S))
    lo, hi = X[S].min(0), X[S].max(0)
    q = lo + 0.5 * ((hi - lo) / 1.0)
    seed = min(S, key=lambda s: (_c4(X[s], q), s))
    chosen = [seed]
    while len(chosen) < k:
        rest = [s for s in S if s not in chosen]
        dist = {s: min(_c4(X[s], X[c]) for c in chosen) for s in rest}
        far = max(rest, key=lambda s: (dist[s], -s))
        chosen.append(far)
    return sorted(chosen)


def test_spec_line_example():
    # {0, 1, ..., 10} on a line, k = 3: the middle point, then both ends
    X = np.arange(11, dtype=float).reshape(-1, 1)
    assert list(oracle.fps(X, np.arange(11), 3)) == [0, 5, 10]


def test_seed_is_nearest_to_box_centre_not_centroid():
    # the centroid 3.5 (nearest point: 3, index 3) differs from the box centre 5 (nearest: 6, index 4)
    X = np.array([[0.0], [1.0], [1.0], [3.0], [6.0], [10.0]])
    assert list(oracle.fps(X, np.arange(6), 1)) == [4]
    # equidistant from the centre: the lowest index wins
    X = np.array([[0.0], [4.0], [6.0], [10.0]])
    assert list(oracle.fps(X, np.arange(4), 1)) == [1]


def test_ties_go_to_the_lowest_index():
    # unit square corners + centre: centre first, then the four corners tie at 0.5 -> corner 0,
    # then the three others tie again at 0.5 (distance to the centre) -> corner 1
    X = np.array([[0, 0], [1, 0], [0, 1], [1, 1], [0.5, 0.5]], float)
    assert list(oracle.fps(X, np.arange(5), 3)) == [0, 1, 4]


def test_pass_through_and_subset():
    X = np.random.default_rng(0).random((50, 3))
    S = np.array([7, 3, 11, 3 + 40])
    assert list(oracle.fps(X, S, 8)) == sorted(S)
    out = oracle.fps(X, np.arange(50), 12)
    assert len(out) == 12 and np.all(np.diff(out) > 0) and set(out) <= set(range(50))


@pytest.mark.parametrize("seed,n,d,k", [(1, 30, 2, 7), (2, 40, 3, 10), (3, 25, 1, 6), (4, 60, 5, 16)])
def test_against_brute_force(seed, n, d, k):
    rng = np.random.default_rng(seed)
    X = rng.random((n, d))
    X[5:10] = X[0:5]  # a few duplicate points (distinct indices, equal coordinates)
    S = rng.permutation(n)[: n - 3]
    assert list(oracle.fps(X, S, k)) == _fps_brute(X, S, k)


def test_lattice_with_exact_ties_against_brute_force():
    g = np.arange(6) / 6.0
    X = np.stack(np.meshgrid(g, g, indexing="ij"), -1).reshape(-1, 2)
    assert list(oracle.fps(X, np.arange(len(X)), 9)) == _fps_brute(X, np.arange(len(X)), 9)


def test_hidr_with_fps_pipeline():
    """HiDR with FPS (the paper's first DataReduct option): X_i^* subset of X_i with min(r, |S_i|)
    points, and the H^2 error falls as id_tol falls."""
    pts = synth.points(1, 3000)
    x = synth.matvec_vector(1, 3000)
    rows = np.arange(0, 3000, 7)
    errs = []
    for tol in (1e-2, 1e-4, 1e-6):
        o = oracle.OracleH2(pts, 32, 0.5, reduct=1)
        r = o.build(synth.KERNEL_GAUSSIAN, 0.5, tol, 27)
        xo, xi = o.export(oracle.XS_OFF), o.export(oracle.XS_IDX)
        nodes = o.export(oracle.NODES).reshape(-1, 7)
        for i in range(len(nodes)):
            sel = xi[xo[i]:xo[i + 1]]
            assert np.all((sel >= nodes[i, 1]) & (sel < nodes[i, 2]))
        y = o.matvec(x, rows)
        yd = oracle.dense_rows(pts, synth.KERNEL_GAUSSIAN, 0.5, x, rows)
        errs.append(np.linalg.norm(y - yd) / np.linalg.norm(yd))
        o.close()
    assert errs[0] > errs[1] > errs[2], errs


# ---- surface-based DataReduct (reading C7) -------------------------------------------
def _surface_brute(X, S, k):
    """Plain numpy version of reading C7, written from the paper's description."""
    S = list(S)
    if len(S) <= k:
        return sorted(set(S))
    d = X.shape[1]
    lo, hi = X[S].min(0), X[S].max(0)
    w = hi - lo
    cen = lo + 0.5 * (w / 1.0)
    out = []
    for e, gam in enumerate((0.3, 0.6, 1.2)):
        M = k // 3 + (1 if e < k % 3 else 0)
        for j in range(M):
            if d == 2:
                t = 2.0 * np.pi * j / M
                u = np.array([np.cos(t), np.sin(t)])
            else:
                z = 1.0 - (2.0 * j + 1.0) / M
                rho = np.sqrt(1.0 - z * z)
                f = j * (np.pi * (3.0 - np.sqrt(5.0)))
                u = np.array([rho * np.cos(f), rho * np.sin(f), z])
            q = cen + (gam * w) * u
            out.append(min(S, key=lambda s: (_c4(X[s], q), s)))
    return sorted(set(out))


def test_surface_k3_axis_points():
    # k = 3 in 2-D: one reference point per ellipsoid, at angle 0: (c + gamma w, c_y) on the x axis
    xs = np.linspace(0.0, 1.0, 11)
    X = np.stack([np.concatenate([xs, xs]), np.concatenate([np.full(11, 0.4), np.full(11, 0.6)])], 1)
    # box [0,1] x [0.4,0.6]: centre (0.5, 0.5); gamma 0.3 -> x = 0.8, 0.6 -> x = 1.1, 1.2 -> x = 1.7
    out = oracle.surface(X, np.arange(22), 3)
    assert list(out) == [8, 10]  # (0.8, 0.4) (lower index of the tie with row 0.6) and (1.0, 0.4)


@pytest.mark.parametrize("seed,n,d,k", [(1, 80, 2, 9), (2, 120, 3, 12), (3, 60, 2, 5), (4, 200, 3, 27)])
def test_surface_against_brute_force(seed, n, d, k):
    X = np.random.default_rng(seed).random((n, d))
    S = np.random.default_rng(seed + 10).permutation(n)[: n - 5]
    out = oracle.surface(X, S, k)
    assert list(out) == _surface_brute(X, S, k)
    assert len(out) <= k and set(out) <= set(S)


def test_surface_rejects_other_dimensions():
    with pytest.raises(ValueError):
        oracle.surface(np.random.default_rng(0).random((30, 4)), np.arange(30), 6)
