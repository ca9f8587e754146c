"""Pins for oracle steps A (partition) and B (admissibility + lists).

Each check fixes the oracle against something other than itself: values the paper prints
(P:150-151), hand-derived trees, an independent recursive centre-split partition on
dyadic inputs, an O(N^2) brute-force list definition in exact rational arithmetic,
and the tiling invariant.
"""
import os
from fractions import Fraction

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_1d_interaction_lists.txt")


def _tree(orc, pts, q, tau=0.5):
    h = orc.OracleH2(pts, q, tau)
    return h, h.nodes()


# ---------------------------------------------------------------- A. partition

def test_single_point_is_root_leaf(orc):
    h, nd = _tree(orc, np.array([[0.3, 0.7]]), q=4)
    assert h.info()["nnodes"] == 1 and nd["is_leaf"][0] == 1
    assert (nd["begin"][0], nd["end"][0]) == (0, 1)
    off, idx = h.nf()
    assert list(idx) == [0] and len(h.il()[1]) == 0           # nearfield(root) = {root}


def test_identical_points_single_leaf(orc):
    h, nd = _tree(orc, np.full((50, 3), 0.25), q=4)             # W = 0: one root leaf (A3)
    assert h.info()["nnodes"] == 1 and list(h.perm) == list(range(50))


def test_equispaced_16_binary_tree(orc):
    # 16 equispaced points on [0,1], q=2 -> complete binary tree of depth 3, 8 leaves of 2
    h, nd = _tree(orc, synth.equispaced_1d(16), q=2)
    assert h.info()["nnodes"] == 15 and h.info()["depth"] == 3
    leaves = np.flatnonzero(nd["is_leaf"])
    assert list(leaves) == list(range(7, 15))
    assert all(nd["end"][i] - nd["begin"][i] == 2 for i in leaves)
    assert list(nd["level"]) == [0, 1, 1, 2, 2, 2, 2] + [3] * 8


def test_grid_64_leaf_width(orc):
    # 64 uniform 1-D grid points, q=4 -> leaves of width 1/16 (16 leaves of 4 points)
    h, nd = _tree(orc, synth.equispaced_1d(64), q=4)
    leaves = np.flatnonzero(nd["is_leaf"])
    assert len(leaves) == 16 and set(nd["level"][leaves]) == {4}
    assert all(nd["end"][i] - nd["begin"][i] == 4 for i in leaves)


def _recursive_split(pts, idx, lo, w, q, level, maxlevel, out):
    """Independent partition: recursive centre split with comparisons x >= mid."""
    if len(idx) <= q or level == maxlevel:
        out.append((level, frozenset(idx)))
        return
    half = w / 2
    mid = lo + half
    groups = {}
    for i in idx:
        code = tuple(bool(pts[i, k] >= mid[k]) for k in range(pts.shape[1]))
        groups.setdefault(code, []).append(i)
    for code, sub in groups.items():
        _recursive_split(pts, sub, lo + half * np.array(code, float), half, q, level + 1, maxlevel, out)


@pytest.mark.parametrize("d,n,q", [(1, 300, 3), (2, 500, 5), (3, 600, 7)])
def test_partition_equals_recursive_split_on_dyadic_points(orc, d, n, q):
    rng = np.random.default_rng(7 + d)
    pts = rng.integers(0, 2 ** 12 + 1, size=(n, d)) / 2.0 ** 12
    pts[0] = 0.0
    pts[1] = 1.0                          # bbox = [0,1]^d: centre splits are exact dyadic numbers
    h, nd = _tree(orc, pts, q)
    perm = h.perm
    ours = set()
    for i in np.flatnonzero(nd["is_leaf"]):
        ours.add((int(nd["level"][i]), frozenset(perm[nd["begin"][i]:nd["end"][i]].tolist())))
    ref = []
    _recursive_split(pts, list(range(n)), np.zeros(d), 1.0, q, 0, h.info()["L"], ref)
    assert ours == set(ref)


@pytest.mark.parametrize("d", [1, 2, 3, 5])
def test_perm_coverage_and_ranges(orc, d):
    pts = synth.clustered(700, d, seed=11 + d)
    h, nd = _tree(orc, pts, q=9)
    perm = h.perm
    assert sorted(perm.tolist()) == list(range(700))                       # permutation
    assert np.array_equal(h.tree_points(), pts[perm])                       # S:86 round trip
    cover = np.zeros(700, int)
    for i in np.flatnonzero(nd["is_leaf"]):
        cover[nd["begin"][i]:nd["end"][i]] += 1
        assert nd["end"][i] - nd["begin"][i] <= 9 or nd["level"][i] == h.info()["L"]
    assert (cover == 1).all()                                               # each point once
    for i in np.flatnonzero(nd["is_leaf"] == 0):                            # parent = concat(children)
        ch = range(nd["first_child"][i], nd["first_child"][i] + nd["nchild"][i])
        assert nd["begin"][ch[0]] == nd["begin"][i] and nd["end"][ch[-1]] == nd["end"][i]
        for a, b in zip(ch[:-1], ch[1:]):
            assert nd["end"][a] == nd["begin"][b]
        assert all(nd["parent"][c] == i and nd["level"][c] == nd["level"][i] + 1 for c in ch)
        assert all(nd["end"][c] > nd["begin"][c] for c in ch)               # no empty children


# ---------------------------------------------------------------- B. admissibility and lists

def test_paper_interaction_lists_golden(orc):
    """IL(4) = {6,7}, IL(10) = {8,12,13} (1-based level-order ids)."""
    h, nd = _tree(orc, synth.equispaced_1d(16), q=2, tau=0.5)
    off, idx = h.il()
    with open(GOLDEN) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            node, lst = line.split(":")
            i = int(node) - 1
            expect = [int(t) - 1 for t in lst.split()]
            assert sorted(idx[off[i]:off[i + 1]].tolist()) == expect


def test_spec_admissibility_examples(orc):
    # S:60-62 on the 1-D binary tree over [0,1], tau = 0.5 (cells at level 2)
    assert orc.admissible([0], 2, [2], 2, 0.5)          # [0,1/4] vs [1/2,3/4]: 1/4+1/4 <= 2*.5*1/2
    assert not orc.admissible([0], 2, [1], 2, 0.5)      # adjacent
    assert not orc.admissible([3], 2, [3], 2, 0.5)      # self pair
    # cross-level: leaf at level 1 ([0,1/2]) vs level-3 cell [7/8,1]: 1/2+1/8 <= 2*.5*(15/16-1/4)
    assert orc.admissible([0], 1, [7], 3, 0.5)
    assert not orc.admissible([0], 1, [4], 3, 0.5)


def _frac_box(W, rlo, cell, level):
    w = Fraction(W) / (2 ** level)
    a = [Fraction(r) + (Fraction(int(c)) + Fraction(1, 2)) * w for r, c in zip(rlo, cell)]
    return w, a


def _adm_frac(bi, bj, d, tau):
    """Eq.(2.1), diam = box diagonal sqrt(d) w (B1), both sides squared, exact rationals:
    sqrt(d) (w_i + w_j) <= 2 tau |a_i - a_j|  <=>  d (w_i + w_j)^2 <= 4 tau^2 |a_i - a_j|^2."""
    (wi, ai), (wj, aj) = bi, bj
    dist2 = sum((x - y) ** 2 for x, y in zip(ai, aj))
    return d * (wi + wj) ** 2 <= 4 * Fraction(tau) ** 2 * dist2


def _boxes(h, nd):
    info = h.info()
    pts = h.pts
    lo, hi = pts.min(0), pts.max(0)
    c = (lo + hi) * 0.5
    W = float((hi - lo).max())
    rlo = c - W * 0.5
    cells = h.cells()
    return [_frac_box(W, rlo, cells[i], nd["level"][i]) for i in range(info["nnodes"])]


@pytest.mark.parametrize("d,side,q,tau", [(1, 64, 4, 0.5), (2, 16, 4, 0.5), (3, 8, 8, 0.5),
                                          (2, 16, 4, 0.7), (2, 16, 4, 0.3)])
def test_lists_equal_bruteforce_definition_on_complete_trees(orc, d, side, q, tau):
    """IL(i) = {j same level : adm(i,j) and not adm(p(i),p(j))}; NF on leaves."""
    g = np.arange(side) / (side - 1)
    pts = np.stack(np.meshgrid(*([g] * d), indexing="ij"), -1).reshape(-1, d)
    h, nd = _tree(orc, pts, q, tau)
    assert len(set(nd["level"][nd["is_leaf"] == 1])) == 1                  # complete tree
    B = _boxes(h, nd)
    nn = len(B)
    lvl, par = nd["level"], nd["parent"]
    off, idx = h.il()
    noff, nidx = h.nf()
    depth = lvl.max()

    def adm(i, j):
        return _adm_frac(B[i], B[j], d, tau)

    far_anc = {}
    for i in range(nn):
        want = set()
        for j in range(nn):
            if lvl[j] != lvl[i] or i == j and lvl[i] == 0:
                continue
            if adm(i, j) and (lvl[i] == 0 or not adm(par[i], par[j])):
                want.add(j)
        assert set(idx[off[i]:off[i + 1]].tolist()) == want, i
    leaves = [i for i in range(nn) if lvl[i] == depth]
    for i in leaves:
        want = set()
        for j in leaves:
            a, b, ok = i, j, True
            while a >= 0:
                if adm(a, b):
                    ok = False
                    break
                a, b = par[a], par[b]
            if ok:
                want.add(j)
        assert set(nidx[noff[i]:noff[i + 1]].tolist()) == want


@pytest.mark.parametrize("d,n,q,tau,seed", [(1, 400, 3, 0.5, 1), (2, 500, 6, 0.5, 2), (3, 600, 9, 0.5, 3),
                                            (2, 500, 4, 0.7, 4), (3, 500, 5, 0.3, 5), (2, 300, 1, 0.5, 6)])
def test_tiling_exactly_once_and_admissibility(orc, d, n, q, tau, seed):
    """S:83 tiling on adaptive trees; every IL pair admissible (exact rationals), its parent
    pair not; every NF pair not admissible; symmetry of both lists."""
    pts = synth.clustered(n, d, seed=seed, k=3, sigma=0.08)
    h, nd = _tree(orc, pts, q, tau)
    B = _boxes(h, nd)
    off, idx = h.il()
    noff, nidx = h.nf()
    cover = np.zeros((n, n), np.int32)
    b, e = nd["begin"], nd["end"]
    nn = len(B)
    pairs = set()
    for i in range(nn):
        for j in idx[off[i]:off[i + 1]]:
            cover[b[i]:e[i], b[j]:e[j]] += 1
            pairs.add((i, int(j)))
            assert _adm_frac(B[i], B[j], d, tau)
    for (i, j) in pairs:
        assert (j, i) in pairs
    npairs = set()
    for i in range(nn):
        for j in nidx[noff[i]:noff[i + 1]]:
            assert nd["is_leaf"][i] and nd["is_leaf"][j]
            assert not _adm_frac(B[i], B[int(j)], d, tau)
            cover[b[i]:e[i], b[j]:e[j]] += 1
            npairs.add((i, int(j)))
    for (i, j) in npairs:
        assert (j, i) in npairs
    assert (cover == 1).all()
