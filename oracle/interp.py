"""Interpolation-based H^2 -- the baseline of the paper's memory comparison (section 6.3).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): imported by tests/ and tools/interp_compare.py;
the product path never imports it.  Plain numpy, fp64, no blocking or reordering beyond the
definitions below; kernel blocks come from the C oracle (oracle.kernel_block, step J).

What it computes (Eq. (2.2)): interpolating kappa(x, y) in x at r nodes
Q = {q_1..q_r},  kappa(x, y) ~= sum_a kappa(q_a, y) L_a(x),  gives K_{X_i Y_i} ~= U_i K_{Q_i Y_i} with
U_i = [L_a(x)]_{x in X_i, a = 1..r}.  "In three dimensions, the number of interpolation nodes is k^3
if k interpolation nodes are used in each dimension": Q_i is a tensor grid of p
Chebyshev nodes per dimension, r = p^d.  Readings (Q1-Q4):
  Q1  the interpolation box of node i is its cell of the tree (root cube of the partition, width
      W 2^-l at level l); the nodes are the Chebyshev points of the first kind
      t_a = c + (w/2) z_a, z_a = cos((2a + 1) pi / (2p)), a = 0..p-1;
  Q2  multi-index alpha = sum_c a_c p^c (dimension 0 fastest); L_alpha(x) = prod_c l_{a_c}(x_c) with
      the 1-D Lagrange polynomial l_a(u) = prod_{b != a} (u - z_b) / (z_a - z_b) of u = (x - c)/(w/2);
  Q3  nested bases: a non-leaf node's U holds the stacked transfers R_c = [L^(p)_alpha(q)]_{q in Q_c}
      of its children (child order) -- the layout of the data-driven U_p (Xbar_p = the children's
      skeletons), with the children's Chebyshev nodes in place of their skeletons;
  Q4  a node has a basis (k_i = r) iff it or an ancestor has an admissible pair (as the data-driven
      k_i > 0 iff Y_i^* is non-empty); coupling blocks B_ij = K(Q_i, Q_j) for (i, j) in IL
      (symmetric kernels: stored for i < j), nearfield blocks K(X_i, X_j) as the data-driven build.
Memory = the stored entries of U (leaves and transfers), the coupling blocks and the nearfield
blocks, symmetric blocks once -- "the cost for storing the hierarchical representation".
"""
from __future__ import annotations

import math

import numpy as np

from . import OracleH2, kernel_block


def cheb_ref(p: int) -> np.ndarray:
    """Q1: z_a = cos((2a + 1) pi / (2p)), a = 0..p-1 (Chebyshev points of the first kind on [-1, 1])."""
    a = np.arange(p, dtype=np.float64)
    return np.cos((2.0 * a + 1.0) * math.pi / (2.0 * p))


def lagrange_1d(z: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Q2: l_a(u) = prod_{b != a} (u - z_b) / (z_a - z_b), b ascending; shape (len(u), p)."""
    u = np.asarray(u, np.float64)
    p = len(z)
    out = np.ones((u.shape[0], p), np.float64)
    for a in range(p):
        for b in range(p):
            if b != a:
                out[:, a] = out[:, a] * ((u - z[b]) / (z[a] - z[b]))
    return out


def multi_index(p: int, d: int) -> np.ndarray:
    """Q2: row alpha holds (a_0, .., a_{d-1}) with alpha = sum_c a_c p^c."""
    al = np.arange(p ** d)
    return np.stack([(al // p ** c) % p for c in range(d)], axis=1)


def lagrange_nd(X: np.ndarray, center: np.ndarray, half: float, z: np.ndarray) -> np.ndarray:
    """L_alpha(x) over the box [center - half, center + half]^d: shape (len(X), p^d)."""
    X = np.asarray(X, np.float64)
    d = X.shape[1]
    p = len(z)
    mi = multi_index(p, d)
    out = np.ones((X.shape[0], p ** d), np.float64)
    for c in range(d):
        lc = lagrange_1d(z, (X[:, c] - center[c]) / half)
        out = out * lc[:, mi[:, c]]
    return out


def cheb_points(center: np.ndarray, half: float, z: np.ndarray) -> np.ndarray:
    """Q_i: q_alpha = center + half * (z_{a_0}, .., z_{a_{d-1}}); shape (p^d, d)."""
    d = len(center)
    mi = multi_index(len(z), d)
    return np.stack([center[c] + half * z[mi[:, c]] for c in range(d)], axis=1)


def root_box(pts: np.ndarray):
    """The partition's root cube (reading A1): W = max extent, rlo = bbox centre - W/2."""
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    W = float(np.max(hi - lo))
    return (lo + hi) * 0.5 - W * 0.5, W


class InterpH2:
    """Interpolation-based H^2 on the tree and lists of an OracleH2 (steps A, B)."""

    def __init__(self, o: OracleH2, p: int, kid: int, param: float):
        self.o, self.p, self.kid, self.param = o, int(p), int(kid), float(param)
        d = o.d
        self.d, self.r = d, self.p ** d
        nd = o.nodes()
        self.level, self.begin, self.end = nd["level"], nd["begin"], nd["end"]
        self.parent, self.first_child, self.nchild, self.is_leaf = (nd["parent"], nd["first_child"], nd["nchild"],
                                                                     nd["is_leaf"])
        self.nn = len(self.level)
        self.X = o.tree_points()
        self.il_off, self.il_idx = o.il()
        self.nf_off, self.nf_idx = o.nf()
        rlo, W = root_box(o.pts)
        self.z = cheb_ref(self.p)
        cells = o.cells()
        # Q1: the node boxes (levels in order: ids are level-order, parents before children)
        self.center = np.zeros((self.nn, d))
        self.half = np.zeros(self.nn)
        for i in range(self.nn):
            w = math.ldexp(W, -int(self.level[i]))
            self.center[i] = (rlo + cells[i] * w) + 0.5 * w
            self.half[i] = 0.5 * w
        # Q4: bases exist where the node or an ancestor has an admissible pair
        self.k = np.zeros(self.nn, np.int64)
        for i in range(self.nn):
            far = self.il_off[i + 1] > self.il_off[i] or (self.parent[i] >= 0 and self.k[self.parent[i]] > 0)
            self.k[i] = self.r if far else 0
        self.Q = {i: cheb_points(self.center[i], self.half[i], self.z) for i in range(self.nn) if self.k[i] > 0}
        # U_i: leaves L(X_i); non-leaves the stacked transfers of their children (Q3)
        self.U = {}
        for i in range(self.nn):
            if self.k[i] == 0:
                continue
            if self.is_leaf[i]:
                rows = self.X[self.begin[i]:self.end[i]]
            else:
                ch = range(self.first_child[i], self.first_child[i] + self.nchild[i])
                rows = np.vstack([self.Q[c] for c in ch])
            self.U[i] = lagrange_nd(rows, self.center[i], self.half[i], self.z)

    def transfer(self, c: int) -> np.ndarray:
        """R_c = rows of U_parent(c) for child c: L^(parent)_alpha(Q_c), r x r."""
        p = self.parent[c]
        j = c - self.first_child[p]
        return self.U[p][j * self.r:(j + 1) * self.r]

    def memory_entries(self) -> dict:
        """Stored entries: U (leaves + transfers), coupling (symmetric: i < j), nearfield (i <= j)."""
        u = sum(v.size for v in self.U.values())
        cp = 0
        for i in range(self.nn):
            for j in self.il_idx[self.il_off[i]:self.il_off[i + 1]]:
                if j > i:
                    cp += int(self.k[i] * self.k[j])
        nf = 0
        for i in range(self.nn):
            for j in self.nf_idx[self.nf_off[i]:self.nf_off[i + 1]]:
                if j >= i:
                    nf += int((self.end[i] - self.begin[i]) * (self.end[j] - self.begin[j]))
        return {"u": int(u), "coupling": cp, "nearfield": nf, "total": int(u) + cp + nf}

    def matvec(self, x: np.ndarray) -> np.ndarray:
        """y = K~ x, x and y in the original point order."""
        perm = self.o.perm
        xt = np.asarray(x, np.float64)[perm]
        r = self.r
        z = np.zeros((self.nn, r))
        for i in range(self.nn - 1, -1, -1):  # up: children (higher ids) before parents
            if self.k[i] == 0:
                continue
            if self.is_leaf[i]:
                z[i] = self.U[i].T @ xt[self.begin[i]:self.end[i]]
            else:
                ch = range(self.first_child[i], self.first_child[i] + self.nchild[i])
                z[i] = self.U[i].T @ np.concatenate([z[c] for c in ch])
        yh = np.zeros((self.nn, r))
        for i in range(self.nn):
            for j in self.il_idx[self.il_off[i]:self.il_off[i + 1]]:
                yh[i] += kernel_block(self.kid, self.param, self.Q[i], self.Q[j]) @ z[j]
        yt = np.zeros(len(xt))
        for i in range(self.nn):  # down: parents before children
            if self.k[i] == 0:
                continue
            if self.parent[i] >= 0 and self.k[self.parent[i]] > 0:
                yh[i] += self.transfer(i) @ yh[self.parent[i]]
            if self.is_leaf[i]:
                yt[self.begin[i]:self.end[i]] += self.U[i] @ yh[i]
        for i in range(self.nn):
            Xi = self.X[self.begin[i]:self.end[i]]
            for j in self.nf_idx[self.nf_off[i]:self.nf_off[i + 1]]:
                Xj = self.X[self.begin[j]:self.end[j]]
                yt[self.begin[i]:self.end[i]] += kernel_block(self.kid, self.param, Xi, Xj) @ xt[self.begin[j]:self.end[j]]
        y = np.empty_like(yt)
        y[perm] = yt
        return y
