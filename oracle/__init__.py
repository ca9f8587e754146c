"""ctypes wrapper of the fp64 CPU oracle (oracle/h2_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  The product path (paper_2206_01885_b200) never imports it.
Step letters (A..I) and readings follow DESIGN.md "Oracle"; the C file cites PAPER.md per step.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "h2_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC", "-std=gnu11"]

PERM, NODES, CELLS, IL_OFF, IL_IDX, NF_OFF, NF_IDX = 1, 2, 3, 4, 5, 6, 7
XS_OFF, XS_IDX, YS_OFF, YS_IDX, K, SK_OFF, SK_IDX, U_OFF, U, XBAR_N, TREE_X, CHILD_OFF = (
    8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19)
# the non-symmetric path's column bases (Algorithm 2 line 11, second getBasis)
K_COL, SKC_OFF, SKC_IDX, V_OFF, V, XBARC_N = 20, 21, 22, 23, 24, 25
KERNEL_MQSHIFT = 7  # sqrt(1 + c |x - y + a|^2), non-symmetric

_DTYPES = {PERM: np.int32, NODES: np.int32, CELLS: np.int64, IL_OFF: np.int64, IL_IDX: np.int32,
           NF_OFF: np.int64, NF_IDX: np.int32, XS_OFF: np.int64, XS_IDX: np.int32, YS_OFF: np.int64,
           YS_IDX: np.int32, K: np.int32, SK_OFF: np.int64, SK_IDX: np.int32, U_OFF: np.int64,
           U: np.float64, XBAR_N: np.int32, TREE_X: np.float64, CHILD_OFF: np.int32, K_COL: np.int32,
           SKC_OFF: np.int64, SKC_IDX: np.int32, V_OFF: np.int64, V: np.float64, XBARC_N: np.int32}


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc, -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        vp, i32, i64, f64 = C.c_void_p, C.c_int, C.c_int64, C.c_double
        L.orc_new.restype = vp
        L.orc_new.argtypes = [vp, i32, i32, i32, f64]
        L.orc_free.argtypes = [vp]
        L.orc_hidr.argtypes = [vp, i32]
        L.orc_calibrate.argtypes = [vp, i32, f64, f64]
        L.orc_calib_level.argtypes = [i32, i32, f64, f64, f64, f64, i32]
        L.orc_calib_trial.restype = f64
        L.orc_calib_trial.argtypes = [i32, i32, f64, f64, f64, f64, i32, i32, vp]
        L.orc_calib_trial_ex.restype = f64
        L.orc_calib_trial_ex.argtypes = [i32, i32, f64, f64, f64, f64, i32, i32, vp, vp, vp, vp, vp]
        L.orc_calib_points.argtypes = [i32, f64, f64, i32, vp, vp]
        L.orc_calib_levels.argtypes = [vp, vp]
        L.orc_id_sweep.argtypes = [vp, i32, f64, f64]
        L.orc_export.restype = i64
        L.orc_export.argtypes = [vp, i32, vp, i64]
        L.orc_info.argtypes = [vp, vp, vp, vp]
        L.orc_matvec_rows.argtypes = [vp, vp, vp, i64, vp]
        L.orc_dense_rows.argtypes = [vp, i32, i32, i32, f64, vp, vp, i64, vp]
        L.orc_kernel_block.argtypes = [i32, f64, vp, i32, vp, i32, i32, vp]
        L.orc_fill.restype = i64
        L.orc_fill.argtypes = [vp, vp, i64, vp]
        L.orc_vol.argtypes = [vp, i32, vp, i32, i32, vp]
        L.orc_fps.argtypes = [vp, i32, vp, i32, i32, vp]
        L.orc_set_reduct.argtypes = [vp, i32]
        L.orc_set_nonsym.argtypes = [vp, i32]
        L.orc_set_srrqr.argtypes = [vp, f64]
        L.orc_srrqr_count.restype = i64
        L.orc_srrqr_count.argtypes = [vp]
        L.orc_id_srrqr.argtypes = [vp, i32, i32, f64, f64, vp, vp, vp]
        L.orc_set_kernel_shift.argtypes = [vp, i32]
        L.orc_calib_level_tr.argtypes = [i32, i32, f64, f64, f64, f64, i32, i32]
        L.orc_surface.argtypes = [vp, i32, vp, i32, i32, vp]
        L.orc_cpqr.argtypes = [vp, i32, i32, f64, vp]
        L.orc_id.argtypes = [vp, i32, i32, f64, vp, vp]
        L.orc_admissible.argtypes = [vp, i32, vp, i32, i32, f64]
        L.orc_kernel.restype = f64
        L.orc_kernel.argtypes = [i32, f64, vp, vp, i32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def num_threads() -> int:
    return int(lib().orc_num_threads())


# ------------------------------------------------------------------------------------------
# standalone steps
# ------------------------------------------------------------------------------------------

def kernel(kid: int, param: float, x, y) -> float:
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return float(lib().orc_kernel(kid, param, _p(x), _p(y), x.size))


def vol(X: np.ndarray, S, k: int) -> np.ndarray:
    """C. Vol(S, k) over point-major coordinates X (indices S into X)."""
    X = np.ascontiguousarray(X, np.float64)
    S = np.ascontiguousarray(S, np.int32)
    out = np.empty(max(1, min(len(S), k)), np.int32)
    c = lib().orc_vol(_p(X), X.shape[1], _p(S), len(S), int(k), _p(out))
    return out[:c].copy()


def fps(X: np.ndarray, S, k: int) -> np.ndarray:
    """C'. farthest point sampling FPS(S, k) (reading C6) over point-major coordinates X."""
    X = np.ascontiguousarray(X, np.float64)
    S = np.ascontiguousarray(S, np.int32)
    out = np.empty(max(1, min(len(S), k)), np.int32)
    c = lib().orc_fps(_p(X), X.shape[1], _p(S), len(S), int(k), _p(out))
    return out[:c].copy()


def surface(X: np.ndarray, S, k: int) -> np.ndarray:
    """C''. surface-based DataReduct (reading C7; d = 2 or 3)."""
    X = np.ascontiguousarray(X, np.float64)
    S = np.ascontiguousarray(S, np.int32)
    out = np.empty(max(1, min(len(S), k)), np.int32)
    c = lib().orc_surface(_p(X), X.shape[1], _p(S), len(S), int(k), _p(out))
    if c < 0:
        raise ValueError("surface DataReduct needs d = 2 or 3")
    return out[:c].copy()


def cpqr(M: np.ndarray, tol: float):
    """F. CPQR of M (rows x cols). Returns (k, piv, Mout) with Mout[:k,:k]=R11, Mout[:k,k:]=T."""
    rows, cols = M.shape
    Mf = np.asfortranarray(M, np.float64).copy(order="F")
    piv = np.empty(cols, np.int32)
    k = lib().orc_cpqr(Mf.ctypes.data_as(C.c_void_p), rows, cols, float(tol), _p(piv))
    return int(k), piv, Mf


def interp_decomp(A: np.ndarray, tol: float):
    """F. ID of A (nx x ny): A ~= U A[skel]. Returns (skel, U)."""
    A = np.ascontiguousarray(A, np.float64)
    nx, ny = A.shape
    skel = np.empty(max(1, min(nx, ny)), np.int32)
    Uf = np.zeros(max(1, nx * min(nx, ny)), np.float64)
    k = lib().orc_id(_p(A), nx, ny, float(tol), _p(skel), _p(Uf))
    U = Uf[: nx * k].reshape(k, nx).T.copy()
    return skel[:k].copy(), U


def interp_decomp_srrqr(A: np.ndarray, tol: float, f: float):
    """F with SRRQR swaps: A ~= U A[skel] with max |G| <= f.  Returns (skel, U, swaps)."""
    A = np.ascontiguousarray(A, np.float64)
    nx, ny = A.shape
    skel = np.empty(max(1, min(nx, ny)), np.int32)
    Uf = np.zeros(max(1, nx * min(nx, ny)), np.float64)
    sw = np.zeros(1, np.int32)
    k = lib().orc_id_srrqr(_p(A), nx, ny, float(tol), float(f), _p(skel), _p(Uf), _p(sw))
    U = Uf[: nx * k].reshape(k, nx).T.copy()
    return skel[:k].copy(), U, int(sw[0])


def admissible(ci, li: int, cj, lj: int, tau: float) -> bool:
    ci = np.ascontiguousarray(ci, np.int64)
    cj = np.ascontiguousarray(cj, np.int64)
    return bool(lib().orc_admissible(_p(ci), li, _p(cj), lj, ci.size, float(tau)))


def calib_level(d, kid, param, eps, tau, w, level, tr: int = 0) -> int:
    """r of one level (tr = 1: the transposed kernel kappa(y, x), the column-basis orientation)."""
    return int(lib().orc_calib_level_tr(d, kid, param, eps, tau, w, level, int(tr)))


def set_kernel_shift(a) -> None:
    """The shift a of kernel 7 (sqrt(1 + c |x - y + a|^2)); global to the oracle library."""
    a = np.ascontiguousarray(a, np.float64)
    lib().orc_set_kernel_shift(_p(a), a.size)


def calib_trial(d, kid, param, eps, tau, w, level, m):
    G = np.zeros(1, np.int64)
    e = lib().orc_calib_trial(d, kid, param, eps, tau, w, level, m, _p(G))
    return float(e), int(G[0])


def calib_points(d, tau, w, level):
    """E4/E6: the calibration point sets (Z1, Z2) of one level, each 256 x d."""
    Z1 = np.empty((256, d), np.float64)
    Z2 = np.empty((256, d), np.float64)
    lib().orc_calib_points(d, float(tau), float(w), int(level), _p(Z1), _p(Z2))
    return Z1, Z2


def calib_trial_ex(d, kid, param, eps, tau, w, level, m) -> dict:
    """One calibration trial with its internals: e, G = m^d, the ID rank k, the skeleton rows
    (indices into Z1) and the columns Z2* (indices into Z2)."""
    G = np.zeros(1, np.int64)
    k = np.zeros(1, np.int32)
    ns = np.zeros(1, np.int32)
    skel = np.zeros(256, np.int32)
    sel = np.zeros(256, np.int32)
    e = lib().orc_calib_trial_ex(d, kid, param, eps, tau, w, level, m, _p(G), _p(k), _p(skel), _p(sel), _p(ns))
    return dict(e=float(e), G=int(G[0]), k=int(k[0]), skel=skel[:k[0]].copy(), sel=sel[:ns[0]].copy())


def dense_rows(pts: np.ndarray, kid: int, param: float, x: np.ndarray, rows) -> np.ndarray:
    """I. exact (K x)[rows] over all n points (original order)."""
    pts = np.ascontiguousarray(pts, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    rows = np.ascontiguousarray(rows, np.int64)
    out = np.empty(len(rows), np.float64)
    lib().orc_dense_rows(_p(pts), pts.shape[0], pts.shape[1], kid, float(param), _p(x), _p(rows),
                         len(rows), _p(out))
    return out


def kernel_block(kid: int, param: float, A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """J. the dense block K(A_a, B_b) of two point-major sets (kappa as orc_kernel)."""
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    out = np.empty((A.shape[0], B.shape[0]), np.float64)
    if out.size:
        lib().orc_kernel_block(kid, float(param), _p(A), A.shape[0], _p(B), B.shape[0], A.shape[1], _p(out))
    return out


# ------------------------------------------------------------------------------------------
# the oracle H^2 object
# ------------------------------------------------------------------------------------------

class OracleH2:
    """A (partition) + B (lists) on construction; then calibrate / hidr / id_sweep / matvec."""

    def __init__(self, pts: np.ndarray, q: int, tau: float = 0.5, reduct: int = 0, nonsym: bool = False,
                 srrqr_f: float = 0.0):
        """reduct: the DataReduct of HiDR, 0 volume-based (reading C1), 1 farthest point sampling (C6),
        2 surface-based (C7).  nonsym: build row AND column bases and every ordered block (Algorithm 2
        with X^(row) != X^(col); required for kernel 7, allowed for symmetric kernels)."""
        self.pts = np.ascontiguousarray(pts, np.float64)
        self.n, self.d = self.pts.shape
        self._h = lib().orc_new(_p(self.pts), self.n, self.d, int(q), float(tau))
        if not self._h:
            raise ValueError("orc_new rejected the arguments")
        lib().orc_set_reduct(self._h, int(reduct))
        lib().orc_set_nonsym(self._h, int(bool(nonsym)))
        lib().orc_set_srrqr(self._h, float(srrqr_f))
        self.nonsym = bool(nonsym)
        self.q, self.tau = q, tau
        self.kid, self.param = None, 0.0

    def close(self):
        if self._h:
            lib().orc_free(self._h)
            self._h = None

    __del__ = close

    def export(self, what: int) -> np.ndarray:
        need = lib().orc_export(self._h, what, None, 0)
        if need < 0:
            raise RuntimeError(f"oracle stage for export {what} has not run")
        a = np.empty(max(need, 1), _DTYPES[what])
        lib().orc_export(self._h, what, _p(a), need)
        return a[:need]

    def info(self) -> dict:
        a = np.zeros(11, np.int64)
        W = np.zeros(1, np.float64)
        ts = np.zeros(8, np.float64)
        lib().orc_info(self._h, _p(a), _p(W), _p(ts))
        keys = ["n", "d", "q", "nnodes", "depth", "L", "r", "n_il", "n_nf", "max_S", "max_T"]
        out = {k: int(v) for k, v in zip(keys, a)}
        out["W"] = float(W[0])
        out["t_stage"] = dict(zip(["partition", "lists", "calibrate", "hidr", "id", "fill"], ts[:6].tolist()))
        return out

    # --- structure accessors ---
    @property
    def perm(self):
        return self.export(PERM)

    def nodes(self) -> dict:
        a = self.export(NODES).reshape(-1, 7)
        return {k: a[:, i].copy() for i, k in enumerate(
            ["level", "begin", "end", "parent", "first_child", "nchild", "is_leaf"])}

    def cells(self):
        return self.export(CELLS).reshape(-1, self.d)

    def csr(self, off_what, idx_what):
        return self.export(off_what), self.export(idx_what)

    def il(self):
        return self.csr(IL_OFF, IL_IDX)

    def nf(self):
        return self.csr(NF_OFF, NF_IDX)

    def xstar(self):
        return self.csr(XS_OFF, XS_IDX)

    def ystar(self):
        return self.csr(YS_OFF, YS_IDX)

    def skeletons(self):
        return self.csr(SK_OFF, SK_IDX)

    def skeletons_col(self):
        return self.csr(SKC_OFF, SKC_IDX)

    def tree_points(self):
        return self.export(TREE_X).reshape(-1, self.d)

    # --- stages ---
    def calibrate(self, kid: int, param: float, eps: float) -> int:
        return int(lib().orc_calibrate(self._h, kid, float(param), float(eps)))

    def srrqr_swaps(self) -> int:
        """SRRQR swaps made by the last id_sweep (srrqr_f > 0)."""
        return int(lib().orc_srrqr_count(self._h))

    def calib_levels(self) -> np.ndarray:
        """E4: the per-level r of the last calibrate() (0 where a level has no admissible pair)."""
        out = np.zeros(64, np.int32)
        c = lib().orc_calib_levels(self._h, _p(out))
        return out[:c].copy()

    def hidr(self, r: int):
        if lib().orc_hidr(self._h, int(r)) != 0:
            raise RuntimeError("orc_hidr failed")

    def id_sweep(self, kid: int, param: float, id_tol: float):
        self.kid, self.param = kid, float(param)
        if lib().orc_id_sweep(self._h, kid, float(param), float(id_tol)) != 0:
            raise RuntimeError("orc_id_sweep needs hidr first")

    def build(self, kid: int, param: float, id_tol: float, r: int | None = None) -> int:
        """Algorithm 2: (tree, lists done) -> calibrate -> HiDR -> ID sweep.  Returns r."""
        if r is None:
            r = self.calibrate(kid, param, id_tol)
        self.hidr(r)
        self.id_sweep(kid, param, id_tol)
        return r

    def fill(self, store: bool = False):
        """G. evaluates all symmetric-once blocks; returns (entries, checksum[, buffer])."""
        cs = np.zeros(1, np.float64)
        total = lib().orc_fill(self._h, None, 0, _p(cs)) if not store else None
        if store:
            need = lib().orc_fill(self._h, None, -1, _p(cs))
            buf = np.empty(max(need, 1), np.float64)
            total = lib().orc_fill(self._h, _p(buf), need, _p(cs))
            return int(total), float(cs[0]), buf[:total]
        return int(total), float(cs[0])

    def matvec(self, x: np.ndarray, rows=None) -> np.ndarray:
        """H. K~ x (x in original order); rows: original row indices (None = all)."""
        x = np.ascontiguousarray(x, np.float64)
        if rows is None:
            y = np.empty(self.n, np.float64)
            rc = lib().orc_matvec_rows(self._h, _p(x), None, 0, _p(y))
        else:
            rows = np.ascontiguousarray(rows, np.int64)
            y = np.empty(len(rows), np.float64)
            rc = lib().orc_matvec_rows(self._h, _p(x), _p(rows), len(rows), _p(y))
        if rc != 0:
            raise RuntimeError("matvec needs id_sweep first")
        return y
