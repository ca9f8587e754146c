"""Thin Python binding of the B200 H^2 library (C ABI: include/h2.h).

Argument marshalling only: every step of the build and the matvec runs in the CUDA kernels of
paper_2206_01885_b200/lib/libh2b200.so.  There is no CPU fallback: if the library is missing or
no CUDA device is present the calls raise.  PyTorch is used by callers only for device memory
and streams (pass tensor.data_ptr() / torch.cuda.current_stream().cuda_stream).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libh2b200.so")

H2_KERNEL_COULOMB, H2_KERNEL_GAUSSIAN, H2_KERNEL_MATERN32, H2_KERNEL_LAPLACE, H2_KERNEL_BUMP, H2_KERNEL_COSDOT = \
    1, 2, 3, 4, 5, 6
H2_KERNEL_MQSHIFT = 7  # sqrt(1 + c |x - y + a|^2), non-symmetric; kernel_params = (c, a_0, ..., a_{d-1})
H2_STORE_AUTO, H2_STORE_ALL, H2_STORE_ON_THE_FLY = 0, 1, 2
H2_REDUCT_VOLUME, H2_REDUCT_FPS, H2_REDUCT_SURFACE = 0, 1, 2  # HiDR DataReduct (h2_options.reduct)

EXPORT = dict(PERM=1, NODES=2, IL_OFF=4, IL_IDX=5, NF_OFF=6, NF_IDX=7, XS_OFF=8, XS_IDX=9, YS_OFF=10,
              YS_IDX=11, K=12, SK_OFF=13, SK_IDX=14, U_OFF=15, U=16, XBAR_N=17, TREE_X=18, SHARD=19, ID_PATH=21,
              K_COL=22, SKC_OFF=23, SKC_IDX=24, V_OFF=25, V=26, XBARC_N=27, INTERP_Q=28)
_EXPORT_DTYPE = dict(PERM=np.int32, NODES=np.int32, IL_OFF=np.int64, IL_IDX=np.int32, NF_OFF=np.int64,
                     NF_IDX=np.int32, XS_OFF=np.int64, XS_IDX=np.int32, YS_OFF=np.int64, YS_IDX=np.int32,
                     K=np.int32, SK_OFF=np.int64, SK_IDX=np.int32, U_OFF=np.int64, U=np.float64,
                     XBAR_N=np.int32, TREE_X=np.float64, SHARD=np.int64, ID_PATH=np.int32, K_COL=np.int32,
                     SKC_OFF=np.int64, SKC_IDX=np.int32, V_OFF=np.int64, V=np.float64, XBARC_N=np.int32,
                     INTERP_Q=np.float64)

EXPORTED_SYMBOLS = ["h2_build", "h2_build_ex", "h2_rebuild_ex", "h2_options_default", "h2_matvec", "h2_matvec_ex", "h2_free", "h2_last_error",
                    "h2_last_error_message", "h2_info", "h2_export", "h2_sample_blocks", "h2_comm_nccl_unique_id",
                    "h2_comm_init_nccl", "h2_comm_init_nccl_dev", "h2_comm_init_local", "h2_comm_free", "h2_comm_size", "h2_comm_rank",
                    "h2_shard_cut_level", "h2_shard_split"]


class h2_options(C.Structure):
    _fields_ = [("r_override", C.c_int32), ("storage", C.c_int32), ("mem_budget_bytes", C.c_int64),
                ("stream", C.c_void_p), ("points_on_host", C.c_int32), ("timing", C.c_int32),
                ("hidr_brute", C.c_int32), ("comm", C.c_void_p), ("serial_fill", C.c_int32),
                ("reduct", C.c_int32), ("nonsymmetric", C.c_int32), ("srrqr_f", C.c_double),
                ("interp_p", C.c_int32)]


class h2_info_t(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("depth", C.c_int32), ("r", C.c_int32),
                ("nnodes", C.c_int32), ("nleaves", C.c_int32), ("csp", C.c_int32), ("n_il", C.c_int64),
                ("n_nf", C.c_int64), ("coupling_entries", C.c_int64), ("nearfield_entries", C.c_int64),
                ("stored_bytes", C.c_int64), ("coupling_stored", C.c_int32), ("nearfield_stored", C.c_int32),
                ("hidr_dist_evals", C.c_int64), ("id_kernel_evals", C.c_int64), ("kmax", C.c_int32),
                ("gpu_launches", C.c_int32), ("stage_ms", C.c_float * 9), ("hidr_dist_done", C.c_int64),
                ("hidr_up_evals", C.c_int64), ("nonsymmetric", C.c_int32), ("kmax_col", C.c_int32),
                ("srrqr_swaps", C.c_int64)]


STAGES = ["tree", "lists", "calibrate", "hidr_up", "hidr_down", "id_sweep", "coupling_fill", "nearfield_fill",
          "build"]


class H2Error(RuntimeError):
    pass


_lib = None


def lib():
    """Loads libh2b200.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise H2Error(f"{LIB_PATH} not built; run python -m paper_2206_01885_b200.build or "
                          f"__graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.h2_build.restype = vp
        L.h2_build.argtypes = [vp, i64, i32, i32, vp, f64, i32, f64]
        L.h2_build_ex.restype = vp
        L.h2_build_ex.argtypes = [vp, i64, i32, i32, vp, f64, i32, f64, C.POINTER(h2_options)]
        L.h2_options_default.argtypes = [C.POINTER(h2_options)]
        L.h2_rebuild_ex.restype = vp
        L.h2_rebuild_ex.argtypes = [vp, i32, vp, f64, C.POINTER(h2_options)]
        L.h2_matvec.restype = C.c_int
        L.h2_matvec.argtypes = [vp, vp, vp]
        L.h2_matvec_ex.restype = C.c_int
        L.h2_matvec_ex.argtypes = [vp, vp, vp, i64]
        L.h2_free.argtypes = [vp]
        L.h2_last_error.restype = C.c_int
        L.h2_last_error_message.restype = C.c_char_p
        L.h2_info.restype = C.c_int
        L.h2_info.argtypes = [vp, C.POINTER(h2_info_t)]
        L.h2_export.restype = C.c_int
        L.h2_export.argtypes = [vp, C.c_int, vp, C.c_size_t, C.POINTER(C.c_size_t)]
        L.h2_sample_blocks.restype = C.c_int
        L.h2_sample_blocks.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp]
        L.h2_comm_nccl_unique_id.restype = C.c_int
        L.h2_comm_nccl_unique_id.argtypes = [vp]
        L.h2_comm_init_nccl.restype = vp
        L.h2_comm_init_nccl.argtypes = [i32, i32, vp]
        L.h2_comm_init_nccl_dev.restype = vp
        L.h2_comm_init_nccl_dev.argtypes = [i32, i32, vp, i32]
        L.h2_comm_init_local.restype = vp
        L.h2_comm_init_local.argtypes = [i32, i32, i64]
        L.h2_comm_free.argtypes = [vp]
        L.h2_comm_size.restype = i32
        L.h2_comm_size.argtypes = [vp]
        L.h2_comm_rank.restype = i32
        L.h2_comm_rank.argtypes = [vp]
        L.h2_shard_cut_level.restype = i32
        L.h2_shard_cut_level.argtypes = [vp, i32, i32]
        L.h2_shard_split.restype = C.c_int
        L.h2_shard_split.argtypes = [vp, i64, i32, vp]
        _lib = L
    return _lib


def last_error() -> tuple[int, str]:
    L = lib()
    return int(L.h2_last_error()), L.h2_last_error_message().decode()


def _raise():
    code, msg = last_error()
    raise H2Error(f"h2 error {code}: {msg}")


def h2_options_default() -> h2_options:
    o = h2_options()
    lib().h2_options_default(C.byref(o))
    return o


def h2_build(points_ptr: int, n: int, d: int, kernel_id: int, kernel_params, id_tol: float, leaf_size: int,
             admissibility: float = 0.5, options: h2_options | None = None) -> int:
    """Calls h2_build_ex. points_ptr: DEVICE pointer (or HOST when options.points_on_host)."""
    kp = (C.c_double * max(1, len(kernel_params or ())))(*(kernel_params or (0.0,)))
    o = options if options is not None else h2_options_default()
    h = lib().h2_build_ex(C.c_void_p(points_ptr), n, d, kernel_id, kp, id_tol, leaf_size, admissibility,
                          C.byref(o))
    if not h:
        _raise()
    return h


def h2_matvec(h: int, x_ptr: int, y_ptr: int, n: int | None = None) -> None:
    """h2_matvec (or h2_matvec_ex when the caller's length n is given: H2_ERR_DIM_MISMATCH on a
    mismatch)."""
    L = lib()
    rc = (L.h2_matvec(C.c_void_p(h), C.c_void_p(x_ptr), C.c_void_p(y_ptr)) if n is None else
          L.h2_matvec_ex(C.c_void_p(h), C.c_void_p(x_ptr), C.c_void_p(y_ptr), int(n)))
    if rc != 0:
        _raise()


def h2_free(h: int) -> None:
    lib().h2_free(C.c_void_p(h))


def h2_info(h: int) -> dict:
    i = h2_info_t()
    if lib().h2_info(C.c_void_p(h), C.byref(i)) != 0:
        _raise()
    out = {f: getattr(i, f) for f, _ in h2_info_t._fields_ if f != "stage_ms"}
    out["stage_ms"] = dict(zip(STAGES, [float(v) for v in i.stage_ms]))
    return out


def h2_export(h: int, what: str) -> np.ndarray:
    code = EXPORT[what]
    need = C.c_size_t(0)
    L = lib()
    L.h2_export(C.c_void_p(h), code, None, 0, C.byref(need))
    if need.value == 0 and L.h2_last_error() not in (0, -1):
        _raise()
    dt = _EXPORT_DTYPE[what]
    a = np.empty(max(1, need.value // np.dtype(dt).itemsize), dt)
    if L.h2_export(C.c_void_p(h), code, a.ctypes.data_as(C.c_void_p), a.nbytes, C.byref(need)) != 0:
        _raise()
    return a[: need.value // np.dtype(dt).itemsize]


def h2_sample_blocks(h: int, kind, pair, entry):
    kind = np.ascontiguousarray(kind, np.int32)
    pair = np.ascontiguousarray(pair, np.int64)
    entry = np.ascontiguousarray(entry, np.int64)
    m = len(kind)
    val = np.empty(m, np.float64)
    rp = np.empty(m, np.int32)
    cp = np.empty(m, np.int32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    if lib().h2_sample_blocks(C.c_void_p(h), m, p(kind), p(pair), p(entry), p(val), p(rp), p(cp)) != 0:
        _raise()
    return val, rp, cp


def _nccl_hint():
    """Points the library's run-time NCCL lookup at the copy PyTorch ships (if the env is unset)."""
    if os.environ.get("H2_NCCL_LIB"):
        return
    try:
        import nvidia.nccl
        for d in nvidia.nccl.__path__:
            so = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(so):
                os.environ["H2_NCCL_LIB"] = so
                return
    except Exception:
        pass


class H2Comm:
    """Exchange transport of a sharded build (include/h2.h "sharded build").

    H2Comm.nccl(nranks, rank, uid): one process per GPU; uid from H2Comm.nccl_unique_id() on rank 0,
    broadcast by the caller (e.g. torch.distributed.broadcast_object_list).
    H2Comm.local(nranks, rank, key): ranks are host threads of this process sharing `key`."""

    def __init__(self, ptr: int):
        if not ptr:
            _raise()
        self.ptr = ptr

    @staticmethod
    def nccl_unique_id() -> bytes:
        _nccl_hint()
        buf = (C.c_ubyte * 128)()
        if lib().h2_comm_nccl_unique_id(buf) != 0:
            _raise()
        return bytes(buf)

    @classmethod
    def nccl(cls, nranks: int, rank: int, uid: bytes, device: int | None = None) -> "H2Comm":
        """device: the CUDA device of this rank (h2_comm_init_nccl_dev); None = the current one."""
        _nccl_hint()
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        if device is None:
            return cls(lib().h2_comm_init_nccl(nranks, rank, buf))
        return cls(lib().h2_comm_init_nccl_dev(nranks, rank, buf, int(device)))

    @classmethod
    def local(cls, nranks: int, rank: int, key: int) -> "H2Comm":
        return cls(lib().h2_comm_init_local(nranks, rank, key))

    @property
    def size(self) -> int:
        return int(lib().h2_comm_size(C.c_void_p(self.ptr)))

    @property
    def rank(self) -> int:
        return int(lib().h2_comm_rank(C.c_void_p(self.ptr)))

    def close(self):
        if getattr(self, "ptr", None):
            lib().h2_comm_free(C.c_void_p(self.ptr))
            self.ptr = None


def shard_cut_level(level_counts, nranks: int) -> int:
    """h2_shard_cut_level (host only)."""
    c = np.ascontiguousarray(level_counts, np.int64)
    return int(lib().h2_shard_cut_level(c.ctypes.data_as(C.c_void_p), len(c), nranks))


def shard_split(weights, nranks: int) -> np.ndarray:
    """h2_shard_split (host only): first[q], q = 0..nranks."""
    w = np.ascontiguousarray(weights, np.int64)
    first = np.empty(nranks + 1, np.int64)
    if lib().h2_shard_split(w.ctypes.data_as(C.c_void_p), len(w), nranks, first.ctypes.data_as(C.c_void_p)) != 0:
        _raise()
    return first


class H2Matrix:
    """Owning wrapper: builds on the GPU from a torch CUDA tensor (n x d fp64) or a numpy array."""

    def __init__(self, points, kernel_id: int, kernel_params=(), id_tol: float = 1e-6, leaf_size: int = 64,
                 admissibility: float = 0.5, r: int = 0, storage: int = H2_STORE_AUTO, stream=None,
                 timing: bool = False, mem_budget_bytes: int = 0, hidr_brute: bool = False,
                 comm: H2Comm | None = None, reduct: int = H2_REDUCT_VOLUME, nonsymmetric: bool = False,
                 srrqr_f: float = 0.0, interp_p: int = 0):
        import torch
        o = h2_options_default()
        o.srrqr_f = float(srrqr_f)
        o.interp_p = int(interp_p)
        o.reduct = int(reduct)
        o.nonsymmetric = int(bool(nonsymmetric))
        if comm is not None:
            o.comm = C.c_void_p(comm.ptr)
            self._comm = comm
        o.hidr_brute = int(bool(hidr_brute))
        o.r_override = int(r)
        o.storage = int(storage)
        o.timing = int(bool(timing))
        o.mem_budget_bytes = int(mem_budget_bytes)
        if stream is None:
            stream = torch.cuda.current_stream()
        o.stream = C.c_void_p(stream.cuda_stream)
        if isinstance(points, np.ndarray):
            pts = np.ascontiguousarray(points, np.float64)
            o.points_on_host = 1
            self._keep = pts
            ptr = pts.ctypes.data
        else:
            assert points.is_cuda and points.dtype == torch.float64 and points.is_contiguous()
            self._keep = points
            ptr = points.data_ptr()
        self.n, self.d = int(points.shape[0]), int(points.shape[1])
        self.stream = stream
        self.id_tol = id_tol
        self.h = h2_build(ptr, self.n, self.d, kernel_id, list(kernel_params), id_tol, leaf_size, admissibility, o)

    def rebuild(self, kernel_id: int, kernel_params=(), id_tol: float | None = None, storage: int = H2_STORE_AUTO,
                timing: bool = False) -> "H2Matrix":
        """h2_rebuild_ex: the same points, tree, lists and HiDR representor sets, another kernel."""
        o = h2_options_default()
        o.storage = int(storage)
        o.timing = int(bool(timing))
        o.stream = C.c_void_p(self.stream.cuda_stream)
        if getattr(self, "_comm", None) is not None:
            o.comm = C.c_void_p(self._comm.ptr)
        kp = list(kernel_params)
        kpa = (C.c_double * max(1, len(kp)))(*(kp or [0.0]))
        tol = self.id_tol if id_tol is None else id_tol
        h = lib().h2_rebuild_ex(C.c_void_p(self.h), kernel_id, kpa, tol, C.byref(o))
        if not h:
            _raise()
        out = H2Matrix.__new__(H2Matrix)
        out.h, out.n, out.d, out.stream, out._keep, out.id_tol = h, self.n, self.d, self.stream, self._keep, tol
        if getattr(self, "_comm", None) is not None:
            out._comm = self._comm
        return out

    def matvec(self, x):
        """y = K~ x for a CUDA float64 contiguous vector of length n (original point order)."""
        import torch
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()
                and x.dim() == 1):
            raise H2Error("matvec: x must be a contiguous 1-D float64 CUDA tensor")
        y = torch.empty_like(x)
        h2_matvec(self.h, x.data_ptr(), y.data_ptr(), x.numel())
        return y

    def info(self) -> dict:
        return h2_info(self.h)

    def export(self, what: str) -> np.ndarray:
        return h2_export(self.h, what)

    def close(self):
        if getattr(self, "h", None):
            h2_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
