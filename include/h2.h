/*
 * h2.h -- C ABI of the B200-native data-driven H^2 construction (arxiv 2206.01885, "HiDR").
 *
 * The library (paper_2206_01885_b200/lib/libh2b200.so) builds, on one NVIDIA B200 (sm_100a), the
 * H^2 representation of Algorithm 2:
 *
 *   a1-a3  adaptive partition tree: cubified bounding box, Morton quantisation, device radix sort,
 *          level-order nodes (readings A1-A4 in DESIGN.md)
 *   a4     interaction / nearfield lists by a level-synchronous dual traversal of Eq.(2.1)
 *          (readings B1-B4)
 *   a5     r1 = r2 = r calibrated from id_tol (Algorithm 2 line 2; readings E1-E6)
 *   a6-a7  HiDR bottom-up / top-down sweeps with volume-based DataReduct (Algorithm 1 P:331-362,
 *          P:430-433; readings C1-C5, D1-D2)
 *   a8     per level, kernel block K(Xbar_i, Y_i^*) + column-pivoted-QR interpolative decomposition
 *          -> skeletons X^_i, leaf bases U_i, transfer matrices R_c (Eqs.(4.1)-(4.4), P:570-604;
 *          Algorithm 2 lines 10-14; readings F1-F6)
 *   a9     coupling blocks B_ij = K(X^_i, X^_j), (i,j) admissible
 *   a10    nearfield blocks K(X_i, X_j) of the leaf nearfield pairs (reading G1)
 *
 * and applies it to vectors (h2_matvec, the four-pass H^2 product; accuracy checks).
 *
 * Conventions for every call:
 *   - Pointers documented DEVICE must be CUDA device (or managed) memory of the current device;
 *     HOST pointers are ordinary host memory.  The caller keeps ownership of every pointer it
 *     passes; the library only reads inputs during the call and never retains them.
 *   - The handle owns all device memory it allocates; it is immutable after the build, freed by
 *     h2_free.
 *   - On failure a call returns NULL (builders) or a negative H2_ERR_* code, and the thread-local
 *     h2_last_error()/h2_last_error_message() describe it.  No call aborts the process.
 *   - Symmetric kernels (1-6): row and column bases coincide (V = U, W = R, reading F6) and
 *     symmetric blocks are stored once (i < j coupling, i <= j nearfield).  Non-symmetric kernels
 *     (7), or h2_options.nonsymmetric = 1: Algorithm 2 with separate row and column sets (both
 *     getBasis calls of line 11): row bases U/R, column bases V/W, and every ordered block
 *     B_ij = K(X^_i^(row), X^_j^(col)), K(X_i, X_j) stored.
 */
#ifndef H2_B200_H
#define H2_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- kernels (Table 1; Matern-3/2 from BASELINE.json configs[3]) ---------- */
enum {
  H2_KERNEL_COULOMB = 1,  /* 1/|x-y|, kappa(x,x) = 0.           kernel_params: none (may be NULL) */
  H2_KERNEL_GAUSSIAN = 2, /* exp(-|x-y|^2 / h^2).          kernel_params[0] = h > 0          */
  H2_KERNEL_MATERN32 = 3, /* (1 + sqrt3 r/l) exp(-sqrt3 r/l), r=|x-y|.    kernel_params[0] = l > 0          */
  H2_KERNEL_LAPLACE = 4,  /* exp(-r/l) (P:91 at l = 1).                     kernel_params[0] = l > 0          */
  H2_KERNEL_BUMP = 5,     /* exp(-1/(1 - 0.1 r^2)) for 0.1 r^2 < 1, else 0 (Table 1 kappa_4).
                             kernel_params: none (may be NULL)                                            */
  H2_KERNEL_COSDOT = 6,   /* cos(x . y) (Table 1 kappa_3): symmetric, not a function of |x-y|.
                             kernel_params: none (may be NULL)                                            */
  H2_KERNEL_MQSHIFT = 7   /* sqrt(1 + c |x - y + a|^2), the shifted multiquadric of PAPER §4 (P:711-716,
                             c = 100, a = [0, 20] there): smooth, NOT symmetric (kappa(x,y) != kappa(y,x)).
                             kernel_params: d + 1 values {c > 0, a_0, ..., a_{d-1}}, all finite.
                             Always built on the non-symmetric path.                                      */
};

/* ---- status codes ------------------------------------------------------------------------------ */
enum {
  H2_OK = 0,
  H2_ERR_INVALID_ARG = -1,      /* n<1, d not in [1,8], q<1, tau not in (0,0.7], id_tol not in (0,1), h,l<=0 */
  H2_ERR_NONFINITE = -2,        /* a coordinate is NaN or Inf                                   */
  H2_ERR_UNKNOWN_KERNEL = -3,   /* kernel_id not one of H2_KERNEL_*                                     */
  H2_ERR_OOM = -4,              /* device allocation failed or the storage budget cannot hold the tree  */
  H2_ERR_CUDA = -5,             /* a CUDA runtime error (message carries cudaGetErrorString)            */
  H2_ERR_DIM_MISMATCH = -6,     /* matvec length mismatch                                       */
  H2_ERR_NCCL = -7,             /* collective failure (sharded builds)                                  */
  H2_ERR_INTERNAL = -8          /* an internal consistency check failed                                 */
};

typedef struct h2_handle h2_handle;

/*
 * h2_build -- Algorithm 2 end to end on the current CUDA device.
 *   points         DEVICE, n*d fp64, point-major (points[i*d + k]); read-only during the call.
 *   n              number of points, n >= 1 (n < 2^31).
 *   d              dimension, 1 <= d <= 8.
 *   kernel_id      H2_KERNEL_*.
 *   kernel_params  HOST, kernel parameters (see the enum); may be NULL for Coulomb.
 *   id_tol         in (0,1): the ID stops when the largest residual column norm < id_tol*|R11|
 *                  (reading F2); also the epsilon of the r calibration (reading F5).
 *   leaf_size      q >= 1: a node splits while it holds more than q points.
 *   admissibility  tau in (0, 0.7] of Eq.(2.1); 0.5 is the SPEC default.
 * Returns a handle, or NULL (see h2_last_error).  Work runs on the legacy default stream unless
 * h2_build_ex passes one; the call returns after the device work has completed.
 */
h2_handle* h2_build(const double* points, int64_t n, int32_t d, int32_t kernel_id,
                    const double* kernel_params, double id_tol, int32_t leaf_size, double admissibility);

/* storage policy for the coupling / nearfield blocks (a9, a10) */
enum {
  H2_STORE_AUTO = 0,      /* store every block when it fits in mem_budget_bytes, else evaluate in matvec */
  H2_STORE_ALL = 1,       /* always store (H2_ERR_OOM if it does not fit)                                  */
  H2_STORE_ON_THE_FLY = 2 /* never store; h2_matvec evaluates the blocks (skeleton build a1-a8 only)       */
};

typedef struct h2_options {
  int32_t r_override;      /* > 0: use r1 = r2 = r_override and skip the calibration (a5)          */
  int32_t storage;         /* H2_STORE_*                                                            */
  int64_t mem_budget_bytes;/* AUTO: block-store budget; 0 = free device memory minus 4 GiB          */
  void* stream;            /* cudaStream_t for all work; NULL = legacy default stream               */
  int32_t points_on_host;  /* 1: `points` is a HOST pointer; the H2D copy is part of the call       */
  int32_t timing;          /* 1: record per-stage CUDA-event times (h2_info stage_ms)               */
  int32_t hidr_brute;      /* 1: brute-force top-down Vol instead of the pruned exact kernel (same  */
                           /*    result bit for bit; for A/B checks)                                */
  struct h2_comm* comm;    /* NULL: single GPU.  Otherwise a sharded build over comm's ranks (see   */
                           /*    "sharded build" below): every rank calls h2_build_ex with the same */
                           /*    points and parameters; the comm must outlive the handle.           */
  int32_t serial_fill;     /* 1: run the nearfield fill (a10) after a9 on the main stream instead of */
                           /*    concurrently with a5-a9 on a low-priority side stream (default 0;  */
                           /*    same result; for measuring the fill kernel in isolation)           */
  int32_t reduct;          /* HiDR's DataReduct (PAPER §3.3): H2_REDUCT_VOLUME (default, */
                           /*    the one of all the paper's runs), H2_REDUCT_FPS (farthest   */
                           /*    point sampling) or H2_REDUCT_SURFACE; the last two O(r |S|)/node   */
  int32_t nonsymmetric;    /* 1: the non-symmetric path (row AND column bases, every ordered block)  */
                           /*    for any kernel -- for a symmetric one it reproduces V = U,          */
                           /*    X^(col) = X^(row) bit for bit; H2_KERNEL_MQSHIFT implies it         */
  double srrqr_f;          /* > 0 (>= 1): strong rank-revealing refinement of every ID:  */
                           /*    Gu-Eisenstat swaps at fixed rank until max |G| <= srrqr_f; 0 = the  */
                           /*    plain column-pivoted QR (reading F1).  < 0 or in (0, 1): INVALID_ARG */
  int32_t interp_p;        /* > 0: the INTERPOLATION-based H^2 instead (the baseline of PAPER section  */
                           /*    6.3; Eq. (2.2)): p Chebyshev points of the */
                           /*    first kind per dimension on every tree cell, r = p^d, U_i = L(X_i),  */
                           /*    transfers L^(parent)(Q_c), B_ij = K(Q_i, Q_j) (readings Q1-Q4);      */
                           /*    no calibration / HiDR / ID (id_tol is validated but unused).         */
                           /*    1 <= p <= 16, p^d <= 4096; symmetric kernels, single GPU, no rebuild; */
                           /*    otherwise INVALID_ARG.  0 (default): the data-driven construction.   */
} h2_options;

/* ---- DataReduct of HiDR (h2_options.reduct) ---------------------------------------------------- */
enum {
  H2_REDUCT_VOLUME = 0, /* nearest point to every node of an m^d grid over the tight bounding box (C1-C5) */
  H2_REDUCT_FPS = 1,    /* farthest point sampling from the point nearest the box centre (reading C6)   */
  H2_REDUCT_SURFACE = 2 /* nearest point to reference points on three ellipsoids, gamma 0.3/0.6/1.2
                           (reading C7); d = 2 or 3 only (H2_ERR_INVALID_ARG otherwise)     */
};

/* h2_options with the defaults listed above (r calibrated, AUTO, whole-device budget, timing off) */
void h2_options_default(h2_options* opt);

/* h2_build with options (NULL opt = defaults). */
h2_handle* h2_build_ex(const double* points, int64_t n, int32_t d, int32_t kernel_id,
                       const double* kernel_params, double id_tol, int32_t leaf_size,
                       double admissibility, const h2_options* opt);

/*
 * h2_rebuild_ex -- "HiDR once for all" (§6.1.3): the
 * representor sets X_i^*, Y_i^* depend on the points and the budget r only, so an H^2 of the same
 * points for ANOTHER kernel (or kernel parameter, or id_tol) reuses them.  The new handle copies
 * base's tree, lists and HiDR sets (a1-a4, a6-a7, at base's r) and runs the skeleton sweep and the
 * block fill (a8-a10) for kernel_id / kernel_params / id_tol.  The result equals h2_build_ex of
 * the same points with opt->r_override = base's r, bit for bit in every index set.
 *   base  a handle from h2_build / h2_build_ex / h2_rebuild_ex; only read; stays valid.
 *   opt   as for h2_build_ex (r_override ignored; points_on_host meaningless); opt->comm must be
 *         base's comm (NULL for a single-GPU base): a sharded rebuild is collective.
 * Returns the new handle or NULL (h2_last_error).                                              */
h2_handle* h2_rebuild_ex(const h2_handle* base, int32_t kernel_id, const double* kernel_params, double id_tol,
                         const h2_options* opt);

/*
 * h2_matvec -- y = K~ x, the four-pass H^2 product: upward (z^ = U^T x, z^_p = sum R_c^T z^_c),
 * coupling (y^_i += B_ij z^_j), downward (y^_c += R_c y^_p, y = U y^), nearfield (y_i += D_ij x_j).
 *   x, y   DEVICE, length n fp64, ORIGINAL point order; y is overwritten; x and y must not alias.
 * Blocks not stored (storage policy) are evaluated on the fly.  Runs on the handle's stream and
 * returns after completion.  Returns H2_OK or an H2_ERR_* code.
 */
int h2_matvec(const h2_handle* h, const double* x, double* y);

/* h2_matvec with the caller's vector length: n must equal the handle's point count, else
 * H2_ERR_DIM_MISMATCH and nothing is read or written.  Otherwise as h2_matvec. */
int h2_matvec_ex(const h2_handle* h, const double* x, double* y, int64_t n);

/* frees every device buffer of the handle (the H^2 of Algorithm 2's output: bases,
 * transfer matrices, coupling and nearfield blocks, tree and lists); NULL-safe.  Waits for the
 * handle's outstanding device work first.  Never fails. */
void h2_free(h2_handle* h);

/* thread-local status / message of the last failing call on this thread (H2_OK if none). */
int h2_last_error(void);
const char* h2_last_error_message(void);

/* ---- sharded build (BASELINE north_star) -------------------------------------
 * One rank per GPU.  Every rank builds the tree, the lists and the calibration redundantly (they are
 * deterministic, hence identical).  The cut level c is the shallowest level with >= 64 nodes per
 * rank; its nodes are split into contiguous Morton runs balanced by an integer work estimate
 * (h2_shard_split).  HiDR (Algorithm 1) and the ID sweep (Algorithm 2 lines 10-14,
 * P:474-495) run at levels >= c on the rank's own subtrees and at levels < c on every rank; the
 * X_i^* of every level >= c are exchanged (one allgather) after HiDR up below the cut, and the
 * skeletons X^_i (with k_i) after the ID sweep below the cut.  A rank stores the coupling and
 * nearfield blocks of the rows it owns (nodes whose first point lies in its point range).
 * Per-node results are bit-identical to a single-GPU build.  h2_matvec on a sharded handle is
 * collective (same x on every rank; every rank receives the whole y).
 *
 * Transports (h2_comm):
 *   h2_comm_nccl_unique_id / h2_comm_init_nccl: NCCL over NVLink, one process per GPU (rank 0 makes
 *     the id, the caller broadcasts it, e.g. with torch.distributed).  libnccl is resolved at run
 *     time: the copy the process already loaded (import torch first), or $H2_NCCL_LIB.
 *   h2_comm_init_local: nranks host threads of ONE process (same or different devices) whose
 *     comms share group_key; the exchange is a host barrier + device copies (tests).
 * All return NULL / an H2_ERR_* code on failure (h2_last_error).                                   */
typedef struct h2_comm h2_comm;
int h2_comm_nccl_unique_id(unsigned char id[128]);
h2_comm* h2_comm_init_nccl(int32_t nranks, int32_t rank, const unsigned char id[128]);  /* current device */
/* the same on `device`, which becomes (and stays) the calling thread's current device: every later
 * build / matvec on this comm must run with it current (NCCL binds a communicator to one device) */
h2_comm* h2_comm_init_nccl_dev(int32_t nranks, int32_t rank, const unsigned char id[128], int32_t device);
h2_comm* h2_comm_init_local(int32_t nranks, int32_t rank, int64_t group_key);
void h2_comm_free(h2_comm* comm);  /* NULL-safe; after every handle built on it is freed */
int32_t h2_comm_size(const h2_comm* comm);
int32_t h2_comm_rank(const h2_comm* comm);

/* Host-only planning helpers (no device work; usable without a GPU).
 * h2_shard_cut_level: the shallowest level l with level_counts[l] >= 64*nranks, else the most
 *   populous level (shallowest on ties).
 * h2_shard_split: first[q] (q = 0..nranks) = the smallest t with (w[0]+...+w[t-1])*nranks >=
 *   q*total, first[nranks] = ncut: rank q owns cut nodes [first[q], first[q+1]).  Weights must be
 *   >= 0.  Returns H2_OK or H2_ERR_INVALID_ARG.                                                    */
int32_t h2_shard_cut_level(const int64_t* level_counts, int32_t nlevels, int32_t nranks);
int h2_shard_split(const int64_t* weights, int64_t ncut, int32_t nranks, int64_t* first);

/* ---- introspection --------------------------------------------------------------------------- */
typedef struct h2_info_t {
  int64_t n;
  int32_t d, depth, r, nnodes, nleaves, csp; /* csp = max interaction-list length        */
  int64_t n_il, n_nf;                        /* ordered interaction / nearfield pairs              */
  int64_t coupling_entries, nearfield_entries; /* symmetric-once entry counts                      */
  int64_t stored_bytes;                      /* bytes of stored blocks (0 when on the fly)         */
  int32_t coupling_stored, nearfield_stored; /* 1 when that block class is stored                  */
  int64_t hidr_dist_evals;                   /* sum over nodes of |grid| x |S_i| (+ |T_i|)         */
  int64_t id_kernel_evals;                   /* sum over nodes of |Xbar_i| x |Y_i^*|               */
  int32_t kmax;                              /* max skeleton size                                  */
  int32_t gpu_launches;                      /* kernels launched by the last build                 */
  /* per-stage device milliseconds (when opt.timing): [0] tree a1-a3, [1] lists a4,
   * [2] calibration a5, [3] HiDR up a6, [4] HiDR down a7, [5] ID sweep a8, [6] coupling fill a9,
   * [7] nearfield fill a10, [8] whole build                                                     */
  float stage_ms[9];
  int64_t hidr_dist_done;                    /* distances the pruned top-down Vol evaluated        */
  int64_t hidr_up_evals;                     /* the bottom-up sweep's share of hidr_dist_evals     */
  int32_t nonsymmetric;                      /* 1: separate column bases, every ordered block      */
  int32_t kmax_col;                          /* max column skeleton size (non-symmetric path)      */
  int64_t srrqr_swaps;                       /* SRRQR swaps made (h2_options.srrqr_f > 0)          */
} h2_info_t;

int h2_info(const h2_handle* h, h2_info_t* out);

/* ---- export hooks for the parity tests (all written to HOST buffers) ------------------------- */
enum {
  H2_EXPORT_PERM = 1,     /* int32[n]: tree position -> original index                          */
  H2_EXPORT_NODES = 2,    /* int32[nnodes*7]: level, begin, end, parent, first_child, nchild, leaf */
  H2_EXPORT_IL_OFF = 4,   /* int64[nnodes+1]  CSR of the interaction lists (ordered, sorted)    */
  H2_EXPORT_IL_IDX = 5,   /* int32[n_il]                                                         */
  H2_EXPORT_NF_OFF = 6,   /* int64[nnodes+1]  CSR of the nearfield lists                         */
  H2_EXPORT_NF_IDX = 7,   /* int32[n_nf]                                                         */
  H2_EXPORT_XS_OFF = 8,   /* int64[nnodes+1]  X_i^* (tree-order indices, sorted)                 */
  H2_EXPORT_XS_IDX = 9,
  H2_EXPORT_YS_OFF = 10,  /* int64[nnodes+1]  Y_i^*                                              */
  H2_EXPORT_YS_IDX = 11,
  H2_EXPORT_K = 12,       /* int32[nnodes] skeleton sizes k_i                                    */
  H2_EXPORT_SK_OFF = 13,  /* int64[nnodes+1]  X^_i (tree-order indices, pivot order)             */
  H2_EXPORT_SK_IDX = 14,
  H2_EXPORT_U_OFF = 15,   /* int64[nnodes+1]  U_i / stacked R_c blocks, |Xbar_i| x k_i col-major */
  H2_EXPORT_U = 16,       /* double[...]                                                         */
  H2_EXPORT_XBAR_N = 17,  /* int32[nnodes] |Xbar_i|                                              */
  H2_EXPORT_TREE_X = 18,  /* double[n*d] tree-order coordinates, point-major                     */
  H2_EXPORT_SHARD = 19,   /* int64[5 + 2*(depth+1)]: nranks, rank, cut level, p_lo, p_hi, then per */
                          /* level l the node range [lo_l, hi_l) this rank computed               */
  H2_EXPORT_BLOCK_SAMPLE = 20, /* see h2_sample_blocks                                           */
  H2_EXPORT_ID_PATH = 21, /* int32[nnodes]: the a8 code path of each node's ID: 0..5 staged       */
                          /* shared-memory size classes, 6 mid class (256 threads, 2 CTAs/SM),   */
                          /* 7 lean shared-memory class, 8 / 9 global memory (256 / 1024          */
                          /* threads), 10 thread-block cluster, 11 warp per node, -1 no basis     */
  /* the column bases of the non-symmetric path (as K, SK_*, U_*, XBAR_N for the row bases)       */
  H2_EXPORT_K_COL = 22, H2_EXPORT_SKC_OFF = 23, H2_EXPORT_SKC_IDX = 24, H2_EXPORT_V_OFF = 25,
  H2_EXPORT_V = 26, H2_EXPORT_XBARC_N = 27,
  H2_EXPORT_INTERP_Q = 28 /* double[nnodes*r*d]: the interpolation baseline's Chebyshev nodes, node-major,
                             point-major (slot alpha = sum_c a_c p^c); zeros where k_i = 0             */
};

/* Copies array `what` into host_buf when cap_bytes suffices; *needed_bytes receives its size.
 * Returns H2_OK, or H2_ERR_INVALID_ARG (unknown `what` or buffer too small: *needed_bytes set). */
int h2_export(const h2_handle* h, int what, void* host_buf, size_t cap_bytes, size_t* needed_bytes);

/* Reads stored block entries for parity sampling.  For each s < count: kind[s] = 0 coupling /
 * 1 nearfield, pair[s] = index into the stored pair list of that kind (ordered as the CSR with
 * i < j resp. i <= j; every ordered pair on the non-symmetric path), entry[s] = row-major entry
 * index inside that block (rows: X^_i^(row) resp. X_i; columns: X^_j^(col) resp. X_j).  Writes
 * value[s] (HOST), and row_pt[s], col_pt[s] = the tree-order point indices of that entry
 * (HOST int32).  Returns H2_OK, H2_ERR_INVALID_ARG if a class is not stored or out of range. */
int h2_sample_blocks(const h2_handle* h, int64_t count, const int32_t* kind, const int64_t* pair,
                     const int64_t* entry, double* value, int32_t* row_pt, int32_t* col_pt);

#ifdef __cplusplus
}
#endif
#endif /* H2_B200_H */
