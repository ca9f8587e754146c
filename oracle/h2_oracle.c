/*
 * h2_oracle.c -- plain, slow, obviously-correct fp64 CPU ORACLE for the data-driven H^2
 * construction of arxiv 2206.01885 ("HiDR").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or helper with
 * the CUDA path (paper_2206_01885_b200/csrc), and the CUDA path never calls it.
 *
 * Citations: "P:L" = /root/reference/PAPER.md line L; "S:L" = SPEC.md line L; readings "B1", "C4",
 * "E3", ... are the numbered ambiguity readings listed in DESIGN.md.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no -ffast-math): every floating-point
 * operation is rounded separately, in the order written.  OpenMP is used only across independent
 * nodes of one tree level; the per-node code is sequential and deterministic.
 *
 * Steps (oracle letters follow DESIGN.md "Oracle"):
 *   A  partition (Fig. partition)          orc_new
 *   B  admissibility Eq.(2.1) + interaction/nearfield lists
 *       via dual traversal                             orc_new
 *   C  volume-based DataReduct (used in all runs P:839)       orc_vol
 *   C' farthest point sampling (reading C6)                    orc_fps
 *   C'' surface-based DataReduct (reading C7)                  orc_surface
 *   D  HiDR, Algorithm 1                                     orc_hidr
 *   E  r calibration, Algorithm 2 line 2 + P:628-630                     orc_calibrate
 *   F  getBasis = pivoted-QR ID, Eqs.(4.1)-(4.4), bottom-up
 *      sweep of Algorithm 2 lines 11-12                      orc_id_sweep
 *   G  coupling / nearfield blocks (Algorithm 2)              orc_fill, on the fly in H
 *   H  H^2 matvec, four passes                                   orc_matvec_rows
 *   I  dense rows of K x                                     orc_dense_rows
 *   J  kernel blocks K(A, B) of arbitrary point sets (interpolation baseline) orc_kernel_block
 *
 * Parity pins: see tests/test_oracle_*.py.  Every function here is pinned; the calibration (E) and
 * the top-down composition of D by tests/test_oracle_calib_topdown_pins.py (Eckart-Young and
 * least-squares identities, the pass-through bound, an independent SplitMix64, a hand golden).
 */
#include <limits.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAXD 8

/* ------------------------------------------------------------------------------------------ */
/* small utilities                                                                             */
/* ------------------------------------------------------------------------------------------ */

static double wall(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

/* sort ascending and remove duplicates in place; returns the new length */
static int sort_unique(int* a, int n) {
  if (n <= 1) return n;
  qsort(a, (size_t)n, sizeof(int), cmp_int);
  int m = 1;
  for (int i = 1; i < n; i++)
    if (a[i] != a[m - 1]) a[m++] = a[i];
  return m;
}

/* m^d, saturating at INT64_MAX/2 */
static int64_t ipow_sat(int64_t m, int d) {
  int64_t r = 1;
  for (int k = 0; k < d; k++) {
    if (r > (INT64_MAX / 2) / (m > 0 ? m : 1)) return INT64_MAX / 2;
    r *= m;
  }
  return r;
}

/* ------------------------------------------------------------------------------------------ */
/* kernel functions  (Table 1; Matern-3/2 from BASELINE.json configs[3])    */
/* ------------------------------------------------------------------------------------------ */

enum { ORC_COULOMB = 1, ORC_GAUSSIAN = 2, ORC_MATERN32 = 3, ORC_LAPLACE = 4, ORC_BUMP = 5, ORC_COSDOT = 6,
       ORC_MQSHIFT = 7 };

/* the shift a of the non-symmetric shifted multiquadric (kernel 7); set by orc_set_kernel_shift */
static double g_shift[ORC_MAXD];

void orc_set_kernel_shift(const double* a, int d) {
  for (int k = 0; k < ORC_MAXD; k++) g_shift[k] = k < d ? a[k] : 0.0;
}

static double sqdist(const double* x, const double* y, int d) {
  double s = 0.0;
  for (int k = 0; k < d; k++) {
    double df = x[k] - y[k];
    s = s + df * df;
  }
  return s;
}

/* kappa(x,y) as a function of the squared distance s.  Coulomb kappa(x,x)=0 (reading G2). */
static double kernel_of_s(int kid, double p, double s) {
  switch (kid) {
    case ORC_COULOMB:
      return s == 0.0 ? 0.0 : 1.0 / sqrt(s);
    case ORC_GAUSSIAN: /* exp(-|x-y|^2 / h^2), P:91 / P:967 */
      return exp(-(s / (p * p)));
    case ORC_MATERN32: { /* (1 + sqrt3 r / l) exp(-sqrt3 r / l) */
      double a = sqrt(3.0) * sqrt(s) / p;
      return (1.0 + a) * exp(-a);
    }
    case ORC_LAPLACE: /* exp(-|x-y| / l): the Laplace kernel e^{-|x-y|} of P:91 at l = 1 */
      return exp(-(sqrt(s) / p));
    case ORC_BUMP: { /* kappa_4 of Table 1: exp(-1/(1 - 0.1|x-y|^2)); 0 where
                        0.1|x-y|^2 >= 1 (reading K5: its limit at the edge of its domain) */
      double t = 0.1 * s;
      return t < 1.0 ? exp(-(1.0 / (1.0 - t))) : 0.0;
    }
    default:
      return NAN;
  }
}

double orc_kernel(int kid, double p, const double* x, const double* y, int d) {
  if (kid == ORC_MQSHIFT) { /* sqrt(1 + c |x - y + a|^2), PAPER §4 P:711-716 (c = 100, a = [0, 20]^T
                               there): smooth and NOT symmetric, kappa(x,y) != kappa(y,x) */
    double t = 0.0;
    for (int k = 0; k < d; k++) {
      double df = x[k] - y[k] + g_shift[k];
      t = t + df * df;
    }
    return sqrt(1.0 + p * t);
  }
  if (kid == ORC_COSDOT) { /* kappa_3 of Table 1: cos(x . y), the dot summed in k order */
    double t = 0.0;
    for (int k = 0; k < d; k++) t = t + x[k] * y[k];
    return cos(t);
  }
  return kernel_of_s(kid, p, sqdist(x, y, d));
}

/* ------------------------------------------------------------------------------------------ */
/* C. volume-based DataReduct (readings C2-C5)                                      */
/* ------------------------------------------------------------------------------------------ */

/* Vol(S, k): X is point-major (X[s*d+k]); S holds indices into X (here: tree-order indices).
 * Returns |out| <= k, out sorted ascending, no duplicates.
 *   |S| <= k           : out = S sorted (C5).
 *   m = max{m : m^d <= k}; grid domain = tight bbox of S (C2); cell-centre nodes q (C3);
 *   for each q: argmin_s sum_k (x_sk - q_k)^2, summed k = 0..d-1, no FMA; ties -> lowest
 *   index (C4).  Selected indices are sorted and de-duplicated.                                */
int orc_vol(const double* X, int d, const int* S, int ns, int k, int* out) {
  if (ns <= 0) return 0;
  if (ns <= k) {
    memcpy(out, S, sizeof(int) * (size_t)ns);
    return sort_unique(out, ns);
  }
  int m = 1;
  while (ipow_sat(m + 1, d) <= k) m++;
  double lo[ORC_MAXD], hi[ORC_MAXD], h[ORC_MAXD];
  for (int c = 0; c < d; c++) {
    lo[c] = X[(int64_t)S[0] * d + c];
    hi[c] = lo[c];
  }
  for (int s = 1; s < ns; s++)
    for (int c = 0; c < d; c++) {
      double v = X[(int64_t)S[s] * d + c];
      if (v < lo[c]) lo[c] = v;
      if (v > hi[c]) hi[c] = v;
    }
  for (int c = 0; c < d; c++) h[c] = (hi[c] - lo[c]) / (double)m;
  int64_t G = ipow_sat(m, d);
  int cnt = 0;
  for (int64_t g = 0; g < G; g++) {
    double q[ORC_MAXD];
    int64_t rem = g;
    for (int c = 0; c < d; c++) { /* dimension 0 varies fastest */
      int64_t j = rem % m;
      rem /= m;
      q[c] = lo[c] + ((double)j + 0.5) * h[c];
    }
    double best = INFINITY;
    int bi = INT_MAX;
    for (int s = 0; s < ns; s++) {
      double dist = sqdist(X + (int64_t)S[s] * d, q, d);
      if (dist < best || (dist == best && S[s] < bi)) {
        best = dist;
        bi = S[s];
      }
    }
    out[cnt++] = bi;
  }
  return sort_unique(out, cnt);
}

/* Farthest point sampling, PAPER §3.3: "S is initialized with one point only. Then FPS
 * searches for a point in X\S that is farthest from S and adds the point to S ... until S reaches
 * size k" (reading C6: the first point is the point nearest the centre of the tight bounding box --
 * Vol(S, 1), the m = 1 case of C2-C4 -- distances as in C4, ties of the farthest point -> lowest
 * index).  Returns |out| = min(k, |S|), sorted ascending (C5).                                  */
int orc_fps(const double* X, int d, const int* S, int ns, int k, int* out) {
  if (ns <= 0) return 0;
  if (ns <= k) {
    memcpy(out, S, sizeof(int) * (size_t)ns);
    return sort_unique(out, ns);
  }
  int seed;
  if (orc_vol(X, d, S, ns, 1, &seed) != 1) return -1;
  double* mind = (double*)malloc(sizeof(double) * (size_t)ns);
  int cnt = 0;
  out[cnt++] = seed;
  for (int s = 0; s < ns; s++) mind[s] = S[s] == seed ? -1.0 : sqdist(X + (int64_t)S[s] * d, X + (int64_t)seed * d, d);
  while (cnt < k) {
    double best = -1.0;
    int bs = -1;
    for (int s = 0; s < ns; s++)
      if (mind[s] > best || (mind[s] == best && mind[s] >= 0.0 && S[s] < S[bs])) {
        best = mind[s];
        bs = s;
      }
    if (bs < 0 || best < 0.0) break; /* every point selected */
    const int z = S[bs];
    out[cnt++] = z;
    mind[bs] = -1.0;
    for (int s = 0; s < ns; s++)
      if (mind[s] >= 0.0) {
        const double dz = sqdist(X + (int64_t)S[s] * d, X + (int64_t)z * d, d);
        if (dz < mind[s]) mind[s] = dz;
      }
  }
  free(mind);
  return sort_unique(out, cnt);
}

/* ------------------------------------------------------------------------------------------ */
/* F. getBasis: column-pivoted Householder QR interpolative decomposition (Eqs.(4.1)-(4.4))    */
/* ------------------------------------------------------------------------------------------ */

/* M: rows x cols, column-major (ld = rows).  CPQR of M with residual column norms recomputed
 * at every step, pivot = largest norm (ties -> lowest current position), stop when the largest
 * residual norm < tol * |R11| (reading F2; k = 0 if R11 = 0).  On return piv[] is the column
 * permutation (piv[t] = original column at position t), M[0:k,0:k] holds R11 and M[0:k,k:cols]
 * holds T = R11^{-1} R12, so that  M[:, piv[k:]] ~= M[:, piv[:k]] T.  Returns k.             */
int orc_cpqr(double* M, int rows, int cols, double tol, int* piv) {
  for (int j = 0; j < cols; j++) piv[j] = j;
  int kmax = rows < cols ? rows : cols;
  double r11 = 0.0;
  int k = 0;
  double* v = (double*)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1));
  for (int t = 0; t < kmax; t++) {
    int p = -1;
    double best = -1.0;
    for (int j = t; j < cols; j++) {
      double s = 0.0;
      for (int i = t; i < rows; i++) {
        double a = M[i + (int64_t)rows * j];
        s = s + a * a;
      }
      double nrm = sqrt(s);
      if (nrm > best) {
        best = nrm;
        p = j;
      }
    }
    if (t == 0) {
      r11 = best;
      if (r11 == 0.0) break;
    }
    if (best < tol * r11) break;
    if (p != t) {
      for (int i = 0; i < rows; i++) {
        double a = M[i + (int64_t)rows * t];
        M[i + (int64_t)rows * t] = M[i + (int64_t)rows * p];
        M[i + (int64_t)rows * p] = a;
      }
      int tp = piv[t];
      piv[t] = piv[p];
      piv[p] = tp;
    }
    /* Householder reflector H = I - 2 v v^T / (v^T v) mapping column t to alpha e_t */
    double x0 = M[t + (int64_t)rows * t];
    double alpha = x0 >= 0.0 ? -best : best;
    double vtv = 0.0;
    for (int i = t; i < rows; i++) v[i] = M[i + (int64_t)rows * t];
    v[t] = x0 - alpha;
    for (int i = t; i < rows; i++) vtv = vtv + v[i] * v[i];
    M[t + (int64_t)rows * t] = alpha;
    for (int i = t + 1; i < rows; i++) M[i + (int64_t)rows * t] = 0.0;
    if (vtv > 0.0) {
      for (int j = t + 1; j < cols; j++) {
        double* col = M + (int64_t)rows * j;
        double s = 0.0;
        for (int i = t; i < rows; i++) s = s + v[i] * col[i];
        double f = 2.0 * s / vtv;
        for (int i = t; i < rows; i++) col[i] = col[i] - f * v[i];
      }
    }
    k = t + 1;
  }
  free(v);
  /* T = R11^{-1} R12 by back substitution, stored over R12 */
  for (int c = k; c < cols; c++) {
    double* col = M + (int64_t)rows * c;
    for (int i = k - 1; i >= 0; i--) {
      double s = col[i];
      for (int l = i + 1; l < k; l++) s = s - M[i + (int64_t)rows * l] * col[l];
      col[i] = s / M[i + (int64_t)rows * i];
    }
  }
  return k;
}

/* Strong rank-revealing refinement (SRRQR, PAPER Eq.(4.1): "||G||_max is bounded by a
 * prescribed constant"; Gu & Eisenstat's swaps at fixed rank): given the CPQR of M0 (rows x cols,
 * column-major, untouched) with rank k and pivot order piv, while some |T_ij| > f (T = R11^{-1} R12,
 * k x (cols - k)) swap the skeleton column at position i with the non-skeleton column at position
 * k + j of the largest such entry (each swap multiplies |det R11| by |T_ij| > f > 1, so the loop
 * ends), and refactor: Householder QR without pivoting of the first k columns in the new order,
 * applied to all columns, then T by back substitution.  On return Mout holds R11 / T like orc_cpqr
 * and piv the new order.  Returns the number of swaps.                                            */
int orc_srrqr_swaps(const double* M0, double* Mout, int rows, int cols, int k, double f, int* piv) {
  if (k <= 0 || k >= cols) return 0;
  int swaps = 0;
  double* v = (double*)malloc(sizeof(double) * (size_t)rows);
  for (;;) {
    /* the largest |T_tc| > f; ties -> the lowest original column index, then the lowest t */
    double best = -1.0;
    int bi = -1, bj = -1;
    for (int c = k; c < cols; c++)
      for (int t = 0; t < k; t++) {
        double a = fabs(Mout[t + (int64_t)rows * c]);
        if (a > f && (a > best || (a == best && (piv[c] < piv[bj] || (piv[c] == piv[bj] && t < bi))))) {
          best = a;
          bi = t;
          bj = c;
        }
      }
    if (bj < 0 || swaps >= 64 * k) break;
    int tp = piv[bi];
    piv[bi] = piv[bj];
    piv[bj] = tp;
    swaps++;
    /* refactor: the columns in the new order, QR of the first k, T = R11^{-1} R12 */
    for (int c = 0; c < cols; c++) memcpy(Mout + (int64_t)rows * c, M0 + (int64_t)rows * piv[c], sizeof(double) * (size_t)rows);
    for (int t = 0; t < k; t++) {
      double s2 = 0.0;
      for (int i = t; i < rows; i++) s2 = s2 + Mout[i + (int64_t)rows * t] * Mout[i + (int64_t)rows * t];
      double nrm = sqrt(s2);
      double x0 = Mout[t + (int64_t)rows * t];
      double alpha = x0 >= 0.0 ? -nrm : nrm;
      double vtv = 0.0;
      for (int i = t; i < rows; i++) v[i] = Mout[i + (int64_t)rows * t];
      v[t] = x0 - alpha;
      for (int i = t; i < rows; i++) vtv = vtv + v[i] * v[i];
      Mout[t + (int64_t)rows * t] = alpha;
      for (int i = t + 1; i < rows; i++) Mout[i + (int64_t)rows * t] = 0.0;
      if (vtv > 0.0)
        for (int j = t + 1; j < cols; j++) {
          double* col = Mout + (int64_t)rows * j;
          double sd = 0.0;
          for (int i = t; i < rows; i++) sd = sd + v[i] * col[i];
          double fct = 2.0 * sd / vtv;
          for (int i = t; i < rows; i++) col[i] = col[i] - fct * v[i];
        }
    }
    for (int c = k; c < cols; c++) {
      double* col = Mout + (int64_t)rows * c;
      for (int i = k - 1; i >= 0; i--) {
        double sd = col[i];
        for (int l = i + 1; l < k; l++) sd = sd - Mout[i + (int64_t)rows * l] * col[l];
        col[i] = sd / Mout[i + (int64_t)rows * i];
      }
    }
  }
  free(v);
  return swaps;
}

/* Interpolative decomposition of A (nx x ny, row-major: A[b*ny + a]) by CPQR of A^T, optionally
 * refined by SRRQR swaps (f > 0; orc_id = f 0):
 *   A ~= U A[skel, :],  U (nx x k, column-major) has U[piv[t], t] = 1 (t < k) and
 *   U[piv[c], t] = T[t, c] for c >= k  (Eq.(4.1): K_{X Y*} = P [I; G] K_{X^ Y*}).
 * skel[0:k] = piv[0:k] (positions into the rows of A, pivot order).  Returns k.             */
int orc_id_srrqr(const double* A, int nx, int ny, double tol, double f, int* skel, double* U, int* nswaps) {
  double* M = (double*)malloc(sizeof(double) * (size_t)nx * (size_t)ny + 8);
  int* piv = (int*)malloc(sizeof(int) * (size_t)(nx > 0 ? nx : 1));
  for (int b = 0; b < nx; b++)
    for (int a = 0; a < ny; a++) M[a + (int64_t)ny * b] = A[(int64_t)b * ny + a];
  double* M0 = NULL;
  if (f > 0.0) {
    M0 = (double*)malloc(sizeof(double) * (size_t)nx * (size_t)ny + 8);
    memcpy(M0, M, sizeof(double) * (size_t)nx * (size_t)ny);
  }
  int k = orc_cpqr(M, ny, nx, tol, piv);
  int sw = f > 0.0 ? orc_srrqr_swaps(M0, M, ny, nx, k, f, piv) : 0;
  if (nswaps) *nswaps = sw;
  free(M0);
  for (int t = 0; t < k; t++) skel[t] = piv[t];
  if (U) {
    memset(U, 0, sizeof(double) * (size_t)nx * (size_t)k);
    for (int t = 0; t < k; t++) U[piv[t] + (int64_t)nx * t] = 1.0;
    for (int c = k; c < nx; c++)
      for (int t = 0; t < k; t++) U[piv[c] + (int64_t)nx * t] = M[t + (int64_t)ny * c];
  }
  free(M);
  free(piv);
  return k;
}

int orc_id(const double* A, int nx, int ny, double tol, int* skel, double* U) {
  return orc_id_srrqr(A, nx, ny, tol, 0.0, skel, U, NULL);
}

/* ------------------------------------------------------------------------------------------ */
/* the oracle's H^2 object                                                                     */
/* ------------------------------------------------------------------------------------------ */

typedef struct orc_h2 {
  int n, d, q;
  double tau;
  /* A */
  double W, rlo[ORC_MAXD];
  int L;
  int* perm;     /* tree position -> original index */
  double* X;     /* tree-order coordinates, point-major */
  uint64_t* key; /* sorted Morton keys */
  int nnodes, depth;
  int* lvl_start; /* nodes of level l: [lvl_start[l], lvl_start[l+1]) */
  int *level, *begin, *end, *parent, *first_child, *nchild, *is_leaf;
  int64_t* cell; /* [i*d + k], integer cell coordinates at the node's own level */
  /* B */
  int64_t *il_off, *nf_off;
  int *il_idx, *nf_idx;
  /* D */
  int r;
  int reduct; /* DataReduct: 0 volume-based (C1), 1 farthest point sampling (C6), 2 surface-based (C7) */
  int **xs, **ys;
  int *xs_n, *ys_n;
  int64_t max_S, max_T;
  /* F */
  int kid;
  double kparam, id_tol;
  int* k;
  int** sk;       /* skeleton X^_i, tree indices in pivot order */
  int* xbar_n;    /* |Xbar_i| */
  double** U;     /* |Xbar_i| x k_i, column-major */
  int* child_off; /* offset of node's skeleton rows inside its parent's Xbar */
  int calib_r[64]; /* E: per-level r of the last orc_calibrate (0 = level without an admissible pair) */
  /* non-symmetric path (Algorithm 2 lines 4-12 with separate row / column sets): the
   * column bases V_i (W = stacked V of the children), skeletons X^_i^(col), ranks */
  int nonsym;
  double srrqr_f; /* > 0: SRRQR swaps until ||G||_max <= srrqr_f; 0: plain CPQR (F1) */
  int64_t srrqr_swaps;
  int *k_col, **sk_col, *xbar_col_n, *child_off_col;
  double** V;
  double t_stage[8];
} orc_h2;

/* ------------------------------------------------------------------------------------------ */
/* A. partition (readings A1-A4)                                           */
/* ------------------------------------------------------------------------------------------ */

typedef struct {
  uint64_t key;
  int idx;
} keyidx;

static int cmp_keyidx(const void* a, const void* b) {
  const keyidx* x = (const keyidx*)a;
  const keyidx* y = (const keyidx*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

static void push_node(orc_h2* h, int* cap, int lvl, int b, int e, int par) {
  if (h->nnodes == *cap) {
    *cap = *cap * 2 + 16;
    h->level = realloc(h->level, sizeof(int) * (size_t)*cap);
    h->begin = realloc(h->begin, sizeof(int) * (size_t)*cap);
    h->end = realloc(h->end, sizeof(int) * (size_t)*cap);
    h->parent = realloc(h->parent, sizeof(int) * (size_t)*cap);
    h->first_child = realloc(h->first_child, sizeof(int) * (size_t)*cap);
    h->nchild = realloc(h->nchild, sizeof(int) * (size_t)*cap);
    h->is_leaf = realloc(h->is_leaf, sizeof(int) * (size_t)*cap);
  }
  int i = h->nnodes++;
  h->level[i] = lvl;
  h->begin[i] = b;
  h->end[i] = e;
  h->parent[i] = par;
  h->first_child[i] = -1;
  h->nchild[i] = 0;
  h->is_leaf[i] = 1;
}

static void partition(orc_h2* h, const double* pts) {
  int n = h->n, d = h->d;
  double lo[ORC_MAXD], hi[ORC_MAXD];
  for (int c = 0; c < d; c++) lo[c] = hi[c] = pts[c];
  for (int i = 1; i < n; i++)
    for (int c = 0; c < d; c++) {
      double v = pts[(int64_t)i * d + c];
      if (v < lo[c]) lo[c] = v;
      if (v > hi[c]) hi[c] = v;
    }
  /* root box: cube of width W = max extent, centred on the bbox centre (A1) */
  double W = 0.0;
  for (int c = 0; c < d; c++)
    if (hi[c] - lo[c] > W) W = hi[c] - lo[c];
  h->W = W;
  for (int c = 0; c < d; c++) h->rlo[c] = (lo[c] + hi[c]) * 0.5 - W * 0.5;
  h->L = 63 / d < 30 ? 63 / d : 30; /* A3 */
  if (W == 0.0) h->L = 0;           /* all points identical: one root leaf */
  int L = h->L;
  keyidx* ki = (keyidx*)malloc(sizeof(keyidx) * (size_t)n);
  double s = L > 0 ? ldexp(1.0, L) / W : 0.0;
  int64_t cmax = L > 0 ? ((int64_t)1 << L) - 1 : 0;
  for (int i = 0; i < n; i++) {
    uint64_t key = 0;
    for (int c = 0; c < d && L > 0; c++) {
      /* half-open cells defined by quantisation, clamped at the top (A2) */
      double f = floor((pts[(int64_t)i * d + c] - h->rlo[c]) * s);
      int64_t cell = f < 0.0 ? 0 : (f > (double)cmax ? cmax : (int64_t)f);
      for (int b = 0; b < L; b++) key |= (uint64_t)((cell >> b) & 1) << (d * b + c);
    }
    ki[i].key = key;
    ki[i].idx = i;
  }
  /* stable order by (key, original index) (A4) */
  qsort(ki, (size_t)n, sizeof(keyidx), cmp_keyidx);
  h->perm = (int*)malloc(sizeof(int) * (size_t)n);
  h->key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  h->X = (double*)malloc(sizeof(double) * (size_t)n * (size_t)d);
  for (int t = 0; t < n; t++) {
    h->perm[t] = ki[t].idx;
    h->key[t] = ki[t].key;
    memcpy(h->X + (int64_t)t * d, pts + (int64_t)ki[t].idx * d, sizeof(double) * (size_t)d);
  }
  free(ki);

  /* level-order node ids; a node splits iff count > q and level < L; empty children do not
   * exist; children of a node are the maximal runs of equal key prefix at the next level   */
  int cap = 0;
  h->nnodes = 0;
  push_node(h, &cap, 0, 0, n, -1);
  h->is_leaf[0] = !(n > h->q && L > 0);
  int lcap = 64;
  h->lvl_start = (int*)malloc(sizeof(int) * (size_t)lcap);
  h->lvl_start[0] = 0;
  int l = 0, ls = 0, le = 1;
  while (1) {
    h->lvl_start[l + 1] = le;
    int any = 0;
    for (int i = ls; i < le; i++) {
      if (h->is_leaf[i]) continue;
      int sh = d * (L - l - 1);
      int p = h->begin[i];
      h->first_child[i] = h->nnodes;
      while (p < h->end[i]) {
        uint64_t g = h->key[p] >> sh;
        int e = p;
        while (e < h->end[i] && (h->key[e] >> sh) == g) e++;
        push_node(h, &cap, l + 1, p, e, i);
        int c = h->nnodes - 1;
        h->is_leaf[c] = !((e - p) > h->q && l + 1 < L);
        h->nchild[i]++;
        p = e;
        any = 1;
      }
    }
    if (!any) break;
    ls = le;
    le = h->nnodes;
    l++;
    if (l + 2 >= lcap) {
      lcap *= 2;
      h->lvl_start = realloc(h->lvl_start, sizeof(int) * (size_t)lcap);
    }
  }
  h->depth = l;
  h->lvl_start[l + 1] = h->nnodes;
  /* integer cell coordinates of each node at its own level (de-interleaved key prefix) */
  h->cell = (int64_t*)malloc(sizeof(int64_t) * (size_t)h->nnodes * (size_t)d);
  for (int i = 0; i < h->nnodes; i++) {
    int li = h->level[i];
    uint64_t pre = L > 0 ? h->key[h->begin[i]] >> (d * (L - li)) : 0;
    if (li == 0) pre = 0;
    for (int c = 0; c < d; c++) {
      int64_t v = 0;
      for (int b = 0; b < li; b++) v |= (int64_t)((pre >> (d * b + c)) & 1) << b;
      h->cell[(int64_t)i * d + c] = v;
    }
  }
}

/* ------------------------------------------------------------------------------------------ */
/* B. admissibility Eq.(2.1) and lists (readings B1-B4)                             */
/* ------------------------------------------------------------------------------------------ */

/* diam(X_i) + diam(X_j) <= 2 tau |a_i - a_j| with diam = cell diagonal sqrt(d) w (B1), equality
 * admissible (B2).  Units: the finer node's cell width; doubled centres A = (2c+1) w, so the test
 * is  d (w_i + w_j)^2 <= tau^2 |A_i - A_j|^2, evaluated as  fl(d * fl(w*w)) <= fl(fl(tau*tau) * S),
 * S = sum_k fl(dA_k * dA_k) accumulated in k order.  All integers are exact below 2^53.       */
int orc_admissible(const int64_t* ci, int li, const int64_t* cj, int lj, int d, double tau) {
  int lf = li > lj ? li : lj;
  int64_t wi = (int64_t)1 << (lf - li), wj = (int64_t)1 << (lf - lj);
  double S = 0.0;
  for (int c = 0; c < d; c++) {
    int64_t Ai = (2 * ci[c] + 1) * wi;
    int64_t Aj = (2 * cj[c] + 1) * wj;
    double df = (double)(Ai - Aj);
    S = S + df * df;
  }
  double w = (double)(wi + wj);
  double lhs = (double)d * (w * w);
  double rhs = (tau * tau) * S;
  return lhs <= rhs;
}

typedef struct {
  uint64_t* a;
  int64_t n, cap;
} u64vec;

static void u64_push(u64vec* v, uint64_t x) {
  if (v->n == v->cap) {
    v->cap = v->cap * 2 + 1024;
    v->a = realloc(v->a, sizeof(uint64_t) * (size_t)v->cap);
  }
  v->a[v->n++] = x;
}

/* dual traversal from (root, root) (B3, B4):
 *   admissible -> j in IL(i);  both leaves -> j in NF(i);
 *   otherwise expand the non-leaf side (both sides when neither is a leaf).                   */
static void traverse(const orc_h2* h, int i, int j, u64vec* il, u64vec* nf) {
  const int d = h->d;
  if (orc_admissible(h->cell + (int64_t)i * d, h->level[i], h->cell + (int64_t)j * d, h->level[j],
                     d, h->tau)) {
    u64_push(il, ((uint64_t)i << 32) | (uint32_t)j);
    return;
  }
  int li = h->is_leaf[i], lj = h->is_leaf[j];
  if (li && lj) {
    u64_push(nf, ((uint64_t)i << 32) | (uint32_t)j);
  } else if (li) {
    for (int c = 0; c < h->nchild[j]; c++) traverse(h, i, h->first_child[j] + c, il, nf);
  } else if (lj) {
    for (int c = 0; c < h->nchild[i]; c++) traverse(h, h->first_child[i] + c, j, il, nf);
  } else {
    for (int a = 0; a < h->nchild[i]; a++)
      for (int b = 0; b < h->nchild[j]; b++)
        traverse(h, h->first_child[i] + a, h->first_child[j] + b, il, nf);
  }
}

static void to_csr(u64vec* v, int nnodes, int64_t** off, int** idx) {
  qsort(v->a, (size_t)v->n, sizeof(uint64_t), cmp_u64);
  *off = (int64_t*)calloc((size_t)nnodes + 1, sizeof(int64_t));
  *idx = (int*)malloc(sizeof(int) * (size_t)(v->n > 0 ? v->n : 1));
  for (int64_t e = 0; e < v->n; e++) {
    (*off)[(v->a[e] >> 32) + 1]++;
    (*idx)[e] = (int)(uint32_t)v->a[e];
  }
  for (int i = 0; i < nnodes; i++) (*off)[i + 1] += (*off)[i];
}

static void build_lists(orc_h2* h) {
  u64vec il = {0}, nf = {0};
  traverse(h, 0, 0, &il, &nf);
  to_csr(&il, h->nnodes, &h->il_off, &h->il_idx);
  to_csr(&nf, h->nnodes, &h->nf_off, &h->nf_idx);
  free(il.a);
  free(nf.a);
}

orc_h2* orc_new(const double* pts, int n, int d, int q, double tau) {
  if (n < 1 || d < 1 || d > ORC_MAXD || q < 1 || !(tau > 0.0)) return NULL;
  orc_h2* h = (orc_h2*)calloc(1, sizeof(orc_h2));
  h->n = n;
  h->d = d;
  h->q = q;
  h->tau = tau;
  double t0 = wall();
  partition(h, pts);
  double t1 = wall();
  build_lists(h);
  h->t_stage[0] = t1 - t0;
  h->t_stage[1] = wall() - t1;
  return h;
}

/* ------------------------------------------------------------------------------------------ */
/* D. HiDR, Algorithm 1 (readings D1, D2)                                           */
/* ------------------------------------------------------------------------------------------ */

static void free_lists2(int** a, int n) {
  if (!a) return;
  for (int i = 0; i < n; i++) free(a[i]);
  free(a);
}

/* Surface-based DataReduct, PAPER §3.3: reference points on three ellipsoids centred
 * at the centre of the tight bounding box, principal semi-axes gamma times the box width in each
 * dimension, gamma = 0.3, 0.6, 1.2 (the values of the paper's runs); for every reference point the
 * nearest point of S (C4 distances, ties -> lowest index); sorted and de-duplicated (C5).
 * Reading C7: d = 2 or 3 only.  The k reference points are dealt round-robin to the ellipsoids
 * (ellipsoid e gets floor(k/3) + [e < k mod 3]); on an ellipsoid with M points, point j has the
 * unit direction (cos t, sin t), t = 2 pi j / M in 2-D, and the Fibonacci-sphere direction
 * (rho cos f, rho sin f, z), z = 1 - (2j+1)/M, rho = sqrt(1 - z^2), f = j pi (3 - sqrt 5) in 3-D;
 * the reference point is c_c + (gamma w_c) u_c with c the box centre lo + 0.5 (hi - lo), w = hi - lo.
 * Returns |out| <= k, or -1 for d outside {2, 3}.                                               */
static const double kSurfGamma[3] = {0.3, 0.6, 1.2};

int orc_surface_dirs(int d, int k, double* u) { /* u[(e*k + j)*d + c]; returns the count */
  if (d != 2 && d != 3) return -1;
  int cnt = 0;
  for (int e = 0; e < 3; e++) {
    const int M = k / 3 + (e < k % 3 ? 1 : 0);
    for (int j = 0; j < M; j++) {
      double* v = u + (int64_t)cnt * (d + 1);
      if (d == 2) {
        const double t = 2.0 * M_PI * (double)j / (double)M;
        v[0] = cos(t);
        v[1] = sin(t);
      } else {
        const double z = 1.0 - (2.0 * (double)j + 1.0) / (double)M;
        const double rho = sqrt(1.0 - z * z);
        const double f = (double)j * (M_PI * (3.0 - sqrt(5.0)));
        v[0] = rho * cos(f);
        v[1] = rho * sin(f);
        v[2] = z;
      }
      v[d] = kSurfGamma[e];
      cnt++;
    }
  }
  return cnt;
}

int orc_surface(const double* X, int d, const int* S, int ns, int k, int* out) {
  if (d != 2 && d != 3) return -1;
  if (ns <= 0) return 0;
  if (ns <= k) {
    memcpy(out, S, sizeof(int) * (size_t)ns);
    return sort_unique(out, ns);
  }
  double lo[ORC_MAXD], hi[ORC_MAXD], cen[ORC_MAXD], w[ORC_MAXD];
  for (int c = 0; c < d; c++) lo[c] = hi[c] = X[(int64_t)S[0] * d + c];
  for (int s = 1; s < ns; s++)
    for (int c = 0; c < d; c++) {
      double v = X[(int64_t)S[s] * d + c];
      if (v < lo[c]) lo[c] = v;
      if (v > hi[c]) hi[c] = v;
    }
  for (int c = 0; c < d; c++) {
    w[c] = hi[c] - lo[c];
    cen[c] = lo[c] + 0.5 * (w[c] / 1.0);
  }
  double* u = (double*)malloc(sizeof(double) * (size_t)k * (d + 1));
  const int nq = orc_surface_dirs(d, k, u);
  int cnt = 0;
  for (int g = 0; g < nq; g++) {
    const double* v = u + (int64_t)g * (d + 1);
    double q[ORC_MAXD];
    for (int c = 0; c < d; c++) q[c] = cen[c] + (v[d] * w[c]) * v[c];
    double best = INFINITY;
    int bi = INT_MAX;
    for (int s = 0; s < ns; s++) {
      double dist = sqdist(X + (int64_t)S[s] * d, q, d);
      if (dist < best || (dist == best && S[s] < bi)) {
        best = dist;
        bi = S[s];
      }
    }
    out[cnt++] = bi;
  }
  free(u);
  return sort_unique(out, cnt);
}

/* the DataReduct of HiDR (readings C1, C6) */
static int orc_reduct(const orc_h2* h, const int* S, int ns, int k, int* out) {
  if (h->reduct == 1) return orc_fps(h->X, h->d, S, ns, k, out);
  if (h->reduct == 2) return orc_surface(h->X, h->d, S, ns, k, out);
  return orc_vol(h->X, h->d, S, ns, k, out);
}

void orc_set_reduct(orc_h2* h, int reduct) { h->reduct = reduct; }
/* 1: build row AND column bases (Algorithm 2 line 11, both getBasis calls), blocks for all ordered
 * pairs; required for a non-symmetric kernel, allowed for a symmetric one (then V = U exactly) */
void orc_set_nonsym(orc_h2* h, int nonsym) { h->nonsym = nonsym; }
void orc_set_srrqr(orc_h2* h, double f) { h->srrqr_f = f; }
int64_t orc_srrqr_count(const orc_h2* h) { return h->srrqr_swaps; }

int orc_hidr(orc_h2* h, int r) {
  if (r < 1) return -1;
  double t0 = wall();
  int nn = h->nnodes;
  free_lists2(h->xs, nn);
  free_lists2(h->ys, nn);
  free(h->xs_n);
  free(h->ys_n);
  h->r = r;
  h->xs = (int**)calloc((size_t)nn, sizeof(int*));
  h->ys = (int**)calloc((size_t)nn, sizeof(int*));
  h->xs_n = (int*)calloc((size_t)nn, sizeof(int));
  h->ys_n = (int*)calloc((size_t)nn, sizeof(int));
  int64_t maxS = 0, maxT = 0;
  /* bottom-up (Alg.1 lines 7-13): S_i = X_i at leaves, S_p = U_c X_c^*; X_i^* = Vol(S_i, r1) */
  for (int l = h->depth; l >= 0; l--) {
#pragma omp parallel for schedule(dynamic, 1) reduction(max : maxS)
    for (int i = h->lvl_start[l]; i < h->lvl_start[l + 1]; i++) {
      int ns = 0;
      if (h->is_leaf[i]) ns = h->end[i] - h->begin[i];
      else
        for (int c = 0; c < h->nchild[i]; c++) ns += h->xs_n[h->first_child[i] + c];
      int* S = (int*)malloc(sizeof(int) * (size_t)(ns > 0 ? ns : 1));
      if (h->is_leaf[i]) {
        for (int t = 0; t < ns; t++) S[t] = h->begin[i] + t;
      } else {
        int o = 0;
        for (int c = 0; c < h->nchild[i]; c++) {
          int ch = h->first_child[i] + c;
          memcpy(S + o, h->xs[ch], sizeof(int) * (size_t)h->xs_n[ch]);
          o += h->xs_n[ch];
        }
      }
      if (ns > maxS) maxS = ns;
      int* out = (int*)malloc(sizeof(int) * (size_t)(ns < r ? (ns > 0 ? ns : 1) : r));
      h->xs_n[i] = orc_reduct(h, S, ns, r, out);
      h->xs[i] = out;
      free(S);
    }
  }
  /* top-down (Alg.1 lines 14-21): T_i = Y_p^* U (U_{j in IL(i)} X_j^*), Y_root^* = {} (D1);
   * Y_i^* = Vol(T_i, r2), or {} if T_i = {} (D2: T_i = Y_p^* when IL(i) is empty)            */
  h->ys[0] = (int*)malloc(sizeof(int));
  h->ys_n[0] = 0;
  for (int l = 1; l <= h->depth; l++) {
#pragma omp parallel for schedule(dynamic, 1) reduction(max : maxT)
    for (int i = h->lvl_start[l]; i < h->lvl_start[l + 1]; i++) {
      int p = h->parent[i];
      int64_t nt = h->ys_n[p];
      for (int64_t e = h->il_off[i]; e < h->il_off[i + 1]; e++) nt += h->xs_n[h->il_idx[e]];
      int* T = (int*)malloc(sizeof(int) * (size_t)(nt > 0 ? nt : 1));
      int o = 0;
      memcpy(T, h->ys[p], sizeof(int) * (size_t)h->ys_n[p]);
      o += h->ys_n[p];
      for (int64_t e = h->il_off[i]; e < h->il_off[i + 1]; e++) {
        int j = h->il_idx[e];
        memcpy(T + o, h->xs[j], sizeof(int) * (size_t)h->xs_n[j]);
        o += h->xs_n[j];
      }
      int nu = sort_unique(T, o); /* set union */
      if (nu > maxT) maxT = nu;
      int* out = (int*)malloc(sizeof(int) * (size_t)(nu < r ? (nu > 0 ? nu : 1) : r));
      h->ys_n[i] = orc_reduct(h, T, nu, r, out);
      h->ys[i] = out;
      free(T);
    }
  }
  h->max_S = maxS;
  h->max_T = maxT;
  h->t_stage[3] = wall() - t0;
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* E. calibration of r1 = r2 = r from epsilon (Alg.2 line 2; readings E1-E6)        */
/* ------------------------------------------------------------------------------------------ */

/* SplitMix64 (E6): portable counter-based generator both sides implement from DESIGN.md */
static uint64_t splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

#define ORC_CAL_NPTS 256
#define ORC_CAL_SEED 2206018850ULL

/* The random well-separated point sets of one calibration level (E4, E6): Z1 = 256 points in
 * [0,w]^d, then Z2 = 256 points in [0,w]^d shifted by w/tau in every coordinate, drawn with
 * SplitMix64 from seed 2206018850 + level, point-major, coordinate = ((x >> 11) 2^-53) w (+ w/tau). */
void orc_calib_points(int d, double tau, double w, int level, double* Z1, double* Z2) {
  const int N = ORC_CAL_NPTS;
  uint64_t st = ORC_CAL_SEED + (uint64_t)level;
  for (int i = 0; i < N * d; i++) Z1[i] = (double)(splitmix64(&st) >> 11) * 0x1.0p-53 * w;
  double shift = w / tau;
  for (int i = 0; i < N * d; i++) Z2[i] = (double)(splitmix64(&st) >> 11) * 0x1.0p-53 * w + shift;
}

/* calibration trial at box width w and grid m: returns the relative Frobenius error e (E5) of
 * the ID built from K(Z1, Z2*) applied to the full K(Z1, Z2); *G_out = m^d.  The optional
 * outputs expose the trial for its pins: *k_out the ID rank, skel_out[0:k] the skeleton rows
 * (indices into Z1, pivot order), sel_out[0:*ns_out] the columns Z2* (indices into Z2).       */
/* kappa(x, y), or kappa^T(x, y) = kappa(y, x) when tr (the column-basis orientation of a
 * non-symmetric kernel, Algorithm 2 line 11: getBasis(K_{Y X}^T)) */
static double kern_tr(int kid, double p, const double* x, const double* y, int d, int tr) {
  return tr ? orc_kernel(kid, p, y, x, d) : orc_kernel(kid, p, x, y, d);
}

static double calib_trial_impl(int d, int kid, double p, double eps, double tau, double w, int level, int m,
                               int tr, int64_t* G_out, int* k_out, int* skel_out, int* sel_out, int* ns_out) {
  const int N = ORC_CAL_NPTS;
  double* Z1 = (double*)malloc(sizeof(double) * (size_t)N * (size_t)d);
  double* Z2 = (double*)malloc(sizeof(double) * (size_t)N * (size_t)d);
  orc_calib_points(d, tau, w, level, Z1, Z2);
  int64_t G = ipow_sat(m, d);
  *G_out = G;
  int idx[ORC_CAL_NPTS], sel[ORC_CAL_NPTS];
  for (int i = 0; i < N; i++) idx[i] = i;
  int ns;
  if (G >= N) { /* pass-through: Z2* = Z2 */
    ns = N;
    for (int i = 0; i < N; i++) sel[i] = i;
  } else {
    ns = orc_vol(Z2, d, idx, N, (int)G, sel);
  }
  /* A = K(Z1, Z2*) (N x ns, row-major); ID with inner tolerance 1e-3 eps (E3) */
  double* A = (double*)malloc(sizeof(double) * (size_t)N * (size_t)ns);
  for (int b = 0; b < N; b++)
    for (int a = 0; a < ns; a++)
      A[(int64_t)b * ns + a] = kern_tr(kid, p, Z1 + (int64_t)b * d, Z2 + (int64_t)sel[a] * d, d, tr);
  int skel[ORC_CAL_NPTS];
  double* U = (double*)malloc(sizeof(double) * (size_t)N * (size_t)(ns > 0 ? ns : 1));
  int k = orc_id(A, N, ns, 1e-3 * eps, skel, U);
  /* e = ||K(Z1,Z2) - U K(Z1[skel], Z2)||_F / ||K(Z1,Z2)||_F */
  double num = 0.0, den = 0.0;
  for (int b = 0; b < N; b++)
    for (int c = 0; c < N; c++) {
      double kv = kern_tr(kid, p, Z1 + (int64_t)b * d, Z2 + (int64_t)c * d, d, tr);
      double ap = 0.0;
      for (int t = 0; t < k; t++)
        ap = ap + U[b + (int64_t)N * t] * kern_tr(kid, p, Z1 + (int64_t)skel[t] * d, Z2 + (int64_t)c * d, d, tr);
      double df = kv - ap;
      num = num + df * df;
      den = den + kv * kv;
    }
  if (k_out) *k_out = k;
  if (skel_out) memcpy(skel_out, skel, sizeof(int) * (size_t)k);
  if (sel_out) memcpy(sel_out, sel, sizeof(int) * (size_t)ns);
  if (ns_out) *ns_out = ns;
  free(Z1);
  free(Z2);
  free(A);
  free(U);
  return den > 0.0 ? sqrt(num) / sqrt(den) : 0.0;
}

double orc_calib_trial_ex(int d, int kid, double p, double eps, double tau, double w, int level,
                          int m, int64_t* G_out, int* k_out, int* skel_out, int* sel_out, int* ns_out) {
  return calib_trial_impl(d, kid, p, eps, tau, w, level, m, 0, G_out, k_out, skel_out, sel_out, ns_out);
}

double orc_calib_trial(int d, int kid, double p, double eps, double tau, double w, int level,
                       int m, int64_t* G_out) {
  return calib_trial_impl(d, kid, p, eps, tau, w, level, m, 0, G_out, NULL, NULL, NULL, NULL);
}

/* r for one level and orientation: first m = 1, 2, ... with e < 1e-2 eps, or m^d >= 256 (E2) */
int orc_calib_level_tr(int d, int kid, double p, double eps, double tau, double w, int level, int tr) {
  for (int m = 1;; m++) {
    int64_t G;
    double e = calib_trial_impl(d, kid, p, eps, tau, w, level, m, tr, &G, NULL, NULL, NULL, NULL);
    if (e < 1e-2 * eps || G >= ORC_CAL_NPTS) return (int)G;
  }
}

int orc_calib_level(int d, int kid, double p, double eps, double tau, double w, int level) {
  return orc_calib_level_tr(d, kid, p, eps, tau, w, level, 0);
}

/* r = max over levels holding an admissible pair of that level's r (E4); 1 if none */
int orc_calibrate(orc_h2* h, int kid, double p, double eps) {
  double t0 = wall();
  int r = 1;
  int* has = (int*)calloc((size_t)h->depth + 1, sizeof(int));
  for (int i = 0; i < h->nnodes; i++)
    if (h->il_off[i + 1] > h->il_off[i]) has[h->level[i]] = 1;
  int rl[64] = {0};
#pragma omp parallel for schedule(dynamic, 1)
  for (int l = 0; l <= h->depth; l++)
    if (has[l]) {
      rl[l] = orc_calib_level(h->d, kid, p, eps, h->tau, ldexp(h->W, -l), l);
      if (h->nonsym) { /* reading E7: the column bases need the same accuracy: max of both orientations */
        int rt = orc_calib_level_tr(h->d, kid, p, eps, h->tau, ldexp(h->W, -l), l, 1);
        if (rt > rl[l]) rl[l] = rt;
      }
    }
  for (int l = 0; l <= h->depth; l++)
    if (has[l] && rl[l] > r) r = rl[l];
  for (int l = 0; l < 64; l++) h->calib_r[l] = l <= h->depth && has[l] ? rl[l] : 0;
  free(has);
  h->t_stage[2] = wall() - t0;
  return r;
}

/* ------------------------------------------------------------------------------------------ */
/* F. bottom-up ID sweep (Algorithm 2 lines 10-13; readings F1-F6)                  */
/* ------------------------------------------------------------------------------------------ */

/* One bottom-up getBasis sweep (Algorithm 2 lines 10-12): for every non-root node with
 * Y_i^* != {}, Xbar_i = X_i at a leaf or the children's skeletons (child order); A = kappa(Xbar_i,
 * Y_i^*) (tr = 0: the row bases U_i, getBasis(K_{Xbar Y*})) or kappa(Y_i^*, Xbar_i)^T (tr = 1: the
 * column bases V_i, getBasis(K_{Y* Xbar}^T)); ID -> k, skeleton, U (|Xbar| x k). */
static void id_sweep_one(orc_h2* h, int kid, double p, double id_tol, int tr, int* K, int** SK, double** UU,
                         int* XBN, int* CHO) {
  int d = h->d;
  for (int l = h->depth; l >= 1; l--) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int i = h->lvl_start[l]; i < h->lvl_start[l + 1]; i++) {
      if (h->ys_n[i] == 0) continue; /* F4: empty farfield, no basis */
      /* Xbar_i = X_i at a leaf; concatenation of the children's X^ (child order) otherwise */
      int nx = 0;
      if (h->is_leaf[i]) nx = h->end[i] - h->begin[i];
      else
        for (int c = 0; c < h->nchild[i]; c++) nx += K[h->first_child[i] + c];
      XBN[i] = nx;
      if (nx == 0) continue;
      int* Xb = (int*)malloc(sizeof(int) * (size_t)nx);
      if (h->is_leaf[i]) {
        for (int t = 0; t < nx; t++) Xb[t] = h->begin[i] + t;
      } else {
        int o = 0;
        for (int c = 0; c < h->nchild[i]; c++) {
          int ch = h->first_child[i] + c;
          CHO[ch] = o;
          if (K[ch] > 0) memcpy(Xb + o, SK[ch], sizeof(int) * (size_t)K[ch]);
          o += K[ch];
        }
      }
      int ny = h->ys_n[i];
      /* A = K(Xbar_i, Y_i^*) (or its transposed-kernel version), columns in ascending Y^* order (F3) */
      double* A = (double*)malloc(sizeof(double) * (size_t)nx * (size_t)ny);
      for (int b = 0; b < nx; b++)
        for (int a = 0; a < ny; a++)
          A[(int64_t)b * ny + a] = kern_tr(kid, p, h->X + (int64_t)Xb[b] * d, h->X + (int64_t)h->ys[i][a] * d, d, tr);
      int* skel = (int*)malloc(sizeof(int) * (size_t)(nx < ny ? nx : ny));
      double* U = (double*)malloc(sizeof(double) * (size_t)nx * (size_t)(nx < ny ? nx : ny));
      int nsw = 0;
      int k = orc_id_srrqr(A, nx, ny, id_tol, h->srrqr_f, skel, U, &nsw);
      if (nsw) {
#pragma omp atomic
        h->srrqr_swaps += nsw;
      }
      int* sk = (int*)malloc(sizeof(int) * (size_t)(k > 0 ? k : 1));
      for (int t = 0; t < k; t++) sk[t] = Xb[skel[t]];
      K[i] = k;
      SK[i] = sk;
      UU[i] = U;
      free(skel);
      free(A);
      free(Xb);
    }
  }
}

static void free_basis(int nn, int** k, int*** sk, double*** U, int** xbn, int** cho) {
  if (*sk) free_lists2(*sk, nn);
  if (*U) {
    for (int i = 0; i < nn; i++) free((*U)[i]);
    free(*U);
  }
  free(*k);
  free(*xbn);
  free(*cho);
  *k = NULL;
  *sk = NULL;
  *U = NULL;
  *xbn = NULL;
  *cho = NULL;
}

int orc_id_sweep(orc_h2* h, int kid, double p, double id_tol) {
  if (!h->ys_n) return -1;
  double t0 = wall();
  int nn = h->nnodes;
  h->kid = kid;
  h->kparam = p;
  h->id_tol = id_tol;
  free_basis(nn, &h->k, &h->sk, &h->U, &h->xbar_n, &h->child_off);
  free_basis(nn, &h->k_col, &h->sk_col, &h->V, &h->xbar_col_n, &h->child_off_col);
  h->srrqr_swaps = 0;
  h->k = (int*)calloc((size_t)nn, sizeof(int));
  h->xbar_n = (int*)calloc((size_t)nn, sizeof(int));
  h->child_off = (int*)calloc((size_t)nn, sizeof(int));
  h->sk = (int**)calloc((size_t)nn, sizeof(int*));
  h->U = (double**)calloc((size_t)nn, sizeof(double*));
  id_sweep_one(h, kid, p, id_tol, 0, h->k, h->sk, h->U, h->xbar_n, h->child_off);
  if (h->nonsym) { /* the column bases: second getBasis of Algorithm 2 line 11 */
    h->k_col = (int*)calloc((size_t)nn, sizeof(int));
    h->xbar_col_n = (int*)calloc((size_t)nn, sizeof(int));
    h->child_off_col = (int*)calloc((size_t)nn, sizeof(int));
    h->sk_col = (int**)calloc((size_t)nn, sizeof(int*));
    h->V = (double**)calloc((size_t)nn, sizeof(double*));
    id_sweep_one(h, kid, p, id_tol, 1, h->k_col, h->sk_col, h->V, h->xbar_col_n, h->child_off_col);
  }
  h->t_stage[4] = wall() - t0;
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* G. block evaluation (Algorithm 2; reading G1): symmetric blocks stored once      */
/* ------------------------------------------------------------------------------------------ */

/* Evaluates every coupling block B_ij = K(X^_i, X^_j) (i<j in IL) and nearfield block
 * D_ij = K(X_i, X_j) (i<=j in NF) into `buf` (when non-NULL and large enough, consecutively,
 * row-major) and returns the entry count; `checksum` receives the sum of all entries.
 * Non-symmetric path: every ordered pair, B_ij = K(X^_i^(row), X^_j^(col)).        */
int64_t orc_fill(const orc_h2* h, double* buf, int64_t cap, double* checksum) {
  int d = h->d;
  int nn = h->nnodes;
  const int ns = h->nonsym;
  const int* kc = ns ? h->k_col : h->k;
  int* const* skc = ns ? h->sk_col : h->sk;
  int64_t* off = (int64_t*)calloc((size_t)nn + 1, sizeof(int64_t));
  for (int i = 0; i < nn; i++) {
    int64_t s = 0;
    for (int64_t e = h->il_off[i]; e < h->il_off[i + 1]; e++) {
      int j = h->il_idx[e];
      if (ns || j > i) s += (int64_t)h->k[i] * kc[j];
    }
    for (int64_t e = h->nf_off[i]; e < h->nf_off[i + 1]; e++) {
      int j = h->nf_idx[e];
      if (ns || j >= i) s += (int64_t)(h->end[i] - h->begin[i]) * (h->end[j] - h->begin[j]);
    }
    off[i + 1] = off[i] + s;
  }
  int64_t total = off[nn];
  int store = buf != NULL && cap >= total;
  double cs = 0.0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : cs)
  for (int i = 0; i < nn; i++) {
    int64_t o = off[i];
    for (int64_t e = h->il_off[i]; e < h->il_off[i + 1]; e++) {
      int j = h->il_idx[e];
      if (!ns && j <= i) continue;
      for (int a = 0; a < h->k[i]; a++)
        for (int b = 0; b < kc[j]; b++) {
          double v = orc_kernel(h->kid, h->kparam, h->X + (int64_t)h->sk[i][a] * d, h->X + (int64_t)skc[j][b] * d, d);
          if (store) buf[o] = v;
          o++;
          cs += v;
        }
    }
    for (int64_t e = h->nf_off[i]; e < h->nf_off[i + 1]; e++) {
      int j = h->nf_idx[e];
      if (!ns && j < i) continue;
      for (int a = h->begin[i]; a < h->end[i]; a++)
        for (int b = h->begin[j]; b < h->end[j]; b++) {
          double v = orc_kernel(h->kid, h->kparam, h->X + (int64_t)a * d, h->X + (int64_t)b * d, d);
          if (store) buf[o] = v;
          o++;
          cs += v;
        }
    }
  }
  free(off);
  if (checksum) *checksum = cs;
  return total;
}

/* ------------------------------------------------------------------------------------------ */
/* H. H^2 matvec with blocks evaluated on the fly, optionally on a subset of rows      */
/* ------------------------------------------------------------------------------------------ */

/* y = K~ x.  x in ORIGINAL order (length n).  rows == NULL: all rows, y has length n (original
 * order).  Otherwise y[r] = (K~ x)[rows[r]] for the given ORIGINAL row indices.
 * Passes: up (z^_leaf = U_i^T x_i, z^_p = sum_c R_c^T z^_c), coupling (y^_i += B_ij z^_j),
 * down (y^_c += R_c y^_p, y_i += U_i y^_i), nearfield (y_i += D_ij x_j).                     */
int orc_matvec_rows(const orc_h2* h, const double* x, const int64_t* rows, int64_t nrows, double* y) {
  if (!h->k) return -1;
  int n = h->n, d = h->d, nn = h->nnodes;
  double* xt = (double*)malloc(sizeof(double) * (size_t)n);
  for (int t = 0; t < n; t++) xt[t] = x[h->perm[t]];
  int* inv = (int*)malloc(sizeof(int) * (size_t)n);
  for (int t = 0; t < n; t++) inv[h->perm[t]] = t;
  /* nodes whose y^ is needed: every node (all rows) or the ancestors of the requested rows */
  char* need = (char*)calloc((size_t)nn, 1);
  char* rowmask = (char*)calloc((size_t)n, 1);
  int* leaf_of = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < nn; i++)
    if (h->is_leaf[i])
      for (int t = h->begin[i]; t < h->end[i]; t++) leaf_of[t] = i;
  if (!rows) {
    memset(need, 1, (size_t)nn);
    memset(rowmask, 1, (size_t)n);
  } else {
    for (int64_t r = 0; r < nrows; r++) {
      int t = inv[rows[r]];
      rowmask[t] = 1;
      for (int a = leaf_of[t]; a >= 0; a = h->parent[a]) need[a] = 1;
    }
  }
  double** zh = (double**)calloc((size_t)nn, sizeof(double*));
  double** yh = (double**)calloc((size_t)nn, sizeof(double*));
  for (int i = 0; i < nn; i++) {
    int kz = h->nonsym ? h->k_col[i] : h->k[i];
    zh[i] = (double*)calloc((size_t)(kz > 0 ? kz : 1), sizeof(double));
    yh[i] = (double*)calloc((size_t)(h->k[i] > 0 ? h->k[i] : 1), sizeof(double));
  }
  /* upward pass with the column bases: z^_i = V_i^T x_i (leaf), z^_p = sum_c W_c^T z^_c (V = U, W = R
   * for a symmetric build, reading F6) */
  const int ns = h->nonsym;
  const int* kc = ns ? h->k_col : h->k;
  int* const* skc = ns ? h->sk_col : h->sk;
  double* const* VV = ns ? h->V : h->U;
  const int* xbc = ns ? h->xbar_col_n : h->xbar_n;
  const int* choc = ns ? h->child_off_col : h->child_off;
  for (int l = h->depth; l >= 1; l--) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int i = h->lvl_start[l]; i < h->lvl_start[l + 1]; i++) {
      int k = kc[i];
      if (k == 0) continue;
      int nx = xbc[i];
      const double* U = VV[i];
      for (int c = 0; c < k; c++) {
        double s = 0.0;
        if (h->is_leaf[i]) {
          for (int a = 0; a < nx; a++) s = s + U[a + (int64_t)nx * c] * xt[h->begin[i] + a];
        } else {
          for (int cc = 0; cc < h->nchild[i]; cc++) {
            int ch = h->first_child[i] + cc;
            for (int a = 0; a < kc[ch]; a++) s = s + U[choc[ch] + a + (int64_t)nx * c] * zh[ch][a];
          }
        }
        zh[i][c] = s;
      }
    }
  }
  /* coupling pass over interaction lists, blocks K(X^_i, X^_j) on the fly */
#pragma omp parallel for schedule(dynamic, 4)
  for (int i = 0; i < nn; i++) {
    if (!need[i] || h->k[i] == 0) continue;
    for (int64_t e = h->il_off[i]; e < h->il_off[i + 1]; e++) {
      int j = h->il_idx[e];
      for (int a = 0; a < h->k[i]; a++) {
        double s = 0.0;
        for (int b = 0; b < kc[j]; b++)
          s = s + orc_kernel(h->kid, h->kparam, h->X + (int64_t)h->sk[i][a] * d, h->X + (int64_t)skc[j][b] * d, d) * zh[j][b];
        yh[i][a] = yh[i][a] + s;
      }
    }
  }
  double* yt = (double*)calloc((size_t)n, sizeof(double));
  /* downward pass */
  for (int l = 1; l <= h->depth; l++) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int i = h->lvl_start[l]; i < h->lvl_start[l + 1]; i++) {
      if (!need[i] || h->k[i] == 0) continue;
      int p = h->parent[i];
      if (p >= 0 && h->k[p] > 0) {
        int nxp = h->xbar_n[p];
        for (int a = 0; a < h->k[i]; a++) {
          double s = 0.0;
          for (int c = 0; c < h->k[p]; c++) s = s + h->U[p][h->child_off[i] + a + (int64_t)nxp * c] * yh[p][c];
          yh[i][a] = yh[i][a] + s;
        }
      }
      if (h->is_leaf[i]) {
        int nx = h->xbar_n[i];
        for (int a = 0; a < nx; a++) {
          int t = h->begin[i] + a;
          if (!rowmask[t]) continue;
          double s = 0.0;
          for (int c = 0; c < h->k[i]; c++) s = s + h->U[i][a + (int64_t)nx * c] * yh[i][c];
          yt[t] = yt[t] + s;
        }
      }
    }
  }
  /* nearfield pass, blocks K(X_i, X_j) on the fly */
#pragma omp parallel for schedule(dynamic, 4)
  for (int i = 0; i < nn; i++) {
    if (!h->is_leaf[i] || !need[i]) continue;
    for (int t = h->begin[i]; t < h->end[i]; t++) {
      if (!rowmask[t]) continue;
      double s = 0.0;
      for (int64_t e = h->nf_off[i]; e < h->nf_off[i + 1]; e++) {
        int j = h->nf_idx[e];
        for (int b = h->begin[j]; b < h->end[j]; b++)
          s = s + orc_kernel(h->kid, h->kparam, h->X + (int64_t)t * d, h->X + (int64_t)b * d, d) * xt[b];
      }
      yt[t] = yt[t] + s;
    }
  }
  if (!rows) {
    for (int t = 0; t < n; t++) y[h->perm[t]] = yt[t];
  } else {
    for (int64_t r = 0; r < nrows; r++) y[r] = yt[inv[rows[r]]];
  }
  for (int i = 0; i < nn; i++) {
    free(zh[i]);
    free(yh[i]);
  }
  free(zh);
  free(yh);
  free(yt);
  free(xt);
  free(inv);
  free(need);
  free(rowmask);
  free(leaf_of);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* I. exact dense rows of K x                                                      */
/* ------------------------------------------------------------------------------------------ */

/* out[r] = sum_j kappa(p_rows[r], p_j) x_j over all n points (original order, point-major). */
/* K(A_a, B_b) for point-major A (na x d) and B (nb x d): out[a nb + b] = kappa(A_a, B_b) (the
 * blocks of the interpolation baseline, oracle/interp.py: Eq. (2.2)).                */
void orc_kernel_block(int kid, double p, const double* A, int na, const double* B, int nb, int d, double* out) {
#pragma omp parallel for schedule(static) if ((int64_t)na * nb > 65536)
  for (int a = 0; a < na; a++)
    for (int b = 0; b < nb; b++) out[(int64_t)a * nb + b] = orc_kernel(kid, p, A + (int64_t)a * d, B + (int64_t)b * d, d);
}

void orc_dense_rows(const double* pts, int n, int d, int kid, double p, const double* x,
                    const int64_t* rows, int64_t nrows, double* out) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t r = 0; r < nrows; r++) {
    const double* xr = pts + rows[r] * d;
    double s = 0.0;
    for (int j = 0; j < n; j++) s = s + orc_kernel(kid, p, xr, pts + (int64_t)j * d, d) * x[j];
    out[r] = s;
  }
}

/* ------------------------------------------------------------------------------------------ */
/* export / info / free                                                                        */
/* ------------------------------------------------------------------------------------------ */

enum {
  ORC_PERM = 1, ORC_NODES = 2, ORC_CELLS = 3, ORC_IL_OFF = 4, ORC_IL_IDX = 5, ORC_NF_OFF = 6,
  ORC_NF_IDX = 7, ORC_XS_OFF = 8, ORC_XS_IDX = 9, ORC_YS_OFF = 10, ORC_YS_IDX = 11, ORC_K = 12,
  ORC_SK_OFF = 13, ORC_SK_IDX = 14, ORC_U_OFF = 15, ORC_U = 16, ORC_XBAR_N = 17, ORC_TREE_X = 18,
  ORC_CHILD_OFF = 19, ORC_K_COL = 20, ORC_SKC_OFF = 21, ORC_SKC_IDX = 22, ORC_V_OFF = 23, ORC_V = 24,
  ORC_XBARC_N = 25
};

static int64_t pack_lists(int** a, const int* cnt, int nn, int64_t* off, int* idx) {
  int64_t s = 0;
  for (int i = 0; i < nn; i++) {
    if (off) off[i] = s;
    if (idx && cnt[i] > 0) memcpy(idx + s, a[i], sizeof(int) * (size_t)cnt[i]);
    s += cnt[i];
  }
  if (off) off[nn] = s;
  return s;
}

/* Copies the requested array into buf when cap (in ELEMENTS) suffices; returns its element
 * count (or -1 when the stage that produces it has not run).                                 */
int64_t orc_export(const orc_h2* h, int what, void* buf, int64_t cap) {
  int nn = h->nnodes, n = h->n, d = h->d;
  int64_t need;
  switch (what) {
    case ORC_PERM:
      need = n;
      if (buf && cap >= need) memcpy(buf, h->perm, sizeof(int) * (size_t)n);
      return need;
    case ORC_NODES:
      need = (int64_t)nn * 7;
      if (buf && cap >= need) {
        int* o = (int*)buf;
        for (int i = 0; i < nn; i++) {
          o[i * 7 + 0] = h->level[i];
          o[i * 7 + 1] = h->begin[i];
          o[i * 7 + 2] = h->end[i];
          o[i * 7 + 3] = h->parent[i];
          o[i * 7 + 4] = h->first_child[i];
          o[i * 7 + 5] = h->nchild[i];
          o[i * 7 + 6] = h->is_leaf[i];
        }
      }
      return need;
    case ORC_CELLS:
      need = (int64_t)nn * d;
      if (buf && cap >= need) memcpy(buf, h->cell, sizeof(int64_t) * (size_t)need);
      return need;
    case ORC_TREE_X:
      need = (int64_t)n * d;
      if (buf && cap >= need) memcpy(buf, h->X, sizeof(double) * (size_t)need);
      return need;
    case ORC_IL_OFF:
    case ORC_NF_OFF:
      need = nn + 1;
      if (buf && cap >= need) memcpy(buf, what == ORC_IL_OFF ? h->il_off : h->nf_off, sizeof(int64_t) * (size_t)need);
      return need;
    case ORC_IL_IDX:
    case ORC_NF_IDX: {
      const int64_t* off = what == ORC_IL_IDX ? h->il_off : h->nf_off;
      need = off[nn];
      if (buf && cap >= need) memcpy(buf, what == ORC_IL_IDX ? h->il_idx : h->nf_idx, sizeof(int) * (size_t)need);
      return need;
    }
    case ORC_XS_OFF:
    case ORC_YS_OFF:
    case ORC_XS_IDX:
    case ORC_YS_IDX: {
      int** a = (what == ORC_XS_OFF || what == ORC_XS_IDX) ? h->xs : h->ys;
      int* c = (what == ORC_XS_OFF || what == ORC_XS_IDX) ? h->xs_n : h->ys_n;
      if (!a) return -1;
      if (what == ORC_XS_OFF || what == ORC_YS_OFF) {
        need = nn + 1;
        if (buf && cap >= need) pack_lists(a, c, nn, (int64_t*)buf, NULL);
        return need;
      }
      need = pack_lists(a, c, nn, NULL, NULL);
      if (buf && cap >= need) pack_lists(a, c, nn, NULL, (int*)buf);
      return need;
    }
    case ORC_K:
    case ORC_XBAR_N:
    case ORC_CHILD_OFF:
      if (!h->k) return -1;
      need = nn;
      if (buf && cap >= need)
        memcpy(buf, what == ORC_K ? h->k : (what == ORC_XBAR_N ? h->xbar_n : h->child_off), sizeof(int) * (size_t)nn);
      return need;
    case ORC_SK_OFF:
    case ORC_SK_IDX:
      if (!h->k) return -1;
      if (what == ORC_SK_OFF) {
        need = nn + 1;
        if (buf && cap >= need) pack_lists(h->sk, h->k, nn, (int64_t*)buf, NULL);
        return need;
      }
      need = pack_lists(h->sk, h->k, nn, NULL, NULL);
      if (buf && cap >= need) pack_lists(h->sk, h->k, nn, NULL, (int*)buf);
      return need;
    case ORC_U_OFF:
    case ORC_U: {
      if (!h->k) return -1;
      int64_t s = 0;
      for (int i = 0; i < nn; i++) {
        if (what == ORC_U_OFF && buf && cap >= nn + 1) ((int64_t*)buf)[i] = s;
        int64_t sz = (int64_t)h->xbar_n[i] * h->k[i];
        if (what == ORC_U && buf && sz > 0 && h->U[i]) {
          /* filled below once total known */
        }
        s += sz;
      }
      if (what == ORC_U_OFF) {
        if (buf && cap >= nn + 1) ((int64_t*)buf)[nn] = s;
        return nn + 1;
      }
      if (buf && cap >= s) {
        int64_t o = 0;
        for (int i = 0; i < nn; i++) {
          int64_t sz = (int64_t)h->xbar_n[i] * h->k[i];
          if (sz > 0) memcpy((double*)buf + o, h->U[i], sizeof(double) * (size_t)sz);
          o += sz;
        }
      }
      return s;
    }
    case ORC_K_COL:
    case ORC_XBARC_N:
      if (!h->k_col) return -1;
      need = nn;
      if (buf && cap >= need) memcpy(buf, what == ORC_K_COL ? h->k_col : h->xbar_col_n, sizeof(int) * (size_t)nn);
      return need;
    case ORC_SKC_OFF:
    case ORC_SKC_IDX:
      if (!h->k_col) return -1;
      if (what == ORC_SKC_OFF) {
        need = nn + 1;
        if (buf && cap >= need) pack_lists(h->sk_col, h->k_col, nn, (int64_t*)buf, NULL);
        return need;
      }
      need = pack_lists(h->sk_col, h->k_col, nn, NULL, NULL);
      if (buf && cap >= need) pack_lists(h->sk_col, h->k_col, nn, NULL, (int*)buf);
      return need;
    case ORC_V_OFF:
    case ORC_V: {
      if (!h->k_col) return -1;
      int64_t s = 0;
      for (int i = 0; i < nn; i++) {
        if (what == ORC_V_OFF && buf && cap >= nn + 1) ((int64_t*)buf)[i] = s;
        s += (int64_t)h->xbar_col_n[i] * h->k_col[i];
      }
      if (what == ORC_V_OFF) {
        if (buf && cap >= nn + 1) ((int64_t*)buf)[nn] = s;
        return nn + 1;
      }
      if (buf && cap >= s) {
        int64_t o = 0;
        for (int i = 0; i < nn; i++) {
          int64_t sz = (int64_t)h->xbar_col_n[i] * h->k_col[i];
          if (sz > 0) memcpy((double*)buf + o, h->V[i], sizeof(double) * (size_t)sz);
          o += sz;
        }
      }
      return s;
    }
    default:
      return -1;
  }
}

/* info: [n, d, q, nnodes, depth, L, r, n_il, n_nf, max_S, max_T] as int64 */
void orc_info(const orc_h2* h, int64_t* out, double* W, double* t_stage) {
  out[0] = h->n;
  out[1] = h->d;
  out[2] = h->q;
  out[3] = h->nnodes;
  out[4] = h->depth;
  out[5] = h->L;
  out[6] = h->r;
  out[7] = h->il_off[h->nnodes];
  out[8] = h->nf_off[h->nnodes];
  out[9] = h->max_S;
  out[10] = h->max_T;
  if (W) *W = h->W;
  if (t_stage) memcpy(t_stage, h->t_stage, sizeof(h->t_stage));
}

/* per-level r of the last orc_calibrate (E4): out[l] for l = 0..depth (0 = no admissible pair) */
int orc_calib_levels(const orc_h2* h, int* out) {
  for (int l = 0; l <= h->depth; l++) out[l] = h->calib_r[l];
  return h->depth + 1;
}

void orc_free(orc_h2* h) {
  if (!h) return;
  int nn = h->nnodes;
  free(h->perm);
  free(h->X);
  free(h->key);
  free(h->lvl_start);
  free(h->level);
  free(h->begin);
  free(h->end);
  free(h->parent);
  free(h->first_child);
  free(h->nchild);
  free(h->is_leaf);
  free(h->cell);
  free(h->il_off);
  free(h->il_idx);
  free(h->nf_off);
  free(h->nf_idx);
  free_lists2(h->xs, nn);
  free_lists2(h->ys, nn);
  free(h->xs_n);
  free(h->ys_n);
  free_lists2(h->sk, nn);
  if (h->U) {
    for (int i = 0; i < nn; i++) free(h->U[i]);
    free(h->U);
  }
  free(h->k);
  free(h->xbar_n);
  free(h->child_off);
  free_basis(nn, &h->k_col, &h->sk_col, &h->V, &h->xbar_col_n, &h->child_off_col);
  free(h);
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
