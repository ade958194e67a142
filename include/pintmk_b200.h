/*
 * pintmk_b200.h -- C-ABI of the B200-native all-at-once space-time MLK solve.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `pintmk` (arXiv 2401.00228): solver.multilevel_solve -> fgmres ->
 * apply_preconditioner -> {matvec, restrict, forward_solve, interpolate}.
 * Reference paths below are relative to /root/reference/pkg/src/pintmk/.
 *
 * The reference is pure Python over numpy/scipy with one Cython seam
 * (_chain.pyx: factor_tridiag / march_chain).  Its duck-typed seams are the
 * methods the entry points below replace; each entry cites the reference
 * method it stands in for.  Every entry:
 *   - takes caller-allocated DEVICE buffers (fp64, row-major (slices, m) with
 *     x fastest, exactly the reference's (n_steps+1, n) layout,
 *     stepper.py:93-94);
 *   - is stream-ordered on `stream` (a cudaStream_t; NULL = legacy stream);
 *   - returns 0 on success, a cudaError_t value (< 1000) on a CUDA failure, or
 *     one of the PMK_ERR_* codes below on a bad argument.  The Python mirror
 *     maps PMK_ERR_ARG/PMK_ERR_SHAPE to ValueError (reference convention,
 *     e.g. stepper.py:28-34, solver.py:114-115) and everything else to
 *     RuntimeError.
 * No entry point allocates device memory except pmk_hier_create (a few KB of
 * Krylov scalars); all vectors belong to the caller.
 */
#ifndef PINTMK_B200_H
#define PINTMK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *pmk_stream_t; /* cudaStream_t */

enum {
  PMK_OK = 0,
  PMK_ERR_ARG = 1001,         /* null pointer / out-of-range scalar */
  PMK_ERR_SHAPE = 1002,       /* inconsistent sizes */
  PMK_ERR_UNSUPPORTED = 1003, /* stencil / coarse kind not supported */
  PMK_ERR_STATE = 1004        /* call order violated (e.g. step before begin) */
};

/* Coarsest-level direct solver kinds (pmk_coarse.kind). */
enum { PMK_COARSE_DST = 1, PMK_COARSE_DENSE = 2, PMK_COARSE_EIG = 3, PMK_COARSE_PCR = 4,
       PMK_COARSE_LINE = 5 };

/*
 * Spatial operator in "right-product" form: (v @ M)_i = sum_j M[j,i] v_j,
 * i.e. M^T applied to v, which is what the reference matvec computes
 * (stepper.py:102, `blocks @ self.diag`).  Five slots in ascending column
 * order, S (i-nx), W (i-1), C (i), E (i+1), N (i+nx); slots whose neighbour
 * lies outside the grid are skipped.  Products are accumulated in that order
 * with separately rounded multiply and add, the order scipy's csc_matvecs
 * uses for the same product.
 */
typedef struct pmk_stencil {
  int32_t var;        /* 0: constant coefficients c[5]; 1: per-point coef */
  double c[5];        /* constant coefficients, slots S W C E N */
  const double *coef; /* device [5][m] per-point coefficients (var = 1) */
} pmk_stencil;

/*
 * One level's block lower-bidiagonal system [I; -B, D; ...; -B, D]
 * (stepper.py:66-105).  diag_t holds D^T and sub_t holds B^T so that
 * out_k = D^T v_k - B^T v_{k-1}; rows listed in `dropped` add B^T v_{k-1}
 * back (stepper.py:103-104).
 */
typedef struct pmk_level {
  int32_t dim;     /* 1 or 2 */
  int32_t nx, ny;  /* ny = 1 in 1-D; m = nx*ny */
  int32_t n_steps; /* slices = n_steps + 1 */
  pmk_stencil diag_t;
  pmk_stencil sub_t;
  const uint8_t *dropped; /* device [n_steps+1] 0/1 mask, or NULL */
} pmk_level;

/*
 * Intergrid pair between a level and the next coarser one.
 * TimePair (intergrid.py:37-63): group_of = NULL, y_* = NULL.
 * TimeSpacePair (intergrid.py:79-120): Z injection through group_of and the
 * Y^T averaging as a CSR over coarse points with ascending fine indices.
 */
typedef struct pmk_pair {
  int32_t nu;              /* time coarsening factor (1 = pure space move) */
  int32_t n_T;             /* coarse steps; fine rows = nu*n_T + 1 */
  int32_t m_fine, m_coarse;
  const int32_t *group_of; /* device [m_fine] coarse index of each fine point */
  const int32_t *y_ptr;    /* device [m_coarse+1] */
  const int32_t *y_idx;    /* device [nnz] fine indices, ascending per row */
  const double *y_val;     /* device [nnz] Y entries (1/|group|) */
  /* MgritPair (intergrid.py:134-167), mgrit != 0: restriction injects every
   * nu-th row; interpolation sets out[nu K] = w[K] and propagates
   * out[nu K + j] = (psi^{-1} phi)^j w[K], j < nu, which is diagonal in the
   * sine basis of the (pristine) fine level: ratio[mode] = beta / delta.
   * Sine tables as in pmk_coarse (fft_* non-NULL: FFT path with fft_scale,
   * else the dense sx/sy GEMM path).  Scratch: work0/work1/work2 of
   * n_T*m_fine doubles, coarse_out of (n_T+1)*m_fine (the coarse solve's
   * output inside the preconditioner). */
  int32_t mgrit;
  int32_t dim, nx, ny;
  const double *sx, *sy, *fft_x, *fft_y;
  double fft_scale;
  const double *ratio;
  double *work0, *work1, *work2, *coarse_out;
  /* Weighted space pair (z_ptr != NULL; group_of = NULL): an extension with
   * no reference counterpart -- BASELINE config 4 names full-weighting
   * restriction and bilinear interpolation, the reference only agglomerates
   * (intergrid.py:79-131).  Restriction is the time sum followed by the Y^T
   * CSR above with general weights; interpolation applies the CSR Z over
   * fine points (z_ptr [m_fine+1], z_idx coarse indices ascending, z_val
   * weights) and repeats in time.  In the solver the coarse solution goes to
   * coarse_out ((n_T+1) m_coarse doubles) and its space interpolation
   * ((n_T+1) m_fine) is the iteration's child vector. */
  const int32_t *z_ptr, *z_idx;
  const double *z_val;
} pmk_pair;

/*
 * Coarsest-level block forward substitution (stepper.py:114-146):
 *   out_0 = rhs_0,
 *   out_k = D^{-1} (rhs_k + [k not dropped] * C out_{k-1}),
 * with C = B in 1-D (_chain.pyx:64-71) and C = B^T in 2-D (stepper.py:144).
 * DST: D and C are simultaneously diagonal in the orthonormal sine basis
 *      (pristine Dirichlet Laplacian levels); delta/beta are their
 *      eigenvalues per mode (p fastest).  One launch chain: x-transform,
 *      y-transform, segmented per-mode recurrence, inverse transforms.
 * EIG: D = I - K and B = I + b K with K = I (x) Kx + Ky (x) I, Kx, Ky
 *      tridiagonal (every agglomerated level: intergrid.py:202-227 groups are
 *      a tensor product; the odd-grid 3-wide last group makes K
 *      non-symmetric).  V = Vy (x) Vx (eigenvectors of K) diagonalises D and
 *      B: dense transforms as fp64 GEMMs over all slices (sx = Vx^{-T} and
 *      ix = Vx^T right operands, sy = Vy^{-1} and iy = Vy left operands),
 *      the per-mode recurrence, and in 2-D (B^T coupling) a low-rank mode
 *      coupling b V^{-1} (K^T - K) V applied by a cluster-per-chain kernel:
 *      n_cx points with rows cx_h [n_cx][nx] (physical extraction) and
 *      cx_u [n_cx][nx] (mode injection), likewise cy_* along y.  Chains
 *      start at seg_start[0..n_seg) (rows; the first is 1).
 * DENSE: explicit D^{-1} (m x m, row-major) for 5-point operators that are
 *      not separable (m <= 8192).
 * PCR: 1-D levels (D tridiagonal, any coefficients; the reference's Thomas
 *      chain, _chain.pyx:15-82): parallel cyclic reduction with the matrix
 *      part factored once -- pcr_alpha/pcr_gamma [pcr_levels][m] multiply the
 *      right-hand side entries at distance 2^l below / above, pcr_inv [m]
 *      are the reciprocal final pivots.  One CTA per chain, one launch.
 * LINE: 2-D 5-point operators of any size that are not separable (the
 *      reference's per-slice SuperLU solve, stepper.py:140-145,
 *      linalg.py:35-68): block Thomas over grid lines.  line_g holds the
 *      inverted Schur blocks G_j = (T_j - L_j G_{j-1} U_{j-1})^{-1} split by
 *      rows over the line_cs CTAs of a chain's cluster, R = ceil(nx/line_cs)
 *      rows each: [ny][line_cs][R][nx] with entry (j, g, r, c) = G_j[g R + r, c]
 *      (0 past row nx); line_l / line_u [m] are the couplings D[i, i-nx] /
 *      D[i, i+nx].  One cluster per chain, one launch; work0 holds
 *      n_seg * 2 m doubles.
 * PCR, LINE and DENSE take `coupling` (C in row form) and the chain table.
 */
typedef struct pmk_coarse {
  int32_t kind;
  int32_t dim, nx, ny, n_steps;
  const uint8_t *dropped; /* device [n_steps+1] or NULL (exact chain) */
  const double *sx;       /* DST GEMM path: [nx][nx] (unused, may be NULL, with fft_x) */
  const double *sy;       /* DST GEMM path: [ny][ny] (dim 2) */
  const double *delta;    /* DST: [m] eigenvalues of D */
  const double *beta;     /* DST: [m] eigenvalues of C */
  const double *dinv;     /* DENSE: [m][m] */
  pmk_stencil coupling;   /* DENSE: C as a stencil in row form */
  double *work0, *work1;  /* device scratch, (n_steps+1)*m doubles each */
  /* DST via FFT (n+1 a power of two): per direction [N] complex four-step
   * twiddles w_N^{n2 k1} at [k1*N2 + n2] (N2 = 2^floor(log2 N / 2)) followed
   * by [N] complex (cos, sin)(pi p/N) (pmk_dst.cu); NULL selects
   * the dense sine-matrix GEMM path (sx/sy).  With the FFT path delta/beta
   * are ordered x-mode slow, y-mode fast, and fft_scale (= 4/(N_x N_y), or
   * 2/N_x in 1-D) folds the orthonormalisation into the recurrence. */
  const double *fft_x, *fft_y;
  double fft_scale;
  /* EIG (and the DST GEMM path): inverse transforms; NULL = sx / sy */
  const double *ix, *iy;
  int32_t n_cx, n_cy; /* EIG 2-D coupling correction points (<= 8 each) */
  const double *cx_h, *cx_u, *cy_h, *cy_u;
  double coupling_b;  /* b in B = I + b K */
  const int32_t *seg_start; /* device [n_seg] first row of each chain */
  int32_t n_seg;
  int32_t pcr_levels;       /* PCR: ceil(log2 m) reduction strides */
  const double *pcr_alpha, *pcr_gamma, *pcr_inv;
  const double *line_g, *line_l, *line_u; /* LINE */
  int32_t line_cs;          /* LINE: CTAs per chain (cluster size, 1..8) */
} pmk_coarse;

/* ---------------------------------------------------------------- per-op */

/* BlockBidiagonalSystem.matvec (stepper.py:96-105). */
int pmk_stmv(const pmk_level *L, const double *v, double *out,
             pmk_stream_t stream);

/* TimePair.restrict / TimeSpacePair.restrict (intergrid.py:51-56, 106-112).
 * scratch: (n_T+1)*m_fine doubles, only used for space pairs (may be NULL
 * for time pairs). */
int pmk_restrict(const pmk_pair *P, const double *v, double *vh,
                 double *scratch, pmk_stream_t stream);

/* TimePair.interpolate / TimeSpacePair.interpolate (intergrid.py:58-63,
 * 114-120). */
int pmk_interpolate(const pmk_pair *P, const double *w, double *out,
                    pmk_stream_t stream);

/* Fused solver.py:336-339: vh = Y^T (A v - mu v).  v is read as
 * v_raw[i] / *v_scale when v_scale is non-NULL (lazily normalised Krylov
 * basis vector, solver.py:395/420). */
int pmk_stmv_shift_restrict(const pmk_level *L, const pmk_pair *P, double mu,
                            const double *v_raw, const double *v_scale,
                            double *vh, double *scratch, pmk_stream_t stream);

/* Fused solver.py:349,359,403: x = v - Z vt ; w = A x.  x may be NULL (not
 * stored).  v read as v_raw / *v_scale when v_scale is non-NULL. */
int pmk_interp_sub_stmv(const pmk_level *L, const pmk_pair *P,
                        const double *v_raw, const double *v_scale,
                        const double *vt, double *x, double *w,
                        pmk_stream_t stream);

/* BlockBidiagonalSystem.forward_solve on the coarsest level
 * (stepper.py:114-146, _chain.pyx:37-82, linalg.py:62-68). */
int pmk_coarsest_solve(const pmk_coarse *C, const double *rhs, double *out,
                       pmk_stream_t stream);

/* Deterministic reductions (np.dot / np.linalg.norm at solver.py:381,407,
 * 412).  result is a DEVICE scalar.  Fixed grid, fixed summation order:
 * bitwise reproducible run to run. */
int pmk_dot(const double *a, const double *b, int64_t n, double *result,
            pmk_stream_t stream);
int pmk_nrm2(const double *a, int64_t n, double *result, pmk_stream_t stream);

/* FineSystem.relative_residual numerator (stepper.py:191-193):
 * result = || rhs - A u ||_2 (device scalar).  tmp: N doubles. */
int pmk_residual_nrm2(const pmk_level *L, const double *u, const double *rhs,
                      double *tmp, double *result, pmk_stream_t stream);

/* Restart step of the FGMRES(m) wrapper (the
 * reference fgmres has no restart, solver.py:366-367, so this replaces the
 * wrapper's `r = b - hier.fine.matvec(x)` and `np.linalg.norm(r)`):
 * r = rhs - A u stored, *result = ||r||_2 (device scalar).  r may not alias
 * u or rhs. */
int pmk_residual(const pmk_level *L, const double *u, const double *rhs,
                 double *r, double *result, pmk_stream_t stream);

/* y += a x (the wrapper's `x = x + dx`; a = 1 rounds once per element like
 * numpy's addition).  x and y may not alias. */
int pmk_axpy(double a, const double *x, double *y, int64_t n,
             pmk_stream_t stream);

/* ----------------------------------------------------- native FGMRES/MLK */

typedef struct pmk_hier pmk_hier;

/* A level hierarchy (solver.py:84-102): levels 0..n_levels-1, the last one
 * being the coarsest direct solve.  mu: the shift (solver.py:47). */
pmk_hier *pmk_hier_create(int32_t n_levels, double mu);
void pmk_hier_destroy(pmk_hier *H);

/* Level idx < n_levels-1: its system, its pair to idx+1 and the inner
 * FGMRES budget (solver.py:219-235; ignored for idx 0).  The coarsest level
 * is described by pmk_hier_set_coarse. */
int pmk_hier_set_level(pmk_hier *H, int32_t idx, const pmk_level *L,
                       const pmk_pair *P, int32_t budget);
int pmk_hier_set_coarse(pmk_hier *H, const pmk_coarse *C);

/* Buffers of an inner level (1 <= idx < n_levels-1), or of the coarsest
 * (idx = n_levels-1: rhs only).  rhs receives the parent's restriction;
 * v_slots[budget] receive the normalised Krylov vectors v_0..v_{budget-1};
 * w_buf holds the unnormalised new vector of each iteration; child_out[budget]
 * (size of level idx+1) receive the child solve of each iteration;
 * ts_scratch ((n_T+1)*m_fine doubles) is required for space pairs. */
int pmk_hier_set_buffers(pmk_hier *H, int32_t idx, double *rhs,
                         double *const *v_slots, double *const *child_out,
                         int32_t n_slots, double *w_buf, double *ts_scratch);

/* fgmres (solver.py:362-456) driven one iteration at a time.
 * begin: beta = ||rhs||.  step j: one iteration (preconditioner
 * solver.py:323-359, matvec, MGS, Givens): its first pass stores the
 * normalised basis vector v_j into v_out (rhs/beta for j = 0, else the
 * previous step's w / h[j][j-1]); the unnormalised next vector goes to w_next
 * (may be the previous step's w_next, never the rhs) and the child solve to
 * child_out (for an MGRIT pair: its interpolation, fine-level size).  tol > 0 stops the device-side iteration once rel <= tol
 * (solver.py:438); tol = 0 is the reference's tol=None.  finish: back substitution
 * and x = sum_i y_i x_i with x_i = v_i - Z vt_i recomputed (no stored
 * preconditioned vectors). */
int pmk_fgmres_begin(pmk_hier *H, int32_t idx, const double *rhs,
                     int32_t max_iter, double tol, pmk_stream_t stream);
int pmk_fgmres_step(pmk_hier *H, int32_t idx, int32_t j, double *v_out,
                    double *w_next, double *child_out, pmk_stream_t stream);
/* 1 when the solver keeps a lazy basis (the default ICWY path; PMK_LAZY=0
 * or PMK_MGS=classic turn it off): step j then keeps its w_next as the raw
 * basis vector j+1 (so w_next must be a fresh buffer every step; v_0 is the
 * rhs itself), never writes a normalised copy unless v_out is non-NULL (it may
 * be NULL), and every consumer uses RN(raw * RN(1/scale)) -- the values the
 * normalised basis would hold.  0: v_out (required) receives v_j and w_next
 * may be reused across steps. */
int32_t pmk_lazy_basis(void);
int pmk_fgmres_finish(pmk_hier *H, int32_t idx, double *x,
                      pmk_stream_t stream);
/* Non-blocking stop test: snapshot enqueues a copy of the level's fgmres
 * scalars into pinned host slot `slot` (0..3) in stream order; after the
 * caller has synchronised with that point (e.g. an event recorded right
 * after), snapshot_read returns {beta, rel, n_iter, breakdown} as of then.
 * Lets a driver enqueue step j+1 before it knows whether step j converged
 * (a converged invocation turns later steps into no-ops on the device). */
int pmk_fgmres_snapshot(pmk_hier *H, int32_t idx, int32_t slot,
                        pmk_stream_t stream);
int pmk_fgmres_snapshot_read(pmk_hier *H, int32_t idx, int32_t slot,
                             double *scalars);
/* finish restricted to the time slices [row_begin, row_end) of x (row_begin a
 * multiple of the level's coarsening factor nu); the call with row_begin = 0
 * also runs the back substitution, so it must come first.  Lets the caller
 * stream the finished part of x (e.g. to the host) while the rest is
 * assembled.  Same result as pmk_fgmres_finish. */
int pmk_fgmres_finish_rows(pmk_hier *H, int32_t idx, double *x,
                           int32_t row_begin, int32_t row_end,
                           pmk_stream_t stream);
/* Copies the level's fgmres state to the host (synchronises the stream):
 * scalars[4] = {beta, rel, n_iter, breakdown}; hist[cap] (residual history),
 * hraw[(cap+1)*cap] (unrotated Hessenberg, row-major, ld = cap) and y[cap]
 * may be NULL.  *cap (if non-NULL) receives the capacity. */
int pmk_fgmres_state(pmk_hier *H, int32_t idx, double *scalars, double *hist,
                     double *hraw, double *y, int32_t *cap,
                     pmk_stream_t stream);

/* fgmres(hier, idx, rhs, tol=None, max_iter=budget) for an inner level,
 * entirely on the device (no host synchronisation): the recursion of
 * solver.py:347-348. Reads the level's registered rhs buffer. */
int pmk_fgmres_fixed(pmk_hier *H, int32_t idx, double *x,
                     pmk_stream_t stream);

/* apply_preconditioner (solver.py:323-359) at level idx < n_levels-1:
 * out = v - Z A_H^{-1} Y^T (A v - mu v).  Uses the registered buffers of
 * level idx+1 and child_out as the coarse-correction buffer (fine-level size
 * for an MGRIT pair). */
int pmk_apply_preconditioner(pmk_hier *H, int32_t idx, const double *v,
                             double *child_out, double *out,
                             pmk_stream_t stream);

/* ------------------------------------------------------------ accounting */

/* Every kernel launch of the library is counted.  pmk_profile_begin(1)
 * additionally brackets each launch with a CUDA event pair (on the launch
 * stream) and records its algorithmic bytes / flops; pmk_profile_end
 * synchronises the device and writes, per category c < *n_categories,
 * stats[4c .. 4c+3] = {launches, total ms, algorithmic bytes, flops}. */
int pmk_profile_begin(int32_t with_events);
int pmk_profile_end(double *stats, int32_t max_categories,
                    int32_t *n_categories);
/* Same records split by attribution (phase ledger, parcost.py:63-122): rows
 * of 7 doubles {level, hint, category, launches, total ms, bytes, flops},
 * one per (level, hint, category) seen; level = the hierarchy level whose
 * work issued the launch (-1: stand-alone call, n_levels-1: coarsest solve),
 * hint = -1 none, 1 restriction, 2 interpolation (MGRIT ideal interpolation).
 * Ends the profile like pmk_profile_end; PMK_ERR_ARG if max_rows is too
 * small (*n_rows tells the size; the records are consumed either way). */
int pmk_profile_end_levels(double *rows, int32_t max_rows, int32_t *n_rows);
const char *pmk_profile_category(int32_t idx);
int64_t pmk_launch_count(void);

/* Diagnostics: out[i] = x[i] / d through the kernels' reciprocal-based
 * correctly rounded division (must equal IEEE x / d bitwise). */
int pmk_div_check(const double *x, double d, int64_t n, double *out,
                  pmk_stream_t stream);

/* The coarsest transforms' batched GEMM, exposed for tests and
 * measurement: C[b] = A[b] B[b] for b < batch, row-major fp64 (element
 * strides stride_* between batches), on the fp64 tensor cores (DMMA). */
int pmk_dgemm(int32_t M, int32_t N, int32_t K, const double *A, int32_t lda,
              int64_t stride_a, const double *B, int32_t ldb, int64_t stride_b,
              double *C, int32_t ldc, int64_t stride_c, int32_t batch,
              pmk_stream_t stream);

/* Library identification (for the loaded-.so checks). */
const char *pmk_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PINTMK_B200_H */
