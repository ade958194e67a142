// pmk_internal.cuh -- shared device helpers and launcher declarations.
//
// All arithmetic is fp64.  Where the reference performs a separately rounded
// multiply and add (numpy / scipy compiled without FMA contraction), the
// kernels use __dmul_rn / __dadd_rn / __dsub_rn explicitly, and the
// translation units on the solver path are compiled with -fmad=false, so the
// only rounding differences left against the reference are the reductions
// (np.dot / OpenBLAS order) and the coarsest direct solve.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/pintmk_b200.h"

namespace pmk {

constexpr int kSMs = 148;
// Fixed grid of every elementwise reduction kernel: deterministic partial
// count independent of the vector length.
constexpr int kRedBlocks = 4 * kSMs;  // 592
constexpr int kRedThreads = 256;
// Upper bound on partial sums produced by any reduction-carrying launch.
constexpr int kMaxPartials = 8 * kSMs;  // 1184

#define PMK_RETURN_IF(cond, code) \
  do {                            \
    if (cond) return (code);      \
  } while (0)

#define PMK_CUDA_TRY(expr)                      \
  do {                                          \
    cudaError_t _e = (expr);                    \
    if (_e != cudaSuccess) return (int)_e;      \
  } while (0)

#define PMK_LAUNCH_CHECK() PMK_CUDA_TRY(cudaGetLastError())

// Opt-in bounds checks (make BOUNDS=1): print the offending index and trap.
#ifdef PMK_BOUNDS
#define PMK_CHECK_IDX(i, n, tag)                                                           \
  do {                                                                                     \
    if ((long long)(i) < 0 || (long long)(i) >= (long long)(n)) {                          \
      printf("PMK OOB %s idx %lld n %lld block %d thread %d\n", tag, (long long)(i),      \
             (long long)(n), (int)blockIdx.x, (int)threadIdx.x);                           \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define PMK_CHECK_IDX(i, n, tag) \
  do {                           \
  } while (0)
#endif

__device__ __forceinline__ bool is_live(const int *live) {
  return live == nullptr || *live != 0;
}

// x / d, correctly rounded (bitwise __ddiv_rn), for a divisor d reused over
// many x: y = RN(1/d) is computed once (`rcp`).  q0 = RN(x y) is within two
// ulps; one FMA correction q1 = RN(q0 + (x - d q0) y) is faithful (its error
// is |eps (x/d - q0)| + 1/2 ulp with |eps| <= 2^-53); Markstein's theorem
// then makes q2 = RN(q1 + (x - d q1) y) the correctly rounded quotient (the
// residuals are exact FMAs).  With d in [2^-100, 2^100] (div_ok) and |x| in
// [2^-800, 2^800] the quotient and the residuals stay normal; other x (and
// zeros) take the IEEE division.  Checked bitwise against IEEE division by
// tests/test_gpu_parity.py (pmk_div_check).
__device__ __forceinline__ double div_by(double x, double d, double rcp) {
  const unsigned ex = (unsigned)(__double2hiint(x) >> 20) & 0x7ffu;
  if (ex < 1023u - 800u || ex > 1023u + 800u) return x == 0.0 ? x : __ddiv_rn(x, d);
  const double q0 = __dmul_rn(x, rcp);
  const double q1 = __fma_rn(__fma_rn(-d, q0, x), rcp, q0);
  return __fma_rn(__fma_rn(-d, q1, x), rcp, q1);
}
// Divisor usable by div_by (normal, not near the exponent limits).
__host__ __device__ __forceinline__ bool div_ok(double d) {
  return d >= 0x1p-100 && d <= 0x1p100;
}

// Deterministic block reduction: warp xor-tree, then warp 0 over the warp
// sums.  Every block running this on the same inputs gets the same bits.
// blockDim.x must be a multiple of 32 (<= 1024).
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();  // protect sh against a previous call
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = (lane < nw) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, o));
  }
  return r;  // valid in warp 0
}

// Sum of `n` partials in a fixed order; every calling block obtains the same
// value (broadcast through shared memory) provided blockDim.x is the same.
__device__ __forceinline__ double reduce_partials(const double *partials, int n) {
  __shared__ double res;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc = __dadd_rn(acc, partials[i]);
  double s = block_sum(acc);
  if (threadIdx.x == 0) res = s;
  __syncthreads();
  return res;
}

// ------------------------------------------------------------ accounting
// RAII bracket around one kernel launch: counts it and, while profiling is
// on, records a CUDA event pair plus the launch's algorithmic bytes/flops.
namespace prof {
enum Cat {
  kMV = 0,    // plain space-time matvec
  kMVR,       // matvec + shift + restrict
  kIMV,       // interpolate + subtract + matvec (+ dot)
  kMGS,       // fused MGS pass
  kRed,       // stand-alone reductions
  kSmall,     // begin / finish_col / backsolve (single block)
  kAsm,       // solution assembly
  kGemm,      // coarsest sine-transform GEMMs
  kRec,       // coarsest per-mode recurrence
  kCoarseMisc,// coarsest dense chain / row copy
  kXfer,      // stand-alone restrict / interpolate / agglomeration gather
  kDst,       // coarsest FFT sine transforms (pmk_dst.cu)
  kChain,     // coarsest chains in one launch: EIG 2-D mode chain, DENSE, PCR, LINE
  kNumCat
};
struct Scope {
  Scope(int cat, double bytes, double flops, cudaStream_t s);
  ~Scope();
  int rec;
  cudaStream_t stream;
};
// Attribution of recorded launches (phase ledger, reference parcost.py:63-122):
// the hierarchy level whose work is being issued, and an optional phase hint.
enum Hint { kHintNone = -1, kHintRestrict = 1, kHintInterp = 2 };
struct Tag {
  Tag(int level, int hint = kHintNone);
  ~Tag();
  int prev_level, prev_hint;
};
}  // namespace prof

// ------------------------------------------------------------------ march
// Parameters of the fused space-time stencil kernels (pmk_march.cu).
enum MarchMode { kModeMV = 0, kModeMVR = 1, kModeIMV = 2 };

struct MarchParams {
  int nx, ny, m, n_steps;
  pmk_stencil P, Q;  // P = D^T (on v_k), Q = B^T (on v_{k-1})
  const uint8_t *dropped;
  const double *v;        // input (raw)
  const double *v_scale;  // device scalar divisor or nullptr
  double *out;            // MV: out, IMV: w
  // MVR
  double mu;
  int nu;
  int inject;          // MVR: MGRIT injection (vh_K = s_{nu K}) instead of the time sum
  int exact_scale;     // v / *v_scale correctly rounded (register path); else the
                       // TMA path multiplies by the rounded reciprocal (<= 1 ulp)
  int fma;             // in-solver passes: the stencil sums, shift and dot may use
                       // fused multiply-add (off: bitwise the reference's product)
  double *vh;          // (n_T+1, m) time-summed (fine spatial)
  double *vh_partials; // optional: per-block partial sums of vh^2 (TMA path only;
                       // launch_march reports 0 partials when it is not produced)
  double *v_norm_out;  // optional: the normalised input v = v_raw / scale
  // MVR "sub" mode (deferred orthogonalisation, fgmres_fixed): the input is
  // w - (*v_sub_coef) v_sub, staged together (both level-size); it is stored
  // into v_norm_out (the next raw basis vector) with per-block partials of
  // its ||.||^2 in vn_partials; v_scale must be NULL (outputs unscaled).
  const double *v_sub;
  const double *v_sub_coef;
  double *vn_partials;
  // IMV
  const double *vt;
  const int32_t *group_of;
  int m_coarse;
  double *x_out;  // optional
  const double *v0;
  const double *v0_scale;
  double *partials;  // one per block (dot(w, v0))
  // optional (IMV, v != v0): partial <w, v> at pj[b] and <v, v0> at
  // pj[kMaxPartials + b], b < *n_partials, read off the staged input v (the
  // ICWY dot pass then skips v_0 and v_j).  Produced by the 2-D TMA path
  // only; the launcher reports whether it did in *pj_done (host pointer).
  double *pj;
  int *pj_done;
  // with pj and v == v0 (j = 0): slot 0 receives ||w||^2 partials instead
  // (budget-1 inner levels: h_10^2 = ||w||^2 - h_00^2, no update pass)
  int pj_wsq;
  const int *live;
};

// Constant stencil with equal off-diagonal slots (S = W = E = N; 1-D: the
// absent S/N slots are ignored when zero).
inline bool iso_stencil(const pmk_stencil &st) {
  if (st.var) return false;
  const double o = st.c[1];
  return st.c[3] == o && (st.c[0] == o || st.c[0] == 0.0) && (st.c[4] == o || st.c[4] == 0.0);
}

// Launch one fused march.  Returns the number of partials written (IMV) via
// *n_partials when non-null.
int launch_march(int mode, const MarchParams &p, cudaStream_t s, int *n_partials);
// TMA-pipelined variant (pmk_march_tma.cu); *handled = 0 asks for the
// register fallback.
int launch_march_tma(int mode, const MarchParams &p, cudaStream_t s, int *n_partials,
                     double bytes, int cat, int *handled);

// ---------------------------------------------------------------- krylov
int launch_dot_partials(const double *a, const double *a_scale, const double *b,
                        const double *b_scale, int64_t n, double *partials,
                        const int *live, cudaStream_t s);
int launch_diffsq_partials(const double *a, const double *b, int64_t n, double *partials,
                           cudaStream_t s, double *r_out = nullptr);
int launch_axpy(double a, const double *x, double *y, int64_t n, cudaStream_t s);
int launch_div_check(const double *x, double d, int64_t n, double *out, cudaStream_t s);
int launch_reduce_to_scalar(const double *partials, int n, double *out, int do_sqrt,
                            cudaStream_t s);

// ---------------------------------------------------------------- coarse
int launch_dst_rows(const double *in, double *out, int n, int64_t rows, const double *tables,
                    const int *live, cudaStream_t s, int64_t rows_per_slice = 0,
                    int64_t out_slice_stride = 0);
// MGRIT pair (pmk_coarse.cu): injection restriction / ideal interpolation
int mgrit_restrict(const pmk_pair &P, const double *v, double *vh, const int *live,
                   cudaStream_t s);
int mgrit_interpolate(const pmk_pair &P, const double *w, double *out, const int *live,
                      cudaStream_t s);
int launch_dst_cols(const double *in, double *out, int nx, int ny, int slices,
                    const double *tables, const int *live, cudaStream_t s);
// batched row-major fp64 GEMM C[b] = A[b] B[b] (DMMA; PMK_GEMM=simt: CUDA cores)
int launch_gemm(int M, int N, int K, const double *A, int lda, int64_t sA, const double *B,
                int ldb, int64_t sB, double *C, int ldc, int64_t sC, int batch, cudaStream_t s);
// per-slice direct solves without a common eigenbasis (pmk_lines.cu)
int launch_pcr_chains(const pmk_coarse &C, const double *rhs, double *out, const int *live,
                      cudaStream_t s);
int launch_line_chains(const pmk_coarse &C, const double *rhs, double *out, const int *live,
                       cudaStream_t s);
int coarse_solve(const pmk_coarse &C, const double *rhs, double *out, const int *live,
                 cudaStream_t s, const double *out_scale = nullptr);

// --------------------------------------------------------------- transfer
int launch_ts_gather(const pmk_pair &P, const double *fine, double *coarse, const int *live,
                     cudaStream_t s);
int launch_restrict_time(const pmk_pair &P, const double *v, double *vh, cudaStream_t s);
int launch_interpolate(const pmk_pair &P, const double *w, double *out, cudaStream_t s);
// weighted space pair (pmk_pair z_*): Z over space, repeated `nu` times in time
int launch_interpolate_z(const pmk_pair &P, const double *w, double *out, int nu,
                         const int *live, cudaStream_t s);

}  // namespace pmk
