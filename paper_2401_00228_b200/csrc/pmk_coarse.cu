// pmk_coarse.cu -- coarsest-level block forward substitution (reference
// stepper.py:114-146, _chain.pyx:37-82, linalg.py:62-68).
//
//   out_0 = rhs_0
//   out_k = D^{-1} (rhs_k + [k not dropped] C out_{k-1})
//
// DST path (pristine Dirichlet-Laplacian levels, i.e. every level reached by
// time moves only): D = I - a dt A and C = I + (1-a) dt A are simultaneously
// diagonal in the orthonormal sine basis S (S = S^T = S^{-1}).  The solve is
//   R^ = S_y R S_x            (two fp64 GEMMs over all slices at once)
//   u^_k = (r^_k + beta u^_{k-1}) / delta   per mode, segmented at dropped k
//   out = S_y U^ S_x          (two GEMMs)
// so the exact chain (coarsest_n_cgs = 0) and any chunked decoupling
// (perturb_decouple, intergrid.py:299-311) cost the same and are parallel
// over all m modes; the sequential dimension is only the scalar recurrence.
//
// DENSE path (agglomerated levels with non-Toeplitz operators): explicit
// D^{-1}, one stencil + GEMV launch pair per slice.
//
// This translation unit keeps FMA contraction on (DFMA GEMM); the result
// differs from the reference's LU / Thomas solve by rounding only.
#include <cooperative_groups.h>

#include <cstdlib>

#include "pmk_internal.cuh"

namespace pmk {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

// C[b] = A[b] * B[b], all row-major; 256 threads, 4x4 outputs per thread
// (rows ty + 16 i, cols tx + 16 j -> conflict-free shared-memory reads).
__global__ void __launch_bounds__(256)
    dgemm_nn_kernel(int M, int N, int K, const double *__restrict__ A, int lda, int64_t sA,
                    const double *__restrict__ B, int ldb, int64_t sB, double *__restrict__ C,
                    int ldc, int64_t sC, int batch, const int *live) {
  if (!is_live(live)) return;
  __shared__ double As[2][BK][BM + 1];
  __shared__ double Bs[2][BK][BN];
  const int mtiles = (M + BM - 1) / BM;
  // grid-stride over (batch, M tile): gridDim.y / .z stay within their limits
  for (int64_t bt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y; bt < (int64_t)batch * mtiles;
       bt += (int64_t)gridDim.z * gridDim.y) {
  const int bz = (int)(bt / mtiles);
  const double *__restrict__ Ab = A + bz * sA;
  const double *__restrict__ Bb = B + bz * sB;
  double *__restrict__ Cb = C + bz * sC;
  const int m0 = (int)(bt % mtiles) * BM, n0 = blockIdx.x * BN;
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  double ra[4], rb[4];
  auto gload = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = (t >> 4) + 16 * q, c = t & 15;
      const int gm = m0 + r, gk = k0 + c;
      ra[q] = (gm < M && gk < K) ? Ab[(int64_t)gm * lda + gk] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = (t >> 6) + 4 * q, c = t & 63;
      const int gk = k0 + r, gn = n0 + c;
      rb[q] = (gk < K && gn < N) ? Bb[(int64_t)gk * ldb + gn] : 0.0;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) As[buf][t & 15][(t >> 4) + 16 * q] = ra[q];
#pragma unroll
    for (int q = 0; q < 4; ++q) Bs[buf][(t >> 6) + 4 * q][t & 63] = rb[q];
  };

  const int nk = (K + BK - 1) / BK;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) gload((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (kt + 1 < nk) sstore(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn < N) Cb[(int64_t)gm * ldc + gn] = acc[i][j];
    }
  }
  __syncthreads();  // (shared tiles are reused by the next (batch, tile))
  }
}

// Same product on the fp64 tensor cores: mma.sync m8n8k4 (SASS DMMA.8x8x4).
// CTA tile 64 x 64, 4 warps of 32 x 32 (4 x 4 MMA tiles, 32 accumulators per
// thread), K staged 16 at a time through shared memory (register double
// buffering of the next tile's loads).  Fragment layouts (PTX ISA, m8n8k4
// .f64): A a0 = A[g][t], B b0 = B[t][g], C {c0, c1} = C[g][2t], C[g][2t+1]
// with g = lane / 4, t = lane % 4.  Shared strides are chosen so that every
// fragment load is the 2-wavefront minimum: A m-major with row stride 20,
// B k-major with row stride 72.
constexpr int TM = 64, TN = 64, TK = 16, SA = TK + 4, SB = TN + 8;

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128)
    dmma_gemm_kernel(int M, int N, int K, const double *__restrict__ A, int lda, int64_t sA,
                     const double *__restrict__ B, int ldb, int64_t sB, double *__restrict__ C,
                     int ldc, int64_t sC, int batch, const int *live) {
  if (!is_live(live)) return;
  __shared__ double As[2][TM][SA];
  __shared__ double Bs[2][TK][SB];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane >> 2, tg = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int mtiles = (M + TM - 1) / TM;
  for (int64_t bt = (int64_t)blockIdx.z * gridDim.y + blockIdx.y; bt < (int64_t)batch * mtiles;
       bt += (int64_t)gridDim.z * gridDim.y) {
    const int bz = (int)(bt / mtiles);
    const double *__restrict__ Ab = A + bz * sA;
    const double *__restrict__ Bb = B + bz * sB;
    double *__restrict__ Cb = C + bz * sC;
    const int m0 = (int)(bt % mtiles) * TM, n0 = blockIdx.x * TN;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double ra[8], rb[8];
    auto gload = [&](int k0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = t + 128 * q;
        const int r = e >> 4, c = e & 15;  // A: 64 rows x 16 k
        const int gm = m0 + r, gk = k0 + c;
        ra[q] = (gm < M && gk < K) ? Ab[(int64_t)gm * lda + gk] : 0.0;
        const int rk = e >> 6, cn = e & 63;  // B: 16 k x 64 columns
        const int bk = k0 + rk, bn = n0 + cn;
        rb[q] = (bk < K && bn < N) ? Bb[(int64_t)bk * ldb + bn] : 0.0;
      }
    };
    auto sstore = [&](int buf) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = t + 128 * q;
        As[buf][e >> 4][e & 15] = ra[q];
        Bs[buf][e >> 6][e & 63] = rb[q];
      }
    };
    const int nk = (K + TK - 1) / TK;
    gload(0);
    sstore(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
      const int buf = kt & 1;
      if (kt + 1 < nk) gload((kt + 1) * TK);
#pragma unroll
      for (int ks = 0; ks < TK; ks += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = As[buf][wm + 8 * i + g][ks + tg];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][ks + tg][wn + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j], af[i], bf[j]);
      }
      if (kt + 1 < nk) sstore(buf ^ 1);
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gm = m0 + wm + 8 * i + g;
      if (gm >= M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn + 8 * j + 2 * tg + h;
          if (gn < N) Cb[(int64_t)gm * ldc + gn] = acc[i][j][h];
        }
    }
  }
}

// PMK_GEMM=simt selects the CUDA-core kernel (A/B); default: DMMA
bool gemm_simt() {
  static const bool on = [] {
    const char *e = getenv("PMK_GEMM");
    return e && e[0] == 's';
  }();
  return on;
}

int gemm(int M, int N, int K, const double *A, int lda, int64_t sA, const double *B, int ldb,
         int64_t sB, double *C, int ldc, int64_t sC, int batch, const int *live, cudaStream_t s) {
  if (!gemm_simt()) {
    const int mt = (M + TM - 1) / TM;
    dim3 grid((N + TN - 1) / TN, mt < 4096 ? mt : 4096, batch < 1024 ? batch : 1024);
    prof::Scope scope(prof::kGemm, 8.0 * batch * ((double)M * N * 2.0) + 8.0 * (double)K * N,
                      2.0 * M * N * (double)K * batch, s);
    dmma_gemm_kernel<<<grid, 128, 0, s>>>(M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC, batch,
                                          live);
    PMK_LAUNCH_CHECK();
    return 0;
  }
  const int mtiles = (M + BM - 1) / BM;
  const int gy = mtiles < 4096 ? mtiles : 4096;
  const int gz = batch < 1024 ? batch : 1024;
  dim3 grid((N + BN - 1) / BN, gy, gz);
  const double flops = 2.0 * M * N * (double)K * batch;
  const double bytes = 8.0 * batch * ((double)M * N * 2.0) + 8.0 * (double)K * N;
  prof::Scope scope(prof::kGemm, bytes, flops, s);
  dgemm_nn_kernel<<<grid, 256, 0, s>>>(M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC, batch, live);
  PMK_LAUNCH_CHECK();
  return 0;
}

// Segmented per-mode first-order recurrence, in place on X ((n+1) x m).
// Loads are batched ahead of the dependent chain (the store to X would
// otherwise serialise them).
constexpr int kRecBatch = 8;
__global__ void __launch_bounds__(256)
    dst_recurrence_kernel(double *X, const double *delta, const double *beta,
                          const uint8_t *dropped, int n_steps, int m, double scale,
                          const int *live, const double *out_scale = nullptr) {
  if (!is_live(live)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (out_scale) scale *= *out_scale;  // (the solve is linear in the rhs)
  // multiply by 1/delta: high modes decay through the subnormal range, where
  // an IEEE division takes the slow path
  const double d = 1.0 / delta[i], b = beta[i];
  double u = X[i] * scale;  // transformed rhs_0 == transformed out_0
  X[i] = u;
  for (int k0 = 1; k0 <= n_steps; k0 += kRecBatch) {
    double r[kRecBatch];
#pragma unroll
    for (int q = 0; q < kRecBatch; ++q) {
      const int k = k0 + q;
      r[q] = (k <= n_steps) ? X[(int64_t)k * m + i] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kRecBatch; ++q) {
      const int k = k0 + q;
      if (k > n_steps) break;
      const bool cut = dropped && dropped[k];
      const double rq = r[q] * scale;
      u = cut ? rq * d : fma(b, u, rq) * d;
      X[(int64_t)k * m + i] = u;
    }
  }
}

// Chunked form of the same recurrence for few modes (1-D coarsest levels):
// u_k = a_k u_{k-1} + b_k with a_k = beta/delta (0 at dropped rows) and
// b_k = scale r^_k / delta.  Pass 1: every (mode, chunk) runs the chunk from a
// zero state and stores its end value and the chunk's product of a_k.  Pass
// 2: every (mode, chunk) combines the carries of the preceding chunks (at
// most n_chunks steps), then re-runs its chunk from the carried state.
__global__ void rec_chunk_pass1(const double *X, const double *delta, const double *beta,
                                const uint8_t *dropped, int n_steps, int m, double scale,
                                int clen, int nch, double *carryB, double *carryA,
                                const int *live) {
  if (!is_live(live)) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m * nch) return;
  const int i = (int)(t % m), c = (int)(t / m);
  const double d = 1.0 / delta[i], a = beta[i] * d;
  const int k0 = 1 + c * clen, k1 = min(n_steps + 1, k0 + clen);
  double u = 0.0, P = 1.0;
  for (int k = k0; k < k1; ++k) {
    const bool cut = dropped && dropped[k];
    const double bk = X[(int64_t)k * m + i] * scale * d;
    u = cut ? bk : fma(a, u, bk);
    P = cut ? 0.0 : P * a;
  }
  carryB[t] = u;
  carryA[t] = P;
}

__global__ void rec_chunk_pass2(double *X, const double *delta, const double *beta,
                                const uint8_t *dropped, int n_steps, int m, double scale,
                                int clen, int nch, const double *carryB, const double *carryA,
                                const int *live) {
  if (!is_live(live)) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)m * nch) return;
  const int i = (int)(t % m), c = (int)(t / m);
  const double d = 1.0 / delta[i], a = beta[i] * d;
  double u = X[i] * scale;  // slice 0 (transformed rhs_0)
  for (int q = 0; q < c; ++q) u = fma(carryA[(int64_t)q * m + i], u, carryB[(int64_t)q * m + i]);
  const int k0 = 1 + c * clen, k1 = min(n_steps + 1, k0 + clen);
  for (int k = k0; k < k1; ++k) {
    const bool cut = dropped && dropped[k];
    const double bk = X[(int64_t)k * m + i] * scale * d;
    u = cut ? bk : fma(a, u, bk);
    X[(int64_t)k * m + i] = u;
  }
  if (c == 0) X[i] = X[i] * scale;
}

// Recurrence launcher: per-mode sequential scan when there are enough modes
// to fill the GPU, chunked two-pass scan otherwise.
int run_recurrence(const pmk_coarse &C, double *X, int m, double scale, double *scratch,
                   const int *live, cudaStream_t s) {
  const int64_t N = (int64_t)(C.n_steps + 1) * m;
  prof::Scope rs(prof::kRec, 16.0 * N, 0.0, s);
  if (m >= 16 * 1024 || !scratch || C.n_steps < 64) {
    dst_recurrence_kernel<<<(m + 255) / 256, 256, 0, s>>>(X, C.delta, C.beta, C.dropped,
                                                         C.n_steps, m, scale, live);
    PMK_LAUNCH_CHECK();
    return 0;
  }
  int nch = (int)((64LL * 1024 + m - 1) / m);  // ~64 K threads
  if (nch > C.n_steps / 8) nch = C.n_steps / 8;
  const int clen = (C.n_steps + nch - 1) / nch;
  nch = (C.n_steps + clen - 1) / clen;
  double *cB = scratch, *cA = scratch + (int64_t)m * nch;
  const int64_t th = (int64_t)m * nch;
  rec_chunk_pass1<<<(int)((th + 255) / 256), 256, 0, s>>>(X, C.delta, C.beta, C.dropped,
                                                          C.n_steps, m, scale, clen, nch, cB, cA,
                                                          live);
  PMK_LAUNCH_CHECK();
  rec_chunk_pass2<<<(int)((th + 255) / 256), 256, 0, s>>>(X, C.delta, C.beta, C.dropped,
                                                          C.n_steps, m, scale, clen, nch, cB, cA,
                                                          live);
  PMK_LAUNCH_CHECK();
  return 0;
}

__global__ void copy_row_kernel(const double *src, double *dst, int m, const int *live,
                                const double *scale = nullptr) {
  if (!is_live(live)) return;
  const double c = scale ? *scale : 1.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    dst[i] = scale ? __dmul_rn(src[i], c) : src[i];
}

// b = rhs_k + [k not dropped] * C out_{k-1}  (row-form 5-slot stencil)
__global__ void coupling_kernel(const double *rhs_k, const double *prev, double *b, pmk_stencil C,
                                int nx, int ny, const uint8_t *dropped, int k, const int *live) {
  if (!is_live(live)) return;
  const int m = nx * ny;
  const bool cut = dropped && dropped[k];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    if (cut) {
      b[i] = rhs_k[i];
      continue;
    }
    const int y = i / nx, x = i - y * nx;
    double cs, cw, cc, ce, cn;
    if (C.var) {
      cs = C.coef[i];
      cw = C.coef[m + i];
      cc = C.coef[2 * m + i];
      ce = C.coef[3 * m + i];
      cn = C.coef[4 * m + i];
    } else {
      cs = C.c[0];
      cw = C.c[1];
      cc = C.c[2];
      ce = C.c[3];
      cn = C.c[4];
    }
    double acc = 0.0;
    if (y > 0) acc = __dadd_rn(acc, __dmul_rn(cs, prev[i - nx]));
    if (x > 0) acc = __dadd_rn(acc, __dmul_rn(cw, prev[i - 1]));
    acc = __dadd_rn(acc, __dmul_rn(cc, prev[i]));
    if (x < nx - 1) acc = __dadd_rn(acc, __dmul_rn(ce, prev[i + 1]));
    if (y < ny - 1) acc = __dadd_rn(acc, __dmul_rn(cn, prev[i + nx]));
    b[i] = __dadd_rn(rhs_k[i], acc);
  }
}

// out = Dinv * b, one warp per row.
__global__ void gemv_kernel(const double *__restrict__ Dinv, const double *__restrict__ b,
                            double *__restrict__ out, int m, const int *live) {
  if (!is_live(live)) return;
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= m) return;
  const double *r = Dinv + (int64_t)row * m;
  double acc = 0.0;
  for (int j = lane; j < m; j += 32) acc = fma(r[j], b[j], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[row] = acc;
}

// DENSE chain (5-point operators that are not separable): every chain of
// the level advances one row per step in ONE cooperative launch -- phase A
// forms b = rhs_k + [k not cut] C out_{k-1} for all chains, phase B applies
// D^{-1} (a warp per (chain, row) dot product), grid-wide barriers between
// phases.  Independent chains (perturb_decouple) run side by side.
__global__ void __launch_bounds__(256)
    dense_chain_kernel(const double *__restrict__ rhs, double *__restrict__ out,
                       const double *__restrict__ Dinv, pmk_stencil Cst, int nx, int ny,
                       const uint8_t *dropped, const int32_t *seg_start, int n_seg, int n_steps,
                       double *__restrict__ b, const int *live) {
  namespace cg = cooperative_groups;
  if (!is_live(live)) return;
  cg::grid_group grid = cg::this_grid();
  const int m = nx * ny;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  const int64_t gwarp = gtid >> 5, nwarps = gsz >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t i = gtid; i < m; i += gsz) out[i] = rhs[i];  // out_0 = rhs_0
  int maxlen = 0;
  for (int sg = 0; sg < n_seg; ++sg) {
    const int end = (sg + 1 < n_seg) ? seg_start[sg + 1] : n_steps + 1;
    maxlen = max(maxlen, end - seg_start[sg]);
  }
  grid.sync();
  const int64_t work = (int64_t)n_seg * m;
  for (int t = 0; t < maxlen; ++t) {
    for (int64_t e = gtid; e < work; e += gsz) {
      const int sg = (int)(e / m), i = (int)(e - (int64_t)sg * m);
      const int a = seg_start[sg];
      const int end = (sg + 1 < n_seg) ? seg_start[sg + 1] : n_steps + 1;
      const int k = a + t;
      if (k >= end) continue;
      const double *rk = rhs + (int64_t)k * m;
      if (t == 0 && dropped && dropped[k]) {
        b[e] = rk[i];
        continue;
      }
      const double *prev = out + (int64_t)(k - 1) * m;
      const int y = i / nx, x = i - y * nx;
      double cs_, cw, cc, ce, cn;
      if (Cst.var) {
        cs_ = Cst.coef[i];
        cw = Cst.coef[m + i];
        cc = Cst.coef[2 * m + i];
        ce = Cst.coef[3 * m + i];
        cn = Cst.coef[4 * m + i];
      } else {
        cs_ = Cst.c[0];
        cw = Cst.c[1];
        cc = Cst.c[2];
        ce = Cst.c[3];
        cn = Cst.c[4];
      }
      double acc = 0.0;
      if (y > 0) acc = __dadd_rn(acc, __dmul_rn(cs_, prev[i - nx]));
      if (x > 0) acc = __dadd_rn(acc, __dmul_rn(cw, prev[i - 1]));
      acc = __dadd_rn(acc, __dmul_rn(cc, prev[i]));
      if (x < nx - 1) acc = __dadd_rn(acc, __dmul_rn(ce, prev[i + 1]));
      if (y < ny - 1) acc = __dadd_rn(acc, __dmul_rn(cn, prev[i + nx]));
      b[e] = __dadd_rn(rk[i], acc);
    }
    grid.sync();
    for (int64_t w = gwarp; w < work; w += nwarps) {
      const int sg = (int)(w / m), row = (int)(w - (int64_t)sg * m);
      const int a = seg_start[sg];
      const int end = (sg + 1 < n_seg) ? seg_start[sg + 1] : n_steps + 1;
      const int k = a + t;
      if (k >= end) continue;
      const double *dr = Dinv + (int64_t)row * m;
      const double *bs = b + (int64_t)sg * m;
      double acc = 0.0;
      for (int j = lane; j < m; j += 32) acc = fma(dr[j], bs[j], acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) out[(int64_t)k * m + row] = acc;
    }
    grid.sync();
  }
}

// dst[K * dstride + doff + i] = src[K * sstride + soff + i], i < m, K < rows
__global__ void strided_rows_copy_kernel(const double *src, int64_t sstride, int64_t soff,
                                         double *dst, int64_t dstride, int64_t doff, int m,
                                         int rows, const int *live) {
  if (!is_live(live)) return;
  for (int K = blockIdx.y; K < rows; K += gridDim.y)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
      dst[K * dstride + doff + i] = src[K * sstride + soff + i];
}

// work2[e] = scale * work1[e] * ratio[e % m]^j
__global__ void mode_power_kernel(const double *w1, double *w2, const double *ratio, int m,
                                  int64_t n, int j, double scale, const int *live) {
  if (!is_live(live)) return;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double r = ratio[e % m];
    double f = scale;
    for (int q = 0; q < j; ++q) f *= r;
    w2[e] = w1[e] * f;
  }
}

int strided_copy(const double *src, int64_t sstride, int64_t soff, double *dst, int64_t dstride,
                 int64_t doff, int m, int rows, const int *live, cudaStream_t s) {
  dim3 grid((m + 255) / 256 < 64 ? (m + 255) / 256 : 64, rows < 4096 ? rows : 4096);
  prof::Scope sc(prof::kXfer, 16.0 * m * (double)rows, 0.0, s);
  strided_rows_copy_kernel<<<grid, 256, 0, s>>>(src, sstride, soff, dst, dstride, doff, m, rows,
                                                live);
  PMK_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------- EIG chain
// Mode-space block forward substitution of a 2-D EIG level whose slices are
// coupled by B^T != B (stepper.py:144 on an agglomerated odd grid):
//   z_k = (r_k + beta z_{k-1} + b C(z_{k-1})) / delta,   C = I (x) Cx + Cy (x) I,
//   Cx z_row = sum_c u_c (h_c . z_row)   (points c of K^T - K, see pmk_coarse),
// in place on X ((n_steps+1) x ny x nx modes, y-mode slow).  One thread
// cluster per chain (segment); CTA g of the cluster owns mode rows
// [g RQ, g RQ + RQ), thread p owns mode column p, so z, 1/delta and beta of
// its RQ modes stay in registers for the whole chain.  Per step: the row dots
// h_c . z_row are warp-transposed sums (31 shuffles for 32 values) completed
// across warps in shared memory; the column dots h_c . z_col are thread-local
// over the CTA's rows, completed across the cluster through distributed
// shared memory after one cluster barrier.  Buffers alternate by step parity,
// so that barrier is the only cluster-wide synchronisation per step.
struct EigChainArgs {
  double *X;
  const double *delta, *beta;
  const uint8_t *dropped;
  const int32_t *seg_start;
  int n_seg, n_steps, nx, ny, n_cx, n_cy;
  const double *cx_h, *cx_u, *cy_h, *cy_u;
  double b;
  const int *live;
};

// v[i] over the 32 lanes -> lane l returns sum_lanes v[l] (fixed order)
template <int NV>
__device__ __forceinline__ double warp_transpose_sum(double (&v)[NV], int base) {
  static_assert(NV % 32 == 0, "");
  double w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) w[i] = v[base + i];
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const double send = up ? w[i] : w[i + o];
      const double keep = up ? w[i + o] : w[i];
      w[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return w[0];
}

template <int RQ, int NC>
__global__ void __launch_bounds__(256) eig_chain_kernel(EigChainArgs a) {
  namespace cg = cooperative_groups;
  if (!is_live(a.live)) return;
  cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks();
  const int g = (int)cluster.block_rank();
  const int seg = blockIdx.x / G;
  if (seg >= a.n_seg) return;  // (whole clusters only: uniform)
  const int nx = a.nx, ny = a.ny;
  const int64_t m = (int64_t)nx * ny;
  const int p = threadIdx.x;
  const bool colok = p < nx;
  const int NT = blockDim.x, NW = NT >> 5, warp = p >> 5, lane = p & 31;
  const int q0 = g * RQ;
  constexpr int NV = ((RQ * NC + 31) / 32) * 32;
  extern __shared__ double sm[];
  double *cxh = sm;                       // [NC][nx]
  double *cxu = cxh + NC * nx;            // [NC][nx]
  double *cyh = cxu + NC * nx;            // [NC][ny]
  double *cyu = cyh + NC * ny;            // [NC][ny]
  double *dpart = cyu + NC * ny;          // [2][NW][NV]
  double *dsum = dpart + 2 * NW * NV;     // [2][NV]
  double *epart = dsum + 2 * NV;          // [2][NC][NT]  (read by the cluster)
  for (int i = threadIdx.x; i < NC * nx; i += NT) {
    const int c = i / nx, x = i - c * nx;
    cxh[i] = c < a.n_cx ? a.cx_h[(int64_t)c * nx + x] : 0.0;
    cxu[i] = c < a.n_cx ? a.cx_u[(int64_t)c * nx + x] : 0.0;
  }
  for (int i = threadIdx.x; i < NC * ny; i += NT) {
    const int c = i / ny, y = i - c * ny;
    cyh[i] = c < a.n_cy ? a.cy_h[(int64_t)c * ny + y] : 0.0;
    cyu[i] = c < a.n_cy ? a.cy_u[(int64_t)c * ny + y] : 0.0;
  }
  double invd[RQ], bt[RQ], z[RQ], r[RQ];
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    const int y = q0 + q;
    const bool ok = colok && y < ny;
    const int64_t i = (int64_t)y * nx + p;
    invd[q] = ok ? 1.0 / a.delta[i] : 0.0;
    bt[q] = ok ? a.beta[i] : 0.0;
  }
  const int k0 = a.seg_start[seg];
  const int k1 = (seg + 1 < a.n_seg) ? a.seg_start[seg + 1] : a.n_steps + 1;
  auto load_rows = [&](int k, double (&dst)[RQ]) {
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      const int y = q0 + q;
      dst[q] = (colok && y < ny) ? a.X[(int64_t)k * m + (int64_t)y * nx + p] : 0.0;
    }
  };
  load_rows(k0 - 1, z);  // previous slice (used only when k0 is not a cut)
  load_rows(k0, r);
  __syncthreads();
  double hx[NC], ux[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    hx[c] = colok ? cxh[c * nx + p] : 0.0;
    ux[c] = colok ? cxu[c * nx + p] : 0.0;
  }
  for (int k = k0; k < k1; ++k) {
    double rn[RQ];
    if (k + 1 < k1) load_rows(k + 1, rn);
    const bool cut = (k == k0) && a.dropped && a.dropped[k];
    if (cut) {
#pragma unroll
      for (int q = 0; q < RQ; ++q) z[q] = r[q] * invd[q];
    } else {
      const int buf = k & 1;
      // row dots: value j = q * NC + c
      double v[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) v[j] = 0.0;
#pragma unroll
      for (int q = 0; q < RQ; ++q)
#pragma unroll
        for (int c = 0; c < NC; ++c) v[q * NC + c] = hx[c] * z[q];
#pragma unroll
      for (int b0 = 0; b0 < NV; b0 += 32) {
        const double sum = warp_transpose_sum<NV>(v, b0);
        dpart[(buf * NW + warp) * NV + b0 + lane] = sum;
      }
      // column partials over this CTA's rows
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double e = 0.0;
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
          const int y = q0 + q;
          if (y < ny) e = fma(cyh[c * ny + y], z[q], e);
        }
        epart[(buf * NC + c) * NT + p] = e;
      }
      cluster.sync();  // dpart (CTA) and epart (cluster) complete
      for (int j = threadIdx.x; j < NV; j += NT) {
        double sacc = 0.0;
        for (int w = 0; w < NW; ++w) sacc += dpart[(buf * NW + w) * NV + j];
        dsum[buf * NV + j] = sacc;
      }
      double e[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) e[c] = 0.0;
      for (int gg = 0; gg < G; ++gg) {
        const double *peer = cluster.map_shared_rank(epart, gg);
#pragma unroll
        for (int c = 0; c < NC; ++c) e[c] += peer[(buf * NC + c) * NT + p];
      }
      __syncthreads();  // dsum
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        const int y = q0 + q;
        double corr = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          corr = fma(ux[c], dsum[buf * NV + q * NC + c], corr);
          if (y < ny) corr = fma(cyu[c * ny + y], e[c], corr);
        }
        z[q] = fma(a.b, corr, fma(bt[q], z[q], r[q])) * invd[q];
      }
    }
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      const int y = q0 + q;
      if (colok && y < ny) a.X[(int64_t)k * m + (int64_t)y * nx + p] = z[q];
    }
    if (k + 1 < k1) {
#pragma unroll
      for (int q = 0; q < RQ; ++q) r[q] = rn[q];
    }
  }
  cluster.sync();  // no CTA leaves while a peer may still read its epart
}

template <int RQ, int NC>
int launch_eig_chain_t(const EigChainArgs &a, int G, cudaStream_t s) {
  const int NT = ((a.nx + 31) / 32) * 32;
  const int NW = NT / 32;
  constexpr int NV = ((RQ * NC + 31) / 32) * 32;
  const size_t smem =
      sizeof(double) * (2 * NC * (size_t)a.nx + 2 * NC * (size_t)a.ny + 2 * (size_t)NW * NV +
                        2 * NV + 2 * (size_t)NC * NT);
  auto fn = eig_chain_kernel<RQ, NC>;
  static bool attr_done = false;
  if (!attr_done) {
    PMK_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    PMK_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.n_seg * G), 1, 1);
  cfg.blockDim = dim3((unsigned)NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PMK_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, a));
  return 0;
}

int launch_eig_chain(const pmk_coarse &C, double *X, const int *live, cudaStream_t s) {
  const int nx = C.nx, ny = C.ny;
  PMK_RETURN_IF(nx > 256 || C.n_cx > 8 || C.n_cy > 8 || !C.seg_start || C.n_seg < 1,
                PMK_ERR_UNSUPPORTED);
  EigChainArgs a;
  a.X = X;
  a.delta = C.delta;
  a.beta = C.beta;
  a.dropped = C.dropped;
  a.seg_start = C.seg_start;
  a.n_seg = C.n_seg;
  a.n_steps = C.n_steps;
  a.nx = nx;
  a.ny = ny;
  a.n_cx = C.n_cx;
  a.n_cy = C.n_cy;
  a.cx_h = C.cx_h;
  a.cx_u = C.cx_u;
  a.cy_h = C.cy_h;
  a.cy_u = C.cy_u;
  a.b = C.coupling_b;
  a.live = live;
  const int nc = C.n_cx > C.n_cy ? C.n_cx : C.n_cy;
  // rows per CTA: the smallest that keeps the cluster within 8 CTAs (16 at most)
  int rq = 4;
  while (rq < 32 && (ny + rq - 1) / rq > 8) rq *= 2;
  const int G = (ny + rq - 1) / rq;
  PMK_RETURN_IF(G > 16, PMK_ERR_UNSUPPORTED);
  const int64_t N = (int64_t)(C.n_steps + 1) * nx * ny;
  prof::Scope sc(prof::kChain, 16.0 * N, 0.0, s);
#define PMK_EIG_CASE(R, NCV) \
  if (rq == R && nc <= NCV) return launch_eig_chain_t<R, NCV>(a, G, s);
  PMK_EIG_CASE(4, 2) PMK_EIG_CASE(4, 4) PMK_EIG_CASE(4, 8)
  PMK_EIG_CASE(8, 2) PMK_EIG_CASE(8, 4) PMK_EIG_CASE(8, 8)
  PMK_EIG_CASE(16, 2) PMK_EIG_CASE(16, 4)
  PMK_EIG_CASE(32, 2)
#undef PMK_EIG_CASE
  return PMK_ERR_UNSUPPORTED;
}

}  // namespace

int launch_gemm(int M, int N, int K, const double *A, int lda, int64_t sA, const double *B,
                int ldb, int64_t sB, double *C, int ldc, int64_t sC, int batch, cudaStream_t s) {
  return gemm(M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC, batch, nullptr, s);
}

// MgritPair.restrict (intergrid.py:152-155): vh[K] = v[nu K].
int mgrit_restrict(const pmk_pair &P, const double *v, double *vh, const int *live,
                   cudaStream_t s) {
  const int64_t m = P.m_fine;
  return strided_copy(v, (int64_t)P.nu * m, 0, vh, m, 0, (int)m, P.n_T + 1, live, s);
}

// MgritPair.interpolate (intergrid.py:157-167): out[nu K] = w[K]; rows
// nu K + j (j < nu) = (psi^{-1} phi)^j w[K], applied as ratio^j in the sine
// basis of the fine grid: one forward transform of w[0..n_T), then per j a
// scaled copy and an inverse transform written into the strided rows.
int mgrit_interpolate(const pmk_pair &P, const double *w, double *out, const int *live,
                      cudaStream_t s) {
  const int nx = P.nx, ny = (P.dim == 2) ? P.ny : 1;
  const int m = nx * ny, nT = P.n_T, nu = P.nu;
  const int64_t Nw = (int64_t)nT * m;
  PMK_RETURN_IF(!P.ratio || !P.work0 || !P.work1 || !P.work2, PMK_ERR_ARG);
  int rc = strided_copy(w, m, 0, out, (int64_t)nu * m, 0, m, nT + 1, live, s);
  if (rc || nu == 1 || nT == 0) return rc;
  const bool fft = P.fft_x != nullptr && (ny == 1 || P.fft_y != nullptr);
  // forward transform of w[0..n_T) -> work1 (modes, y-mode slow)
  if (fft) {
    if (ny == 1) {
      rc = launch_dst_rows(w, P.work1, nx, nT, P.fft_x, live, s);
    } else {
      rc = launch_dst_rows(w, P.work0, nx, (int64_t)nT * ny, P.fft_x, live, s);
      if (!rc) rc = launch_dst_cols(P.work0, P.work1, nx, ny, nT, P.fft_y, live, s);
    }
  } else {
    PMK_RETURN_IF(!P.sx || (ny > 1 && !P.sy), PMK_ERR_ARG);
    if (ny == 1) {
      rc = gemm(nT, nx, nx, w, nx, 0, P.sx, nx, 0, P.work1, nx, 0, 1, live, s);
    } else {
      rc = gemm(nT * ny, nx, nx, w, nx, 0, P.sx, nx, 0, P.work0, nx, 0, 1, live, s);
      if (!rc) rc = gemm(ny, nx, ny, P.sy, ny, 0, P.work0, nx, m, P.work1, nx, m, nT, live, s);
    }
  }
  if (rc) return rc;
  const double scale = fft ? P.fft_scale : 1.0;
  for (int j = 1; j < nu; ++j) {
    {
      prof::Scope sc(prof::kXfer, 16.0 * Nw, 0.0, s);
      const int64_t g = (Nw + 255) / 256 < 16 * kSMs ? (Nw + 255) / 256 : 16 * kSMs;
      mode_power_kernel<<<(int)g, 256, 0, s>>>(P.work1, P.work2, P.ratio, m, Nw, j, scale, live);
    }
    PMK_LAUNCH_CHECK();
    double *dst = out + (int64_t)j * m;  // rows nu K + j, slice stride nu m
    if (fft) {
      if (ny == 1) {
        rc = launch_dst_rows(P.work2, dst, nx, nT, P.fft_x, live, s, 1, (int64_t)nu * m);
      } else {
        rc = launch_dst_cols(P.work2, P.work0, nx, ny, nT, P.fft_y, live, s);
        if (!rc)
          rc = launch_dst_rows(P.work0, dst, nx, (int64_t)nT * ny, P.fft_x, live, s, ny,
                               (int64_t)nu * m);
      }
    } else {
      if (ny == 1) {
        rc = gemm(1, nx, nx, P.work2, nx, m, P.sx, nx, 0, dst, nx, (int64_t)nu * m, nT, live, s);
      } else {
        rc = gemm(ny, nx, ny, P.sy, ny, 0, P.work2, nx, m, P.work0, nx, m, nT, live, s);
        if (!rc)
          rc = gemm(ny, nx, nx, P.work0, nx, m, P.sx, nx, 0, dst, nx, (int64_t)nu * m, nT, live,
                    s);
      }
    }
    if (rc) return rc;
  }
  return 0;
}

int coarse_solve(const pmk_coarse &C, const double *rhs, double *out, const int *live,
                 cudaStream_t s, const double *out_scale) {
  const int nx = C.nx, ny = (C.dim == 2) ? C.ny : 1;
  const int m = nx * ny;
  const int rows = C.n_steps + 1;
  const int64_t N = (int64_t)rows * m;
  // out_scale (output of the solve for rhs / scale's reciprocal): 2-D FFT path
  PMK_RETURN_IF(out_scale && !(C.kind == PMK_COARSE_DST && C.fft_x && ny > 1), PMK_ERR_ARG);
  if (C.kind == PMK_COARSE_DST && C.fft_x) {
    // FFT sine transforms (pmk_dst.cu): every pass streams the vector once.
    PMK_RETURN_IF(!C.delta || !C.beta || !C.work0, PMK_ERR_ARG);
    int rc;
    if (ny == 1) {
      rc = launch_dst_rows(rhs, C.work0, nx, rows, C.fft_x, live, s);
      if (rc) return rc;
      rc = run_recurrence(C, C.work0, m, C.fft_scale, C.work1, live, s);
      if (rc) return rc;
      rc = launch_dst_rows(C.work0, out, nx, rows, C.fft_x, live, s);
      if (rc) return rc;
    } else {
      PMK_RETURN_IF(!C.fft_y || !C.work1, PMK_ERR_ARG);
      // x then y (modes [k][q][p], q slow), recurrence, y then x
      rc = launch_dst_rows(rhs, C.work0, nx, (int64_t)rows * ny, C.fft_x, live, s);
      if (rc) return rc;
      rc = launch_dst_cols(C.work0, C.work1, nx, ny, rows, C.fft_y, live, s);
      if (rc) return rc;
      {
        prof::Scope rs(prof::kRec, 16.0 * N, 0.0, s);
        dst_recurrence_kernel<<<(m + 255) / 256, 256, 0, s>>>(C.work1, C.delta, C.beta,
                                                             C.dropped, C.n_steps, m,
                                                             C.fft_scale, live, out_scale);
      }
      PMK_LAUNCH_CHECK();
      rc = launch_dst_cols(C.work1, C.work0, nx, ny, rows, C.fft_y, live, s);
      if (rc) return rc;
      rc = launch_dst_rows(C.work0, out, nx, (int64_t)rows * ny, C.fft_x, live, s);
      if (rc) return rc;
    }
    {
      prof::Scope cs(prof::kCoarseMisc, 16.0 * m, 0.0, s);
      copy_row_kernel<<<(m + 255) / 256, 256, 0, s>>>(rhs, out, m, live,
                                                      out_scale);  // stepper.py:118
    }
    PMK_LAUNCH_CHECK();
    return 0;
  }
  if (C.kind == PMK_COARSE_DST || C.kind == PMK_COARSE_EIG) {
    // dense transforms as GEMMs over all slices: forward R Fx (rows), Fy R_k
    // (per slice); inverse Iy Z_k, then Z Ix.  Sine basis: F = I = S.
    PMK_RETURN_IF(!C.sx || !C.delta || !C.beta || !C.work0, PMK_ERR_ARG);
    const double *ixm = C.ix ? C.ix : C.sx;
    const bool chain = C.kind == PMK_COARSE_EIG && ny > 1 && (C.n_cx > 0 || C.n_cy > 0);
    if (ny == 1) {
      int rc = gemm(rows, nx, nx, rhs, nx, 0, C.sx, nx, 0, C.work0, nx, 0, 1, live, s);
      if (rc) return rc;
      rc = run_recurrence(C, C.work0, m, 1.0, C.work1, live, s);
      if (rc) return rc;
      rc = gemm(rows, nx, nx, C.work0, nx, 0, ixm, nx, 0, out, nx, 0, 1, live, s);
      if (rc) return rc;
    } else {
      PMK_RETURN_IF(!C.sy || !C.work1, PMK_ERR_ARG);
      const double *iym = C.iy ? C.iy : C.sy;
      // X Fx over all (slice, y) rows
      int rc = gemm(rows * ny, nx, nx, rhs, nx, 0, C.sx, nx, 0, C.work0, nx, 0, 1, live, s);
      if (rc) return rc;
      // Fy X_k per slice
      rc = gemm(ny, nx, ny, C.sy, ny, 0, C.work0, nx, m, C.work1, nx, m, rows, live, s);
      if (rc) return rc;
      if (chain) {
        if (C.n_steps > 0) rc = launch_eig_chain(C, C.work1, live, s);
        if (rc) return rc;
      } else {
        prof::Scope rs(prof::kRec, 16.0 * N, 0.0, s);
        dst_recurrence_kernel<<<(m + 255) / 256, 256, 0, s>>>(C.work1, C.delta, C.beta,
                                                             C.dropped, C.n_steps, m, 1.0, live);
      }
      PMK_LAUNCH_CHECK();
      rc = gemm(ny, nx, ny, iym, ny, 0, C.work1, nx, m, C.work0, nx, m, rows, live, s);
      if (rc) return rc;
      rc = gemm(rows * ny, nx, nx, C.work0, nx, 0, ixm, nx, 0, out, nx, 0, 1, live, s);
      if (rc) return rc;
    }
    // out_0 = rhs_0 exactly (stepper.py:118)
    {
      prof::Scope cs(prof::kCoarseMisc, 16.0 * m, 0.0, s);
      copy_row_kernel<<<(m + 255) / 256, 256, 0, s>>>(rhs, out, m, live);
    }
    PMK_LAUNCH_CHECK();
    return 0;
  }
  if (C.kind == PMK_COARSE_PCR || C.kind == PMK_COARSE_LINE) {
    {
      prof::Scope cs(prof::kCoarseMisc, 16.0 * m, 0.0, s);
      copy_row_kernel<<<(m + 255) / 256, 256, 0, s>>>(rhs, out, m, live);  // stepper.py:118
    }
    PMK_LAUNCH_CHECK();
    if (C.n_steps < 1) return 0;
    return C.kind == PMK_COARSE_PCR ? launch_pcr_chains(C, rhs, out, live, s)
                                    : launch_line_chains(C, rhs, out, live, s);
  }
  if (C.kind == PMK_COARSE_DENSE && C.seg_start && C.n_seg >= 1) {
    PMK_RETURN_IF(!C.dinv || !C.work0, PMK_ERR_ARG);
    static int blocks = 0;
    if (!blocks) {
      int b = 0;
      PMK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, dense_chain_kernel, 256, 0));
      blocks = (b > 0 ? b : 1) * kSMs;
    }
    const double steps = (double)(C.n_steps + 1);
    prof::Scope cs(prof::kChain, 8.0 * m * (double)m * C.n_seg + 32.0 * m * steps,
                   2.0 * m * (double)m * steps, s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PMK_CUDA_TRY(cudaLaunchKernelEx(&cfg, dense_chain_kernel, rhs, out, C.dinv, C.coupling, nx,
                                    ny, C.dropped, C.seg_start, C.n_seg, C.n_steps, C.work0,
                                    live));
    return 0;
  }
  if (C.kind == PMK_COARSE_DENSE) {  // (no chain table: one launch pair per slice)
    PMK_RETURN_IF(!C.dinv || !C.work0, PMK_ERR_ARG);
    {
      prof::Scope cs(prof::kCoarseMisc, 16.0 * m, 0.0, s);
      copy_row_kernel<<<(m + 255) / 256, 256, 0, s>>>(rhs, out, m, live);
    }
    PMK_LAUNCH_CHECK();
    const int cb = (m + 255) / 256 < 4 * kSMs ? (m + 255) / 256 : 4 * kSMs;
    const int gb = (m * 32 + 255) / 256;
    for (int k = 1; k <= C.n_steps; ++k) {
      {
        prof::Scope c1(prof::kCoarseMisc, 32.0 * m, 0.0, s);
        coupling_kernel<<<cb, 256, 0, s>>>(rhs + (int64_t)k * m, out + (int64_t)(k - 1) * m,
                                         C.work0, C.coupling, nx, ny, C.dropped, k, live);
      }
      PMK_LAUNCH_CHECK();
      prof::Scope c2(prof::kCoarseMisc, 8.0 * m * (double)m + 16.0 * m, 2.0 * m * (double)m, s);
      gemv_kernel<<<gb, 256, 0, s>>>(C.dinv, C.work0, out + (int64_t)k * m, m, live);
      PMK_LAUNCH_CHECK();
    }
    return 0;
  }
  return PMK_ERR_UNSUPPORTED;
}

}  // namespace pmk
