// pmk_lines.cu -- coarsest-level chains by per-slice direct solves that need
// no common eigenbasis (reference stepper.py:114-146, linalg.py:35-68,
// _chain.pyx:15-82):
//
//   PCR   1-D levels: D is tridiagonal.  Parallel cyclic reduction whose
//         matrix part (the reduction multipliers of every stride and the
//         final pivots) is factored once on the host, as the reference
//         factors once with factor_tridiag; a slice's solve is then
//         log2(m) shared-memory sweeps of the right-hand side only.  One
//         CTA per independent chain (perturb_decouple segments), all chains
//         in one launch.
//   LINE  2-D 5-point levels of any size whose operator is not separable
//         (a caller's own SpatialOperator): block-tridiagonal by grid lines,
//         block Thomas with the inverted Schur blocks G_j formed once on the
//         host (the SuperLU factorisation's role, linalg.py:42-55).  A slice
//         is 2 ny dense nx x nx products; one CTA per chain, one launch.
#include "pmk_internal.cuh"

namespace pmk {

namespace {

__device__ __forceinline__ double stencil_row_1d(const pmk_stencil &C, int m, int i,
                                                 const double *prev) {
  double cw, cc, ce;
  if (C.var) {
    cw = C.coef[m + i];
    cc = C.coef[2 * m + i];
    ce = C.coef[3 * m + i];
  } else {
    cw = C.c[1];
    cc = C.c[2];
    ce = C.c[3];
  }
  double acc = cc * prev[i];
  if (i > 0) acc = fma(cw, prev[i - 1], acc);
  if (i < m - 1) acc = fma(ce, prev[i + 1], acc);
  return acc;
}

// One CTA per chain.  Shared memory: x (previous slice), r0, r1 (ping-pong),
// m doubles each.  E = elements per thread (compile-time so that the next
// slice's right-hand side can wait in registers while this slice reduces).
template <int E>
__global__ void __launch_bounds__(1024)
    pcr_chain_kernel(const double *__restrict__ rhs, double *__restrict__ out, int m, int n_steps,
                     const double *__restrict__ alpha, const double *__restrict__ gamma,
                     const double *__restrict__ inv, int levels, pmk_stencil C,
                     const uint8_t *__restrict__ dropped, const int32_t *__restrict__ seg_start,
                     int n_seg, const int *live) {
  if (!is_live(live)) return;
  extern __shared__ double sh[];
  double *x = sh, *r0 = sh + m, *r1 = sh + 2 * m;
  const int sg = blockIdx.x;
  const int first = seg_start[sg];
  const int end = (sg + 1 < n_seg) ? seg_start[sg + 1] : n_steps + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  const bool cut = dropped && dropped[first];
  // previous slice of the chain's first row: out_0 = rhs_0 for the first
  // chain; cut chains start from nothing (stepper.py:107-112)
  double nxt[E], piv[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = tid + e * nt;
    if (i < m) {
      x[i] = cut ? 0.0 : rhs[(int64_t)(first - 1) * m + i];
      nxt[e] = rhs[(int64_t)first * m + i];
      piv[e] = inv[i];
    }
  }
  __syncthreads();
  for (int k = first; k < end; ++k) {
    const bool couple = !(k == first && cut);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = tid + e * nt;
      if (i < m) r0[i] = couple ? nxt[e] + stencil_row_1d(C, m, i, x) : nxt[e];
    }
    if (k + 1 < end) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = tid + e * nt;
        if (i < m) nxt[e] = rhs[(int64_t)(k + 1) * m + i];
      }
    }
    __syncthreads();
    double *src = r0, *dst = r1;
    for (int l = 0; l < levels; ++l) {
      const int s = 1 << l;
      const double *al = alpha + (int64_t)l * m, *ga = gamma + (int64_t)l * m;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = tid + e * nt;
        if (i < m) {
          double v = src[i];
          if (i - s >= 0) v = fma(__ldg(al + i), src[i - s], v);
          if (i + s < m) v = fma(__ldg(ga + i), src[i + s], v);
          dst[i] = v;
        }
      }
      __syncthreads();
      double *t = src;
      src = dst;
      dst = t;
    }
    double *ok = out + (int64_t)k * m;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = tid + e * nt;
      if (i < m) {
        const double v = src[i] * piv[e];
        x[i] = v;
        ok[i] = v;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ LINE
// y = G t for one line: G [nx][nx] row-major in global memory, t in shared
// memory; a warp per output row, lanes across columns.
__device__ __forceinline__ void line_gemv(const double *__restrict__ G, const double *t, int nx,
                                          double *y_sh, int warp, int nw, int lane) {
  for (int r = warp; r < nx; r += nw) {
    const double *g = G + (int64_t)r * nx;
    double acc = 0.0;
    for (int c = lane; c < nx; c += 32) acc = fma(__ldg(g + c), t[c], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y_sh[r] = acc;
  }
}

// One CTA per chain.  Per slice: b = rhs_k + [coupled] C x_{k-1}; forward
// y_j = G_j (b_j - l_j . y_{j-1}); backward x_j = y_j - G_j (u_j . x_{j+1}).
// `ybuf` holds the chain's y lines ([n_seg][m]); x_k goes straight to out.
__global__ void __launch_bounds__(512)
    line_chain_kernel(const double *__restrict__ rhs, double *__restrict__ out, int nx, int ny,
                      int n_steps, const double *__restrict__ G, const double *__restrict__ lo,
                      const double *__restrict__ up, pmk_stencil C,
                      const uint8_t *__restrict__ dropped,
                      const int32_t *__restrict__ seg_start, int n_seg,
                      double *__restrict__ ybuf, const int *live) {
  if (!is_live(live)) return;
  extern __shared__ double sh[];
  double *t = sh, *y = sh + nx;  // the line being multiplied / the product
  const int m = nx * ny;
  const int sg = blockIdx.x;
  const int first = seg_start[sg];
  const int end = (sg + 1 < n_seg) ? seg_start[sg + 1] : n_steps + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const bool cut = dropped && dropped[first];
  double *yb = ybuf + (int64_t)sg * m;
  for (int k = first; k < end; ++k) {
    const bool couple = !(k == first && cut);
    const double *rk = rhs + (int64_t)k * m;
    // out_0 = rhs_0 was written by the launcher's row copy; every other
    // chain's first row is cut and never reads its predecessor
    const double *prev = out + (int64_t)(k - 1) * m;
    double *xk = out + (int64_t)k * m;
    // forward sweep over lines
    for (int j = 0; j < ny; ++j) {
      for (int p = tid; p < nx; p += nt) {
        const int i = j * nx + p;
        double b = rk[i];
        if (couple) {
          double cs_, cw, cc, ce, cn;
          if (C.var) {
            cs_ = C.coef[i];
            cw = C.coef[m + i];
            cc = C.coef[2 * m + i];
            ce = C.coef[3 * m + i];
            cn = C.coef[4 * m + i];
          } else {
            cs_ = C.c[0];
            cw = C.c[1];
            cc = C.c[2];
            ce = C.c[3];
            cn = C.c[4];
          }
          double acc = cc * prev[i];
          if (j > 0) acc = fma(cs_, prev[i - nx], acc);
          if (p > 0) acc = fma(cw, prev[i - 1], acc);
          if (p < nx - 1) acc = fma(ce, prev[i + 1], acc);
          if (j < ny - 1) acc = fma(cn, prev[i + nx], acc);
          b += acc;
        }
        // y still holds y_{j-1} (written by the previous product)
        t[p] = (j > 0) ? fma(-lo[i], y[p], b) : b;
      }
      __syncthreads();
      line_gemv(G + (int64_t)j * nx * nx, t, nx, y, warp, nw, lane);
      __syncthreads();
      for (int p = tid; p < nx; p += nt) yb[j * nx + p] = y[p];
    }
    // backward sweep: x_{ny-1} = y_{ny-1}; y (shared) carries x_{j+1}
    for (int p = tid; p < nx; p += nt) xk[(ny - 1) * nx + p] = y[p];
    for (int j = ny - 2; j >= 0; --j) {
      __syncthreads();
      for (int p = tid; p < nx; p += nt) t[p] = up[j * nx + p] * y[p];
      __syncthreads();
      line_gemv(G + (int64_t)j * nx * nx, t, nx, y, warp, nw, lane);
      __syncthreads();
      for (int p = tid; p < nx; p += nt) {
        const double v = yb[j * nx + p] - y[p];
        y[p] = v;
        xk[j * nx + p] = v;
      }
    }
    __syncthreads();  // x_k complete (global, block scope) before slice k + 1 reads it
  }
}

}  // namespace

int launch_pcr_chains(const pmk_coarse &C, const double *rhs, double *out, const int *live,
                      cudaStream_t s) {
  const int m = C.nx;
  PMK_RETURN_IF(C.dim != 1 || !C.pcr_alpha || !C.pcr_gamma || !C.pcr_inv || !C.seg_start ||
                    C.n_seg < 1 || C.pcr_levels < 0,
                PMK_ERR_ARG);
  const size_t smem = 3 * (size_t)m * sizeof(double);
  PMK_RETURN_IF(smem > 220 * 1024, PMK_ERR_UNSUPPORTED);
  int threads = ((m + 31) / 32) * 32;
  if (threads > 1024) threads = 1024;
  const int E = (m + threads - 1) / threads;
  const double rows = (double)C.n_steps + 1.0;
  prof::Scope sc(prof::kChain, 16.0 * m * rows, (4.0 * C.pcr_levels + 7.0) * m * rows, s);
#define PMK_PCR_CASE(EE)                                                                         \
  case EE: {                                                                                     \
    static bool attr = false;                                                                    \
    if (!attr) {                                                                                 \
      PMK_CUDA_TRY(cudaFuncSetAttribute(pcr_chain_kernel<EE>,                                    \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,             \
                                        220 * 1024));                                            \
      attr = true;                                                                               \
    }                                                                                            \
    pcr_chain_kernel<EE><<<C.n_seg, threads, smem, s>>>(rhs, out, m, C.n_steps, C.pcr_alpha,     \
                                                         C.pcr_gamma, C.pcr_inv, C.pcr_levels,   \
                                                         C.coupling, C.dropped, C.seg_start,     \
                                                         C.n_seg, live);                         \
    break;                                                                                       \
  }
  switch (E) {
    PMK_PCR_CASE(1)
    PMK_PCR_CASE(2)
    PMK_PCR_CASE(3)
    PMK_PCR_CASE(4)
    PMK_PCR_CASE(5)
    PMK_PCR_CASE(6)
    PMK_PCR_CASE(7)
    PMK_PCR_CASE(8)
    PMK_PCR_CASE(9)
    default:
      return PMK_ERR_UNSUPPORTED;
  }
#undef PMK_PCR_CASE
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_line_chains(const pmk_coarse &C, const double *rhs, double *out, const int *live,
                       cudaStream_t s) {
  PMK_RETURN_IF(C.dim != 2 || !C.line_g || !C.line_l || !C.line_u || !C.seg_start ||
                    C.n_seg < 1 || !C.work0,
                PMK_ERR_ARG);
  const int nx = C.nx, ny = C.ny;
  const size_t smem = 2 * (size_t)nx * sizeof(double);
  PMK_RETURN_IF(smem > 48 * 1024, PMK_ERR_UNSUPPORTED);
  const double m = (double)nx * ny, rows = (double)C.n_steps + 1.0;
  prof::Scope sc(prof::kChain, 16.0 * m * rows + 16.0 * m * nx * rows, 4.0 * m * nx * rows, s);
  line_chain_kernel<<<C.n_seg, 512, smem, s>>>(rhs, out, nx, ny, C.n_steps, C.line_g, C.line_l,
                                               C.line_u, C.coupling, C.dropped, C.seg_start,
                                               C.n_seg, C.work0, live);
  PMK_LAUNCH_CHECK();
  return 0;
}

}  // namespace pmk
