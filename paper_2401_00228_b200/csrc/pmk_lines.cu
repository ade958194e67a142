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
//         is 2 ny dense nx x nx products; one thread-block cluster per chain
//         (rows of G_j split over its CTAs, lines exchanged through
//         distributed shared memory), one launch.
#include <cooperative_groups.h>

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
                     int n_seg, const int *live, int stage_tables) {
  if (!is_live(live)) return;
  extern __shared__ double sh[];
  double *x = sh, *r0 = sh + m, *r1 = sh + 2 * m;
  // the multipliers of every stride, staged once per CTA when they fit
  // (2 levels m doubles next to the three rows), else read through L1
  if (stage_tables) {
    double *ta = sh + 3 * m, *tg = ta + (size_t)levels * m;
    for (int i = threadIdx.x; i < levels * m; i += blockDim.x) {
      ta[i] = alpha[i];
      tg[i] = gamma[i];
    }
    alpha = ta;
    gamma = tg;
  }
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
          if (i - s >= 0) v = fma(al[i], src[i - s], v);
          if (i + s < m) v = fma(ga[i], src[i + s], v);
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
// One thread-block cluster of CS CTAs per chain.  CTA g owns rows
// [g R, g R + R) of every Schur-block inverse G_j, stored by the host as
// [j][g][r][c] (row-major chunks).  Per slice:
//   b   = rhs_k + [coupled] C x_{k-1}            (all cluster threads)
//   forward   y_j = G_j (b_j - l_j . y_{j-1}),   j = 0 .. ny-1
//   backward  x_j = y_j - G_j (u_j . x_{j+1}),   j = ny-2 .. 0
// Each product: every CTA forms the full input line t in its own shared
// memory; warp w multiplies rows w, w + 16, ... of the CTA's chunk (lanes
// across columns, a shuffle tree per row) and lanes 0..CS-1 send the result
// to every CTA's line buffer with st.async, which also credits the bytes to
// the receiving CTA's mbarrier: a CTA starts product n + 1 as soon as the nx
// values of product n have landed in its own shared memory -- no cluster-wide
// barrier inside a sweep (cluster.sync costs more than the product itself).
// Line buffers and mbarriers alternate with the product's parity; a peer can
// only send product n + 2 after it has received this CTA's product n + 1,
// i.e. after this CTA has read buffer n & 1 for the last time.
// Nothing a product reads from global memory depends on the previous product
// (G, l, u, b, y), so it is fetched into registers one product ahead: RW rows
// per warp x NQ columns per lane of G (RW = 0: streamed instead, long lines).
struct LineArgs {
  const double *rhs;
  double *out;
  int nx, ny, n_steps, R;
  const double *G, *lo, *up;
  pmk_stencil C;
  const uint8_t *dropped;
  const int32_t *seg_start;
  int n_seg;
  double *work;  // [n_seg][2][m]: b lines, y lines
  const int *live;
};

constexpr int kLineThreads = 512, kLineWarps = kLineThreads / 32, kLinePE = 3;

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void send_f64(uint32_t remote, double v, uint32_t remote_bar) {
  asm volatile(
      "st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
          remote),
      "l"(__double_as_longlong(v)), "r"(remote_bar)
      : "memory");
}
__device__ __forceinline__ void bar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int RW, int NQ>
__global__ void __launch_bounds__(kLineThreads) line_chain_kernel(LineArgs a) {
  namespace cg = cooperative_groups;
  if (!is_live(a.live)) return;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), g = (int)cl.block_rank();
  const int nx = a.nx, ny = a.ny, R = a.R, m = nx * ny;
  extern __shared__ double sh[];
  __shared__ __align__(8) unsigned long long bars[2];
  double *t = sh;
  double *const line0 = sh + nx, *const line1 = sh + 2 * nx;
  const int sg = blockIdx.x / CS;
  const int first = a.seg_start[sg];
  const int end = (sg + 1 < a.n_seg) ? a.seg_start[sg + 1] : a.n_steps + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = g * R;
  const bool cut = a.dropped && a.dropped[first];
  double *bbuf = a.work + (int64_t)sg * 2 * m, *ybuf = bbuf + m;
  const int64_t gstride = (int64_t)nx * R;  // one (j, g) chunk
  const uint32_t bar0 = smem_addr(&bars[0]), bar1 = smem_addr(&bars[1]);
  // this lane's peer (lanes 0 .. CS-1): its line buffers and mbarriers
  uint32_t peer_line0 = 0, peer_line1 = 0, peer_bar0 = 0, peer_bar1 = 0;
  if (lane < CS) {
    peer_line0 = peer_addr(smem_addr(line0), lane);
    peer_line1 = peer_addr(smem_addr(line1), lane);
    peer_bar0 = peer_addr(bar0, lane);
    peer_bar1 = peer_addr(bar1, lane);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  constexpr int RWc = RW > 0 ? RW : 1, NQc = RW > 0 ? NQ : 1;
  double gq[RWc][NQc];              // G_j values of this thread's rows / columns
  double p0[kLinePE], p1[kLinePE];  // next line: (b, l) forward, (u, -) backward
  double yq[RWc] = {};              // backward: y_j of this warp's rows (lane 0)
  auto row_of = [&](int i) { return warp + i * kLineWarps; };
  auto row_ok = [&](int i) { return row_of(i) < R && row0 + row_of(i) < nx; };
  auto fetch_g = [&](int j) {
    if (RW > 0) {
      const double *Gc = a.G + ((int64_t)j * CS + g) * gstride;
#pragma unroll
      for (int i = 0; i < RWc; ++i)
#pragma unroll
        for (int q = 0; q < NQc; ++q) {
          const int c = lane + 32 * q;
          gq[i][q] = (row_ok(i) && c < nx) ? __ldg(Gc + (int64_t)row_of(i) * nx + c) : 0.0;
        }
    }
  };
  uint32_t n = 0;  // products issued so far (all CTAs of the cluster in step)
  // wait for the nx values of product q in this CTA's line buffer q & 1
  auto wait_product = [&](uint32_t q) { bar_wait((q & 1) ? bar1 : bar0, (q >> 1) & 1); };
  // One product: t is ready in shared memory (block barrier passed).  Row r's
  // result is fin(r, sum) -- sent to every CTA's line buffer n & 1.
  auto product = [&](int j, auto &&prefetch, auto &&fin) {
    const uint32_t dst_line = (n & 1) ? peer_line1 : peer_line0;
    const uint32_t dst_bar = (n & 1) ? peer_bar1 : peer_bar0;
    if (RW > 0) {
      double res[RWc];
#pragma unroll
      for (int i = 0; i < RWc; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < NQc; ++q) {
          const int c = lane + 32 * q;
          if (c < nx) acc = fma(gq[i][q], t[c], acc);
        }
        res[i] = acc;
      }
      double ycur[RWc];
#pragma unroll
      for (int i = 0; i < RWc; ++i) ycur[i] = yq[i];
      prefetch();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < RWc; ++i) res[i] += __shfl_xor_sync(0xffffffffu, res[i], o);
#pragma unroll
      for (int i = 0; i < RWc; ++i)
        if (row_ok(i)) {
          const int idx = row0 + row_of(i);
          double v = 0.0;
          if (lane == 0) v = fin(idx, res[i], ycur[i]);
          v = __shfl_sync(0xffffffffu, v, 0);
          if (lane < CS) send_f64(dst_line + 8u * idx, v, dst_bar);
        }
    } else {
      const double *Gc = a.G + ((int64_t)j * CS + g) * gstride;
      for (int rl = warp; rl < R && row0 + rl < nx; rl += kLineWarps) {
        double acc = 0.0;
#pragma unroll 4
        for (int c = lane; c < nx; c += 32)
          acc = fma(__ldg(Gc + (int64_t)rl * nx + c), t[c], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const int idx = row0 + rl;
        double v = 0.0;
        if (lane == 0) v = fin(idx, acc, 0.0);
        v = __shfl_sync(0xffffffffu, v, 0);
        if (lane < CS) send_f64(dst_line + 8u * idx, v, dst_bar);
      }
      prefetch();
    }
    ++n;
  };
  for (int k = first; k < end; ++k) {
    const bool couple = !(k == first && cut);
    const double *rk = a.rhs + (int64_t)k * m;
    // out_0 = rhs_0 was written by the launcher's row copy; every other
    // chain's first row is cut and never reads its predecessor
    const double *prev = a.out + (int64_t)(k - 1) * m;
    double *xk = a.out + (int64_t)k * m;
    fetch_g(0);
    for (int i = g * kLineThreads + tid; i < m; i += CS * kLineThreads) {
      double b = rk[i];
      if (couple) {
        const int j = i / nx, p = i - j * nx;
        double cs_, cw, cc, ce, cn;
        if (a.C.var) {
          cs_ = a.C.coef[i];
          cw = a.C.coef[m + i];
          cc = a.C.coef[2 * m + i];
          ce = a.C.coef[3 * m + i];
          cn = a.C.coef[4 * m + i];
        } else {
          cs_ = a.C.c[0];
          cw = a.C.c[1];
          cc = a.C.c[2];
          ce = a.C.c[3];
          cn = a.C.c[4];
        }
        double acc = cc * prev[i];
        if (j > 0) acc = fma(cs_, prev[i - nx], acc);
        if (p > 0) acc = fma(cw, prev[i - 1], acc);
        if (p < nx - 1) acc = fma(ce, prev[i + 1], acc);
        if (j < ny - 1) acc = fma(cn, prev[i + nx], acc);
        b += acc;
      }
      bbuf[i] = b;
    }
    cl.sync();  // b complete (global memory, cluster scope)
#pragma unroll
    for (int e = 0; e < kLinePE; ++e) {
      const int p = tid + e * kLineThreads;
      p0[e] = p < nx ? bbuf[p] : 0.0;
      p1[e] = 0.0;
    }
    // forward sweep
    for (int j = 0; j < ny; ++j) {
      if (j > 0) wait_product(n - 1);
      if (tid == 0) bar_expect((n & 1) ? bar1 : bar0, 8u * (uint32_t)nx);
      const double *yp = ((n - 1) & 1) ? line1 : line0;  // y_{j-1}
#pragma unroll
      for (int e = 0; e < kLinePE; ++e) {
        const int p = tid + e * kLineThreads;
        if (p < nx) t[p] = (j > 0) ? fma(-p1[e], yp[p], p0[e]) : p0[e];
      }
      __syncthreads();
      // next product's operands: line j + 1 forward, or the first backward one
      const int jn = (j + 1 < ny) ? j + 1 : ny - 2;
      product(
          j,
          [&]() {
            if (jn < 0) return;
            fetch_g(jn);
#pragma unroll
            for (int e = 0; e < kLinePE; ++e) {
              const int p = tid + e * kLineThreads;
              if (p < nx) {
                if (j + 1 < ny) {
                  p0[e] = bbuf[jn * nx + p];
                  p1[e] = a.lo[jn * nx + p];
                } else {
                  p0[e] = a.up[jn * nx + p];
                }
              }
            }
            if (RW > 0 && j + 1 == ny && lane == 0) {  // y of the first backward product
#pragma unroll
              for (int i = 0; i < RWc; ++i)
                if (row_ok(i)) yq[i] = ybuf[jn * nx + row0 + row_of(i)];
            }
          },
          [&](int idx, double y, double) {
            ybuf[j * nx + idx] = y;
            if (j == ny - 1) xk[j * nx + idx] = y;  // x_{ny-1} = y_{ny-1}
            return y;
          });
    }
    // backward sweep: the previous product's line is x_{j+1}
    for (int j = ny - 2; j >= 0; --j) {
      wait_product(n - 1);
      if (tid == 0) bar_expect((n & 1) ? bar1 : bar0, 8u * (uint32_t)nx);
      const double *xp = ((n - 1) & 1) ? line1 : line0;
#pragma unroll
      for (int e = 0; e < kLinePE; ++e) {
        const int p = tid + e * kLineThreads;
        if (p < nx) t[p] = p0[e] * xp[p];
      }
      __syncthreads();
      product(
          j,
          [&]() {
            if (j == 0) return;
            fetch_g(j - 1);
#pragma unroll
            for (int e = 0; e < kLinePE; ++e) {
              const int p = tid + e * kLineThreads;
              if (p < nx) p0[e] = a.up[(j - 1) * nx + p];
            }
            if (RW > 0 && lane == 0) {
#pragma unroll
              for (int i = 0; i < RWc; ++i)
                if (row_ok(i)) yq[i] = ybuf[(j - 1) * nx + row0 + row_of(i)];
            }
          },
          [&](int idx, double s, double yj) {
            // y_j: fetched one product ahead (RW > 0), written by this thread
            const double v = (RW > 0 ? yj : ybuf[j * nx + idx]) - s;
            xk[j * nx + idx] = v;
            return v;
          });
    }
    wait_product(n - 1);  // every product is consumed: parities stay in step
    cl.sync();            // x_k complete (global memory, cluster scope)
  }
}

}  // namespace

int launch_pcr_chains(const pmk_coarse &C, const double *rhs, double *out, const int *live,
                      cudaStream_t s) {
  const int m = C.nx;
  PMK_RETURN_IF(C.dim != 1 || !C.pcr_alpha || !C.pcr_gamma || !C.pcr_inv || !C.seg_start ||
                    C.n_seg < 1 || C.pcr_levels < 0,
                PMK_ERR_ARG);
  size_t smem = 3 * (size_t)m * sizeof(double);
  PMK_RETURN_IF(smem > 220 * 1024, PMK_ERR_UNSUPPORTED);
  const size_t tabs = 2 * (size_t)C.pcr_levels * m * sizeof(double);
  const int stage_tables = (C.pcr_levels > 0 && smem + tabs <= 220 * 1024) ? 1 : 0;
  if (stage_tables) smem += tabs;
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
                                                         C.n_seg, live, stage_tables);           \
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
                    C.n_seg < 1 || !C.work0 || C.line_cs < 1 || C.line_cs > 8,
                PMK_ERR_ARG);
  const int nx = C.nx, ny = C.ny, CS = C.line_cs;
  const int R = (nx + CS - 1) / CS;
  PMK_RETURN_IF(nx > kLinePE * kLineThreads, PMK_ERR_UNSUPPORTED);
  const size_t smem = 3 * (size_t)nx * sizeof(double);
  const int rw = (R + kLineWarps - 1) / kLineWarps;  // rows per warp
  const int nq = (nx + 31) / 32;                      // columns per lane
  const double m = (double)nx * ny, rows = (double)C.n_steps + 1.0;
  prof::Scope sc(prof::kChain, 16.0 * m * rows + 16.0 * m * nx * rows, 4.0 * m * nx * rows, s);
  LineArgs a;
  a.rhs = rhs;
  a.out = out;
  a.nx = nx;
  a.ny = ny;
  a.n_steps = C.n_steps;
  a.R = R;
  a.G = C.line_g;
  a.lo = C.line_l;
  a.up = C.line_u;
  a.C = C.coupling;
  a.dropped = C.dropped;
  a.seg_start = C.seg_start;
  a.n_seg = C.n_seg;
  a.work = C.work0;
  a.live = live;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C.n_seg * CS), 1, 1);
  cfg.blockDim = dim3((unsigned)kLineThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // register-resident G: RW rows per warp x NQ columns per lane (<= 32 values)
#define PMK_LINE_TRY(RWv, NQv)                                                     \
  if (rw <= RWv && nq <= NQv) {                                                    \
    PMK_CUDA_TRY(cudaLaunchKernelEx(&cfg, line_chain_kernel<RWv, NQv>, a));        \
    return 0;                                                                      \
  }
  PMK_LINE_TRY(1, 2)
  PMK_LINE_TRY(1, 4)
  PMK_LINE_TRY(2, 4)
  PMK_LINE_TRY(1, 8)
  PMK_LINE_TRY(2, 8)
  PMK_LINE_TRY(4, 4)
  PMK_LINE_TRY(4, 8)
  PMK_LINE_TRY(8, 4)
  PMK_LINE_TRY(1, 16)
  PMK_LINE_TRY(2, 16)
#undef PMK_LINE_TRY
  PMK_CUDA_TRY(cudaLaunchKernelEx(&cfg, line_chain_kernel<0, 0>, a));
  return 0;
}

}  // namespace pmk
