// pmk_dst.cu -- fast sine transforms for the coarsest-level solve.
//
// The coarsest forward substitution (reference stepper.py:114-146) is
// diagonal in the sine basis (pmk_coarse.cu).  This file replaces the dense
// fp64 GEMMs that applied the basis (2 (n_x + n_y) flop per unknown per
// transform, compute-bound) by O(n log n) DST-I transforms.
//
// DST-I of length n = N - 1 (N a power of two), X_p = sum_j x_j sin(pi j p/N),
// through one N-point complex FFT: with z the odd extension of x (length 2N),
// w_j = z_{2j} + i z_{2j+1}, W = FFT_N(w),
//   X_p = [ c (a_r - b_r) + s (a_i + b_i) - (a_i - b_i) ] / 4,
//   A = W_p, B = W_{N-p}, c + i s = e^{i pi p / N}
// (the real-input split of the length-2N transform of z, whose bins are
// -2i X_p).
//
// FFT_N as a register four-step, N = N1 * N2 (N1 >= N2, both <= 32):
//   lane (group h, n2) loads w[N2 n1 + n2], n1 < N1, straight from the input
//   (consecutive lanes read consecutive pairs), runs an N1-point FFT in
//   registers, multiplies by w_N^{n2 k1}, and stores its column to a padded
//   shared buffer; each lane then runs N1/N2 N2-point FFTs over rows of that
//   buffer in registers and writes W in natural order back for the unpack.
//   Shared-memory traffic is ~3 N complex accesses per transform (a radix-2
//   shared-memory FFT moves ~5 N log2 N); 32 / N2 transforms run per warp,
//   synchronised with __syncwarp only.
// x-direction: rows contiguous, groups of N2 lanes per row.
// y-direction: a CTA stages a (ny x 16) column tile of one slice (coalesced
// 128-byte row segments) and transforms its 16 columns from shared memory.
// Unnormalised: applying it twice gives (N/2) x; the solver folds the
// orthonormal factors into the recurrence.
#include <cmath>
#include <mutex>

#include "pmk_internal.cuh"

namespace pmk {
namespace {

#ifndef PMK_DST_WARPS
#define PMK_DST_WARPS 8
#endif
#ifndef PMK_DST_COLTILE
#define PMK_DST_COLTILE 16
#endif
constexpr int kDstWarps = PMK_DST_WARPS;
constexpr int kColTile = PMK_DST_COLTILE;
// Row transforms: smaller CTAs under a register cap keep more warps resident
// (the kernel is latency-bound at 114 registers x 8 warps x 2 CTAs = 16 warps
// per SM): 6 warps x 3 CTAs = 18 warps at 96 registers, no spills up to
// N = 256 (longer transforms keep their registers).  c5_c coarsest solve
// (tools/coarse_probe.py): 0.472 ms vs 0.499 (8 warps x 2 CTAs), 0.478 (5 x 4),
// 0.479 (4 x 5).  The
// column kernel's shared-memory tile keeps it at 2 CTAs either way.
#ifndef PMK_DST_ROW_WARPS
#define PMK_DST_ROW_WARPS 6
#endif
#ifndef PMK_DST_ROW_BLOCKS
#define PMK_DST_ROW_BLOCKS 3
#endif
constexpr int kRowWarps = PMK_DST_ROW_WARPS;
constexpr int kRowBlocks = PMK_DST_ROW_BLOCKS;

// e^{-2 pi i j / 32}, j < 32: radix-2 twiddles of every in-register FFT
// (length L <= 32 uses entries j * 32 / L).
__constant__ double2 c_tw32[32];

__device__ __forceinline__ double2 cmul(double2 v, double2 w) {
  return make_double2(fma(v.x, w.x, -v.y * w.y), fma(v.x, w.y, v.y * w.x));
}

template <int L>
struct Log2 {
  static constexpr int value = 1 + Log2<L / 2>::value;
};
template <>
struct Log2<1> {
  static constexpr int value = 0;
};

// In-register radix-2 DIF FFT of length L: natural order in, bit-reversed
// order out (a[i] = A[bitrev(i)]).  One template instantiation per stage so
// that every register index is a compile-time constant (the array must not
// fall back to local memory).
template <int L, int S>
struct DifStage {
  static __device__ __forceinline__ void run(double2 (&a)[L]) {
    constexpr int half = 1 << (S - 1);
#pragma unroll
    for (int g = 0; g < L; g += 2 * half) {
#pragma unroll
      for (int pos = 0; pos < half; ++pos) {
        const double2 u = a[g + pos], v = a[g + pos + half];
        a[g + pos] = make_double2(u.x + v.x, u.y + v.y);
        const double2 d = make_double2(u.x - v.x, u.y - v.y);
        a[g + pos + half] = (pos == 0) ? d : cmul(d, c_tw32[pos * (32 >> S)]);
      }
    }
    DifStage<L, S - 1>::run(a);
  }
};
template <int L>
struct DifStage<L, 0> {
  static __device__ __forceinline__ void run(double2 (&)[L]) {}
};

template <int L>
__device__ __forceinline__ void fft_reg_dif(double2 (&a)[L]) {
  DifStage<L, Log2<L>::value>::run(a);
}

// compile-time bit reversal of B-bit indices (register subscripts)
template <int B>
struct ConstBrev {
  static constexpr __host__ __device__ int of(int v) {
    int r = 0;
    for (int b = 0; b < B; ++b) r |= ((v >> b) & 1) << (B - 1 - b);
    return r;
  }
};

__device__ __forceinline__ int brev_bits(int v, int bits) {
  return bits ? (int)(__brev((unsigned)v) >> (32 - bits)) : 0;
}

template <int LOGN>
struct Plan {
  static constexpr int N = 1 << LOGN;
  static constexpr int N2 = 1 << (LOGN / 2);  // lanes per transform
  static constexpr int N1 = N / N2;           // registers per lane (>= N2)
  static constexpr int TPW = 32 / N2;         // transforms per warp
  static constexpr int BS = N1 * (N2 + 1);    // padded buffer per transform (double2)
};

// One DST-I of length N - 1 by the N2 lanes of one group.  get(j) returns
// x_{j+1}; put(p, X_p) receives p = 1..N-1.  buf: the group's buffer.
template <int LOGN, typename Get, typename Put>
__device__ __forceinline__ void dst_group(Get get, Put put, double2 *buf, const double2 *tw2,
                                          const double2 *post, int n2) {
  using P = Plan<LOGN>;
  constexpr int N = P::N, N1 = P::N1, N2 = P::N2;
  auto z = [&](int q) -> double {  // odd extension, q in [0, 2N)
    if (q == 0 || q == N) return 0.0;
    return q < N ? get(q - 1) : -get(2 * N - q - 1);
  };
  // step 1: column FFTs (length N1) in registers
  double2 a[N1];
#pragma unroll
  for (int n1 = 0; n1 < N1; ++n1) {
    const int mq = N2 * n1 + n2;
    a[n1] = make_double2(z(2 * mq), z(2 * mq + 1));
  }
  fft_reg_dif<N1>(a);  // a[i] = A[k1 = bitrev(i)]
  // twiddle w_N^{n2 k1}; transpose through the padded buffer
  constexpr int LG1 = Log2<N1>::value, LG2 = Log2<N2>::value;
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    const int k1 = brev_bits(i, LG1);
    const double2 t = (i == 0) ? a[i] : cmul(a[i], tw2[k1 * N2 + n2]);
    buf[k1 * (N2 + 1) + n2] = t;
  }
  __syncwarp();
  // step 2: row FFTs (length N2); lane n2 owns k1 = n2 + N2 r
  double2 c[N1 / N2][N2];
#pragma unroll
  for (int r = 0; r < N1 / N2; ++r) {
    const int k1 = n2 + N2 * r;
#pragma unroll
    for (int q = 0; q < N2; ++q) c[r][q] = buf[k1 * (N2 + 1) + q];
    fft_reg_dif<N2>(c[r]);  // c[r][i] = C[k1][k2 = bitrev(i)]
  }
  // Unpack X_p = [c (a_r - b_r) + s (a_i + b_i) - (a_i - b_i)] / 4 with
  // A = W_p, B = W_{N-p}.  Lane n2 holds W_k for k = k1 + N1 k2, k1 = n2 +
  // N2 r (register c[r][bitrev(k2)]); W_{N-p} sits in lane (N2 - n2) mod N2
  // at (r', k2') = (R-1-r, N2-1-k2), or for lane 0 at (R-r mod R, ...) in its
  // own registers -- a register shuffle instead of a shared-memory round trip.
  constexpr int RR = N1 / N2;
  const int src = (threadIdx.x & 31) - n2 + ((N2 - n2) & (N2 - 1));
#pragma unroll
  for (int r = 0; r < RR; ++r) {
#pragma unroll
    for (int i = 0; i < N2; ++i) {
      const int k2 = ConstBrev<LG2>::of(i);
      const int ib = ConstBrev<LG2>::of(N2 - 1 - k2);   // partner register, lanes != 0
      const int r0 = (r == 0) ? 0 : RR - r;              // lane 0: own registers
      const int i0 = ConstBrev<LG2>::of((r == 0) ? ((N2 - k2) & (N2 - 1)) : N2 - 1 - k2);
      double2 B;
      B.x = __shfl_sync(0xffffffffu, c[RR - 1 - r][ib].x, src);
      B.y = __shfl_sync(0xffffffffu, c[RR - 1 - r][ib].y, src);
      if (n2 == 0) B = c[r0][i0];
      const int p = n2 + N2 * r + N1 * k2;
      if (p != 0) {
        const double2 A = c[r][i], cs = post[p];
        put(p, 0.25 * (cs.x * (A.x - B.x) + cs.y * (A.y + B.y) - (A.y - B.y)));
      }
    }
  }
  __syncwarp();
}

// Shared layout: [tw2: N] [post: N] [group buffers] ([tile]) (double2 units)
template <int LOGN>
__device__ __forceinline__ void load_tables(double2 *tw2, double2 *post, const double2 *gtw2,
                                            const double2 *gpost) {
  constexpr int N = 1 << LOGN;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    tw2[i] = gtw2[i];
    post[i] = gpost[i];
  }
}

template <int LOGN>
__global__ void __launch_bounds__(32 * kRowWarps, LOGN <= 8 ? kRowBlocks : 1)
    dst_rows_kernel(const double *__restrict__ in, double *__restrict__ out, int64_t rows,
                    int64_t rps, int64_t oss, const double2 *gtw2, const double2 *gpost,
                    const int *live) {
  if (!is_live(live)) return;
  using P = Plan<LOGN>;
  constexpr int N = P::N, n = N - 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2 *tw2 = reinterpret_cast<double2 *>(smem_raw);
  double2 *post = tw2 + N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = lane / P::N2, n2 = lane % P::N2;
  double2 *buf = post + N + (warp * P::TPW + h) * P::BS;
  load_tables<LOGN>(tw2, post, gtw2, gpost);
  __syncthreads();
  const int64_t per_iter = (int64_t)gridDim.x * kRowWarps * P::TPW;
  for (int64_t r0 = ((int64_t)blockIdx.x * kRowWarps + warp) * P::TPW; r0 < rows;
       r0 += per_iter) {
    const int64_t r = r0 + h;
    const bool ok = r < rows;
    const int64_t rr = ok ? r : 0;
    const double *x = in + rr * n;
    // output row: slice rr / rps at stride oss (contiguous when oss = rps * n)
    double *y = out + (rr / rps) * oss + (rr % rps) * n;
    dst_group<LOGN>([&](int j) { return ok ? __ldg(x + j) : 0.0; },
                    [&](int p, double v) {
                      if (ok) y[p - 1] = v;
                    },
                    buf, tw2, post, n2);
  }
}

template <int LOGN>
__global__ void __launch_bounds__(32 * kDstWarps)
    dst_cols_kernel(const double *__restrict__ in, double *__restrict__ out, int nx, int slices,
                    const double2 *gtw2, const double2 *gpost, const int *live) {
  if (!is_live(live)) return;
  using P = Plan<LOGN>;
  constexpr int N = P::N, ny = N - 1;
  constexpr int TS = kColTile + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2 *tw2 = reinterpret_cast<double2 *>(smem_raw);
  double2 *post = tw2 + N;
  double2 *bufs = post + N;
  double *tile = reinterpret_cast<double *>(bufs + kDstWarps * P::TPW * P::BS);  // [ny][TS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = lane / P::N2, n2 = lane % P::N2;
  double2 *buf = bufs + (warp * P::TPW + h) * P::BS;
  load_tables<LOGN>(tw2, post, gtw2, gpost);
  const int xblocks = (nx + kColTile - 1) / kColTile;
  const int64_t m = (int64_t)nx * ny;
  constexpr int GROUPS = kDstWarps * P::TPW;
  for (int64_t item = blockIdx.x; item < (int64_t)slices * xblocks; item += gridDim.x) {
    const int64_t k = item / xblocks;
    const int x0 = (int)(item - k * xblocks) * kColTile;
    const int cw = min(kColTile, nx - x0);
    const double *src = in + k * m + x0;
    // stage the tile: all of a thread's loads issued before the first use
    constexpr int kThreads = 32 * kDstWarps;
    constexpr int ITEMS = (ny * kColTile + kThreads - 1) / kThreads;
    double vals[ITEMS];
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int idx = threadIdx.x + u * kThreads;
      const int yy = idx / kColTile, c = idx - yy * kColTile;
      vals[u] = (idx < ny * kColTile && c < cw) ? __ldg(src + (int64_t)yy * nx + c) : 0.0;
    }
    __syncthreads();  // previous tile stored; tables loaded
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int idx = threadIdx.x + u * kThreads;
      const int yy = idx / kColTile, c = idx - yy * kColTile;
      if (idx < ny * kColTile) tile[yy * TS + c] = vals[u];
    }
    __syncthreads();
    for (int c0 = 0; c0 < cw; c0 += GROUPS) {
      const int c = c0 + warp * P::TPW + h;
      const bool ok = c < cw;
      double *col = tile + (ok ? c : 0);
      dst_group<LOGN>([&](int j) { return ok ? col[j * TS] : 0.0; },
                      [&](int p, double v) {
                        if (ok) col[(p - 1) * TS] = v;
                      },
                      buf, tw2, post, n2);
    }
    __syncthreads();
    double *dst = out + k * m + x0;
    for (int idx = threadIdx.x; idx < ny * kColTile; idx += blockDim.x) {
      const int yy = idx / kColTile, c = idx - yy * kColTile;
      if (c < cw) dst[(int64_t)yy * nx + c] = tile[yy * TS + c];
    }
  }
}

std::once_flag g_tw_once;
int g_tw_rc = -1;
int init_constants() {
  std::call_once(g_tw_once, [] {
    double2 h[32];
    for (int j = 0; j < 32; ++j) {
      const double ang = -2.0 * 3.14159265358979323846 * j / 32.0;
      h[j] = make_double2(std::cos(ang), std::sin(ang));
    }
    g_tw_rc = (int)cudaMemcpyToSymbol(c_tw32, h, sizeof(h));
  });
  return g_tw_rc;
}

template <int LOGN, bool COLS>
int run_dst(const double *in, double *out, int64_t rows_or_slices, int nx, const double *tables,
            const int *live, cudaStream_t s, int64_t rps = 0, int64_t oss = 0) {
  using P = Plan<LOGN>;
  constexpr int N = P::N;
  const int rc0 = init_constants();
  if (rc0) return rc0;
  constexpr int kWarps = COLS ? kDstWarps : kRowWarps;
  size_t smem = (size_t)(2 * N + kWarps * P::TPW * P::BS) * sizeof(double2);
  if (COLS) smem += (size_t)(N - 1) * (kColTile + 1) * sizeof(double);
  void (*kern)(const double *, double *, int, int, const double2 *, const double2 *,
               const int *) = dst_cols_kernel<LOGN>;
  void (*kern_r)(const double *, double *, int64_t, int64_t, int64_t, const double2 *,
                 const double2 *, const int *) = dst_rows_kernel<LOGN>;
  static int occ = -1;
  if (occ < 0) {
    int b = 0;
    if (COLS) {
      PMK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      PMK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 32 * kDstWarps, smem));
    } else {
      PMK_CUDA_TRY(cudaFuncSetAttribute(kern_r, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      PMK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern_r, 32 * kRowWarps, smem));
    }
    occ = b > 0 ? b : 1;
  }
  const double2 *tw2 = reinterpret_cast<const double2 *>(tables);
  const double2 *post = tw2 + N;
  double elems;
  int64_t need;
  if (COLS) {
    need = rows_or_slices * ((nx + kColTile - 1) / kColTile);
    elems = (double)rows_or_slices * nx * (N - 1);
  } else {
    need = (rows_or_slices + kRowWarps * P::TPW - 1) / (kRowWarps * P::TPW);
    elems = (double)rows_or_slices * (N - 1);
  }
  const double units = elems / (N - 1);
  const int grid = (int)(need < (int64_t)occ * kSMs ? need : (int64_t)occ * kSMs);
  prof::Scope scope(prof::kDst, 16.0 * elems, units * (5.0 * N * LOGN + 8.0 * N), s);
  if (COLS)
    kern<<<grid, 32 * kDstWarps, smem, s>>>(in, out, nx, (int)rows_or_slices, tw2, post, live);
  else {
    if (rps <= 0) {
      rps = rows_or_slices;
      oss = rows_or_slices * (N - 1);
    }
    kern_r<<<grid, 32 * kRowWarps, smem, s>>>(in, out, rows_or_slices, rps, oss, tw2, post,
                                              live);
  }
  PMK_LAUNCH_CHECK();
  return 0;
}

int log2_exact(int n1) {
  int l = 0;
  while ((1 << l) < n1) ++l;
  return ((1 << l) == n1) ? l : -1;
}

}  // namespace

// DST of every contiguous row of length n (n + 1 = 2^2 .. 2^10).  tables:
// [N] w_N^{n2 k1} at [k1 * N2 + n2] (N2 = 2^floor(log2(N)/2)), then [N]
// (cos, sin)(pi p / N), interleaved complex.
int launch_dst_rows(const double *in, double *out, int n, int64_t rows, const double *tables,
                    const int *live, cudaStream_t s, int64_t rps, int64_t oss) {
  switch (log2_exact(n + 1)) {
    case 2: return run_dst<2, false>(in, out, rows, 0, tables, live, s, rps, oss);
    case 3: return run_dst<3, false>(in, out, rows, 0, tables, live, s, rps, oss);
    case 4: return run_dst<4, false>(in, out, rows, 0, tables, live, s, rps, oss);
    case 5: return run_dst<5, false>(in, out, rows, 0, tables, live, s, rps, oss);
    case 6: return run_dst<6, false>(in, out, rows, 0, tables, live, s, rps, oss);
    case 7: return run_dst<7, false>(in, out, rows, 0, tables, live, s, rps, oss);
    case 8: return run_dst<8, false>(in, out, rows, 0, tables, live, s, rps, oss);
    case 9: return run_dst<9, false>(in, out, rows, 0, tables, live, s, rps, oss);
    case 10: return run_dst<10, false>(in, out, rows, 0, tables, live, s, rps, oss);
  }
  return PMK_ERR_UNSUPPORTED;
}

// DST along y of (slices, ny, nx) data, ny + 1 = 2^2 .. 2^9.
int launch_dst_cols(const double *in, double *out, int nx, int ny, int slices,
                    const double *tables, const int *live, cudaStream_t s) {
  switch (log2_exact(ny + 1)) {
    case 2: return run_dst<2, true>(in, out, slices, nx, tables, live, s);
    case 3: return run_dst<3, true>(in, out, slices, nx, tables, live, s);
    case 4: return run_dst<4, true>(in, out, slices, nx, tables, live, s);
    case 5: return run_dst<5, true>(in, out, slices, nx, tables, live, s);
    case 6: return run_dst<6, true>(in, out, slices, nx, tables, live, s);
    case 7: return run_dst<7, true>(in, out, slices, nx, tables, live, s);
    case 8: return run_dst<8, true>(in, out, slices, nx, tables, live, s);
    case 9: return run_dst<9, true>(in, out, slices, nx, tables, live, s);
  }
  return PMK_ERR_UNSUPPORTED;
}

}  // namespace pmk
