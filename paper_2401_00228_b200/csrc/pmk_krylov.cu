// pmk_krylov.cu -- FGMRES building blocks on the device (reference
// solver.py:362-456) and the stand-alone intergrid transfers
// (intergrid.py:51-63, 106-120).
//
// Krylov basis vectors: the reference appends b / beta and w / h[j+1, j]
// (solver.py:395, 420).  Here the last orthogonalisation pass leaves w
// unnormalised and the next iteration's K-MVR pass -- which reads it anyway --
// scales it (multiply by RN(1/h), within 1 ulp of the division; PMK_MGS=classic
// divides exactly) and writes the normalised v_j as a by-product (+8 B/unknown
// instead of a separate 16 B scale pass).  Every other reader (K-IMV, the
// orthogonalisation, assembly) reads v_j scale-free.
//
// All reductions are two-level with a fixed grid (kRedBlocks) and a fixed
// summation order, so results are bitwise reproducible.  The second level is
// folded into the prologue of the next consumer kernel: every block of the
// consumer sums the same partials in the same order, so no separate reduce
// launch and no host round trip is needed between MGS passes.
#include <math.h>

#include "pmk_internal.cuh"
#include "pmk_krylov.cuh"

namespace pmk {
namespace {

__device__ __forceinline__ double ld_scaled(const double *p, int64_t i, double sc, bool has) {
  const double v = p[i];
  return has ? __ddiv_rn(v, sc) : v;
}

// ------------------------------------------------------------ reductions
__global__ void __launch_bounds__(kRedThreads)
    dot_partials_kernel(const double *a, const double *as, const double *b, const double *bs,
                        int64_t n, double *partials, const int *live) {
  if (!is_live(live)) return;
  const double sa = as ? *as : 1.0, sb = bs ? *bs : 1.0;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = ld_scaled(a, i, sa, as != nullptr);
    const double y = ld_scaled(b, i, sb, bs != nullptr);
    acc = __dadd_rn(acc, __dmul_rn(x, y));
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// Vectorised variant: 16-byte loads, two vectors per thread per trip
// (unscaled, 16-byte aligned operands).
__global__ void __launch_bounds__(kRedThreads)
    dot_partials_vec_kernel(const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                            double *partials, const int *live) {
  if (!is_live(live)) return;
  const double2 *a2 = reinterpret_cast<const double2 *>(a);
  const double2 *b2 = reinterpret_cast<const double2 *>(b);
  const int64_t n2 = n >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < n2; i += 2 * stride) {
    const double2 x0 = __ldg(a2 + i), x1 = __ldg(a2 + i + stride);
    const double2 y0 = __ldg(b2 + i), y1 = __ldg(b2 + i + stride);
    acc = __dadd_rn(acc, __dmul_rn(x0.x, y0.x));
    acc = __dadd_rn(acc, __dmul_rn(x0.y, y0.y));
    acc = __dadd_rn(acc, __dmul_rn(x1.x, y1.x));
    acc = __dadd_rn(acc, __dmul_rn(x1.y, y1.y));
  }
  for (; i < n2; i += stride) {
    const double2 x0 = __ldg(a2 + i), y0 = __ldg(b2 + i);
    acc = __dadd_rn(acc, __dmul_rn(x0.x, y0.x));
    acc = __dadd_rn(acc, __dmul_rn(x0.y, y0.y));
  }
  if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1)
    acc = __dadd_rn(acc, __dmul_rn(a[n - 1], b[n - 1]));
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// partial sums of (a - b)^2 with r = a - b rounded first (stepper.py:192-193)
__global__ void __launch_bounds__(kRedThreads)
    diffsq_partials_kernel(const double *a, const double *b, int64_t n, double *partials,
                           double *r_out) {
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double r = __dsub_rn(a[i], b[i]);
    if (r_out) r_out[i] = r;  // (may alias b: each element is read before it is written)
    acc = __dadd_rn(acc, __dmul_rn(r, r));
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void reduce_scalar_kernel(const double *partials, int n, double *out, int do_sqrt) {
  const double s = reduce_partials(partials, n);
  if (threadIdx.x == 0) *out = do_sqrt ? sqrt(s) : s;
}

// ------------------------------------------------------------ fgmres state
// begin: beta = ||b|| from the partials, init g, flags (solver.py:381-396).
__global__ void begin_kernel(KState *st, const double *partials, int n_partials,
                             const int *parent_live) {
  const bool entered = is_live(parent_live);
  const double ss = entered ? reduce_partials(partials, n_partials) : 0.0;
  if (threadIdx.x == 0) {
    st->entered = entered ? 1 : 0;
    st->n_iter = 0;
    st->breakdown = 0;
    if (!entered) {
      st->live = 0;
      return;
    }
    const double beta = sqrt(ss);
    st->beta = beta;
    st->vscale[0] = beta;
    st->vrcp[0] = st->lazy ? __drcp_rn(beta) : 1.0;
    st->g[0] = beta;
    st->rel = 1.0;
    st->live = (beta == 0.0) ? 0 : 1;  // solver.py:382-383: zero rhs -> x = 0
  }
}

// One fused MGS pass (solver.py:405-408) for basis index l of column j:
//   h[l][j] = <w, v_l>            (from the previous pass' partials)
//   w      -= h[l][j] * v_l
//   partial <w, v_{l+1}>          (or <w, w> on the last pass, solver.py:412)
// Streams w, v_l, v_{l+1} as 16-byte vectors, two vectors per thread per
// trip with all six loads issued before any use (memory-level parallelism:
// 96 B in flight per thread).  Requires 16-byte aligned w / v_l / v_{l+1}
// (checked on the host; the scalar variant below handles the rest).
__global__ void __launch_bounds__(kRedThreads)
    mgs_pass_vec_kernel(KState *st, int ld, int l, int j, double *__restrict__ w,
                        const double *__restrict__ vl, const double *__restrict__ vn, int64_t n,
                        const double *prev, int n_prev, double *partials) {
  if (!st->live) return;
  const double h = reduce_partials(prev, n_prev);
  if (blockIdx.x == 0 && threadIdx.x == 0) st->h[l * ld + j] = h;
  const bool last = (vn == nullptr);
  const int64_t n2 = n >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double2 *w2 = reinterpret_cast<double2 *>(w);
  const double2 *l2 = reinterpret_cast<const double2 *>(vl);
  const double2 *z2 = reinterpret_cast<const double2 *>(last ? w : vn);
  double acc = 0.0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < n2; i += 2 * stride) {
    const double2 a0 = w2[i], a1 = w2[i + stride];
    const double2 b0 = __ldg(l2 + i), b1 = __ldg(l2 + i + stride);
    double2 c0, c1;
    if (!last) {
      c0 = __ldg(z2 + i);
      c1 = __ldg(z2 + i + stride);
    }
    double2 r0, r1;
    r0.x = __dsub_rn(a0.x, __dmul_rn(h, b0.x));
    r0.y = __dsub_rn(a0.y, __dmul_rn(h, b0.y));
    r1.x = __dsub_rn(a1.x, __dmul_rn(h, b1.x));
    r1.y = __dsub_rn(a1.y, __dmul_rn(h, b1.y));
    w2[i] = r0;
    w2[i + stride] = r1;
    if (last) {
      c0 = r0;
      c1 = r1;
    }
    acc = __dadd_rn(acc, __dmul_rn(r0.x, c0.x));
    acc = __dadd_rn(acc, __dmul_rn(r0.y, c0.y));
    acc = __dadd_rn(acc, __dmul_rn(r1.x, c1.x));
    acc = __dadd_rn(acc, __dmul_rn(r1.y, c1.y));
  }
  for (; i < n2; i += stride) {
    const double2 a0 = w2[i];
    const double2 b0 = __ldg(l2 + i);
    double2 r0;
    r0.x = __dsub_rn(a0.x, __dmul_rn(h, b0.x));
    r0.y = __dsub_rn(a0.y, __dmul_rn(h, b0.y));
    w2[i] = r0;
    const double2 c0 = last ? r0 : __ldg(z2 + i);
    acc = __dadd_rn(acc, __dmul_rn(r0.x, c0.x));
    acc = __dadd_rn(acc, __dmul_rn(r0.y, c0.y));
  }
  if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) {
    const int64_t t = n - 1;
    const double r = __dsub_rn(w[t], __dmul_rn(h, vl[t]));
    w[t] = r;
    acc = __dadd_rn(acc, __dmul_rn(r, last ? r : vn[t]));
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// Scalar variant (unaligned operands or lazily scaled inputs).
__global__ void __launch_bounds__(kRedThreads)
    mgs_pass_kernel(KState *st, int ld, int l, int j, double *w, const double *vl,
                    const double *vl_scale, const double *vn, const double *vn_scale, int64_t n,
                    const double *prev, int n_prev, double *partials) {
  if (!st->live) return;
  const double h = reduce_partials(prev, n_prev);
  if (blockIdx.x == 0 && threadIdx.x == 0) st->h[l * ld + j] = h;
  const double sl = vl_scale ? *vl_scale : 1.0;
  const bool last = (vn == nullptr);
  const double sn = (!last && vn_scale) ? *vn_scale : 1.0;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = ld_scaled(vl, i, sl, vl_scale != nullptr);
    const double wn = __dsub_rn(w[i], __dmul_rn(h, v));
    w[i] = wn;
    const double z = last ? wn : ld_scaled(vn, i, sn, vn_scale != nullptr);
    acc = __dadd_rn(acc, __dmul_rn(wn, z));
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// ------------------------------------------------- one-reduce MGS (ICWY)
// The reference orthogonalises w against v_0..v_j one vector at a time
// (solver.py:405-408): h_i = <w^(i), v_i>, w^(i+1) = w^(i) - h_i v_i, which
// streams ~4 vectors per basis vector.  In exact arithmetic
//   h_i = <w, v_i> - sum_{l<i} h_l <v_l, v_i>,   i.e.  (I + L) h = V^T w
// with L the strictly lower triangle of the basis Gram matrix, so h follows
// from ONE pass of dot products (V^T w, plus the new Gram row <v_j, v_i>
// while v_j streams by anyway) and w from ONE update pass applying the
// subtractions in the reference's order with the reference's per-element
// rounding.  This is the inverse-compact-WY form of MGS (Swirydowicz et al.,
// "Low synchronization Gram-Schmidt and GMRES algorithms"), whose loss of
// orthogonality is that of MGS; ~2 vectors per basis vector are streamed.
// Update passes take up to kGroup basis vectors each, dot passes kDotGroup
// (two accumulators per vector).

// Deterministic block reduction of NV per-thread values; thread v < NV
// writes value v's block sum to out[v * out_stride].
template <int NV>
__device__ __forceinline__ void block_sum_multi(double (&a)[NV], double *out, int out_stride) {
  __shared__ double red[kRedThreads / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double x = a[v];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) red[warp][v] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double x = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) x = __dadd_rn(x, red[w][threadIdx.x]);
    out[(int64_t)threadIdx.x * out_stride] = x;
  }
}

__device__ __forceinline__ double dot2(double acc, double2 a, double2 b) {
  acc = __dadd_rn(acc, __dmul_rn(a.x, b.x));
  return __dadd_rn(acc, __dmul_rn(a.y, b.y));
}

// Partials of <w, v_q> (slot q), <vj, v_q> (slot kDotGroup + q) for the
// group, and <w, vj> (slot 2 kDotGroup); slot s at partials[s * gridDim.x].
// Aligned operands: CNT vectors, U element steps per trip so that ~12
// 16-byte loads are in flight per thread whatever the group size.
template <int CNT>
__global__ void __launch_bounds__(kRedThreads)
    icwy_dots_vec_kernel(const KState *st, const double *__restrict__ w,
                         const double *__restrict__ vj, MultiVec V, int64_t n,
                         double *partials) {
  if (!st->live) return;
  constexpr int U = (12 / (CNT + 2)) > 1 ? 12 / (CNT + 2) : 1;
  double aw[CNT], ag[CNT], awj[1] = {0.0};
#pragma unroll
  for (int q = 0; q < CNT; ++q) aw[q] = ag[q] = 0.0;
  const double2 *w2 = reinterpret_cast<const double2 *>(w);
  const double2 *j2 = reinterpret_cast<const double2 *>(vj);
  const double2 *c2[CNT];
#pragma unroll
  for (int q = 0; q < CNT; ++q) c2[q] = reinterpret_cast<const double2 *>(V.v[q]);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n2 = n >> 1;
  int64_t i = t0;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 a[U], b[U], c[U][CNT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = __ldg(w2 + i + u * stride);
      b[u] = __ldg(j2 + i + u * stride);
#pragma unroll
      for (int q = 0; q < CNT; ++q) c[u][q] = __ldg(c2[q] + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      awj[0] = dot2(awj[0], a[u], b[u]);
#pragma unroll
      for (int q = 0; q < CNT; ++q) {
        aw[q] = dot2(aw[q], a[u], c[u][q]);
        ag[q] = dot2(ag[q], b[u], c[u][q]);
      }
    }
  }
  for (; i < n2; i += stride) {
    const double2 a = __ldg(w2 + i), b = __ldg(j2 + i);
    awj[0] = dot2(awj[0], a, b);
#pragma unroll
    for (int q = 0; q < CNT; ++q) {
      const double2 c = __ldg(c2[q] + i);
      aw[q] = dot2(aw[q], a, c);
      ag[q] = dot2(ag[q], b, c);
    }
  }
  if ((n & 1) && t0 == stride - 1) {
    const double a = w[n - 1], b = vj[n - 1];
    awj[0] = __dadd_rn(awj[0], __dmul_rn(a, b));
#pragma unroll
    for (int q = 0; q < CNT; ++q) {
      const double c = V.v[q][n - 1];
      aw[q] = __dadd_rn(aw[q], __dmul_rn(a, c));
      ag[q] = __dadd_rn(ag[q], __dmul_rn(b, c));
    }
  }
  double *out = partials + blockIdx.x;
  block_sum_multi<CNT>(aw, out, gridDim.x);
  __syncthreads();
  block_sum_multi<CNT>(ag, out + (int64_t)kDotGroup * gridDim.x, gridDim.x);
  __syncthreads();
  block_sum_multi<1>(awj, out + (int64_t)2 * kDotGroup * gridDim.x, gridDim.x);
}

// <w, v_q> only (slot q at partials[q * gridDim.x]), up to kGroup vectors:
// the Gram row of v_j came from the update pass that produced v_j.
template <int CNT>
__global__ void __launch_bounds__(kRedThreads)
    icwy_dotsw_vec_kernel(const KState *st, const double *__restrict__ w, MultiVec V, int64_t n,
                          double *partials) {
  if (!st->live) return;
  constexpr int U = (12 / (CNT + 1)) > 1 ? 12 / (CNT + 1) : 1;
  double aw[CNT];
#pragma unroll
  for (int q = 0; q < CNT; ++q) aw[q] = 0.0;
  const double2 *w2 = reinterpret_cast<const double2 *>(w);
  const double2 *c2[CNT];
#pragma unroll
  for (int q = 0; q < CNT; ++q) c2[q] = reinterpret_cast<const double2 *>(V.v[q]);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n2 = n >> 1;
  int64_t i = t0;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 a[U], c[U][CNT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = __ldg(w2 + i + u * stride);
#pragma unroll
      for (int q = 0; q < CNT; ++q) c[u][q] = __ldg(c2[q] + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int q = 0; q < CNT; ++q) aw[q] = dot2(aw[q], a[u], c[u][q]);
    }
  }
  for (; i < n2; i += stride) {
    const double2 a = __ldg(w2 + i);
#pragma unroll
    for (int q = 0; q < CNT; ++q) aw[q] = dot2(aw[q], a, __ldg(c2[q] + i));
  }
  if ((n & 1) && t0 == stride - 1) {
    const double a = w[n - 1];
#pragma unroll
    for (int q = 0; q < CNT; ++q) aw[q] = __dadd_rn(aw[q], __dmul_rn(a, V.v[q][n - 1]));
  }
  block_sum_multi<CNT>(aw, partials + blockIdx.x, gridDim.x);
}

// Any alignment, runtime group size.
__global__ void __launch_bounds__(kRedThreads)
    icwy_dots_kernel(const KState *st, const double *__restrict__ w,
                     const double *__restrict__ vj, MultiVec V, int count, int64_t n,
                     double *partials) {
  if (!st->live) return;
  double aw[kDotGroup], ag[kDotGroup], awj[1] = {0.0};
#pragma unroll
  for (int q = 0; q < kDotGroup; ++q) aw[q] = ag[q] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double a = w[i], b = vj[i];
    awj[0] = __dadd_rn(awj[0], __dmul_rn(a, b));
#pragma unroll
    for (int q = 0; q < kDotGroup; ++q)
      if (q < count) {
        const double c = V.v[q][i];
        aw[q] = __dadd_rn(aw[q], __dmul_rn(a, c));
        ag[q] = __dadd_rn(ag[q], __dmul_rn(b, c));
      }
  }
  double *out = partials + blockIdx.x;
  block_sum_multi<kDotGroup>(aw, out, gridDim.x);
  __syncthreads();
  block_sum_multi<kDotGroup>(ag, out + (int64_t)kDotGroup * gridDim.x, gridDim.x);
  __syncthreads();
  block_sum_multi<1>(awj, out + (int64_t)2 * kDotGroup * gridDim.x, gridDim.x);
}

// warp-level deterministic sum of n partials (fixed lane order + xor tree)
__device__ __forceinline__ double warp_reduce_partials(const double *p, int n) {
  const int lane = threadIdx.x & 31;
  double x = 0.0;
  for (int i = lane; i < n; i += 32) x = __dadd_rn(x, p[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// Reduce the dot partials, store Gram row j, solve (I + L) h = c and write
// column j of H (rows 0..j).  One block.
//   c_0 = <w, v_0>: K-IMV partials (c0p, n_c0); for j >= 1 the group passes
//   wrote, per group g (basis o..j-1 in groups of kDotGroup, slots as above),
//   <w, v_i> for i >= 1, <v_j, v_i>, and <w, v_j> (taken from group 0).
//   With pj (o = 1), K-IMV also produced <w, v_j> (pj) and <v_j, v_0>
//   (pj + kMaxPartials) and the group passes start at v_1.
__global__ void __launch_bounds__(1024)
    icwy_solve_kernel(KState *st, int ld, int j, const double *c0p, int n_c0,
                      const double *pj, const double *gp, int n_gp, int ugram = 0) {
  if (!st->live) return;
  extern __shared__ double sh[];  // c[0..j], g[0..j-1]
  double *c = sh, *g = sh + (j + 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gstride = (2 * kDotGroup + 1) * n_gp;  // doubles per group
  const int o = pj ? 1 : 0;                         // first basis vector of group 0
  for (int d = warp; d < 2 * j + 1; d += nw) {
    double x;
    if (d == 0) {
      x = warp_reduce_partials(c0p, n_c0);
    } else if (d < j && ugram) {  // w-only dot passes, kGroup slots per pass
      const int e = d - 1;
      x = warp_reduce_partials(gp + (int64_t)(e / kGroup) * kGroup * n_gp + (e % kGroup) * n_gp,
                               n_gp);
      x = __dmul_rn(x, st->vrcp[d]);
    } else if (d < j) {  // <w, v_d>, 1 <= d < j (dot pass: raw v_d)
      const int e = d - o;
      x = warp_reduce_partials(gp + (int64_t)(e / kDotGroup) * gstride + (e % kDotGroup) * n_gp, n_gp);
      x = __dmul_rn(x, st->vrcp[d]);
    } else if (d == j) {  // <w, v_j> (K-IMV: scaled; dot pass: raw v_j)
      x = pj ? warp_reduce_partials(pj, n_c0)
             : __dmul_rn(warp_reduce_partials(gp + (int64_t)2 * kDotGroup * n_gp, n_gp),
                         st->vrcp[j]);
    } else {  // <v_j, v_i>, i = d - j - 1
      const int i = d - j - 1;
      const int e = i - o;
      if (ugram && i >= 1) {  // from the update pass that produced v_j (raw x raw)
        x = __dmul_rn(warp_reduce_partials(st->ugp + (int64_t)i * kMaxPartials, kRedBlocks),
                      __dmul_rn(st->vrcp[j], st->vrcp[i]));
      } else
      x = (pj && i == 0)
              ? warp_reduce_partials(pj + kMaxPartials, n_c0)
              : __dmul_rn(warp_reduce_partials(gp + (int64_t)(e / kDotGroup) * gstride +
                                                   (kDotGroup + e % kDotGroup) * n_gp,
                                               n_gp),
                          __dmul_rn(st->vrcp[j], st->vrcp[i]));
    }
    if (lane == 0) {
      if (d <= j)
        c[d] = x;
      else
        g[d - j - 1] = x;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < j; i += blockDim.x) st->gram[(int64_t)j * ld + i] = g[i];
  if (warp != 0) return;
  // forward substitution, row i of L = Gram row i (stored at iteration i)
  double *h = st->h;
  for (int i = 0; i <= j; ++i) {
    const double *Li = (i == j) ? g : st->gram + (int64_t)i * ld;
    double x = 0.0;
    for (int l = lane; l < i; l += 32) x = __dadd_rn(x, __dmul_rn(Li[l], c[l]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
    // c[l] for l < i already holds h_l
    const double hi = __dsub_rn(c[i], x);
    __syncwarp();
    if (lane == 0) {
      c[i] = hi;
      h[(int64_t)i * ld + j] = hi;
      st->hv[i] = __dmul_rn(hi, st->vrcp[i]);  // update coefficient (lazy: h_i / scale_i)
    }
    __syncwarp();
  }
}

// h[j+1][j] = ||w||, breakdown test, Givens update (solver.py:412-440), by
// one block (all its threads take part in the reduction).
__device__ __forceinline__ void finish_col_block(KState *st, int ld, int j,
                                                 const double *partials, int n_partials,
                                                 double tol, bool pyth = false) {
  double ss = reduce_partials(partials, n_partials);
  if (threadIdx.x != 0) return;
  // pyth (column 0 of a budget-1 solve): the partials are ||w||^2 of the
  // unorthogonalised w; ||w - h_00 v_0||^2 = ||w||^2 - h_00^2.  Only
  // h_00^2 + h_10^2 = ||w||^2 enters the one-column least squares (y_0 =
  // beta h_00 / ||w||^2), so the cancellation for h_10 << ||w|| does not.
  if (pyth) ss = fmax(__dsub_rn(ss, __dmul_rn(st->h[0], st->h[0])), 0.0);
  double *h = st->h;
  const double hn = sqrt(ss);
  h[(j + 1) * ld + j] = hn;
  for (int l = 0; l <= j + 1; ++l) st->hraw[l * ld + j] = h[l * ld + j];
  st->n_iter = j + 1;
  double cn2 = 0.0;  // np.linalg.norm(h[:j+2, j])
  for (int l = 0; l <= j + 1; ++l) cn2 = __dadd_rn(cn2, __dmul_rn(h[l * ld + j], h[l * ld + j]));
  const double col_norm = sqrt(cn2);
  const bool breakdown = hn <= 1e-14 * fmax(col_norm, 1e-300);
  if (!breakdown) {
    st->vscale[j + 1] = hn;
    st->vrcp[j + 1] = st->lazy ? __drcp_rn(hn) : 1.0;
  }
  double *cs = st->cs, *sn = st->sn, *g = st->g;
  for (int l = 0; l < j; ++l) {
    const double a = h[l * ld + j], b = h[(l + 1) * ld + j];
    const double tmp = __dadd_rn(__dmul_rn(cs[l], a), __dmul_rn(sn[l], b));
    h[(l + 1) * ld + j] = __dadd_rn(__dmul_rn(-sn[l], a), __dmul_rn(cs[l], b));
    h[l * ld + j] = tmp;
  }
  const double hjj = h[j * ld + j], hj1 = h[(j + 1) * ld + j];
  const double denom = hypot(hjj, hj1);
  cs[j] = __ddiv_rn(hjj, denom);
  sn[j] = __ddiv_rn(hj1, denom);
  h[j * ld + j] = denom;
  h[(j + 1) * ld + j] = 0.0;
  g[j + 1] = __dmul_rn(-sn[j], g[j]);
  g[j] = __dmul_rn(cs[j], g[j]);
  const double rel = __ddiv_rn(fabs(g[j + 1]), st->beta);
  st->rel = rel;
  st->hist[j] = rel;
  if (breakdown) {
    st->breakdown = 1;
    st->live = 0;
  } else if (tol > 0.0 && rel <= tol) {
    st->live = 0;  // converged (solver.py:438-440)
  }
}

__global__ void finish_col_kernel(KState *st, int ld, int j, const double *partials,
                                  int n_partials, double tol, bool pyth = false) {
  if (!st->live) return;
  finish_col_block(st, ld, j, partials, n_partials, tol, pyth);
}

// w -= sum_q h[i0+q][j] v_q (ascending q, the reference's per-element
// rounding); with `partials`, the partial sums of ||w||^2 of the result.
template <int CNT, bool GRAM = false>
__global__ void __launch_bounds__(kRedThreads)
    icwy_update_vec_kernel(KState *st, int ld, int j, int i0, MultiVec V,
                           double *__restrict__ w, int64_t n, double *partials, bool store,
                           bool finish, double tol) {
  if (!st->live) return;
  constexpr int U = (12 / (CNT + 1)) > 1 ? 12 / (CNT + 1) : 1;
  double hq[CNT];
  const double2 *c2[CNT];
#pragma unroll
  for (int q = 0; q < CNT; ++q) {  // h_q (x vrcp_q for a lazy basis), icwy_solve
    hq[q] = st->hv[i0 + q];
    c2[q] = reinterpret_cast<const double2 *>(V.v[q]);
  }
  double acc[1] = {0.0};
  double ag[GRAM ? CNT : 1];  // GRAM: <w', raw_q>, the next basis vector's Gram row
#pragma unroll
  for (int q = 0; q < (GRAM ? CNT : 1); ++q) ag[q] = 0.0;
  double2 *w2 = reinterpret_cast<double2 *>(w);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n2 = n >> 1;
  int64_t i = t0;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 a[U], c[U][CNT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = w2[i + u * stride];
#pragma unroll
      for (int q = 0; q < CNT; ++q) c[u][q] = __ldg(c2[q] + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int q = 0; q < CNT; ++q) {
        a[u].x = __dsub_rn(a[u].x, __dmul_rn(hq[q], c[u][q].x));
        a[u].y = __dsub_rn(a[u].y, __dmul_rn(hq[q], c[u][q].y));
      }
      if (store) w2[i + u * stride] = a[u];
      if (partials) acc[0] = dot2(acc[0], a[u], a[u]);
      if constexpr (GRAM) {
#pragma unroll
        for (int q = 0; q < CNT; ++q) ag[q] = dot2(ag[q], a[u], c[u][q]);
      }
    }
  }
  for (; i < n2; i += stride) {
    double2 a = w2[i];
#pragma unroll
    for (int q = 0; q < CNT; ++q) {
      const double2 c = __ldg(c2[q] + i);
      a.x = __dsub_rn(a.x, __dmul_rn(hq[q], c.x));
      a.y = __dsub_rn(a.y, __dmul_rn(hq[q], c.y));
    }
    if (store) w2[i] = a;
    if (partials) acc[0] = dot2(acc[0], a, a);
    if constexpr (GRAM) {
#pragma unroll
      for (int q = 0; q < CNT; ++q) ag[q] = dot2(ag[q], a, __ldg(c2[q] + i));
    }
  }
  if ((n & 1) && t0 == stride - 1) {
    double a = w[n - 1];
#pragma unroll
    for (int q = 0; q < CNT; ++q) a = __dsub_rn(a, __dmul_rn(hq[q], V.v[q][n - 1]));
    if (store) w[n - 1] = a;
    if (partials) acc[0] = __dadd_rn(acc[0], __dmul_rn(a, a));
    if constexpr (GRAM) {
#pragma unroll
      for (int q = 0; q < CNT; ++q) ag[q] = __dadd_rn(ag[q], __dmul_rn(a, V.v[q][n - 1]));
    }
  }
  if constexpr (GRAM) {
    block_sum_multi<CNT>(ag, st->ugp + (int64_t)i0 * kMaxPartials + blockIdx.x, kMaxPartials);
    __syncthreads();
  }
  if (partials) block_sum_multi<1>(acc, partials + blockIdx.x, gridDim.x);
  if (finish) {  // last block to finish runs finish_col (fixed-order reduction)
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
      __threadfence();
      finish_col_block(st, ld, j, partials, gridDim.x, tol);
      if (threadIdx.x == 0) st->ticket = 0;
    }
  }
}

__global__ void __launch_bounds__(kRedThreads)
    icwy_update_kernel(const KState *st, int ld, int j, int i0, MultiVec V, int count,
                       double *__restrict__ w, int64_t n, double *partials, bool store) {
  if (!st->live) return;
  double hq[kGroup];
#pragma unroll
  for (int q = 0; q < kGroup; ++q)
    hq[q] = (q < count) ? st->hv[i0 + q] : 0.0;
  double acc[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double a = w[i];
#pragma unroll
    for (int q = 0; q < kGroup; ++q)
      if (q < count) a = __dsub_rn(a, __dmul_rn(hq[q], V.v[q][i]));
    if (store) w[i] = a;
    if (partials) acc[0] = __dadd_rn(acc[0], __dmul_rn(a, a));
  }
  if (partials) block_sum_multi<1>(acc, partials + blockIdx.x, gridDim.x);
}


// Back substitution (solver.py:442-444).
__global__ void backsolve_kernel(KState *st, int ld, const double *out_scale) {
  if (!st->entered || threadIdx.x != 0) return;
  const int n = st->n_iter;
  const double *h = st->h, *g = st->g;
  double *y = st->y;
  for (int i = n - 1; i >= 0; --i) {
    double d = 0.0;
    for (int k = i + 1; k < n; ++k) d = __dadd_rn(d, __dmul_rn(h[i * ld + k], y[k]));
    y[i] = __ddiv_rn(__dsub_rn(g[i], d), h[i * ld + i]);
  }
  // the caller wants the solution for rhs * out_scale (linear in the rhs)
  if (out_scale)
    for (int i = 0; i < n; ++i) y[i] = __dmul_rn(y[i], *out_scale);
}

// x = sum_i y_i x_i with x_i = v_i - Z vt_i recomputed (solver.py:445-447,
// 359).  `first` > 0 continues an accumulation already in x.  Grid: x over
// the in-slice index, y over slices (coarse row K computed once per slice).
__global__ void __launch_bounds__(256)
    assemble_kernel(const KState *st, AssembleArgs a, double *x, int rows, int m, int nu,
                    int m_coarse, const int32_t *group_of, int first) {
  if (!st->entered) return;
  const int n_iter = st->n_iter;
  const int hi = min(n_iter, first + a.count);
  if (first > 0 && first >= n_iter) return;
  __shared__ double ys[kAsmChunk], sc[kAsmChunk];  // y_l and the lazy-basis scales
  for (int q = threadIdx.x; q < kAsmChunk; q += blockDim.x) {
    ys[q] = (first + q < hi) ? st->y[first + q] : 0.0;
    sc[q] = (first + q < hi) ? st->vrcp[first + q] : 1.0;
  }
  __syncthreads();
  for (int k = blockIdx.y; k < rows; k += gridDim.y) {
    const int K = (k == 0) ? 0 : (k - 1) / nu + 1;
    const int64_t base = (int64_t)k * m;
    const int64_t cbase = (int64_t)K * m_coarse;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
      const int64_t e = base + i;
      const int64_t ci = cbase + (group_of ? group_of[i] : i);
      double acc = (first == 0) ? 0.0 : x[e];
      for (int l = first; l < hi; ++l) {
        const int q = l - first;
        const double vl = __dmul_rn(__ldg(a.v[q] + e), sc[q]);  // (lazy basis)
        const double xl = __dsub_rn(vl, __ldg(a.vt[q] + ci));
        acc = __dadd_rn(acc, __dmul_rn(ys[q], xl));
      }
      x[e] = acc;
    }
  }
}

// Same sum for a time-only coarse mapping with nu = 2 (group_of == nullptr),
// for the few-vector assemblies of the inner levels; templated on the
// vector count.  Grid y runs over coarse slices K: a block owns the fine
// slices of K (slice 0 alone for K = 0, else 2K-1 and 2K), and each thread
// loads, for U elements of the slice, the coarse value vt_q once and both
// fine values v_q up front (3 U CNT loads in flight), so every coarse value
// is read once and no load waits behind a store.
template <int CNT>
__global__ void __launch_bounds__(256)
    assemble_pair_kernel(const KState *st, AssembleArgs a, double *x, int rows, int m,
                         int first) {
  if (!st->entered) return;
  constexpr int U = (12 / (3 * CNT)) > 1 ? 12 / (3 * CNT) : 1;
  const int n_iter = st->n_iter;
  if (first > 0 && first >= n_iter) return;
  const int hi = min(n_iter, first + CNT);
  double y[CNT], sc[CNT];  // sc: lazy-basis scales (1 for a normalised basis)
#pragma unroll
  for (int q = 0; q < CNT; ++q) {
    y[q] = (first + q < hi) ? st->y[first + q] : 0.0;
    sc[q] = (first + q < hi) ? st->vrcp[first + q] : 1.0;
  }
  const int chunk = 256 * U;
  const int n_coarse = rows / 2 + 1;  // K = 0 and the pairs (2K-1, 2K)
  for (int K = blockIdx.y; K < n_coarse; K += gridDim.y) {
    const int64_t cbase = (int64_t)K * m;
    const int k0 = (K == 0) ? 0 : 2 * K - 1;
    const bool two = K > 0 && k0 + 1 < rows;  // (a row-range view may end on 2K-1)
    for (int i0 = blockIdx.x * chunk; i0 < m; i0 += gridDim.x * chunk) {
      double tt[U][CNT], v0[U][CNT], v1[U][CNT], a0[U], a1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + threadIdx.x + u * 256;
        const bool ok = i < m;
        const int64_t e0 = (int64_t)k0 * m + i, e1 = e0 + m;
        a0[u] = (first == 0 || !ok) ? 0.0 : x[e0];
        a1[u] = (first == 0 || !ok || !two) ? 0.0 : x[e1];
#pragma unroll
        for (int q = 0; q < CNT; ++q) {
          const bool on = ok && first + q < hi;
          tt[u][q] = on ? __ldg(a.vt[q] + cbase + i) : 0.0;
          v0[u][q] = on ? __ldg(a.v[q] + e0) : 0.0;
          v1[u][q] = (on && two) ? __ldg(a.v[q] + e1) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + threadIdx.x + u * 256;
        if (i >= m) continue;
        const int64_t e0 = (int64_t)k0 * m + i;
        double s0 = a0[u], s1 = a1[u];
#pragma unroll
        for (int q = 0; q < CNT; ++q)
          if (first + q < hi) {
            s0 = __dadd_rn(s0, __dmul_rn(y[q], __dsub_rn(__dmul_rn(v0[u][q], sc[q]), tt[u][q])));
            s1 = __dadd_rn(s1, __dmul_rn(y[q], __dsub_rn(__dmul_rn(v1[u][q], sc[q]), tt[u][q])));
          }
        x[e0] = s0;
        if (two) x[e0 + m] = s1;
      }
    }
  }
}

// ------------------------------------------------------------- transfers
__global__ void restrict_time_kernel(const double *v, double *vh, int nu, int n_T, int m) {
  const int64_t total = (int64_t)(n_T + 1) * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t K = e / m, i = e - K * m;
    if (K == 0) {
      vh[e] = v[i];
    } else {
      const int64_t base = ((K - 1) * nu + 1) * m + i;
      double acc = v[base];
      for (int q = 1; q < nu; ++q) acc = __dadd_rn(acc, v[base + (int64_t)q * m]);
      vh[e] = acc;
    }
  }
}

// Y^T gather: out[K, c] = sum_{j in group c, ascending} Y[j, c] * fine[K, j]
// (the csc_matvecs order of `summed @ y_space`, intergrid.py:109-111).
__global__ void ts_gather_kernel(const double *fine, double *coarse, const int32_t *ptr,
                                 const int32_t *idx, const double *val, int n_rows, int m_fine,
                                 int m_coarse, const int *live) {
  if (!is_live(live)) return;
  const int64_t total = (int64_t)n_rows * m_coarse;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t K = e / m_coarse;
    const int c = (int)(e - K * m_coarse);
    const double *row = fine + K * m_fine;
    double acc = 0.0;
    for (int q = ptr[c]; q < ptr[c + 1]; ++q) acc = __dadd_rn(acc, __dmul_rn(val[q], row[idx[q]]));
    coarse[e] = acc;
  }
}

__global__ void interpolate_kernel(const double *w, double *out, int nu, int n_T, int m_fine,
                                   int m_coarse, const int32_t *group_of) {
  const int64_t total = (int64_t)(nu * n_T + 1) * m_fine;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / m_fine, i = e - k * m_fine;
    const int64_t K = (k == 0) ? 0 : (k - 1) / nu + 1;
    out[e] = w[K * m_coarse + (group_of ? (int64_t)group_of[i] : i)];
  }
}

// Weighted space interpolation (pmk_pair z_*): out[k, i] = sum_q z_val[q] *
// w[K(k), z_idx[q]], K(k) = coarse slice of fine slice k (nu = 1: the space
// interpolation of every coarse slice, the solver's child vector).
__global__ void interpolate_z_kernel(const double *w, double *out, int nu, int rows, int m_fine,
                                     int m_coarse, const int32_t *ptr, const int32_t *idx,
                                     const double *val, const int *live) {
  if (!is_live(live)) return;
  const int64_t total = (int64_t)rows * m_fine;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / m_fine;
    const int i = (int)(e - k * m_fine);
    const int64_t K = (k == 0) ? 0 : (k - 1) / nu + 1;
    const double *row = w + K * m_coarse;
    double acc = 0.0;
    for (int q = ptr[i]; q < ptr[i + 1]; ++q) acc = __dadd_rn(acc, __dmul_rn(val[q], row[idx[q]]));
    out[e] = acc;
  }
}

__global__ void div_check_kernel(const double *x, double d, int64_t n, double *out) {
  const double rcp = __drcp_rn(d);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = div_by(x[i], d, rcp);
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 16 * kSMs) g = 16 * kSMs;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

// ------------------------------------------------------------ launchers
int launch_dot_partials(const double *a, const double *a_scale, const double *b,
                        const double *b_scale, int64_t n, double *partials, const int *live,
                        cudaStream_t s) {
  prof::Scope scope(prof::kRed, (a == b ? 8.0 : 16.0) * (double)n, 0.0, s);
  auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!a_scale && !b_scale && al(a) && al(b)) {
    dot_partials_vec_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(a, b, n, partials, live);
    PMK_LAUNCH_CHECK();
    return 0;
  }
  dot_partials_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(a, a_scale, b, b_scale, n, partials,
                                                         live);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_diffsq_partials(const double *a, const double *b, int64_t n, double *partials,
                           cudaStream_t s, double *r_out) {
  prof::Scope scope(prof::kRed, (r_out ? 24.0 : 16.0) * (double)n, 0.0, s);
  diffsq_partials_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(a, b, n, partials, r_out);
  PMK_LAUNCH_CHECK();
  return 0;
}

// y += a x (the restart update x <- x + dx of the FGMRES(m) wrapper, SURVEY
// section 8(c)); one rounding per element, as numpy's x + dx.
__global__ void __launch_bounds__(256)
    axpy_kernel(double a, const double *__restrict__ x, double *__restrict__ y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (a == 1.0) ? __dadd_rn(y[i], x[i]) : fma(a, x[i], y[i]);
}

int launch_axpy(double a, const double *x, double *y, int64_t n, cudaStream_t s) {
  prof::Scope scope(prof::kAsm, 24.0 * (double)n, 0.0, s);
  axpy_kernel<<<grid_for(n, 256), 256, 0, s>>>(a, x, y, n);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_reduce_to_scalar(const double *partials, int n, double *out, int do_sqrt,
                            cudaStream_t s) {
  prof::Scope scope(prof::kSmall, 0.0, 0.0, s);
  reduce_scalar_kernel<<<1, kRedThreads, 0, s>>>(partials, n, out, do_sqrt);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_begin(KState *st, const double *partials, int n_partials, const int *parent_live,
                 cudaStream_t s) {
  prof::Scope scope(prof::kSmall, 0.0, 0.0, s);
  begin_kernel<<<1, kRedThreads, 0, s>>>(st, partials, n_partials, parent_live);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_mgs_pass(KState *st, int ld, int l, int j, double *w, const double *vl,
                    const double *vl_scale, const double *vn, const double *vn_scale, int64_t n,
                    const double *prev, int n_prev, double *partials, cudaStream_t s) {
  prof::Scope scope(prof::kMGS, (vn ? 32.0 : 24.0) * (double)n, 0.0, s);
  auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!vl_scale && !vn_scale && al(w) && al(vl) && (!vn || al(vn))) {
    mgs_pass_vec_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(st, ld, l, j, w, vl, vn, n, prev,
                                                           n_prev, partials);
    PMK_LAUNCH_CHECK();
    return 0;
  }
  mgs_pass_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(st, ld, l, j, w, vl, vl_scale, vn, vn_scale,
                                                     n, prev, n_prev, partials);
  PMK_LAUNCH_CHECK();
  return 0;
}

template <int CNT>
void dots_vec(const KState *st, const double *w, const double *vj, const MultiVec &V, int64_t n,
              double *partials, cudaStream_t s) {
  icwy_dots_vec_kernel<CNT><<<kRedBlocks, kRedThreads, 0, s>>>(st, w, vj, V, n, partials);
}
template <int CNT>
void update_vec(KState *st, int ld, int j, int i0, const MultiVec &V, double *w, int64_t n,
                double *partials, bool store, bool finish, double tol, cudaStream_t s,
                bool gram = false) {
  if (gram)
    icwy_update_vec_kernel<CNT, true><<<kRedBlocks, kRedThreads, 0, s>>>(
        st, ld, j, i0, V, w, n, partials, store, finish, tol);
  else
    icwy_update_vec_kernel<CNT, false><<<kRedBlocks, kRedThreads, 0, s>>>(
        st, ld, j, i0, V, w, n, partials, store, finish, tol);
}
template <int CNT>
void dotsw_vec(const KState *st, const double *w, const MultiVec &V, int64_t n,
               double *partials, cudaStream_t s) {
  icwy_dotsw_vec_kernel<CNT><<<kRedBlocks, kRedThreads, 0, s>>>(st, w, V, n, partials);
}

#define PMK_CASES8(F) F(1) F(2) F(3) F(4) F(5) F(6) F(7) F(8)
#define PMK_CASES16(F) PMK_CASES8(F) F(9) F(10) F(11) F(12) F(13) F(14) F(15) F(16)

// Orthogonalise w against v[0..j] (ICWY form, see icwy_dots_vec_kernel) and
// leave the partials of ||w||^2 in `norm_partials` (*n_norm of them).  All
// passes use the fixed kRedBlocks grid (deterministic partial layout).
int launch_icwy_mgs(KState *st, int ld, int j, double *w, const double *const *v, int64_t n,
                    const double *c0p, int n_c0, const double *pj, double *dot_partials,
                    double *norm_partials, int *n_norm, bool keep_w, cudaStream_t s, double tol,
                    bool fuse_finish, bool *finished, bool ugram_in, bool ugram_out,
                    bool *ugram_done) {
  if (finished) *finished = false;
  if (ugram_done) *ugram_done = false;
  auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  bool vec = al(w);
  for (int i = 0; i <= j; ++i) vec = vec && al(v[i]);
  const int64_t gstride = (int64_t)(2 * kDotGroup + 1) * kRedBlocks;
  if (j < 1) pj = nullptr;
  const bool ug = ugram_in && vec && pj && j >= 2;
  // ug: the Gram row of v_j is already in st->ugp; the dot passes need
  // <w, v_i>, 0 < i < j, only (w and up to kGroup basis vectors per pass)
  for (int i0 = 1, gi = 0; ug && i0 < j; i0 += kGroup, ++gi) {
    const int cnt = (j - i0 < kGroup) ? j - i0 : kGroup;
    MultiVec V{};
    for (int q = 0; q < cnt; ++q) V.v[q] = v[i0 + q];
    prof::Scope scope(prof::kMGS, 8.0 * (cnt + 1) * (double)n, 4.0 * cnt * (double)n, s);
    double *part = dot_partials + (int64_t)gi * kGroup * kRedBlocks;
    switch (cnt) {
#define PMK_DOTSW_CASE(C)                   \
  case C:                                   \
    dotsw_vec<C>(st, w, V, n, part, s);     \
    break;
      PMK_CASES16(PMK_DOTSW_CASE)
#undef PMK_DOTSW_CASE
      default:
        return PMK_ERR_ARG;
    }
    PMK_LAUNCH_CHECK();
  }
  // with pj the K-IMV pass already produced every dot involving v_0 or v_j
  // except the Gram entries <v_j, v_i>, 0 < i < j
  for (int i0 = pj ? 1 : 0, gi = 0; !ug && i0 < j; i0 += kDotGroup, ++gi) {
    const int cnt = (j - i0 < kDotGroup) ? j - i0 : kDotGroup;
    MultiVec V{};
    for (int q = 0; q < cnt; ++q) V.v[q] = v[i0 + q];
    prof::Scope scope(prof::kMGS, 8.0 * (cnt + 2) * (double)n, 4.0 * (2 * cnt + 1) * (double)n,
                      s);
    double *part = dot_partials + gi * gstride;
    if (vec) {
      switch (cnt) {
#define PMK_DOTS_CASE(C)                        \
  case C:                                       \
    dots_vec<C>(st, w, v[j], V, n, part, s);    \
    break;
#if PMK_DOT_GROUP > 8
        PMK_CASES16(PMK_DOTS_CASE)
#else
        PMK_CASES8(PMK_DOTS_CASE)
#endif
#undef PMK_DOTS_CASE
        default:
          return PMK_ERR_ARG;
      }
    } else {
      icwy_dots_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(st, w, v[j], V, cnt, n, part);
    }
    PMK_LAUNCH_CHECK();
  }
  {
    prof::Scope scope(prof::kSmall, 0.0, 0.0, s);
    icwy_solve_kernel<<<1, 1024, (2 * j + 1) * sizeof(double), s>>>(
        st, ld, j, c0p, n_c0, pj, dot_partials, kRedBlocks, ug ? 1 : 0);
    PMK_LAUNCH_CHECK();
  }
  for (int i0 = 0; i0 <= j; i0 += kGroup) {
    const int cnt = (j + 1 - i0 < kGroup) ? j + 1 - i0 : kGroup;
    const bool last = i0 + cnt > j;
    MultiVec V{};
    for (int q = 0; q < cnt; ++q) V.v[q] = v[i0 + q];
    const bool store = keep_w || !last;
    const bool fin = last && fuse_finish && vec;
    if (fin && finished) *finished = true;
    // one pass over all of v_0..v_j: it can leave the next vector's Gram row
    const bool gram = ugram_out && vec && store && i0 == 0 && last;
    if (gram && ugram_done) *ugram_done = true;
    prof::Scope scope(prof::kMGS, 8.0 * (cnt + (store ? 2 : 1)) * (double)n,
                      2.0 * (cnt + (last ? 1 : 0)) * (double)n, s);
    double *part = last ? norm_partials : nullptr;
    if (vec) {
      switch (cnt) {
#define PMK_UPD_CASE(C)                                \
  case C:                                              \
    update_vec<C>(st, ld, j, i0, V, w, n, part, store, fin, tol, s, gram); \
    break;
        PMK_CASES16(PMK_UPD_CASE)
#undef PMK_UPD_CASE
        default:
          return PMK_ERR_ARG;
      }
    } else {
      icwy_update_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(st, ld, j, i0, V, cnt, w, n, part,
                                                            store);
    }
    PMK_LAUNCH_CHECK();
  }
  *n_norm = kRedBlocks;
  return 0;
}

int launch_icwy_solve(KState *st, int ld, int j, const double *c0p, int n_c0,
                      cudaStream_t s) {
  PMK_RETURN_IF(j != 0, PMK_ERR_ARG);  // column 0: h_00 = <w, v_0> only
  prof::Scope scope(prof::kSmall, 0.0, 0.0, s);
  icwy_solve_kernel<<<1, 1024, sizeof(double), s>>>(st, ld, 0, c0p, n_c0, nullptr, nullptr, 0);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_finish_col(KState *st, int ld, int j, const double *partials, int n_partials,
                      double tol, cudaStream_t s, bool pyth) {
  PMK_RETURN_IF(pyth && j != 0, PMK_ERR_ARG);
  prof::Scope scope(prof::kSmall, 0.0, 0.0, s);
  finish_col_kernel<<<1, kRedThreads, 0, s>>>(st, ld, j, partials, n_partials, tol, pyth);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_backsolve(KState *st, int ld, cudaStream_t s, const double *out_scale) {
  prof::Scope scope(prof::kSmall, 0.0, 0.0, s);
  backsolve_kernel<<<1, 32, 0, s>>>(st, ld, out_scale);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_assemble(const KState *st, const AssembleArgs &a, double *x, int64_t n, int m, int nu,
                    int m_coarse, const int32_t *group_of, int first, cudaStream_t s) {
  const double nc = (double)(n / m - 1) / nu + 1.0;  // coarse rows
  prof::Scope scope(prof::kAsm,
                    a.count * (8.0 * (double)n + 8.0 * nc * m_coarse) + (first ? 16.0 : 8.0) * n,
                    0.0, s);
  const int rows = (int)(n / m);
  if (!group_of && nu == 2 && m_coarse == m && a.count >= 1 && a.count <= 8) {
    const int u = (12 / (3 * a.count)) > 1 ? 12 / (3 * a.count) : 1;
    const int xb = (m + 256 * u - 1) / (256 * u);
    const int target = 8 * kSMs * 8;  // ~8 waves of 8 resident blocks per SM
    const int n_coarse = rows / 2 + 1;  // K = 0 and the pairs (2K-1, 2K)
    int yb = (target + xb - 1) / xb;
    if (yb > n_coarse) yb = n_coarse;
    dim3 grid(xb, yb < 1 ? 1 : yb);
    switch (a.count) {
#define PMK_ASM_CASE(C)                                                             \
  case C:                                                                           \
    assemble_pair_kernel<C><<<grid, 256, 0, s>>>(st, a, x, rows, m, first);         \
    break;
      PMK_ASM_CASE(1) PMK_ASM_CASE(2) PMK_ASM_CASE(3) PMK_ASM_CASE(4)
      PMK_ASM_CASE(5) PMK_ASM_CASE(6) PMK_ASM_CASE(7) PMK_ASM_CASE(8)
#undef PMK_ASM_CASE
    }
    PMK_LAUNCH_CHECK();
    return 0;
  }
  dim3 grid((m + 255) / 256, rows < 1024 ? rows : 1024);
  if (grid.x > 64) grid.x = 64;
  assemble_kernel<<<grid, 256, 0, s>>>(st, a, x, rows, m, nu, m_coarse, group_of, first);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_div_check(const double *x, double d, int64_t n, double *out, cudaStream_t s) {
  if (!div_ok(d)) return PMK_ERR_ARG;
  div_check_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, d, n, out);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_restrict_time(const pmk_pair &P, const double *v, double *vh, cudaStream_t s) {
  const int64_t n = (int64_t)(P.n_T + 1) * P.m_fine;
  prof::Scope scope(prof::kXfer, 8.0 * n + 8.0 * (double)(P.nu * P.n_T + 1) * P.m_fine, 0.0, s);
  restrict_time_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, vh, P.nu, P.n_T, P.m_fine);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_ts_gather(const pmk_pair &P, const double *fine, double *coarse, const int *live,
                     cudaStream_t s) {
  const int64_t n = (int64_t)(P.n_T + 1) * P.m_coarse;
  prof::Scope scope(prof::kXfer, 8.0 * n + 8.0 * (double)(P.n_T + 1) * P.m_fine, 0.0, s);
  ts_gather_kernel<<<grid_for(n, 256), 256, 0, s>>>(fine, coarse, P.y_ptr, P.y_idx, P.y_val,
                                                    P.n_T + 1, P.m_fine, P.m_coarse, live);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_interpolate_z(const pmk_pair &P, const double *w, double *out, int nu,
                         const int *live, cudaStream_t s) {
  const int rows = nu * P.n_T + 1;
  const int64_t n = (int64_t)rows * P.m_fine;
  prof::Scope scope(prof::kXfer, 8.0 * n + 8.0 * (double)(P.n_T + 1) * P.m_coarse, 0.0, s);
  interpolate_z_kernel<<<grid_for(n, 256), 256, 0, s>>>(w, out, nu, rows, P.m_fine, P.m_coarse,
                                                        P.z_ptr, P.z_idx, P.z_val, live);
  PMK_LAUNCH_CHECK();
  return 0;
}

int launch_interpolate(const pmk_pair &P, const double *w, double *out, cudaStream_t s) {
  if (P.z_ptr) return launch_interpolate_z(P, w, out, P.nu, nullptr, s);
  const int64_t n = (int64_t)(P.nu * P.n_T + 1) * P.m_fine;
  prof::Scope scope(prof::kXfer, 8.0 * n + 8.0 * (double)(P.n_T + 1) * P.m_coarse, 0.0, s);
  interpolate_kernel<<<grid_for(n, 256), 256, 0, s>>>(w, out, P.nu, P.n_T, P.m_fine, P.m_coarse,
                                                      P.group_of);
  PMK_LAUNCH_CHECK();
  return 0;
}

}  // namespace pmk
