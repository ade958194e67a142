// pmk_march.cu -- fused space-time stencil kernels (K-MV, K-MVR, K-IMV).
//
// The block lower-bidiagonal operator of a level (reference
// stepper.py:96-105) is applied as ONE stencil sweep over all time slices:
//
//     out_0 = v_0,   out_k = D^T v_k - B^T v_{k-1}  (+ B^T v_{k-1} if dropped)
//
// Each thread owns one grid column x and R consecutive rows, and marches
// forward in time over a chunk of slices.  Per slice it loads its R+2 rows
// once (coalesced across the warp), gets the x-neighbours through warp
// shuffles (lanes 0/31 load one halo value), and computes D^T v_k and
// B^T v_k together; B^T v_k is kept in registers for slice k+1.  Every input
// element is therefore read from DRAM once and every output written once:
// 16 B per space-time unknown for the plain matvec.
//
// The stencil sums run in ascending column order (S, W, C, E, N) with
// separately rounded products, which is the order scipy's csc_matvecs uses
// for `blocks @ diag` -- the GPU matvec is bitwise identical to the
// reference's.
//
// Fused variants (one DRAM pass each):
//   MVR  solver.py:336-339      vh = restrict(A v - mu v)  (time sum over nu
//                               slices in registers; intergrid.py:51-56)
//   IMV  solver.py:349,359,403  x = v - interpolate(vt); w = A x; and the
//                               partial dot(w, v_0) that seeds MGS
//                               (solver.py:407, l = 0)
#include <cstdlib>

#include "pmk_internal.cuh"

namespace pmk {
namespace {

constexpr unsigned kFull = 0xffffffffu;

struct Coef5 {
  double s, w, c, e, n;
};

__device__ __forceinline__ double stencil5(const Coef5 &a, bool hs, double vs, bool hw, double vw,
                                           double vc, bool he, double ve, bool hn, double vn) {
  // scipy csc_matvecs order: y = 0; y += a_j * x_j for ascending j.
  double acc = 0.0;
  if (hs) acc = __dadd_rn(acc, __dmul_rn(a.s, vs));
  if (hw) acc = __dadd_rn(acc, __dmul_rn(a.w, vw));
  acc = __dadd_rn(acc, __dmul_rn(a.c, vc));
  if (he) acc = __dadd_rn(acc, __dmul_rn(a.e, ve));
  if (hn) acc = __dadd_rn(acc, __dmul_rn(a.n, vn));
  return acc;
}

__device__ __forceinline__ Coef5 load_coef(const pmk_stencil &st, bool in, int64_t i, int m) {
  if (!st.var) return Coef5{st.c[0], st.c[1], st.c[2], st.c[3], st.c[4]};
  if (!in) return Coef5{0, 0, 0, 0, 0};
  const double *c = st.coef;
  return Coef5{c[i], c[m + i], c[2 * (int64_t)m + i], c[3 * (int64_t)m + i],
               c[4 * (int64_t)m + i]};
}

template <int MODE>
__device__ __forceinline__ double fetch(const MarchParams &p, double vsc, int k, int y, int x) {
  const int64_t i = (int64_t)y * p.nx + x;
  PMK_CHECK_IDX(i, p.m, "fetch.i");
  PMK_CHECK_IDX((int64_t)k * p.m + i, (int64_t)(p.n_steps + 1) * p.m, "fetch.v");
  double u = p.v[(int64_t)k * p.m + i];
  if (p.v_scale) u = __ddiv_rn(u, vsc);
  if (MODE == kModeIMV) {
    const int K = (k == 0) ? 0 : (k - 1) / p.nu + 1;
    const int64_t gi = p.group_of ? (int64_t)p.group_of[i] : i;
    PMK_CHECK_IDX((int64_t)K * p.m_coarse + gi,
                  (int64_t)(p.n_steps / p.nu + 1) * p.m_coarse, "fetch.vt");
    u = __dsub_rn(u, p.vt[(int64_t)K * p.m_coarse + gi]);
  }
  return u;
}

template <int DIM, int MODE, int R, bool VAR>
__global__ void __launch_bounds__(256)
    march_kernel(const MarchParams p, int BX, int gx, int gy, int upc, int n_chunks) {
  if (!is_live(p.live)) return;
  const int U = (MODE == kModeMVR) ? p.nu : 1;
  const int n_units = p.n_steps / U + 1;
  const int tiles = gx * gy;
  const int64_t n_items = (int64_t)tiles * n_chunks;
  const int lane = threadIdx.x & 31;
  const double vsc = p.v_scale ? *p.v_scale : 1.0;
  const double v0sc = (MODE == kModeIMV && p.v0_scale) ? *p.v0_scale : 1.0;
  double dot = 0.0;

  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int tile = (int)(item % tiles);
    const int chunk = (int)(item / tiles);
    const int x = (tile % gx) * BX + threadIdx.x;
    const int y0 = (tile / gx) * R;
    const bool xin = x < p.nx;
    const int U0 = chunk * upc;
    const int U1 = min(n_units, U0 + upc);
    const int kb = (U0 == 0) ? 0 : U * (U0 - 1) + 1;
    const int ke = U * (U1 - 1) + 1;

    Coef5 pc[VAR ? R : 1], qc[VAR ? R : 1];
    if constexpr (VAR) {
      // Either operator may be per-point while the other is constant (e.g.
      // theta = 1 makes B = I, whose stored pattern is only the diagonal).
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int y = y0 + r;
        const bool in = xin && y < p.ny;
        const int64_t i = (int64_t)y * p.nx + x;
        pc[r] = load_coef(p.P, in, i, p.m);
        qc[r] = load_coef(p.Q, in, i, p.m);
      }
    } else {
      pc[0] = Coef5{p.P.c[0], p.P.c[1], p.P.c[2], p.P.c[3], p.P.c[4]};
      qc[0] = Coef5{p.Q.c[0], p.Q.c[1], p.Q.c[2], p.Q.c[3], p.Q.c[4]};
    }

    double qprev[R];
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      qprev[r] = 0.0;
      acc[r] = 0.0;
    }

    const int kstart = (kb > 0) ? kb - 1 : 0;
    for (int k = kstart; k < ke; ++k) {
      const bool prime = k < kb;
      double u[R + 2];
#pragma unroll
      for (int r = 0; r < R + 2; ++r) {
        const int y = y0 - 1 + r;
        const bool ok = (DIM == 2 || r == 1) && xin && y >= 0 && y < p.ny;
        u[r] = ok ? fetch<MODE>(p, vsc, k, y, x) : 0.0;
      }
      double hal[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int y = y0 + r;
        const int hx = (lane == 0) ? x - 1 : x + 1;
        const bool need = (lane == 0 || lane == 31) && y < p.ny && hx >= 0 && hx < p.nx;
        hal[r] = need ? fetch<MODE>(p, vsc, k, y, hx) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double c = u[r + 1];
        double l = __shfl_up_sync(kFull, c, 1);
        double rr = __shfl_down_sync(kFull, c, 1);
        if (lane == 0) l = hal[r];
        if (lane == 31) rr = hal[r];
        const int y = y0 + r;
        const bool hs = DIM == 2 && y > 0;
        const bool hn = DIM == 2 && y < p.ny - 1;
        const bool hw = x > 0;
        const bool he = x < p.nx - 1;
        const Coef5 &a = pc[VAR ? r : 0];
        const Coef5 &b = qc[VAR ? r : 0];
        const double Pu = stencil5(a, hs, u[r], hw, l, c, he, rr, hn, u[r + 2]);
        const double Qu = stencil5(b, hs, u[r], hw, l, c, he, rr, hn, u[r + 2]);
        const bool valid = xin && y < p.ny;
        if (!prime && valid) {
          double o;
          if (k == 0) {
            o = c;  // identity block row (stepper.py:100)
          } else {
            o = __dsub_rn(Pu, qprev[r]);
            if (p.dropped && p.dropped[k]) o = __dadd_rn(o, qprev[r]);  // stepper.py:103-104
          }
          const int64_t i = (int64_t)y * p.nx + x;
          const int64_t e = (int64_t)k * p.m + i;
          PMK_CHECK_IDX(e, (int64_t)(p.n_steps + 1) * p.m, "store.e");
          if (MODE == kModeMV) {
            p.out[e] = o;
          } else if (MODE == kModeMVR) {
            if (p.v_norm_out) p.v_norm_out[e] = c;  // basis vector b/beta, w/h (solver.py:395,420)
            const double sv = __dsub_rn(o, __dmul_rn(p.mu, c));  // s -= mu * v
            if (p.inject) {
              if (k % p.nu == 0) p.vh[(int64_t)(k / p.nu) * p.m + i] = sv;
            } else if (k == 0) {
              p.vh[i] = sv;
            } else {
              const int pos = (k - 1) % p.nu;
              acc[r] = (pos == 0) ? sv : __dadd_rn(acc[r], sv);
              if (pos == p.nu - 1) p.vh[(int64_t)((k - 1) / p.nu + 1) * p.m + i] = acc[r];
            }
          } else {  // IMV
            if (p.x_out) p.x_out[e] = c;
            if (p.out) p.out[e] = o;
            if (p.partials) {
              double v0v = p.v0[e];
              if (p.v0_scale) v0v = __ddiv_rn(v0v, v0sc);
              dot = __dadd_rn(dot, __dmul_rn(o, v0v));
            }
          }
        }
        qprev[r] = Qu;
      }
    }
  }
  if (MODE == kModeIMV && p.partials) {
    const double s = block_sum(dot);
    if (threadIdx.x == 0) p.partials[blockIdx.x] = s;
  }
}

struct Geometry {
  int BX, gx, gy, upc, n_chunks, grid;
};

template <int DIM, int MODE, int R, bool VAR>
int run(const MarchParams &p, cudaStream_t s, int *n_partials, double bytes, int cat) {
  auto kern = march_kernel<DIM, MODE, R, VAR>;
  static int occ = -1;
  if (occ < 0) {
    int b = 0;
    PMK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 0));
    occ = b > 0 ? b : 1;
  }
  // Block width: 256 columns (fewer for narrow grids, multiple of 32).
  int BX = ((p.nx + 31) / 32) * 32;
  if (BX > 256) BX = 256;
  const int gx = (p.nx + BX - 1) / BX;
  const int gy = (DIM == 2) ? (p.ny + R - 1) / R : 1;
  const int U = (MODE == kModeMVR) ? p.nu : 1;
  const int n_units = p.n_steps / U + 1;
  const int tiles = gx * gy;
  int grid_cap = occ * kSMs;
  if (MODE == kModeIMV && grid_cap > kMaxPartials) grid_cap = kMaxPartials;
  // Time chunking: enough items for ~8 per resident block, at most 32 units
  // per chunk (prime overhead 1/upc of a slice read, served from L2).
  const int64_t target = 8LL * grid_cap;
  int64_t upc = ((int64_t)n_units * tiles) / (target > 0 ? target : 1);
  if (upc < 1) upc = 1;
  if (upc > 32) upc = 32;
  const int n_chunks = (int)((n_units + upc - 1) / upc);
  const int64_t n_items = (int64_t)tiles * n_chunks;
  const int grid = (int)(n_items < grid_cap ? n_items : grid_cap);
  prof::Scope scope(cat, bytes, 0.0, s);
  // BX threads per block (whole warps: the x-neighbours come from shuffles).
  march_kernel<DIM, MODE, R, VAR><<<grid, BX, 0, s>>>(p, BX, gx, gy, (int)upc, n_chunks);
  PMK_LAUNCH_CHECK();
  if (n_partials) *n_partials = grid;
  return 0;
}

template <int MODE>
int dispatch(const MarchParams &p, cudaStream_t s, int *n_partials, double b, int c) {
  const bool var = p.P.var || p.Q.var;
  if (p.ny == 1) {
    return var ? run<1, MODE, 1, true>(p, s, n_partials, b, c)
               : run<1, MODE, 1, false>(p, s, n_partials, b, c);
  }
  return var ? run<2, MODE, 2, true>(p, s, n_partials, b, c)
             : run<2, MODE, 8, false>(p, s, n_partials, b, c);
}

// Algorithmic DRAM bytes of one launch.
double march_bytes(int mode, const MarchParams &p, int *cat) {
  const double N = (double)(p.n_steps + 1) * p.m;
  if (mode == kModeMV) {
    *cat = prof::kMV;
    return 16.0 * N;
  }
  if (mode == kModeMVR) {
    *cat = prof::kMVR;
    double b = 8.0 * N + 8.0 * (double)(p.n_steps / p.nu + 1) * p.m;
    if (p.v_norm_out) b += 8.0 * N;
    if (p.v_sub) b += 8.0 * N;
    return b;
  }
  *cat = prof::kIMV;
  double b = 8.0 * N + 8.0 * (double)(p.n_steps / p.nu + 1) * p.m_coarse;
  if (p.out) b += 8.0 * N;
  if (p.x_out) b += 8.0 * N;
  if (p.partials) b += 8.0 * N;
  return b;
}

}  // namespace

int launch_march(int mode, const MarchParams &p, cudaStream_t s, int *n_partials) {
  if (mode != kModeMV && mode != kModeMVR && mode != kModeIMV) return PMK_ERR_ARG;
  if (p.pj_done) *p.pj_done = 0;
  int cat = 0;
  const double bytes = march_bytes(mode, p, &cat);
  static const bool force_reg = getenv("PMK_MARCH_REG") != nullptr;
  if (!force_reg) {
    int handled = 0;
    const int rc = launch_march_tma(mode, p, s, n_partials, bytes, cat, &handled);
    if (rc || handled) return rc;
  }
  if (p.v_sub) return PMK_ERR_UNSUPPORTED;  // sub mode: TMA path only
  switch (mode) {
    case kModeMV:
      return dispatch<kModeMV>(p, s, n_partials, bytes, cat);
    case kModeMVR: {
      MarchParams q = p;
      q.vh_partials = nullptr;  // ||vh||^2 partials are a TMA-path product
      const int rc = dispatch<kModeMVR>(q, s, nullptr, bytes, cat);
      if (n_partials) *n_partials = 0;
      return rc;
    }
    default:
      return dispatch<kModeIMV>(p, s, n_partials, bytes, cat);
  }
}

}  // namespace pmk
