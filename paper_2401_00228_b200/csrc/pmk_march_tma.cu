// pmk_march_tma.cu -- TMA-pipelined fused space-time stencil kernels
// (K-MV, K-MVR, K-IMV; same semantics and rounding as pmk_march.cu).
//
// Data movement: every input space-time vector is described by a 1-D TMA
// tensor map over its N doubles (out-of-range box elements are zero-filled,
// so no end-of-array cases exist).  A box must start 16-byte aligned (an odd
// fp64 coordinate raises an illegal-instruction fault on sm_100a), so each
// row box is issued at the even coordinate at or below the row start and the
// consumer applies the row's parity shift; a tile is therefore at most 255
// columns wide (single tile) or 252 plus halo (wider rows).  A CTA owns a tile of R grid
// rows x up to 256 columns and streams consecutive time slices of it through
// an S-stage shared-memory ring: one elected thread issues, per slice, R+2
// row boxes (256 doubles = 2 KB each; the rows above/below are the halo)
// with cp.async.bulk.tensor, completion tracked by an mbarrier per stage.
// The copy engine keeps S slices in flight per CTA while the threads
// compute, which is what the register version lacked (it was latency- and
// issue-bound at ~15% of HBM bandwidth).
//
// Compute per slice:
//   pre-pass   each thread transforms one box column in place, once per
//              element: v * RN(1/scale) (lazily normalised basis vector; the
//              normalised value is also stored, solver.py:395/420) or
//              v - Z vt (K-IMV; vt staged through the same ring);
//   stencil    each thread walks its column down the R rows keeping the
//              vertical neighbours in registers (3 shared loads per output),
//              forms D^T u_k and B^T u_k in ascending column order with
//              separately rounded products (bitwise the reference's scipy
//              product), keeps B^T u_k in registers for slice k+1, and
//              writes the mode's outputs with coalesced stores.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include <type_traits>

#include "pmk_internal.cuh"

namespace pmk {
namespace {

constexpr int kBox = 256;  // doubles per TMA box (one tile row)
constexpr int kTmaThreads = 256;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "PMK_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra PMK_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_row(double *dst, const CUtensorMap *map, int coord,
                                        uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2}], [%3];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(coord), "r"(smem_u32(bar))
      : "memory");
}

// Same row box as a plain bulk copy (64-bit global address, no tensor map):
// the vectors whose coordinates exceed int32 (N >= 2^31 doubles).  Without a
// tensor map there is no out-of-range zero fill, so the box is clipped to
// [0, n) (16-byte granules); the clipped elements sit at row positions the
// kernels never read (x = -1 of the first row, past the end of the last).
// Returns the bytes requested.
__device__ __forceinline__ uint32_t bulk_bytes(int64_t c, int64_t n) {
  int64_t lo = c < 0 ? 0 : c, hi = c + kBox;
  const int64_t nr = (n + 1) & ~(int64_t)1;  // (16-byte granules)
  if (hi > nr) hi = nr;
  return hi > lo ? (uint32_t)((hi - lo) * 8) : 0u;
}
__device__ __forceinline__ void bulk_row(double *dst, const double *base, int64_t c, int64_t n,
                                         uint64_t *bar) {
  const int64_t lo = c < 0 ? 0 : c;
  const uint32_t bytes = bulk_bytes(c, n);
  if (!bytes) return;
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst + (lo - c))),
      "l"(reinterpret_cast<uint64_t>(base + lo)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct Coef5 {
  double s, w, c, e, n;
};

// Dropped-coupling flags are read a slice ahead through a pointer that is
// always valid (stride 0 over a zero byte when the level has no dropped
// rows), so the load is never predicated off: a predicated-off load keeps its
// scoreboard until the memory pipe retires it, which stalled its consumer
// behind every other load sharing that scoreboard.
__device__ const uint8_t g_no_drop = 0;

__device__ __forceinline__ Coef5 coef_at(const pmk_stencil &st, int64_t i, int m) {
  if (!st.var) return Coef5{st.c[0], st.c[1], st.c[2], st.c[3], st.c[4]};
  const double *c = st.coef;
  return Coef5{__ldg(c + i), __ldg(c + m + i), __ldg(c + 2 * (int64_t)m + i),
               __ldg(c + 3 * (int64_t)m + i), __ldg(c + 4 * (int64_t)m + i)};
}

__device__ __forceinline__ double stencil5(const Coef5 &a, bool hs, double vs, bool hw, double vw,
                                           double vc, bool he, double ve, bool hn, double vn) {
  double acc = 0.0;  // scipy csc_matvecs order: ascending column index
  if (hs) acc = __dadd_rn(acc, __dmul_rn(a.s, vs));
  if (hw) acc = __dadd_rn(acc, __dmul_rn(a.w, vw));
  acc = __dadd_rn(acc, __dmul_rn(a.c, vc));
  if (he) acc = __dadd_rn(acc, __dmul_rn(a.e, ve));
  if (hn) acc = __dadd_rn(acc, __dmul_rn(a.n, vn));
  return acc;
}

struct TmaGeom {
  int bulk;         // 1: plain bulk copies from p.v / p.vt / p.v_sub (no tensor maps)
  int64_t n_v, n_vt;  // their lengths (bulk clipping)
  int single;  // 1: one column tile per row, box starts at x = 0
  int tile_w;  // output columns per tile (1-D: per segment)
  int nseg;    // 1-D: column segments per row
  int gx, gy;  // column tiles, row groups
  int upc, n_chunks;
};

// IMVK (in-solver K-IMV only) fixes the launch-uniform dot-product flags at
// compile time, so the row loop carries no test of them: 0 = read them from
// the parameters; 1 = j = 0 (v is v_0), <w, v_0> only; 2 = j = 0 plus ||w||^2
// (budget-1 levels); 3 = j >= 1 with the pj dots <w, v_j>, <v_j, v_0>; 4 =
// j >= 1, <w, v_0> only.  For the in-solver K-MVR, IMVK = 1 is the common
// contract -- v not stored (lazy basis; the sub mode always stores it),
// time-sum restriction (no MGRIT injection) -- likewise fixed at compile time.
template <int MODE, int DIM, int R, int S, bool VAR, bool GATHER, bool SCALED, bool FMA,
          int IMVK = 0>
__global__ void __launch_bounds__(kTmaThreads)
    march_tma_kernel(const MarchParams p, const __grid_constant__ CUtensorMap tm_v,
                     const __grid_constant__ CUtensorMap tm_vt, const TmaGeom g) {
  // K-MVR "sub" mode (MarchParams::v_sub; GATHER, meaningless for K-MVR,
  // selects it): the staged input is w - c v_sub, v_sub staged alongside
  constexpr bool kSub = MODE == kModeMVR && GATHER;
  constexpr int NB = ((MODE == kModeIMV && !GATHER) || kSub) ? 2 : 1;
  constexpr int ROWS = (DIM == 2) ? R + 2 : 1;
  constexpr int RO = (DIM == 2) ? R : 1;  // output rows per tile
  // TMA tensor destinations must be 128-byte aligned; dynamic shared memory
  // follows the static part at an unspecified alignment, so align by hand.
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // (offset arithmetic on the shared pointer keeps shared-space loads)
  double *smem = reinterpret_cast<double *>(
      smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t bars[S];

  if (!is_live(p.live)) return;
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int nx = p.nx, ny = p.ny, m = p.m;
  const int U = (MODE == kModeMVR) ? p.nu : 1;
  const int n_units = p.n_steps / U + 1;
  const int tiles = g.gx * g.gy;
  const int64_t n_items = (int64_t)tiles * g.n_chunks;
  // normalisation of a lazily scaled basis vector: multiply by RN(1 / scale)
  // (within 1 ulp of the division; exact_scale launches take the register path)
  const double vrcp = SCALED ? __drcp_rn(*p.v_scale) : 1.0;
  double dot = 0.0;
  double dwj = 0.0, dgj = 0.0;  // K-IMV with pj: <w, v>, <v, v0>
  // (in-solver variant only; run_tma reports it through p.pj_done)
  constexpr bool kPj = MODE == kModeIMV && DIM == 2 && FMA && !VAR && !GATHER;
  const bool wantj = IMVK ? IMVK == 3 : (kPj && p.pj != nullptr && !p.pj_wsq);
  const bool wantw = IMVK ? IMVK == 2 : (kPj && p.pj != nullptr && p.pj_wsq);  // ||w||^2 into slot 0
  // In-solver (FMA) launches honour a fixed contract, checked by the
  // launcher: K-IMV writes w (p.out) and the <w, v_0> partials and no x;
  // K-MVR writes the normalised v (p.v_norm_out).  Compile-time flags keep
  // the per-row null tests (and their constant-bank reloads) out of the loop.
  constexpr bool kSolver = FMA;
  const bool has_out = kSolver ? (MODE != kModeMVR) : (p.out != nullptr);
  const bool has_x = kSolver ? false : (p.x_out != nullptr);
  const bool has_part = kSolver ? (MODE == kModeIMV) : (p.partials != nullptr);
  // (K-MVR's normalised v is optional: with a lazy basis nobody stores it)
  const bool has_vn = (MODE == kModeMVR && IMVK == 1) ? kSub : p.v_norm_out != nullptr;
  const bool mvr_inject = (MODE == kModeMVR && IMVK == 1) ? false : p.inject != 0;
  const bool has_drop = !kSolver;  // (solver launches: no dropped rows, no load)
  // In-solver K-MVR works on the raw (unnormalised) staged values: the
  // operator is linear, so A v - mu v = RN(1/h) (A raw - mu raw) up to
  // rounding; only the stored outputs are scaled (v itself is stored as
  // RN(raw * RN(1/h)), exactly the pre-pass value).  No pre-pass, and one
  // block barrier per slice fewer.
  constexpr bool kLazy = FMA && MODE == kModeMVR && SCALED;
  const double osc = kLazy ? vrcp : 1.0;
  const double csub = kSub ? *p.v_sub_coef : 0.0;
  double wsq = 0.0;  // sub mode: ||w - c v_0||^2 of the stored values
  // j = 0 (v is v_0): <w, v_0> takes the staged input itself, no v_0 stream
  const bool v0_self = IMVK ? IMVK <= 2 : (kPj && p.v0 == p.v);
  // a lazily scaled v_0 (raw rhs, divisor *v0_scale) is scaled at use
  // a lazily scaled v_0 (raw rhs, divisor *v0_scale): the dot products with
  // it are accumulated raw and scaled once at the end (j >= 1; at j = 0 the
  // staged, already scaled input is v_0 itself)
  double vsq = 0.0;  // K-MVR: partial ||vh||^2 of the values this thread stores
  uint32_t it = 0;  // slices consumed by this CTA (ring position)

  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int tile = (int)(item % tiles);
    const int chunk = (int)(item / tiles);
    const int x0 = (tile % g.gx) * g.tile_w;
    const int y0 = (DIM == 2) ? (tile / g.gx) * R : 0;
    const int U0 = chunk * g.upc;
    const int U1 = min(n_units, U0 + g.upc);
    const int kb = (U0 == 0) ? 0 : U * (U0 - 1) + 1;
    const int ke = U * (U1 - 1) + 1;
    const int kstart = (kb > 0) ? kb - 1 : 0;
    const int nsl = ke - kstart;
    const int boxx = g.single ? 0 : x0 - 1;  // grid column of box element 0

    // rows of the tile that exist
    int rlo = 0, rhi = ROWS - 1;
    if (DIM == 2) {
      if (y0 - 1 < 0) rlo = 1;
      if (y0 - 1 + rhi > ny - 1) rhi = ny - 1 - (y0 - 1);
    }
    const uint32_t tx_bytes = (uint32_t)(NB * (rhi - rlo + 1) * kBox * sizeof(double));
    const double *vt_src = kSub ? p.v_sub : p.vt;

    auto issue = [&](int k, int stage) {
      double *sv = smem + (size_t)stage * NB * ROWS * kBox;
      const int K = (k == 0) ? 0 : (k - 1) / p.nu + 1;
      if (g.bulk) {
        uint32_t bytes = 0;
        for (int r = rlo; r <= rhi; ++r) {
          const int y = (DIM == 2) ? y0 - 1 + r : 0;
          const int64_t c = (int64_t)k * m + (int64_t)y * nx + boxx;
          bytes += bulk_bytes(c & ~(int64_t)1, g.n_v);
          if (NB == 2) {
            const int64_t cv = kSub ? c : (int64_t)K * p.m_coarse + (int64_t)y * nx + boxx;
            bytes += bulk_bytes(cv & ~(int64_t)1, g.n_vt);
          }
        }
        mbar_expect_tx(&bars[stage], bytes);
        for (int r = rlo; r <= rhi; ++r) {
          const int y = (DIM == 2) ? y0 - 1 + r : 0;
          const int64_t c = (int64_t)k * m + (int64_t)y * nx + boxx;
          bulk_row(sv + r * kBox, p.v, c & ~(int64_t)1, g.n_v, &bars[stage]);
          if (NB == 2) {
            const int64_t cv = kSub ? c : (int64_t)K * p.m_coarse + (int64_t)y * nx + boxx;
            bulk_row(sv + (ROWS + r) * kBox, vt_src, cv & ~(int64_t)1, g.n_vt, &bars[stage]);
          }
        }
        return;
      }
      mbar_expect_tx(&bars[stage], tx_bytes);
      for (int r = rlo; r <= rhi; ++r) {
        const int y = (DIM == 2) ? y0 - 1 + r : 0;
        const int c = (int)((int64_t)k * m + (int64_t)y * nx + boxx);
        tma_row(sv + r * kBox, &tm_v, c & ~1, &bars[stage]);
        if (NB == 2) {
          const int cv = kSub ? c : (int)((int64_t)K * p.m_coarse + (int64_t)y * nx + boxx);
          tma_row(sv + (ROWS + r) * kBox, &tm_vt, cv & ~1, &bars[stage]);
        }
      }
    };
    if (t == 0) {
      const int pre = nsl < S ? nsl : S;
      for (int q = 0; q < pre; ++q) issue(kstart + q, (int)((it + q) % S));
    }

    // this thread's output column
    const int x = g.single ? t : x0 + t;
    const bool xin = (g.single ? t < nx : t < g.tile_w) && x < nx;
    const bool hw = x > 0, he = x < nx - 1;
    // this thread's pre-pass box element: the one holding its own output
    // column (box element x - boxx, so that the staged input of its outputs
    // stays in registers); on split rows thread kBox-1 takes element 0.
    const int pe = g.single ? t : ((t == kBox - 1) ? 0 : t + 1);
    const int px = boxx + pe;
    const bool pin = pe < kBox - 1 && px >= 0 && px < nx;

    double qprev[RO], acc[RO];
#pragma unroll
    for (int r = 0; r < RO; ++r) {
      qprev[r] = 0.0;
      acc[r] = 0.0;
    }
    Coef5 pcst, qcst;
    if (!VAR) {
      pcst = Coef5{p.P.c[0], p.P.c[1], p.P.c[2], p.P.c[3], p.P.c[4]};
      qcst = Coef5{p.Q.c[0], p.Q.c[1], p.Q.c[2], p.Q.c[3], p.Q.c[4]};
    }

    const int nu = p.nu;
    const int xo = x - boxx;         // box offset of this thread's output column
    const int gx0 = y0 * nx + x;     // in-slice index of (y0, x)
    // Warps whose columns are all interior (no W/E boundary, all in range) on a
    // tile whose rows and row neighbours all exist take the mask-free variant
    // of the stencil pass below (same operations, no neighbour selects).
    const bool tile_interior = DIM == 2 && (R % 2 == 0) && rlo == 0 && y0 + R <= ny - 1;
    // In-solver (FMA) launches take the fused pass on every warp of an interior
    // tile, zeroing the absent W/E neighbours of the first/last column (their
    // products then add +-0) and masking the stores of columns past the grid:
    // no warp of the tile runs the slower masked variant while the others wait
    // for it at the slice barriers.
    const bool warp_fast =
        FMA ? tile_interior : __all_sync(0xffffffffu, tile_interior && xin && hw && he);
    double v0next[RO];
    if (MODE == kModeIMV && has_part && !v0_self) {
      const int kf = (kb > kstart) ? kb : kstart;  // first non-prime slice
#pragma unroll
      for (int r = 0; r < RO; ++r)
        v0next[r] = (xin && kf < ke && y0 + r < ny)
                        ? __ldg(p.v0 + (int64_t)kf * m + gx0 + r * nx)
                        : 0.0;
    }
    int Kc = (kstart == 0) ? 0 : (kstart - 1) / nu + 1;
    int posc = (kstart == 0) ? nu - 1 : (kstart - 1) - (Kc - 1) * nu;
    const uint8_t *dflag = p.dropped ? p.dropped : &g_no_drop;
    const int dstep = p.dropped ? 1 : 0;
    int dnext = (has_drop && kstart < ke) ? dflag[kstart * dstep] : 0;
    for (int i = 0; i < nsl; ++i, ++it) {
      // ---- per-slice uniform quantities
      const int k = kstart + i;
      const bool prime = k < kb;
      const int stage = (int)(it % S);
      double *sv = smem + (size_t)stage * NB * ROWS * kBox;
      // coarse slice K of k and position in its slab (stepped, no division)
      const int K = Kc, pos = posc;
      if (k == 0) {
        Kc = 1;
        posc = 0;
      } else if (++posc == nu) {
        ++Kc;
        posc = 0;
      }
      // dropped coupling of k: loaded one slice ahead, off the critical path
      const bool drop = dnext != 0;
      // (a predicated-off load still holds its scoreboard until the memory
      // pipe retires it, and shares it with the v_0 prefetch: solver
      // launches have no dropped rows and skip the load entirely)
      if (has_drop && k + 1 < ke) dnext = dflag[(k + 1) * dstep];
      const int pk = (int)(((int64_t)k * m + boxx) & 1);  // row parity shifts (issue())
      const int pK = (int)(((int64_t)K * p.m_coarse + boxx) & 1);
      const int64_t kofs = (int64_t)k * m;
      // IMV: v_0 of this slice (prefetched one slice ahead) for the dot
      double v0v[RO];
      double vj[RO];  // the staged input at this thread's outputs (pj dots)
#pragma unroll
      for (int r = 0; r < RO; ++r) vj[r] = 0.0;
      if (MODE == kModeIMV && has_part && !v0_self) {
#pragma unroll
        for (int r = 0; r < RO; ++r) v0v[r] = v0next[r];
        const int kn = k + 1;  // prefetch the next slice of this item
        if (kn < ke && xin) {
          const double *v0k = p.v0 + (int64_t)kn * m + gx0;
#pragma unroll
          for (int r = 0; r < RO; ++r) v0next[r] = (y0 + r < ny) ? __ldg(v0k + r * nx) : 0.0;
        }
      }
      mbar_wait(&bars[stage], (it / S) & 1);
      // ---- pre-pass: u = v / scale  or  u = v - Z vt, once per element
      if (((SCALED && !kLazy) || MODE == kModeIMV || kSub) && pin) {
        const double *vtk = (GATHER && !kSub) ? p.vt + (int64_t)K * p.m_coarse : nullptr;
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          if (r < rlo || r > rhi) continue;
          const int y = (DIM == 2) ? y0 - 1 + r : 0;
          double *cell = sv + r * kBox + pe + ((pk + (y & nx)) & 1);
          double u = *cell;
          if (SCALED) u = __dmul_rn(u, vrcp);
          if (MODE == kModeIMV) {
            if (kPj && r >= 1 && r <= R) vj[r - 1] = u;
            const double z = GATHER ? __ldg(vtk + p.group_of[y * nx + px])
                                    : sv[(ROWS + r) * kBox + pe + ((pK + (y & nx)) & 1)];
            u = __dsub_rn(u, z);
          }
          if (kSub)  // w - c v_0, the update pass's per-element rounding
            u = __dsub_rn(u, __dmul_rn(csub, sv[(ROWS + r) * kBox + pe + ((pk + (y & nx)) & 1)]));
          *cell = u;
        }
      }
      if ((SCALED && !kLazy) || MODE == kModeIMV || kSub) __syncthreads();
      // ---- stencil pass, mask-free variant: every neighbour exists, k >= 1,
      // no dropped coupling.  Tile rows start at even y0 (R even) and box row
      // r holds grid row y0 - 1 + r, odd for even r: its parity shift
      // (pk + y nx) & 1 is pk ^ (nx & 1) on even box rows and pk on odd ones.
      if (warp_fast && k > 0 && !drop) {
        const int sh0 = pk ^ (nx & 1), sh1 = pk;  // box rows 0, 2, ... / 1, 3, ...
        const double *col = sv + xo;
        double up = col[sh0];
        double cur = col[kBox + sh1];
        const bool wn = MODE == kModeMVR && has_vn;
        const bool inj = MODE == kModeMVR && mvr_inject;
        // slice-k base pointers at (y0, x); rows at + r nx
        double *ob = (MODE == kModeMVR ? p.v_norm_out : p.out) + kofs + gx0;
        double *hb = (MODE == kModeMVR) ? p.vh + (int64_t)K * m + gx0 : nullptr;
        const bool closes = pos == nu - 1, opens = pos == 0;
        // The row loop is instantiated per combination of the slice-uniform
        // flags that steer its stores (a tag of 2 keeps the runtime test):
        // inside the unrolled loop each test costs a constant-bank reload, a
        // compare and a branch per row -- half of the ~50 instructions per
        // output of the in-solver K-MVR (profiles/r2_ncu_march.md).
        auto rows = [&](auto wn_t, auto inj_t, auto opens_t, auto closes_t, auto wantj_t) {
          constexpr int kWn = decltype(wn_t)::value, kInj = decltype(inj_t)::value;
          constexpr int kOp = decltype(opens_t)::value, kCl = decltype(closes_t)::value;
          constexpr int kWj = decltype(wantj_t)::value;  // K-IMV: 0 none, 1 pj, 3 ||w||^2
          const bool wn_ = kWn == 2 ? wn : kWn == 1;
          const bool inj_ = kInj == 2 ? inj : kInj == 1;
          const bool opens_ = kOp == 2 ? opens : kOp == 1;
          const bool closes_ = kCl == 2 ? closes : kCl == 1;
          const bool wantj_ = kWj == 2 ? wantj : kWj == 1;
          const bool wantw_ = kWj == 2 ? wantw : kWj == 3;
#pragma unroll
        for (int r = 0; r < RO; ++r) {
          const double *row = col + (r + 1) * kBox + (((r + 1) & 1) ? sh1 : sh0);
          const double dn = col[(r + 2) * kBox + (((r + 2) & 1) ? sh1 : sh0)];
          const double lf = (FMA && !hw) ? 0.0 : row[-1];
          const double rt = (FMA && !he) ? 0.0 : row[1];
          Coef5 a, b;
          if (VAR) {
            a = coef_at(p.P, gx0 + r * nx, m);
            b = coef_at(p.Q, gx0 + r * nx, m);
          } else {
            a = pcst;
            b = qcst;
          }
          double Pu, Qu;
          if (FMA) {
            // in-solver passes on isotropic constant stencils (S = W = E = N,
            // checked by the launcher; every pristine level): the neighbour
            // sum is formed once and shared by D^T u and B^T u
#ifndef PMK_NO_ISO
            const double s4 = (up + lf) + (rt + dn);
            Pu = fma(a.w, s4, a.c * cur);
            Qu = fma(b.w, s4, b.c * cur);
#else  // (A/B: two full 5-point stencils, round-1 form)
            Pu = fma(a.n, dn, fma(a.e, rt, fma(a.c, cur, fma(a.w, lf, __dmul_rn(a.s, up)))));
            Qu = fma(b.n, dn, fma(b.e, rt, fma(b.c, cur, fma(b.w, lf, __dmul_rn(b.s, up)))));
#endif
          } else {  // separately rounded: bitwise the reference's sparse product
            Pu = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a.s, up), __dmul_rn(a.w, lf)),
                                               __dmul_rn(a.c, cur)),
                                     __dmul_rn(a.e, rt)),
                           __dmul_rn(a.n, dn));
            Qu = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(b.s, up), __dmul_rn(b.w, lf)),
                                               __dmul_rn(b.c, cur)),
                                     __dmul_rn(b.e, rt)),
                           __dmul_rn(b.n, dn));
          }
          if (!prime && (!FMA || xin)) {
            const double o = __dsub_rn(Pu, qprev[r]);
            const int64_t gi = kofs + gx0 + r * nx;
            if (MODE == kModeMV) {
              p.out[gi] = o;
            } else if (MODE == kModeMVR) {
              if (wn_) ob[r * nx] = kLazy ? __dmul_rn(cur, osc) : cur;
              if (kSub) wsq = fma(cur, cur, wsq);
              const double sval = FMA ? fma(-p.mu, cur, o) : __dsub_rn(o, __dmul_rn(p.mu, cur));
              if (inj_) {
                if (k % nu == 0) {
                  const double sv = kLazy ? __dmul_rn(sval, osc) : sval;
                  p.vh[(int64_t)(k / nu) * m + gx0 + r * nx] = sv;
                  vsq = __dadd_rn(vsq, __dmul_rn(sv, sv));
                }
              } else {
                acc[r] = opens_ ? sval : __dadd_rn(acc[r], sval);
                if (closes_) {
                  const double av = kLazy ? __dmul_rn(acc[r], osc) : acc[r];
                  hb[r * nx] = av;
                  vsq = __dadd_rn(vsq, __dmul_rn(av, av));
                }
              }
            } else {
              if (has_x) p.x_out[gi] = cur;
              if (has_out) ob[r * nx] = o;
              const double v0r = v0_self ? vj[r] : v0v[r];
              if (has_part) dot = FMA ? fma(o, v0r, dot) : __dadd_rn(dot, __dmul_rn(o, v0r));
              if (wantj_) {
                dwj = fma(o, vj[r], dwj);
                dgj = fma(vj[r], v0r, dgj);
              } else if (wantw_) {
                dwj = fma(o, o, dwj);
              }
            }
          }
          qprev[r] = Qu;
          up = cur;
          cur = dn;
        }
        };
        using std::integral_constant;
        constexpr integral_constant<int, 0> c0{};
        constexpr integral_constant<int, 1> c1{};
        constexpr integral_constant<int, 2> rt{};
        if (MODE == kModeMVR && kSolver && kSub) {  // (sub mode always stores v)
          if (inj) rows(c1, c1, rt, rt, c0);
          else if (opens && closes) rows(c1, c0, c1, c1, c0);
          else if (opens) rows(c1, c0, c1, c0, c0);
          else if (closes) rows(c1, c0, c0, c1, c0);
          else rows(c1, c0, c0, c0, c0);
        } else if (MODE == kModeMVR && kSolver) {
          if (IMVK != 1 && (wn || inj)) rows(rt, rt, rt, rt, c0);
          else if (opens && closes) rows(c0, c0, c1, c1, c0);
          else if (opens) rows(c0, c0, c1, c0, c0);
          else if (closes) rows(c0, c0, c0, c1, c0);
          else rows(c0, c0, c0, c0, c0);
        } else {
          // (K-IMV: the same specialisation on its pj / ||w||^2 flags needs 100
          // registers; capped at the 64 its 4 CTAs per SM allow it spills and
          // runs 30% slower -- its loop keeps the runtime tests)
          rows(rt, rt, rt, rt, rt);
        }
      } else if (xin) {
        // ---- generic variant.  Absent neighbours read as 0: adding their
        // (+-0) products to the partial sum leaves it unchanged, so the sum
        // equals the reference's sparse product.
        const double *col = sv + xo;
        double up = (DIM == 2 && rlo == 0) ? col[(pk + ((y0 - 1) & nx)) & 1] : 0.0;
        double cur = col[((DIM == 2) ? kBox : 0) + ((pk + (y0 & nx)) & 1)];
#pragma unroll
        for (int r = 0; r < RO; ++r) {
          const int y = y0 + r;
          const bool rv = DIM == 1 || y < ny;  // row exists (last tile may be partial)
          const double *row = col + ((DIM == 2) ? (r + 1) * kBox : 0) + ((pk + (y & nx)) & 1);
          const double dn = (DIM == 2 && y < ny - 1)
                                ? col[(r + 2) * kBox + ((pk + ((y + 1) & nx)) & 1)]
                                : 0.0;
          const double lf = hw ? row[-1] : 0.0;
          const double rt = he ? row[1] : 0.0;
          Coef5 a, b;
          if (VAR) {
            a = coef_at(p.P, gx0 + r * nx, m);
            b = coef_at(p.Q, gx0 + r * nx, m);
          } else {
            a = pcst;
            b = qcst;
          }
          double Pu = __dmul_rn(a.s, up), Qu = __dmul_rn(b.s, up);
          if (DIM == 1) {  // no S term in 1-D: start from the W product
            Pu = 0.0;
            Qu = 0.0;
          }
          Pu = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(Pu, __dmul_rn(a.w, lf)), __dmul_rn(a.c, cur)),
                                   __dmul_rn(a.e, rt)),
                         __dmul_rn(a.n, dn));
          Qu = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(Qu, __dmul_rn(b.w, lf)), __dmul_rn(b.c, cur)),
                                   __dmul_rn(b.e, rt)),
                         __dmul_rn(b.n, dn));
          if (!prime && rv) {
            double o;
            if (k == 0) {
              o = cur;  // identity block row (stepper.py:100)
            } else {
              o = __dsub_rn(Pu, qprev[r]);
              if (drop) o = __dadd_rn(o, qprev[r]);  // stepper.py:103-104
            }
            const int gi = gx0 + r * nx;
            if (MODE == kModeMV) {
              p.out[kofs + gi] = o;
            } else if (MODE == kModeMVR) {
              if (has_vn) p.v_norm_out[kofs + gi] = kLazy ? __dmul_rn(cur, osc) : cur;
              if (kSub) wsq = fma(cur, cur, wsq);
              const double sval = __dsub_rn(o, __dmul_rn(p.mu, cur));  // s -= mu v
              if (mvr_inject) {  // MgritPair.restrict: rows 0, nu, 2 nu, ...
                if (k % nu == 0) {
                  const double sv = kLazy ? __dmul_rn(sval, osc) : sval;
                  p.vh[(int64_t)(k / nu) * m + gi] = sv;
                  vsq = __dadd_rn(vsq, __dmul_rn(sv, sv));
                }
              } else {
                acc[r] = (pos == 0 || k == 0) ? sval : __dadd_rn(acc[r], sval);
                if (pos == nu - 1) {
                  const double av = kLazy ? __dmul_rn(acc[r], osc) : acc[r];
                  p.vh[(int64_t)K * m + gi] = av;
                  vsq = __dadd_rn(vsq, __dmul_rn(av, av));
                }
              }
            } else {
              if (has_x) p.x_out[kofs + gi] = cur;
              if (has_out) p.out[kofs + gi] = o;
              const double v0r = v0_self ? vj[r] : v0v[r];
              if (has_part) {
                dot = __dadd_rn(dot, __dmul_rn(o, v0r));
              }
              if (wantj) {
                dwj = fma(o, vj[r], dwj);
                dgj = fma(vj[r], v0r, dgj);
              } else if (wantw) {
                dwj = fma(o, o, dwj);
              }
            }
          }
          qprev[r] = Qu;
          up = cur;
          cur = dn;
        }
      }
      __syncthreads();  // stage fully consumed
      if (t == 0 && i + S < nsl) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + S, stage);
      }
    }
  }
  if (MODE == kModeIMV && p.v0_scale && !v0_self) {
    const double v0rcp = __drcp_rn(*p.v0_scale);
    dot = __dmul_rn(dot, v0rcp);
    dgj = __dmul_rn(dgj, v0rcp);
  }
  if (MODE == kModeIMV && has_part) {
    const double s = block_sum(dot);
    if (threadIdx.x == 0) p.partials[blockIdx.x] = s;
  }
  if (wantj || wantw) {
    const double a = block_sum(dwj);
    const double b = block_sum(dgj);
    if (threadIdx.x == 0) {
      p.pj[blockIdx.x] = a;
      p.pj[kMaxPartials + blockIdx.x] = b;
    }
  }
  if (MODE == kModeMVR && p.vh_partials) {
    const double s = block_sum(vsq);
    if (threadIdx.x == 0) p.vh_partials[blockIdx.x] = s;
  }
  if (kSub) {
    const double s = block_sum(wsq);
    if (threadIdx.x == 0) p.vn_partials[blockIdx.x] = s;
  }
}

// 1-D variant.  A 1-D slice is a single grid row, so one box per slice gave
// each stage only ~200 outputs and the kernel was bound by per-stage
// overhead.  Here a tile is up to R column segments of the row (each <= 252
// columns + halo = one box, the segments of a tile are contiguous), a stage
// holds the tile's boxes of one slice, and the 256 threads cover the tile's
// outputs e = t + 256 u (column x0 + e; segment e / W, box offset e % W + 1).
template <int MODE, int R, int S, bool VAR, bool GATHER, bool SCALED>
__global__ void __launch_bounds__(kTmaThreads)
    march_tma_1d_kernel(const MarchParams p, const __grid_constant__ CUtensorMap tm_v,
                        const __grid_constant__ CUtensorMap tm_vt, const TmaGeom g) {
  constexpr int NB = (MODE == kModeIMV && !GATHER) ? 2 : 1;
  constexpr int SL = (R * (kBox - 4) + kTmaThreads - 1) / kTmaThreads;  // outputs / thread
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double *smem = reinterpret_cast<double *>(
      smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t bars[S];

  if (!is_live(p.live)) return;
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int nx = p.nx, m = p.m;  // m == nx
  const int W = g.tile_w;
  const int U = (MODE == kModeMVR) ? p.nu : 1;
  const int n_units = p.n_steps / U + 1;
  const int tiles = g.gx;
  const int64_t n_items = (int64_t)tiles * g.n_chunks;
  // normalisation of a lazily scaled basis vector: multiply by RN(1 / scale)
  // (within 1 ulp of the division; exact_scale launches take the register path)
  const double vrcp = SCALED ? __drcp_rn(*p.v_scale) : 1.0;
  const double v0rcp = (MODE == kModeIMV && p.v0_scale) ? __drcp_rn(*p.v0_scale) : 1.0;
  double dot = 0.0;
  double vsq = 0.0;  // K-MVR: partial ||vh||^2 of the values this thread stores
  uint32_t it = 0;

  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int tile = (int)(item % tiles);
    const int chunk = (int)(item / tiles);
    const int s0 = tile * R;
    const int cnt = min(R, g.nseg - s0);  // segments (boxes) of this tile
    const int x0 = s0 * W;                // first output column
    const int cntW = min(cnt * W, nx - x0);
    const int U0 = chunk * g.upc;
    const int U1 = min(n_units, U0 + g.upc);
    const int kb = (U0 == 0) ? 0 : U * (U0 - 1) + 1;
    const int ke = U * (U1 - 1) + 1;
    const int kstart = (kb > 0) ? kb - 1 : 0;
    const int nsl = ke - kstart;
    const int boxx = g.single ? 0 : x0 - 1;  // grid column of box 0's element 0
    const int bo = g.single ? 0 : 1;         // box offset of a segment's first output
    const uint32_t tx_bytes = (uint32_t)(NB * cnt * kBox * sizeof(double));

    auto issue = [&](int k, int stage) {
      double *sv = smem + (size_t)stage * NB * R * kBox;
      const int K = (k == 0) ? 0 : (k - 1) / p.nu + 1;
      if (g.bulk) {
        uint32_t bytes = 0;
        for (int r = 0; r < cnt; ++r) {
          bytes += bulk_bytes(((int64_t)k * m + boxx + r * W) & ~(int64_t)1, g.n_v);
          if (NB == 2)
            bytes += bulk_bytes(((int64_t)K * p.m_coarse + boxx + r * W) & ~(int64_t)1, g.n_vt);
        }
        mbar_expect_tx(&bars[stage], bytes);
        for (int r = 0; r < cnt; ++r) {
          bulk_row(sv + r * kBox, p.v, ((int64_t)k * m + boxx + r * W) & ~(int64_t)1, g.n_v,
                   &bars[stage]);
          if (NB == 2)
            bulk_row(sv + (R + r) * kBox, p.vt,
                     ((int64_t)K * p.m_coarse + boxx + r * W) & ~(int64_t)1, g.n_vt, &bars[stage]);
        }
        return;
      }
      mbar_expect_tx(&bars[stage], tx_bytes);
      for (int r = 0; r < cnt; ++r) {
        const int c = (int)((int64_t)k * m + boxx + r * W);
        tma_row(sv + r * kBox, &tm_v, c & ~1, &bars[stage]);
        if (NB == 2) {
          const int cv = (int)((int64_t)K * p.m_coarse + boxx + r * W);
          tma_row(sv + (R + r) * kBox, &tm_vt, cv & ~1, &bars[stage]);
        }
      }
    };
    if (t == 0) {
      const int pre = nsl < S ? nsl : S;
      for (int q = 0; q < pre; ++q) issue(kstart + q, (int)((it + q) % S));
    }

    // this thread's outputs: e = t + 256 u
    int xs[SL], br[SL], bx[SL];
    bool ok[SL];
#pragma unroll
    for (int u = 0; u < SL; ++u) {
      const int e = t + u * kTmaThreads;
      ok[u] = e < cntW;
      xs[u] = x0 + e;
      br[u] = ok[u] ? e / W : 0;
      bx[u] = ok[u] ? e - br[u] * W + bo : 0;
    }
    double qprev[SL], acc[SL], v0next[SL];
#pragma unroll
    for (int u = 0; u < SL; ++u) qprev[u] = acc[u] = v0next[u] = 0.0;
    Coef5 pcst, qcst;
    if (!VAR) {
      pcst = Coef5{p.P.c[0], p.P.c[1], p.P.c[2], p.P.c[3], p.P.c[4]};
      qcst = Coef5{p.Q.c[0], p.Q.c[1], p.Q.c[2], p.Q.c[3], p.Q.c[4]};
    }
    const int nu = p.nu;
    if (MODE == kModeIMV && p.partials) {
      const int kf = (kb > kstart) ? kb : kstart;
#pragma unroll
      for (int u = 0; u < SL; ++u)
        v0next[u] = (ok[u] && kf < ke) ? __ldg(p.v0 + (int64_t)kf * m + xs[u]) : 0.0;
    }
    int Kc = (kstart == 0) ? 0 : (kstart - 1) / nu + 1;
    int posc = (kstart == 0) ? nu - 1 : (kstart - 1) - (Kc - 1) * nu;
    const uint8_t *dflag = p.dropped ? p.dropped : &g_no_drop;
    const int dstep = p.dropped ? 1 : 0;
    int dnext = (kstart < ke) ? dflag[kstart * dstep] : 0;
    for (int i = 0; i < nsl; ++i, ++it) {
      const int k = kstart + i;
      const bool prime = k < kb;
      const int stage = (int)(it % S);
      double *sv = smem + (size_t)stage * NB * R * kBox;
      // coarse slice K of k and position in its slab (stepped, no division)
      const int K = Kc, pos = posc;
      if (k == 0) {
        Kc = 1;
        posc = 0;
      } else if (++posc == nu) {
        ++Kc;
        posc = 0;
      }
      // dropped coupling of k: loaded one slice ahead, off the critical path
      const bool drop = dnext != 0;
      if (k + 1 < ke) dnext = dflag[(k + 1) * dstep];
      const int pk = (int)(((int64_t)k * m + boxx) & 1);  // parity of box 0
      const int pK = (int)(((int64_t)K * p.m_coarse + boxx) & 1);
      const int64_t kofs = (int64_t)k * m;
      double v0v[SL];
      if (MODE == kModeIMV && p.partials) {
#pragma unroll
        for (int u = 0; u < SL; ++u) v0v[u] = v0next[u];
        const int kn = k + 1;
        if (kn < ke) {
#pragma unroll
          for (int u = 0; u < SL; ++u)
            if (ok[u]) v0next[u] = __ldg(p.v0 + (int64_t)kn * m + xs[u]);
        }
      }
      mbar_wait(&bars[stage], (it / S) & 1);
      // ---- pre-pass over the boxes' elements (v / scale or v - Z vt)
      if (SCALED || MODE == kModeIMV) {
        for (int r = 0; r < cnt; ++r) {
          const int px = boxx + r * W + t;
          if (t < kBox - 1 && px >= 0 && px < nx) {
            double *cell = sv + r * kBox + t + ((pk + (r * W)) & 1);
            double u = *cell;
            if (SCALED) u = __dmul_rn(u, vrcp);
            if (MODE == kModeIMV) {
              const double z = GATHER
                                    ? __ldg(p.vt + (int64_t)K * p.m_coarse + p.group_of[px])
                                    : sv[(R + r) * kBox + t + ((pK + (r * W)) & 1)];
              u = __dsub_rn(u, z);
            }
            *cell = u;
          }
        }
        __syncthreads();
      }
      // ---- stencil (W, C, E in ascending column order; no S/N in 1-D)
#pragma unroll
      for (int u = 0; u < SL; ++u) {
        if (!ok[u]) continue;
        const int x = xs[u];
        const double *row = sv + br[u] * kBox + ((pk + (br[u] * W)) & 1) + bx[u];
        const double cur = row[0];
        const double lf = (x > 0) ? row[-1] : 0.0;
        const double rt = (x < nx - 1) ? row[1] : 0.0;
        Coef5 a, b;
        if (VAR) {
          a = coef_at(p.P, x, m);
          b = coef_at(p.Q, x, m);
        } else {
          a = pcst;
          b = qcst;
        }
        const double Pu = __dadd_rn(
            __dadd_rn(__dadd_rn(0.0, __dmul_rn(a.w, lf)), __dmul_rn(a.c, cur)), __dmul_rn(a.e, rt));
        const double Qu = __dadd_rn(
            __dadd_rn(__dadd_rn(0.0, __dmul_rn(b.w, lf)), __dmul_rn(b.c, cur)), __dmul_rn(b.e, rt));
        if (!prime) {
          double o;
          if (k == 0) {
            o = cur;  // identity block row (stepper.py:100)
          } else {
            o = __dsub_rn(Pu, qprev[u]);
            if (drop) o = __dadd_rn(o, qprev[u]);  // stepper.py:103-104
          }
          if (MODE == kModeMV) {
            p.out[kofs + x] = o;
          } else if (MODE == kModeMVR) {
            if (p.v_norm_out) p.v_norm_out[kofs + x] = cur;
            const double sval = __dsub_rn(o, __dmul_rn(p.mu, cur));
            if (p.inject) {
              if (k % nu == 0) {
                p.vh[(int64_t)(k / nu) * m + x] = sval;
                vsq = __dadd_rn(vsq, __dmul_rn(sval, sval));
              }
            } else {
              acc[u] = (pos == 0 || k == 0) ? sval : __dadd_rn(acc[u], sval);
              if (pos == nu - 1) {
                p.vh[(int64_t)K * m + x] = acc[u];
                vsq = __dadd_rn(vsq, __dmul_rn(acc[u], acc[u]));
              }
            }
          } else {
            if (p.x_out) p.x_out[kofs + x] = cur;
            if (p.out) p.out[kofs + x] = o;
            if (p.partials) dot = __dadd_rn(dot, __dmul_rn(o, __dmul_rn(v0v[u], v0rcp)));
          }
        }
        qprev[u] = Qu;
      }
      __syncthreads();  // stage fully consumed
      if (t == 0 && i + S < nsl) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + S, stage);
      }
    }
  }
  if (MODE == kModeIMV && p.partials) {
    const double s = block_sum(dot);
    if (threadIdx.x == 0) p.partials[blockIdx.x] = s;
  }
  if (MODE == kModeMVR && p.vh_partials) {
    const double s = block_sum(vsq);
    if (threadIdx.x == 0) p.vh_partials[blockIdx.x] = s;
  }
}

// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  return fn;
}

bool encode_1d(CUtensorMap *map, const double *base, int64_t n) {
  EncodeTiledFn fn = encoder();
  if (!fn || !base || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  cuuint64_t dims[1] = {(cuuint64_t)n};
  cuuint64_t strides[1] = {0};
  cuuint32_t box[1] = {kBox};
  cuuint32_t estr[1] = {1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, const_cast<double *>(base), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODE, int DIM, int R, int S, bool VAR, bool GATHER, bool SCALED, bool FMA = false,
          int IMVK = 0>
int run_tma(const MarchParams &p, const CUtensorMap &mv, const CUtensorMap &mvt, cudaStream_t s,
            int *n_partials, double bytes, int cat, bool bulk) {
  constexpr int NB = ((MODE == kModeIMV && !GATHER) || (MODE == kModeMVR && GATHER)) ? 2 : 1;
  constexpr int ROWS = (DIM == 2) ? R + 2 : R;
  const size_t smem = (size_t)S * NB * ROWS * kBox * sizeof(double) + 128;
  auto kern = (DIM == 2) ? march_tma_kernel<MODE, DIM, R, S, VAR, GATHER, SCALED, FMA, IMVK>
                         : march_tma_1d_kernel<MODE, R, S, VAR, GATHER, SCALED>;
  static int occ = -1;
  if (occ < 0) {
    PMK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int b = 0;
    PMK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kTmaThreads, smem));
    occ = b > 0 ? b : 1;
  }
  TmaGeom g;
  g.bulk = bulk ? 1 : 0;
  g.n_v = (int64_t)(p.n_steps + 1) * p.m;
  g.n_vt = (MODE == kModeIMV && !GATHER) ? (int64_t)(p.n_steps / p.nu + 1) * p.m_coarse : g.n_v;
  g.single = p.nx <= kBox - 1 ? 1 : 0;  // row + parity shift fits one box
  if (g.single) {
    g.tile_w = p.nx;
  } else {  // halo + shift fit one box (<= 252); balance the tiles of a row
    const int nt = (p.nx + (kBox - 4) - 1) / (kBox - 4);
    g.tile_w = (p.nx + nt - 1) / nt;
  }
  g.nseg = (p.nx + g.tile_w - 1) / g.tile_w;
  g.gx = (DIM == 2) ? g.nseg : (g.nseg + R - 1) / R;  // 1-D: R segments per tile
  g.gy = (DIM == 2) ? (p.ny + R - 1) / R : 1;
  const int U = (MODE == kModeMVR) ? p.nu : 1;
  const int n_units = p.n_steps / U + 1;
  const int tiles = g.gx * g.gy;
  int grid_cap = occ * kSMs;
  if (MODE != kModeMV && grid_cap > kMaxPartials) grid_cap = kMaxPartials;  // partials
  // ~8 work items per resident CTA; chunks of at most 32 units (one extra
  // prime slice per chunk, served from L2).
  static const int ipc = [] {  // work items per resident CTA (tuning knob PMK_IPC)
    const char *e = getenv("PMK_IPC");
    const int v = e ? atoi(e) : 8;
    return v > 0 ? v : 8;
  }();
  int64_t upc = ((int64_t)n_units * tiles) / ((int64_t)ipc * grid_cap);
  if (upc < 2) upc = 2;
  if (upc > 32) upc = 32;
  g.upc = (int)upc;
  g.n_chunks = (int)((n_units + upc - 1) / upc);
  const int64_t n_items = (int64_t)tiles * g.n_chunks;
  const int grid = (int)(n_items < grid_cap ? n_items : grid_cap);
  static const bool dbg = getenv("PMK_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr, "[pmk] tma mode %d dim %d R %d S %d var %d gather %d: nx %d ny %d steps %d "
            "grid %d smem %zu occ %d single %d tile_w %d gx %d gy %d upc %d chunks %d bulk %d\n",
            MODE, DIM, R, S, (int)VAR, (int)GATHER, p.nx, p.ny, p.n_steps, grid, smem, occ,
            g.single, g.tile_w, g.gx, g.gy, g.upc, g.n_chunks, g.bulk);
  prof::Scope scope(cat, bytes, 0.0, s);
  kern<<<grid, kTmaThreads, smem, s>>>(p, mv, mvt, g);
  PMK_LAUNCH_CHECK();
  if (MODE == kModeIMV && DIM == 2 && FMA && !VAR && !GATHER && p.pj && p.pj_done)
    *p.pj_done = 1;
  if (n_partials) *n_partials = grid;
  return 0;
}

}  // namespace

// Returns 1 when the TMA path handled the launch, 0 when the caller should
// use the register path (no driver entry point, unaligned base, N >= 2^31).
int launch_march_tma(int mode, const MarchParams &p_in, cudaStream_t s, int *n_partials,
                     double bytes, int cat, int *handled) {
  *handled = 0;
  MarchParams p = p_in;
  // the in-solver (FMA) instantiations assume isotropic constant stencils
  // (S = W = E = N: every pristine level); others take the exact kernels
  const bool iso = iso_stencil(p.P) && iso_stencil(p.Q);
  if (p.fma && !(p.P.var || p.Q.var) && !iso) {
    if (p.v_sub) return PMK_ERR_ARG;  // (fgmres_fixed only fuses isotropic levels)
    p.fma = 0;
  }
  const int64_t N = (int64_t)(p.n_steps + 1) * p.m;
  const bool gather = (mode == kModeIMV) && p.group_of != nullptr;
  // 1-D tensor-map coordinates are int32: longer vectors (and PMK_TMA_BULK=1,
  // for tests) take plain bulk copies with 64-bit addresses instead
  static const bool force_bulk = [] {
    const char *e = getenv("PMK_TMA_BULK");
    return e && e[0] == '1';
  }();
  const bool bulk = force_bulk || N + 2 * kBox >= (int64_t)1 << 31;
  auto al16 = [](const void *q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  CUtensorMap mv, mvt;
  std::memset(&mv, 0, sizeof(mv));
  std::memset(&mvt, 0, sizeof(mvt));
  if (bulk) {
    if (!al16(p.v) || (mode == kModeIMV && !gather && !al16(p.vt)) ||
        (mode == kModeMVR && p.v_sub && !al16(p.v_sub)))
      return 0;
  } else {
    if (!encode_1d(&mv, p.v, N)) return 0;
    if (mode == kModeIMV && !gather) {
      const int64_t Nc = (int64_t)(p.n_steps / p.nu + 1) * p.m_coarse;
      if (!encode_1d(&mvt, p.vt, Nc)) return 0;
    } else if (mode == kModeMVR && p.v_sub) {
      if (!encode_1d(&mvt, p.v_sub, N)) return 0;
    } else {
      mvt = mv;
    }
  }
  if (p.v_scale && p.exact_scale) return 0;       // correctly rounded division
  const bool var = p.P.var || p.Q.var;

  const bool d2 = p.ny > 1;
  const bool wide1d = !d2 && p.nx > kBox - 1;  // 1-D rows of several segments
  const bool scaled = p.v_scale != nullptr;
  int rc = 0;
#define PMK_RUN(MODE, DIM, R, S, GATHER)                                                        \
  do {                                                                                         \
    if (var) {                                                                                 \
      rc = scaled ? run_tma<MODE, DIM, R, S, true, GATHER, true>(p, mv, mvt, s, n_partials,     \
                                                                 bytes, cat, bulk)                   \
                  : run_tma<MODE, DIM, R, S, true, GATHER, false>(p, mv, mvt, s, n_partials,    \
                                                                  bytes, cat, bulk);                 \
    } else {                                                                                   \
      rc = scaled ? run_tma<MODE, DIM, R, S, false, GATHER, true>(p, mv, mvt, s, n_partials,    \
                                                                  bytes, cat, bulk)                  \
                  : run_tma<MODE, DIM, R, S, false, GATHER, false>(p, mv, mvt, s, n_partials,   \
                                                                   bytes, cat, bulk);                \
    }                                                                                          \
  } while (0)
  // tile rows x ring stages per mode (tuning knob PMK_TMA_CFG=<mvr>,<imv>;
  // mvr 0: 4x3, 1: 4x4, 2: 8x3, 3: 16x2; imv 0: 4x2, 1: 4x3, 2: 8x2, 3: 2x4).
  // Defaults from an ncu sweep of the c5_c fine level (profiles/r1_march_sweep.md):
  // 4-row tiles keep more CTAs resident, which hides the FP64 dependency
  // chains better than taller tiles amortise the per-slice overhead.
  static int cfg_mvr = -1, cfg_imv = -1;
  if (cfg_mvr < 0) {
    cfg_mvr = 0;
    cfg_imv = 0;
    if (const char *e = getenv("PMK_TMA_CFG")) sscanf(e, "%d,%d", &cfg_mvr, &cfg_imv);
  }
  // Plain matvec tile (tuning knob PMK_MV_CFG; 1: 8x3, 2: 16x2, default by
  // size).  16-row tiles x 2 stages (92 registers, 2 CTAs/SM) load 18 rows per
  // 16 outputs instead of 10 per 8: 5.89 vs 5.51 TB/s on the 2.13 GB c5_c
  // vector (16x3: 5.63, 16x4: 4.88, 24x2: 4.35, 4x3: 5.43, 4x4: 5.31, 8x2:
  // 5.47; tools/mv_probe.py); launches of a few tens of microseconds prefer
  // the smaller tile's larger grid (63^2 x 513: 25.0 vs 28.9 us).
  static const int cfg_mv = [] {
    const char *e = getenv("PMK_MV_CFG");
    return e ? atoi(e) : 0;
  }();
  switch (mode) {
    case kModeMV:
      if (d2) {
        const bool tall = cfg_mv ? cfg_mv == 2 : (p.ny >= 64 && N >= ((int64_t)1 << 25));
        if (tall)
          PMK_RUN(kModeMV, 2, 16, 2, false);
        else
          PMK_RUN(kModeMV, 2, 8, 3, false);
      } else if (wide1d) PMK_RUN(kModeMV, 1, 8, 3, false);
      else PMK_RUN(kModeMV, 1, 1, 8, false);
      break;
    case kModeMVR:
      if (p.v_sub) {  // sub mode: 2-D, constant stencils, in-solver, unscaled only
        if (!(d2 && p.fma && !var && !scaled && !p.dropped && p.v_norm_out && p.vn_partials &&
              p.v_sub_coef))
          return PMK_ERR_ARG;
        static const bool tall = [] {  // PMK_SUB_TALL=1: 8-row tiles (2 CTAs/SM)
          const char *e = getenv("PMK_SUB_TALL");
          return e && e[0] == '1';
        }();
        if (tall)
          rc = run_tma<kModeMVR, 2, 8, 2, false, true, false, true>(p, mv, mvt, s, n_partials,
                                                                     bytes, cat, bulk);
        else if (!p.inject)
          rc = run_tma<kModeMVR, 2, 4, 2, false, true, false, true, 1>(p, mv, mvt, s, n_partials,
                                                                        bytes, cat, bulk);
        else
          rc = run_tma<kModeMVR, 2, 4, 2, false, true, false, true>(p, mv, mvt, s, n_partials,
                                                                     bytes, cat, bulk);
        break;
      }
      if (d2) {
        if (p.fma && !var && scaled && !p.dropped && (cfg_mvr == 0 || cfg_mvr >= 4)) {
          // in-solver K-MVR (no pre-pass since the lazy basis, so taller tiles'
          // per-slice savings win over occupancy up to a point): 6-row tiles x
          // 3 stages, 72 registers, 3 CTAs/SM.  Same-box bench A/B, ms of the
          // K-MVR launches of 4 c5_c solves: 6x3 242, 8x3 249 (round 1's pick,
          // -3% vs 4x3), 8x4 284, 10x3 / 12x2 ~400 (ptxas goes to > 200
          // registers), 16x2 397.  PMK_TMA_CFG=4/5/6/7,x: 8x2, 8x3, 4x4, 4x3.
          if (cfg_mvr == 4)
            rc = run_tma<kModeMVR, 2, 8, 2, false, false, true, true>(p, mv, mvt, s, n_partials,
                                                                       bytes, cat, bulk);
          else if (cfg_mvr == 5)
            rc = run_tma<kModeMVR, 2, 8, 3, false, false, true, true>(p, mv, mvt, s, n_partials,
                                                                       bytes, cat, bulk);
          else if (cfg_mvr == 6)
            rc = run_tma<kModeMVR, 2, 4, 4, false, false, true, true>(p, mv, mvt, s, n_partials,
                                                                       bytes, cat, bulk);
          else if (cfg_mvr == 7)
            rc = run_tma<kModeMVR, 2, 4, 3, false, false, true, true>(p, mv, mvt, s, n_partials,
                                                                       bytes, cat, bulk);
          else if (!p.v_norm_out && !p.inject)  // the common contract, fixed at compile time
            rc = run_tma<kModeMVR, 2, 6, 3, false, false, true, true, 1>(p, mv, mvt, s,
                                                                          n_partials, bytes, cat,
                                                                          bulk);
          else
            rc = run_tma<kModeMVR, 2, 6, 3, false, false, true, true>(p, mv, mvt, s, n_partials,
                                                                       bytes, cat, bulk);
          break;
        }
        switch (cfg_mvr) {
          case 1: PMK_RUN(kModeMVR, 2, 4, 4, false); break;
          case 2: PMK_RUN(kModeMVR, 2, 8, 3, false); break;
          case 3: PMK_RUN(kModeMVR, 2, 16, 2, false); break;
          default: PMK_RUN(kModeMVR, 2, 4, 3, false);
        }
      } else if (wide1d) {
        PMK_RUN(kModeMVR, 1, 8, 3, false);
      } else {
        PMK_RUN(kModeMVR, 1, 1, 8, false);
      }
      break;
    case kModeIMV:
      if (d2) {
        if (gather) {
          PMK_RUN(kModeIMV, 2, 4, 3, true);
        } else if (p.fma && !var && cfg_imv == 0 && p.out && !p.x_out && p.partials && p.v0 &&
                   !p.dropped) {
          // in-solver K-IMV, one instantiation per dot-product contract (IMVK)
          const bool self = p.v0 == p.v;
          int kk = self ? ((p.pj && p.pj_wsq) ? 2 : 1) : ((p.pj && !p.pj_wsq) ? 3 : 4);
          // (combinations the solver never asks for keep the runtime flags)
          if ((self && p.pj && !p.pj_wsq) || (!self && p.pj && p.pj_wsq)) kk = 0;
#define PMK_RUN_IMVK(K)                                                                          \
  case K:                                                                                        \
    rc = scaled ? run_tma<kModeIMV, 2, 4, 2, false, false, true, true, K>(p, mv, mvt, s,         \
                                                                          n_partials, bytes, cat, \
                                                                          bulk)                  \
                : run_tma<kModeIMV, 2, 4, 2, false, false, false, true, K>(p, mv, mvt, s,        \
                                                                           n_partials, bytes,    \
                                                                           cat, bulk);           \
    break;
          switch (kk) {
            PMK_RUN_IMVK(1)
            PMK_RUN_IMVK(2)
            PMK_RUN_IMVK(3)
            PMK_RUN_IMVK(4)
            default:
              PMK_RUN_IMVK(0)
          }
#undef PMK_RUN_IMVK
        } else {
          switch (cfg_imv) {
            case 1: PMK_RUN(kModeIMV, 2, 4, 3, false); break;
            case 2: PMK_RUN(kModeIMV, 2, 8, 2, false); break;
            case 3: PMK_RUN(kModeIMV, 2, 2, 4, false); break;
            default: PMK_RUN(kModeIMV, 2, 4, 2, false);
          }
        }
      } else if (wide1d) {
        if (gather) PMK_RUN(kModeIMV, 1, 8, 3, true); else PMK_RUN(kModeIMV, 1, 8, 3, false);
      } else {
        if (gather) PMK_RUN(kModeIMV, 1, 1, 8, true); else PMK_RUN(kModeIMV, 1, 1, 8, false);
      }
      break;
    default:
      return PMK_ERR_ARG;
  }
#undef PMK_RUN
  if (rc == 0) *handled = 1;
  return rc;
}

}  // namespace pmk
