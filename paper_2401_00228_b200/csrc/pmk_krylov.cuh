// pmk_krylov.cuh -- device-resident FGMRES state and launchers.
#pragma once

#include "pmk_internal.cuh"

namespace pmk {

// Device-resident state of one fgmres invocation (solver.py:389-396).
// The header lives in device memory so that every kernel of the iteration
// (including the ones captured in CUDA graphs) reads and updates it without
// host involvement.
struct KState {
  double *h;     // (cap+1) x cap, row-major, ld = cap; rotated in place
  double *hraw;  // unrotated copy (keep_basis, tests)
  double *cs, *sn, *g, *y;
  double *vscale;  // vscale[l]: divisor of raw basis vector l (beta, h[l][l-1])
  // Lazy basis (lazy = 1): basis vector l is stored raw (the rhs, or w of
  // iteration l-1 after its orthogonalisation) and used as RN(raw * vrcp[l]),
  // vrcp[l] = RN(1 / vscale[l]) -- the exact values an explicit normalisation
  // pass would have stored.  lazy = 0: stored normalised, vrcp[l] = 1.
  double *vrcp;
  double *hv;  // current column's update coefficients h_i * vrcp_i (ICWY)
  int lazy;
  unsigned int ticket;  // blocks done in a pass that ends with a fused finish
  // Gram row of the next basis vector, accumulated by the update pass that
  // produces it: partials of <w', raw_i> at ugp[i * kMaxPartials + block]
  double *ugp;
  double *hist;    // residual history rel_j
  double *gram;    // cap x cap, row i = <v_i, v_l>, l < i (ICWY MGS)
  double beta, rel;
  int live;      // iterating (cleared on breakdown / convergence / beta == 0)
  int entered;   // parent was live when this invocation began
  int n_iter;
  int breakdown;
};

constexpr int kAsmChunk = 32;
struct AssembleArgs {
  int count;
  const double *v[kAsmChunk];  // normalised basis vectors
  const double *vt[kAsmChunk];
};

constexpr int kGroup = 16;     // basis vectors per ICWY update pass
#ifndef PMK_DOT_GROUP
#define PMK_DOT_GROUP 8
#endif
constexpr int kDotGroup = PMK_DOT_GROUP;  // basis vectors per ICWY dot pass (ptxas serialises
                               // the loads of larger groups: ~3 TB/s at 12)
struct MultiVec {
  const double *v[kGroup];
};
// dot partial buffer: ceil(cap / kDotGroup) * (2 kDotGroup + 1) * kMaxPartials doubles
// With fuse_finish (and aligned operands) the last block of the last update
// pass also runs finish_col (h[j+1][j], Givens, stop test); *finished tells
// the caller whether it still has to launch it.
// ugram_in: the Gram row of v_j was produced by the previous update pass
// (the dot passes then read w and v_1..v_{j-1} only, 16 vectors per pass);
// ugram_out: this column's single update pass produces the Gram row of the
// next basis vector.  *ugram_done reports whether it did.
int launch_icwy_mgs(KState *st, int ld, int j, double *w, const double *const *v, int64_t n,
                    const double *c0p, int n_c0, const double *pj, double *dot_partials,
                    double *norm_partials, int *n_norm, bool keep_w, cudaStream_t s,
                    double tol = 0.0, bool fuse_finish = false, bool *finished = nullptr,
                    bool ugram_in = false, bool ugram_out = false, bool *ugram_done = nullptr);

int launch_begin(KState *st, const double *partials, int n_partials, const int *parent_live,
                 cudaStream_t s);
int launch_mgs_pass(KState *st, int ld, int l, int j, double *w, const double *vl,
                    const double *vl_scale, const double *vn, const double *vn_scale, int64_t n,
                    const double *prev, int n_prev, double *partials, cudaStream_t s);
// pyth: column 0 from ||w||^2 partials (see finish_col_block)
int launch_finish_col(KState *st, int ld, int j, const double *partials, int n_partials,
                      double tol, cudaStream_t s, bool pyth = false);
int launch_backsolve(KState *st, int ld, cudaStream_t s, const double *out_scale = nullptr);
// column 0's ICWY solve alone (h_00 = <w, v_0>, hv[0]): the deferred update of
// fgmres_fixed's fused first step
int launch_icwy_solve(KState *st, int ld, int j, const double *c0p, int n_c0, cudaStream_t s);
int launch_assemble(const KState *st, const AssembleArgs &a, double *x, int64_t n, int m, int nu,
                    int m_coarse, const int32_t *group_of, int first, cudaStream_t s);

}  // namespace pmk
