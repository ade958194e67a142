// pmk_api.cu -- extern "C" entry points (include/pintmk_b200.h) and the
// native FGMRES / MLK recursion.
//
// The recursion mirrors reference solver.py:323-456 step for step:
//
//   fgmres(level, rhs, tol, max_iter)          solver.py:362-456
//     beta = ||rhs||                            (begin_kernel)
//     for j:
//       x_j = apply_preconditioner(v_j)        solver.py:323-359
//          vh = Y^T (A v_j - mu v_j)           K-MVR (one pass; also stores
//                                              v_j = raw_j / h[j][j-1] or rhs / beta)
//          vt = coarsest forward_solve(vh)     or fgmres(level+1, vh, None, budget)
//          x_j = v_j - Z vt                    fused into K-IMV below
//       w = A x_j                              K-IMV (+ partial <w, v_0>)
//       MGS                                    j+1 fused passes
//       h[j+1,j], breakdown, Givens, rel       finish_col_kernel (device)
//     y = R^{-1} g ; x = sum y_i x_i           backsolve + assemble (x_i recomputed)
//
// Nothing in an inner solve synchronises with the host: the breakdown /
// beta == 0 exits of the reference are device flags that turn the remaining
// launches of that invocation into no-ops.
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <unordered_map>
#include <set>
#include <tuple>
#include <unordered_set>
#include <vector>

#include "pmk_internal.cuh"
#include "pmk_krylov.cuh"

using namespace pmk;

// ------------------------------------------------------------- accounting
namespace {
struct ProfRec {
  int cat, level, hint;
  double bytes, flops;
  cudaEvent_t a, b;
};
thread_local int t_level = -1;  // level being issued (-1: stand-alone call)
thread_local int t_hint = -1;
std::atomic<int64_t> g_launches{0};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_recs;
std::vector<cudaEvent_t> g_pool;
size_t g_pool_used = 0;
const char *kCatNames[prof::kNumCat] = {"march_mv", "march_mvr", "march_imv", "mgs_pass",
                                         "reduce",   "fgmres_small", "assemble", "coarse_gemm",
                                         "coarse_recurrence", "coarse_misc", "transfer",
                                         "coarse_dst", "coarse_chain"};

cudaEvent_t pool_event() {
  if (g_pool_used == g_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    g_pool.push_back(e);
  }
  return g_pool[g_pool_used++];
}
}  // namespace

namespace pmk {
namespace prof {
Scope::Scope(int cat, double bytes, double flops, cudaStream_t s) : rec(-1), stream(s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  ProfRec r{cat, t_level, t_hint, bytes, flops, pool_event(), pool_event()};
  if (!r.a || !r.b) return;
  cudaEventRecord(r.a, s);
  rec = (int)g_recs.size();
  g_recs.push_back(r);
}
Scope::~Scope() {
  if (rec < 0) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  cudaEventRecord(g_recs[rec].b, stream);
}
Tag::Tag(int level, int hint) : prev_level(t_level), prev_hint(t_hint) {
  t_level = level;
  t_hint = hint;
}
Tag::~Tag() {
  t_level = prev_level;
  t_hint = prev_hint;
}
}  // namespace prof
}  // namespace pmk

namespace {

using GraphKey = std::tuple<const double *, const int *, const double *>;

struct LevelRT {
  bool set = false;
  pmk_level L{};
  pmk_pair P{};
  int budget = 0;
  int64_t N = 0;
  // registered buffers (inner levels / coarsest rhs)
  double *rhs = nullptr;
  std::vector<double *> v_slots, child_out;
  double *w_buf = nullptr;
  double *ts_scratch = nullptr;
  // device state
  KState *d_state = nullptr;  // header in device memory
  KState h_state{};           // host copy of the pointers
  void *d_block = nullptr;
  int cap = 0;
  double *partA = nullptr, *partB = nullptr;
  double *partM = nullptr;  // ICWY dot partials
  // ||rhs||^2 partials left by the parent's K-MVR for the next begin (inner
  // levels; rhs_part_n = 0: none, begin computes the norm itself)
  double *rhs_part = nullptr;
  int rhs_part_n = 0;
  double tol = 0.0;
  // CUDA graphs of this level's inner solve, keyed by everything the capture
  // bakes in that varies between calls: the output buffer, the parent's live
  // flag and the output scale (the registered buffers and level states are
  // fixed until drop_graphs)
  std::set<GraphKey> seen;
  std::map<GraphKey, std::pair<cudaGraphExec_t, int64_t>> graphs;
  bool graph_failed = false;
  // current invocation
  const double *rhs_cur = nullptr;   // rhs of this invocation (raw basis vector 0)
  const double *pending = nullptr;   // unnormalised basis vector j (w of iteration j-1)
  std::vector<const double *> v;     // normalised basis vectors, index l
  std::vector<const double *> vt;    // child outputs, iteration j
  const int *parent_live = nullptr;
  // pinned ring of KState snapshots (pmk_fgmres_snapshot / _read)
  KState *snap = nullptr;
  int ugram_col = -1;  // column whose Gram row the last update pass produced
};

}  // namespace

struct pmk_hier {
  int n_levels = 0;
  double mu = 1.0;
  std::vector<LevelRT> lv;
  pmk_coarse coarse{};
  bool has_coarse = false;
  double *coarse_rhs = nullptr;
};

namespace {

// Every captured graph holds device pointers of the levels below it (states,
// registered buffers, the coarsest tables): any change to those invalidates
// all of them.
void drop_graphs(pmk_hier *H) {
  for (auto &R : H->lv) {
    for (auto &kv : R.graphs) cudaGraphExecDestroy(kv.second.first);
    R.graphs.clear();
    R.seen.clear();
    R.graph_failed = false;
  }
}

inline cudaStream_t cs(pmk_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

int64_t level_N(const pmk_level &L) {
  const int64_t m = (int64_t)L.nx * (L.dim == 2 ? L.ny : 1);
  return (int64_t)(L.n_steps + 1) * m;
}

int check_level(const pmk_level *L) {
  PMK_RETURN_IF(!L, PMK_ERR_ARG);
  PMK_RETURN_IF(L->dim != 1 && L->dim != 2, PMK_ERR_ARG);
  PMK_RETURN_IF(L->nx < 1 || L->ny < 1 || L->n_steps < 0, PMK_ERR_SHAPE);
  PMK_RETURN_IF(L->dim == 1 && L->ny != 1, PMK_ERR_SHAPE);
  PMK_RETURN_IF(L->diag_t.var && !L->diag_t.coef, PMK_ERR_ARG);
  PMK_RETURN_IF(L->sub_t.var && !L->sub_t.coef, PMK_ERR_ARG);
  return 0;
}

int check_pair(const pmk_level &L, const pmk_pair *P) {
  PMK_RETURN_IF(!P, PMK_ERR_ARG);
  PMK_RETURN_IF(P->nu < 1 || P->n_T < 0, PMK_ERR_ARG);
  PMK_RETURN_IF(P->nu * P->n_T != L.n_steps, PMK_ERR_SHAPE);
  PMK_RETURN_IF(P->m_fine != L.nx * L.ny, PMK_ERR_SHAPE);
  if (P->mgrit) {
    PMK_RETURN_IF(P->group_of || P->m_coarse != P->m_fine, PMK_ERR_SHAPE);
    PMK_RETURN_IF(!P->ratio || !P->work0 || !P->work1 || !P->work2 || !P->coarse_out,
                  PMK_ERR_ARG);
    PMK_RETURN_IF(!P->fft_x && !P->sx, PMK_ERR_ARG);
    return 0;
  }
  const bool space = P->group_of != nullptr || P->z_ptr != nullptr;
  PMK_RETURN_IF(space && (!P->y_ptr || !P->y_idx || !P->y_val), PMK_ERR_ARG);
  PMK_RETURN_IF(!space && P->m_coarse != P->m_fine, PMK_ERR_SHAPE);
  PMK_RETURN_IF(P->z_ptr && (P->group_of || !P->z_idx || !P->z_val), PMK_ERR_ARG);
  return 0;
}

// weighted space pair (full weighting / bilinear): see pmk_pair z_*
inline bool weighted(const pmk_pair &P) { return P.z_ptr != nullptr; }
// the iteration's child vector is already at the level's spatial size
inline bool child_is_fine_space(const pmk_pair &P) { return P.mgrit || weighted(P); }

MarchParams base_params(const pmk_level &L) {
  MarchParams p;
  std::memset(&p, 0, sizeof(p));
  p.nx = L.nx;
  p.ny = (L.dim == 2) ? L.ny : 1;
  p.m = p.nx * p.ny;
  p.n_steps = L.n_steps;
  p.P = L.diag_t;
  p.Q = L.sub_t;
  p.dropped = L.dropped;
  p.nu = 1;
  p.m_coarse = p.m;
  return p;
}

// K-MVR of level idx into the child's rhs; when the child is an inner FGMRES
// level its ||rhs||^2 partials come out of the same pass.
int mvr_into_child(pmk_hier *H, int idx, const double *v, const double *v_scale,
                   double *v_norm_out, const int *live, cudaStream_t s, bool exact);

// PMK_MGS=classic: sequential MGS passes (bitwise the reference's Hessenberg)
bool classic_mgs() {
  static const bool on = [] {
    const char *e = getenv("PMK_MGS");
    return e && std::strcmp(e, "classic") == 0;
  }();
  return on;
}

// Lazy basis (KState::lazy; the ICWY path, PMK_LAZY=0 turns it off): no
// normalisation pass writes v_j; every consumer scales the raw vector.
bool lazy_basis() {
  static const bool on = [] {
    const char *e = getenv("PMK_LAZY");
    return !classic_mgs() && !(e && e[0] == '0');
  }();
  return on;
}

// Deferred first orthogonalisation in fixed-budget inner solves (PMK_FUSE01=0
// turns it off): see fgmres_fixed.
bool fuse01() {
  static const bool on = [] {
    const char *e = getenv("PMK_FUSE01");
    return lazy_basis() && !(e && e[0] == '0');
  }();
  return on;
}

// vh = Y^T (A v - mu v) ; optionally v_norm_out = v (normalised input)
int do_mvr(const pmk_level &L, const pmk_pair &P, double mu, const double *v,
           const double *v_scale, double *vh, double *scratch, double *v_norm_out,
           const int *live, cudaStream_t s, bool exact = true, double *vh_partials = nullptr,
           int *n_vh = nullptr, const double *v_sub = nullptr,
           const double *v_sub_coef = nullptr, double *vn_partials = nullptr) {
  MarchParams p = base_params(L);
  p.v = v;
  p.v_sub = v_sub;
  p.v_sub_coef = v_sub_coef;
  p.vn_partials = vn_partials;
  p.v_scale = v_scale;
  p.v_norm_out = v_norm_out;
  p.mu = mu;
  p.nu = P.nu;
  p.inject = P.mgrit ? 1 : 0;  // MgritPair.restrict (intergrid.py:152-155)
  p.exact_scale = exact ? 1 : 0;
  p.fma = exact ? 0 : 1;  // in-solver (non-exact) passes may fuse
  const bool space = P.group_of != nullptr || weighted(P);
  PMK_RETURN_IF(space && !scratch, PMK_ERR_ARG);
  p.vh = space ? scratch : vh;
  p.live = live;
  p.vh_partials = space ? nullptr : vh_partials;  // a space pair gathers afterwards
  int np = 0;
  int rc = launch_march(kModeMVR, p, s, &np);
  if (n_vh) *n_vh = (p.vh_partials || p.vn_partials) ? np : 0;
  if (rc) return rc;
  if (space) {
    prof::Tag tag(t_level, prof::kHintRestrict);
    return launch_ts_gather(P, scratch, vh, live, s);
  }
  return 0;
}

// x = v - Z vt ; w = A x ; partial <w, v0>.  For MGRIT pairs vt is the
// already interpolated fine vector (identity coarse mapping).
int do_imv(const pmk_level &L, const pmk_pair &P, const double *v, const double *v_scale,
           const double *vt, double *x, double *w, const double *v0, const double *v0_scale,
           double *partials, int *n_partials, const int *live, cudaStream_t s,
           bool fused = false, double *pj = nullptr, int *pj_done = nullptr, int pj_wsq = 0) {
  MarchParams p = base_params(L);
  p.fma = fused ? 1 : 0;
  p.v = v;
  p.v_scale = v_scale;
  p.nu = P.mgrit ? 1 : P.nu;
  p.vt = vt;
  p.group_of = P.group_of;  // (NULL for weighted pairs: vt is space-interpolated)
  p.m_coarse = child_is_fine_space(P) ? P.m_fine : P.m_coarse;
  p.x_out = x;
  p.out = w;
  p.v0 = v0;
  p.v0_scale = v0_scale;
  p.partials = partials;
  p.pj = pj;
  p.pj_done = pj_done;
  p.pj_wsq = pj_wsq;
  p.live = live;
  return launch_march(kModeIMV, p, s, n_partials);
}

int alloc_state(LevelRT &R, int cap) {
  if (R.cap >= cap && R.d_state) return 0;
  if (R.d_block) {
    cudaFree(R.d_block);
    R.d_block = nullptr;
  }
  const size_t nh = (size_t)(cap + 1) * cap;
  const size_t n_groups = (size_t)(cap + kDotGroup - 1) / kDotGroup;
  const size_t n_dotp = n_groups * (2 * kDotGroup + 1) * kMaxPartials;
  const size_t n_doubles =
      2 * nh + (size_t)cap * cap + 8 * (size_t)(cap + 1) + 4 * kMaxPartials + n_dotp +
      (size_t)(cap + 1) * kMaxPartials;
  const size_t bytes = sizeof(KState) + 64 + n_doubles * sizeof(double);
  PMK_CUDA_TRY(cudaMalloc(&R.d_block, bytes));
  PMK_CUDA_TRY(cudaMemset(R.d_block, 0, bytes));
  char *base = static_cast<char *>(R.d_block);
  R.d_state = reinterpret_cast<KState *>(base);
  double *d = reinterpret_cast<double *>(base + ((sizeof(KState) + 63) / 64) * 64);
  KState h{};
  h.h = d;
  d += nh;
  h.hraw = d;
  d += nh;
  h.cs = d;
  d += cap + 1;
  h.sn = d;
  d += cap + 1;
  h.g = d;
  d += cap + 1;
  h.y = d;
  d += cap + 1;
  h.vscale = d;
  d += cap + 1;
  h.hist = d;
  d += cap + 1;
  h.vrcp = d;
  d += cap + 1;
  h.hv = d;
  d += cap + 1;
  h.ugp = d;
  d += (size_t)(cap + 1) * kMaxPartials;
  h.lazy = lazy_basis() ? 1 : 0;
  R.partA = d;  // K-IMV <w, v_0>, then the pj block (<w, v_j>, <v_j, v_0>)
  d += 3 * kMaxPartials;
  R.partB = d;
  d += kMaxPartials;
  h.gram = d;
  d += (size_t)cap * cap;
  R.partM = d;
  R.h_state = h;
  R.cap = cap;
  PMK_CUDA_TRY(cudaMemcpy(R.d_state, &h, sizeof(KState), cudaMemcpyHostToDevice));
  return 0;
}

inline const int *live_ptr(const LevelRT &R) { return &R.d_state->live; }

constexpr int kSnapSlots = 4;

int fgmres_begin(pmk_hier *H, int idx, const double *rhs, int max_iter, double tol,
                 const int *parent_live, cudaStream_t s) {
  prof::Tag tag(idx);
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.set, PMK_ERR_STATE);
  PMK_RETURN_IF(!rhs || max_iter < 1, PMK_ERR_ARG);
  const void *block = R.d_block;
  int rc = alloc_state(R, max_iter);
  if (rc) return rc;
  if (R.d_block != block && block) drop_graphs(H);  // graphs point into the old block
  R.tol = tol;
  R.parent_live = parent_live;
  if (R.rhs_part_n > 0 && rhs == R.rhs) {
    // ||rhs||^2 partials produced by the parent's K-MVR while writing rhs
    rc = launch_begin(R.d_state, R.rhs_part, R.rhs_part_n, parent_live, s);
    R.rhs_part_n = 0;
  } else {
    rc = launch_dot_partials(rhs, nullptr, rhs, nullptr, R.N, R.partA, parent_live, s);
    if (rc) return rc;
    rc = launch_begin(R.d_state, R.partA, kRedBlocks, parent_live, s);
  }
  if (rc) return rc;
  R.rhs_cur = rhs;
  R.pending = rhs;
  R.v.clear();
  R.ugram_col = -1;
  R.vt.clear();
  return 0;
}

int fgmres_fixed(pmk_hier *H, int idx, double *x, const int *parent_live, cudaStream_t s,
                 const double *out_scale = nullptr);

bool graphs_enabled() {
  static const bool on = [] {
    const char *e = getenv("PMK_GRAPHS");
    return !(e && e[0] == '0');
  }();
  return on && !g_prof_on;
}

// The inner FGMRES recursion below a level (solver.py:347-348) touches only
// registered buffers plus its output, and never synchronises with the host,
// so it is captured once per output buffer into a CUDA graph and replayed
// (the first call runs eagerly so that lazy one-time initialisation -- kernel
// attributes, constant tables -- never happens inside a capture).
int fgmres_fixed_graph(pmk_hier *H, int child, double *out, const int *live, cudaStream_t s,
                       const double *out_scale = nullptr) {
  LevelRT &R = H->lv[child];
  if (!graphs_enabled() || R.graph_failed || s == nullptr || s == cudaStreamLegacy ||
      s == cudaStreamPerThread)
    return fgmres_fixed(H, child, out, live, s, out_scale);
  const GraphKey key{out, live, out_scale};
  auto it = R.graphs.find(key);
  if (it != R.graphs.end()) {
    g_launches.fetch_add(it->second.second);  // the graph's kernel nodes
    PMK_CUDA_TRY(cudaGraphLaunch(it->second.first, s));
    return 0;
  }
  if (!R.seen.count(key)) {
    R.seen.insert(key);
    return fgmres_fixed(H, child, out, live, s, out_scale);
  }
  const int64_t before = g_launches.load();
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    R.graph_failed = true;
    return fgmres_fixed(H, child, out, live, s, out_scale);
  }
  int rc = fgmres_fixed(H, child, out, live, s, out_scale);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &g);
  const int64_t nodes = g_launches.load() - before;
  g_launches.store(before);  // captured launches are counted when replayed
  cudaGraphExec_t exec = nullptr;
  if (rc == 0 && e == cudaSuccess && g &&
      cudaGraphInstantiate(&exec, g, 0) == cudaSuccess) {
    cudaGraphDestroy(g);
    R.graphs[key] = {exec, nodes};
    g_launches.fetch_add(nodes);
    PMK_CUDA_TRY(cudaGraphLaunch(exec, s));
    return 0;
  }
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
  R.graph_failed = true;
  if (rc) return rc;
  return fgmres_fixed(H, child, out, live, s, out_scale);
}

// Child solve of level idx: vt = A_{idx+1}^{-1} vh (approximately); with
// out_scale, the solution for vh * (*out_scale) (every child solve is
// homogeneous in its rhs: the FGMRES iterates scale with it).
int child_solve(pmk_hier *H, int idx, double *out, const int *live, cudaStream_t s,
                const double *out_scale = nullptr) {
  const int child = idx + 1;
  if (child == H->n_levels - 1) {
    PMK_RETURN_IF(!H->has_coarse || !H->coarse_rhs, PMK_ERR_STATE);
    prof::Tag tag(child);
    return coarse_solve(H->coarse, H->coarse_rhs, out, live, s, out_scale);
  }
  if (idx == 0) return fgmres_fixed_graph(H, child, out, live, s, out_scale);
  return fgmres_fixed(H, child, out, live, s, out_scale);
}

// Can child_solve(idx) honour an out_scale?
bool child_scalable(const pmk_hier *H, int idx) {
  const int child = idx + 1;
  if (child == H->n_levels - 1) {
    const pmk_coarse &C = H->coarse;
    return H->has_coarse && C.kind == PMK_COARSE_DST && C.fft_x && C.dim == 2 && C.ny > 1;
  }
  return true;
}

double *child_rhs(pmk_hier *H, int idx) {
  const int child = idx + 1;
  if (child == H->n_levels - 1) return H->coarse_rhs;
  return H->lv[child].rhs;
}

int mvr_into_child(pmk_hier *H, int idx, const double *v, const double *v_scale,
                   double *v_norm_out, const int *live, cudaStream_t s, bool exact) {
  LevelRT &R = H->lv[idx];
  double *vh = child_rhs(H, idx);
  PMK_RETURN_IF(!vh, PMK_ERR_STATE);
  const int child = idx + 1;
  LevelRT *C = (child < H->n_levels - 1) ? &H->lv[child] : nullptr;
  double *part = (C && C->rhs_part) ? C->rhs_part : nullptr;
  int n = 0;
  const int rc = do_mvr(R.L, R.P, H->mu, v, v_scale, vh, R.ts_scratch, v_norm_out, live, s,
                        exact, part, &n);
  if (C) C->rhs_part_n = part ? n : 0;
  return rc;
}

// fuse (fgmres_fixed only): kStepDefer = step 0 stops after h_00 (its w stays
// unorthogonalised in w_next); kStepSub = step 1 starts with the deferred
// update, fused into its K-MVR, which stores v_1 raw into sub_store.
constexpr int kStepPlain = 0, kStepDefer = 1, kStepSub = 2, kStepPyth = 3;

int fgmres_step(pmk_hier *H, int idx, int j, double *v_out, double *w_next, double *child_out,
                cudaStream_t s, bool keep_w = true, int fuse = kStepPlain,
                double *sub_store = nullptr) {
  prof::Tag tag(idx);
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.set || !R.d_state, PMK_ERR_STATE);
  PMK_RETURN_IF(j != (int)R.vt.size() || j >= R.cap, PMK_ERR_STATE);
  const bool lazy = R.h_state.lazy != 0;
  PMK_RETURN_IF((!lazy && !v_out) || !w_next || !child_out, PMK_ERR_ARG);
  PMK_RETURN_IF(w_next == R.rhs_cur || v_out == R.pending, PMK_ERR_ARG);
  // lazy basis: w_next is kept as raw basis vector j+1 and may not be a
  // buffer of the current basis (a fresh buffer per step)
  for (const double *b : R.v) PMK_RETURN_IF(lazy && w_next == b, PMK_ERR_ARG);
  double *vh = child_rhs(H, idx);
  PMK_RETURN_IF(!vh, PMK_ERR_STATE);
  const int *live = live_ptr(R);
  const KState &K = R.h_state;
  // apply_preconditioner (solver.py:336-359) on v_j = raw / scale (in-solver
  // normalisation by reciprocal multiply, <= 1 ulp; the classic mode keeps
  // the reference's division).  Normalised basis: this pass also stores v_j
  // into v_out.  Lazy basis: v_j stays raw (every consumer scales it); v_out,
  // if given, still receives the normalised copy.
  int rc;
  const double *child_scale = nullptr;
  if (fuse == kStepSub) {
    // deferred step-0 update fused into this K-MVR: it stages w_0 and v_0,
    // forms v_1 raw = w_0 - h_00 v_0 (update-pass rounding), stores it, and
    // restricts (A - mu) v_1 raw; then finish_col(0) gives h_10 from the
    // stored values.  The child solve is homogeneous, so it is asked for the
    // solution of (its rhs) / h_10 directly (out_scale = RN(1/h_10)).
    LevelRT *C = (idx + 1 < H->n_levels - 1) ? &H->lv[idx + 1] : nullptr;
    double *part = (C && C->rhs_part) ? C->rhs_part : nullptr;
    int n = 0;
    rc = do_mvr(R.L, R.P, H->mu, R.pending, nullptr, child_rhs(H, idx), R.ts_scratch, sub_store,
                live, s, false, part, &n, R.v[0], K.hv, R.partB);
    if (rc) return rc;
    if (C) C->rhs_part_n = part ? n : 0;
    rc = launch_finish_col(R.d_state, R.cap, 0, R.partB, n, R.tol, s);
    if (rc) return rc;
    R.v.push_back(sub_store);
    child_scale = K.vrcp + 1;
  } else {
    rc = mvr_into_child(H, idx, R.pending, K.vscale + j, v_out, live, s, classic_mgs());
    if (rc) return rc;
    R.v.push_back(lazy ? R.pending : v_out);
  }
  if (R.P.mgrit) {
    // coarse solve into the pair's scratch, then ideal interpolation into the
    // iteration's (fine-size) child_out (intergrid.py:157-167)
    rc = child_solve(H, idx, R.P.coarse_out, live, s);
    if (rc) return rc;
    prof::Tag tag(idx, prof::kHintInterp);
    rc = mgrit_interpolate(R.P, R.P.coarse_out, child_out, live, s);
  } else if (weighted(R.P)) {
    // coarse solve into the pair's scratch, then Z over space into the
    // iteration's child vector ((n_T+1) x m_fine; K-IMV repeats it in time)
    PMK_RETURN_IF(!R.P.coarse_out, PMK_ERR_ARG);
    rc = child_solve(H, idx, R.P.coarse_out, live, s);
    if (rc) return rc;
    prof::Tag tag(idx, prof::kHintInterp);
    rc = launch_interpolate_z(R.P, R.P.coarse_out, child_out, 1, live, s);
  } else {
    rc = child_solve(H, idx, child_out, live, s, child_scale);
  }
  if (rc) return rc;
  // w = A (v_j - Z vt) and partial <w, v_0>   (solver.py:359, 403, 407);
  // for j >= 1 also <w, v_j> and <v_j, v_0> off the staged v_j
  int np = 0, pj_done = 0;
  static const bool pj_on = [] {  // PMK_PJ=0: the dot pass takes v_0 and v_j too
    const char *e = getenv("PMK_PJ");
    return !(e && e[0] == '0');
  }();
  const bool pyth = fuse == kStepPyth && j == 0;  // (budget 1: ||w||^2 instead)
  double *pj = ((j >= 1 || pyth) && !classic_mgs() && pj_on) ? R.partA + kMaxPartials : nullptr;
  rc = do_imv(R.L, R.P, R.v[j], lazy ? K.vscale + j : nullptr, child_out, nullptr, w_next,
              R.v[0], lazy ? K.vscale : nullptr, R.partA, &np, live, s, !classic_mgs(), pj,
              &pj_done, pyth ? 1 : 0);
  if (rc) return rc;
  if (pyth && pj_done) {  // one-column solve: h_00, then h_10 from ||w||^2
    rc = launch_icwy_solve(R.d_state, R.cap, 0, R.partA, np, s);
    if (rc) return rc;
    rc = launch_finish_col(R.d_state, R.cap, 0, pj, np, R.tol, s, true);
    if (rc) return rc;
    R.pending = w_next;
    R.vt.push_back(child_out);
    return 0;
  }
  if (fuse == kStepDefer) {  // h_00 only; update + finish_col(0) follow in step 1
    rc = launch_icwy_solve(R.d_state, R.cap, 0, R.partA, np, s);
    if (rc) return rc;
    R.pending = w_next;
    R.vt.push_back(child_out);
    return 0;
  }
  if (!classic_mgs()) {
    // MGS (solver.py:405-408) in its one-reduce form, ||w|| (solver.py:412);
    // the last step of a fixed-budget inner solve needs only ||w||, not w
    int n_norm = 0;
    bool finished = false;  // (finish_col fused into the last update pass)
    // Gram row of v_{j+1} out of this column's update pass (lazy basis: raw
    // products, scaled in the next ICWY solve), used by the next column
    static const bool ugram_on = [] {
      const char *e = getenv("PMK_UGRAM");
      return !(e && e[0] == '0');
    }();
    const bool ug_in = ugram_on && lazy && R.ugram_col == j;
    const bool ug_out = ugram_on && lazy && keep_w && j + 1 < R.cap;
    bool ug_done = false;
    rc = launch_icwy_mgs(R.d_state, R.cap, j, w_next, R.v.data(), R.N, R.partA, np,
                         pj_done ? pj : nullptr, R.partM, R.partB, &n_norm, keep_w, s, R.tol,
                         true, &finished, ug_in, ug_out, &ug_done);
    R.ugram_col = ug_done ? j + 1 : -1;
    if (rc) return rc;
    if (!finished) rc = launch_finish_col(R.d_state, R.cap, j, R.partB, n_norm, R.tol, s);
    if (rc) return rc;
    R.pending = w_next;
    R.vt.push_back(child_out);
    return 0;
  }
  // MGS one basis vector per pass, exactly the reference's operation order
  double *prev = R.partA, *cur = R.partB;
  int n_prev = np;
  for (int l = 0; l <= j; ++l) {
    const double *vn = (l < j) ? R.v[l + 1] : nullptr;
    rc = launch_mgs_pass(R.d_state, R.cap, l, j, w_next, R.v[l], nullptr, vn, nullptr, R.N, prev,
                         n_prev, cur, s);
    if (rc) return rc;
    double *t = prev;
    prev = cur;
    cur = t;
    n_prev = kRedBlocks;
  }
  rc = launch_finish_col(R.d_state, R.cap, j, prev, n_prev, R.tol, s);
  if (rc) return rc;
  R.pending = w_next;
  R.vt.push_back(child_out);
  return 0;
}

// Back substitution (when row0 == 0) and x = sum_i y_i (v_i - Z vt_i) over
// fine slices [row0, row1).  row0 is a multiple of nu: slice nu J closes
// coarse slice J, so the sub-range starting there is itself a (shorter)
// space-time vector whose slice 0 maps to coarse slice J, exactly the
// assembly's slice mapping -- it runs on offset views.
int fgmres_finish_rows(pmk_hier *H, int idx, double *x, int row0, int row1, cudaStream_t s,
                       const double *out_scale = nullptr) {
  prof::Tag tag(idx);
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.set || !R.d_state, PMK_ERR_STATE);
  PMK_RETURN_IF(!x, PMK_ERR_ARG);
  const int m = R.P.m_fine;
  const int rows = (int)(R.N / m);
  const int nu = R.P.mgrit ? 1 : R.P.nu;
  PMK_RETURN_IF(row0 < 0 || row1 > rows || row0 >= row1 || row0 % nu != 0, PMK_ERR_ARG);
  int rc = 0;
  if (row0 == 0) {
    rc = launch_backsolve(R.d_state, R.cap, s, out_scale);
    if (rc) return rc;
  }
  const int64_t off = (int64_t)row0 * m;
  const int mc = child_is_fine_space(R.P) ? m : R.P.m_coarse;
  const int64_t coff = (int64_t)(row0 / nu) * mc;
  const int64_t n_sub = (int64_t)(row1 - row0) * m;
  const int n = (int)R.vt.size();
  // time pairs with nu = 2 take the pair kernel (<= 8 vectors per pass, every
  // coarse value read once, all loads up front); more vectors are summed in
  // passes of 8 -- two extra x read/write sweeps for 19 vectors still beat
  // the one-pass generic kernel's dependent per-element loop (4.4 TB/s)
  const bool pair = !R.P.mgrit && !R.P.group_of && R.P.nu == 2 && mc == m;
  const int per_pass = pair ? 8 : kAsmChunk;
  int first = 0;
  do {
    AssembleArgs a;
    std::memset(&a, 0, sizeof(a));
    a.count = 0;
    for (int l = first; l < n && a.count < per_pass; ++l) {
      a.v[a.count] = R.v[l] + off;
      a.vt[a.count] = R.vt[l] + coff;
      ++a.count;
    }
    if (R.P.mgrit)  // vt_l are the interpolated fine vectors
      rc = launch_assemble(R.d_state, a, x + off, n_sub, m, 1, m, nullptr, first, s);
    else  // (weighted pairs: vt_l are interpolated in space already)
      rc = launch_assemble(R.d_state, a, x + off, n_sub, m, R.P.nu, mc, R.P.group_of, first, s);
    if (rc) return rc;
    first += per_pass;
  } while (first < n);
  return 0;
}

int fgmres_finish(pmk_hier *H, int idx, double *x, cudaStream_t s,
                  const double *out_scale = nullptr) {
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.set || !R.d_state, PMK_ERR_STATE);
  return fgmres_finish_rows(H, idx, x, 0, (int)(R.N / R.P.m_fine), s, out_scale);
}

int fgmres_fixed(pmk_hier *H, int idx, double *x, const int *parent_live, cudaStream_t s,
                 const double *out_scale) {
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.set || !R.rhs, PMK_ERR_STATE);
  PMK_RETURN_IF((int)R.v_slots.size() < R.budget || (int)R.child_out.size() < R.budget ||
                    !R.w_buf,
                PMK_ERR_STATE);
  int rc = fgmres_begin(H, idx, R.rhs, R.budget, 0.0, parent_live, s);
  if (rc) return rc;
  const bool lazy = R.h_state.lazy != 0;
  // Deferred first orthogonalisation: step 0's update pass (w_0 -= h_00 v_0,
  // 24 B per unknown) is fused into step 1's K-MVR, which reads w_0 and v_0
  // anyway-adjacent (+8 B): 2-D constant-stencil time pairs, lazy basis.
  const bool iso = iso_stencil(R.L.diag_t) && iso_stencil(R.L.sub_t);
  const bool fuse = fuse01() && lazy && R.budget >= 2 && !R.P.mgrit && !R.P.group_of && !R.P.z_ptr &&
                    R.L.dim == 2 && iso && !R.L.dropped && child_scalable(H, idx);
  // budget 1: no update pass at all (h_10 from ||w||^2, see finish_col_block)
  const bool pyth1 = fuse01() && lazy && R.budget == 1 && !R.P.mgrit && !R.P.group_of && !R.P.z_ptr &&
                     R.L.dim == 2 && iso && !R.L.dropped;
  for (int j = 0; j < R.budget; ++j) {
    // lazy basis: v_0 is the rhs, step j's w goes to slot j+1 (it is basis
    // vector j+1), the last step's w only feeds ||w|| (w_buf)
    double *w_next = (lazy && j + 1 < R.budget) ? R.v_slots[j + 1] : R.w_buf;
    int mode = kStepPlain;
    double *store = nullptr;
    if (pyth1) {
      mode = kStepPyth;
    } else if (fuse && j == 0) {
      mode = kStepDefer;
      w_next = R.w_buf;  // w_0 raw, consumed by step 1's K-MVR
    } else if (fuse && j == 1) {
      mode = kStepSub;
      store = R.v_slots[1];  // v_1 raw
      w_next = (2 < R.budget) ? R.v_slots[2] : R.w_buf;
    }
    rc = fgmres_step(H, idx, j, lazy ? nullptr : R.v_slots[j], w_next, R.child_out[j], s,
                     j + 1 < R.budget, mode, store);
    if (rc) return rc;
  }
  return fgmres_finish(H, idx, x, s, out_scale);
}

// Internal scratch for the stand-alone reductions.
std::mutex g_scratch_mu;
double *g_scratch = nullptr;
double *scratch_partials() {
  std::lock_guard<std::mutex> g(g_scratch_mu);
  if (!g_scratch) {
    if (cudaMalloc(&g_scratch, kMaxPartials * sizeof(double)) != cudaSuccess) g_scratch = nullptr;
  }
  return g_scratch;
}

}  // namespace

// ============================================================== C-ABI
extern "C" {

const char *pmk_version(void) { return "pintmk_b200 0.1 sm_100a"; }

int64_t pmk_launch_count(void) { return g_launches.load(); }

int32_t pmk_lazy_basis(void) { return lazy_basis() ? 1 : 0; }

int pmk_div_check(const double *x, double d, int64_t n, double *out, pmk_stream_t stream) {
  PMK_RETURN_IF(!x || !out || n < 0, PMK_ERR_ARG);
  return launch_div_check(x, d, n, out, cs(stream));
}

int pmk_dgemm(int32_t M, int32_t N, int32_t K, const double *A, int32_t lda, int64_t stride_a,
              const double *B, int32_t ldb, int64_t stride_b, double *C, int32_t ldc,
              int64_t stride_c, int32_t batch, pmk_stream_t stream) {
  PMK_RETURN_IF(!A || !B || !C || M < 0 || N < 0 || K < 0 || batch < 0, PMK_ERR_ARG);
  PMK_RETURN_IF(lda < K || ldb < N || ldc < N, PMK_ERR_SHAPE);
  if (M == 0 || N == 0 || batch == 0) return 0;
  return launch_gemm(M, N, K, A, lda, stride_a, B, ldb, stride_b, C, ldc, stride_c, batch,
                     cs(stream));
}

int pmk_profile_begin(int32_t with_events) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_recs.clear();
  g_pool_used = 0;
  g_prof_on = with_events != 0;
  return 0;
}

int pmk_profile_end(double *stats, int32_t max_categories, int32_t *n_categories) {
  PMK_CUDA_TRY(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = false;
  const int nc = prof::kNumCat < max_categories ? prof::kNumCat : max_categories;
  if (stats)
    for (int i = 0; i < 4 * nc; ++i) stats[i] = 0.0;
  for (const ProfRec &r : g_recs) {
    if (r.cat >= nc || !stats) continue;
    float ms = 0.f;
    PMK_CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
    stats[4 * r.cat + 0] += 1.0;
    stats[4 * r.cat + 1] += ms;
    stats[4 * r.cat + 2] += r.bytes;
    stats[4 * r.cat + 3] += r.flops;
  }
  g_recs.clear();
  g_pool_used = 0;
  if (n_categories) *n_categories = nc;
  return 0;
}

int pmk_profile_end_levels(double *rows, int32_t max_rows, int32_t *n_rows) {
  PMK_CUDA_TRY(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = false;
  // aggregate by (level, hint, category), in order of first appearance
  std::vector<std::array<double, 7>> agg;
  std::unordered_map<int64_t, size_t> where;
  for (const ProfRec &r : g_recs) {
    float ms = 0.f;
    PMK_CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
    const int64_t key = ((int64_t)(r.level + 1) << 32) | ((int64_t)(r.hint + 1) << 16) | r.cat;
    auto it = where.find(key);
    if (it == where.end()) {
      it = where.emplace(key, agg.size()).first;
      agg.push_back({(double)r.level, (double)r.hint, (double)r.cat, 0.0, 0.0, 0.0, 0.0});
    }
    auto &a = agg[it->second];
    a[3] += 1.0;
    a[4] += ms;
    a[5] += r.bytes;
    a[6] += r.flops;
  }
  g_recs.clear();
  g_pool_used = 0;
  const int n = (int)agg.size();
  if (n_rows) *n_rows = n;
  PMK_RETURN_IF(rows && n > max_rows, PMK_ERR_ARG);
  if (rows)
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < 7; ++c) rows[7 * i + c] = agg[i][c];
  return 0;
}

const char *pmk_profile_category(int32_t idx) {
  return (idx >= 0 && idx < prof::kNumCat) ? kCatNames[idx] : "";
}

int pmk_stmv(const pmk_level *L, const double *v, double *out, pmk_stream_t stream) {
  int rc = check_level(L);
  if (rc) return rc;
  PMK_RETURN_IF(!v || !out, PMK_ERR_ARG);
  MarchParams p = base_params(*L);
  p.v = v;
  p.out = out;
  return launch_march(kModeMV, p, cs(stream), nullptr);
}

int pmk_restrict(const pmk_pair *P, const double *v, double *vh, double *scratch,
                 pmk_stream_t stream) {
  PMK_RETURN_IF(!P || !v || !vh, PMK_ERR_ARG);
  if (P->mgrit) return mgrit_restrict(*P, v, vh, nullptr, cs(stream));
  if (P->group_of || P->z_ptr) {
    PMK_RETURN_IF(!scratch, PMK_ERR_ARG);
    pmk_pair tp = *P;
    int rc = launch_restrict_time(tp, v, scratch, cs(stream));
    if (rc) return rc;
    return launch_ts_gather(*P, scratch, vh, nullptr, cs(stream));
  }
  return launch_restrict_time(*P, v, vh, cs(stream));
}

int pmk_interpolate(const pmk_pair *P, const double *w, double *out, pmk_stream_t stream) {
  PMK_RETURN_IF(!P || !w || !out, PMK_ERR_ARG);
  if (P->mgrit) return mgrit_interpolate(*P, w, out, nullptr, cs(stream));
  return launch_interpolate(*P, w, out, cs(stream));
}

int pmk_stmv_shift_restrict(const pmk_level *L, const pmk_pair *P, double mu,
                            const double *v_raw, const double *v_scale, double *vh,
                            double *scratch, pmk_stream_t stream) {
  int rc = check_level(L);
  if (rc) return rc;
  rc = check_pair(*L, P);
  if (rc) return rc;
  PMK_RETURN_IF(!v_raw || !vh, PMK_ERR_ARG);
  return do_mvr(*L, *P, mu, v_raw, v_scale, vh, scratch, nullptr, nullptr, cs(stream));
}

int pmk_interp_sub_stmv(const pmk_level *L, const pmk_pair *P, const double *v_raw,
                        const double *v_scale, const double *vt, double *x, double *w,
                        pmk_stream_t stream) {
  int rc = check_level(L);
  if (rc) return rc;
  rc = check_pair(*L, P);
  if (rc) return rc;
  PMK_RETURN_IF(!v_raw || !vt || !w, PMK_ERR_ARG);
  return do_imv(*L, *P, v_raw, v_scale, vt, x, w, v_raw, v_scale, nullptr, nullptr, nullptr,
                cs(stream));
}

int pmk_coarsest_solve(const pmk_coarse *C, const double *rhs, double *out,
                       pmk_stream_t stream) {
  PMK_RETURN_IF(!C || !rhs || !out, PMK_ERR_ARG);
  return coarse_solve(*C, rhs, out, nullptr, cs(stream));
}

int pmk_dot(const double *a, const double *b, int64_t n, double *result, pmk_stream_t stream) {
  PMK_RETURN_IF(!a || !b || !result || n < 0, PMK_ERR_ARG);
  double *part = scratch_partials();
  PMK_RETURN_IF(!part, (int)cudaErrorMemoryAllocation);
  int rc = launch_dot_partials(a, nullptr, b, nullptr, n, part, nullptr, cs(stream));
  if (rc) return rc;
  return launch_reduce_to_scalar(part, kRedBlocks, result, 0, cs(stream));
}

int pmk_nrm2(const double *a, int64_t n, double *result, pmk_stream_t stream) {
  PMK_RETURN_IF(!a || !result || n < 0, PMK_ERR_ARG);
  double *part = scratch_partials();
  PMK_RETURN_IF(!part, (int)cudaErrorMemoryAllocation);
  int rc = launch_dot_partials(a, nullptr, a, nullptr, n, part, nullptr, cs(stream));
  if (rc) return rc;
  return launch_reduce_to_scalar(part, kRedBlocks, result, 1, cs(stream));
}

int pmk_residual_nrm2(const pmk_level *L, const double *u, const double *rhs, double *tmp,
                      double *result, pmk_stream_t stream) {
  int rc = check_level(L);
  if (rc) return rc;
  PMK_RETURN_IF(!u || !rhs || !tmp || !result, PMK_ERR_ARG);
  rc = pmk_stmv(L, u, tmp, stream);
  if (rc) return rc;
  double *part = scratch_partials();
  PMK_RETURN_IF(!part, (int)cudaErrorMemoryAllocation);
  rc = launch_diffsq_partials(rhs, tmp, level_N(*L), part, cs(stream));
  if (rc) return rc;
  return launch_reduce_to_scalar(part, kRedBlocks, result, 1, cs(stream));
}

int pmk_residual(const pmk_level *L, const double *u, const double *rhs, double *r,
                 double *result, pmk_stream_t stream) {
  int rc = check_level(L);
  if (rc) return rc;
  PMK_RETURN_IF(!u || !rhs || !r || !result || r == u || r == rhs, PMK_ERR_ARG);
  rc = pmk_stmv(L, u, r, stream);
  if (rc) return rc;
  double *part = scratch_partials();
  PMK_RETURN_IF(!part, (int)cudaErrorMemoryAllocation);
  rc = launch_diffsq_partials(rhs, r, level_N(*L), part, cs(stream), r);
  if (rc) return rc;
  return launch_reduce_to_scalar(part, kRedBlocks, result, 1, cs(stream));
}

int pmk_axpy(double a, const double *x, double *y, int64_t n, pmk_stream_t stream) {
  PMK_RETURN_IF(!x || !y || n < 0 || x == y, PMK_ERR_ARG);
  if (n == 0) return 0;
  return launch_axpy(a, x, y, n, cs(stream));
}

pmk_hier *pmk_hier_create(int32_t n_levels, double mu) {
  if (n_levels < 2 || mu == 0.0) return nullptr;
  pmk_hier *H = new (std::nothrow) pmk_hier();
  if (!H) return nullptr;
  H->n_levels = n_levels;
  H->mu = mu;
  H->lv.resize(n_levels - 1);
  return H;
}

void pmk_hier_destroy(pmk_hier *H) {
  if (!H) return;
  drop_graphs(H);
  for (auto &R : H->lv) {
    if (R.d_block) cudaFree(R.d_block);
    if (R.rhs_part) cudaFree(R.rhs_part);
    if (R.snap) cudaFreeHost(R.snap);
  }
  delete H;
}

int pmk_hier_set_level(pmk_hier *H, int32_t idx, const pmk_level *L, const pmk_pair *P,
                       int32_t budget) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels - 1, PMK_ERR_ARG);
  int rc = check_level(L);
  if (rc) return rc;
  rc = check_pair(*L, P);
  if (rc) return rc;
  PMK_RETURN_IF(idx > 0 && budget < 1, PMK_ERR_ARG);
  drop_graphs(H);
  LevelRT &R = H->lv[idx];
  R.L = *L;
  R.P = *P;
  R.budget = budget;
  R.N = level_N(*L);
  R.set = true;
  if (idx > 0) return alloc_state(R, budget);
  return 0;
}

int pmk_hier_set_coarse(pmk_hier *H, const pmk_coarse *C) {
  PMK_RETURN_IF(!H || !C, PMK_ERR_ARG);
  PMK_RETURN_IF(C->kind < PMK_COARSE_DST || C->kind > PMK_COARSE_LINE, PMK_ERR_UNSUPPORTED);
  drop_graphs(H);
  H->coarse = *C;
  H->has_coarse = true;
  return 0;
}

int pmk_hier_set_buffers(pmk_hier *H, int32_t idx, double *rhs, double *const *v_slots,
                         double *const *child_out, int32_t n_slots, double *w_buf,
                         double *ts_scratch) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels || !rhs, PMK_ERR_ARG);
  drop_graphs(H);
  if (idx == H->n_levels - 1) {
    H->coarse_rhs = rhs;
    return 0;
  }
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.set, PMK_ERR_STATE);
  PMK_RETURN_IF(n_slots < 0 || (n_slots > 0 && (!v_slots || !child_out || !w_buf)),
                PMK_ERR_ARG);
  PMK_RETURN_IF((R.P.group_of || R.P.z_ptr) && !ts_scratch, PMK_ERR_ARG);
  R.rhs = rhs;
  R.w_buf = w_buf;
  if (idx > 0 && !R.rhs_part)  // the parent's K-MVR leaves ||rhs||^2 partials here
    PMK_CUDA_TRY(cudaMalloc(&R.rhs_part, kMaxPartials * sizeof(double)));
  R.rhs_part_n = 0;
  R.v_slots.assign(v_slots, v_slots + n_slots);
  R.child_out.assign(child_out, child_out + n_slots);
  R.ts_scratch = ts_scratch;
  return 0;
}

int pmk_fgmres_begin(pmk_hier *H, int32_t idx, const double *rhs, int32_t max_iter, double tol,
                     pmk_stream_t stream) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels - 1, PMK_ERR_ARG);
  return fgmres_begin(H, idx, rhs, max_iter, tol, nullptr, cs(stream));
}

int pmk_fgmres_step(pmk_hier *H, int32_t idx, int32_t j, double *v_out, double *w_next,
                    double *child_out, pmk_stream_t stream) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels - 1, PMK_ERR_ARG);
  return fgmres_step(H, idx, j, v_out, w_next, child_out, cs(stream));
}

int pmk_fgmres_finish(pmk_hier *H, int32_t idx, double *x, pmk_stream_t stream) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels - 1, PMK_ERR_ARG);
  return fgmres_finish(H, idx, x, cs(stream));
}

int pmk_fgmres_finish_rows(pmk_hier *H, int32_t idx, double *x, int32_t row_begin,
                           int32_t row_end, pmk_stream_t stream) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels - 1, PMK_ERR_ARG);
  return fgmres_finish_rows(H, idx, x, row_begin, row_end, cs(stream));
}

int pmk_fgmres_state(pmk_hier *H, int32_t idx, double *scalars, double *hist, double *hraw,
                     double *y, int32_t *cap, pmk_stream_t stream) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels - 1, PMK_ERR_ARG);
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.d_state, PMK_ERR_STATE);
  cudaStream_t s = cs(stream);
  KState k;
  PMK_CUDA_TRY(cudaMemcpyAsync(&k, R.d_state, sizeof(KState), cudaMemcpyDeviceToHost, s));
  if (hist)
    PMK_CUDA_TRY(cudaMemcpyAsync(hist, R.h_state.hist, R.cap * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
  if (hraw)
    PMK_CUDA_TRY(cudaMemcpyAsync(hraw, R.h_state.hraw, (size_t)(R.cap + 1) * R.cap * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
  if (y)
    PMK_CUDA_TRY(
        cudaMemcpyAsync(y, R.h_state.y, R.cap * sizeof(double), cudaMemcpyDeviceToHost, s));
  PMK_CUDA_TRY(cudaStreamSynchronize(s));
  if (scalars) {
    scalars[0] = k.beta;
    scalars[1] = k.rel;
    scalars[2] = (double)k.n_iter;
    scalars[3] = (double)k.breakdown;
  }
  if (cap) *cap = R.cap;
  return 0;
}

int pmk_fgmres_snapshot(pmk_hier *H, int32_t idx, int32_t slot, pmk_stream_t stream) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels - 1 || slot < 0 || slot >= kSnapSlots,
                PMK_ERR_ARG);
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.d_state, PMK_ERR_STATE);
  if (!R.snap) PMK_CUDA_TRY(cudaHostAlloc(&R.snap, kSnapSlots * sizeof(KState), 0));
  PMK_CUDA_TRY(cudaMemcpyAsync(R.snap + slot, R.d_state, sizeof(KState), cudaMemcpyDeviceToHost,
                               cs(stream)));
  return 0;
}

int pmk_fgmres_snapshot_read(pmk_hier *H, int32_t idx, int32_t slot, double *scalars) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels - 1 || slot < 0 || slot >= kSnapSlots ||
                    !scalars,
                PMK_ERR_ARG);
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.snap, PMK_ERR_STATE);
  const KState &k = R.snap[slot];
  scalars[0] = k.beta;
  scalars[1] = k.rel;
  scalars[2] = (double)k.n_iter;
  scalars[3] = (double)k.breakdown;
  return 0;
}

int pmk_fgmres_fixed(pmk_hier *H, int32_t idx, double *x, pmk_stream_t stream) {
  PMK_RETURN_IF(!H || idx < 1 || idx >= H->n_levels - 1 || !x, PMK_ERR_ARG);
  return fgmres_fixed(H, idx, x, nullptr, cs(stream));
}

int pmk_apply_preconditioner(pmk_hier *H, int32_t idx, const double *v, double *child_out,
                             double *out, pmk_stream_t stream) {
  PMK_RETURN_IF(!H || idx < 0 || idx >= H->n_levels - 1 || !v || !child_out || !out, PMK_ERR_ARG);
  LevelRT &R = H->lv[idx];
  PMK_RETURN_IF(!R.set, PMK_ERR_STATE);
  cudaStream_t s = cs(stream);
  double *vh = child_rhs(H, idx);
  PMK_RETURN_IF(!vh, PMK_ERR_STATE);
  prof::Tag tag(idx);
  int rc = mvr_into_child(H, idx, v, nullptr, nullptr, nullptr, s, true);
  if (rc) return rc;
  if (R.P.mgrit) {
    rc = child_solve(H, idx, R.P.coarse_out, nullptr, s);
    if (rc) return rc;
    prof::Tag itag(idx, prof::kHintInterp);
    rc = mgrit_interpolate(R.P, R.P.coarse_out, child_out, nullptr, s);
  } else if (weighted(R.P)) {
    PMK_RETURN_IF(!R.P.coarse_out, PMK_ERR_ARG);
    rc = child_solve(H, idx, R.P.coarse_out, nullptr, s);
    if (rc) return rc;
    prof::Tag itag(idx, prof::kHintInterp);
    rc = launch_interpolate_z(R.P, R.P.coarse_out, child_out, 1, nullptr, s);
  } else {
    rc = child_solve(H, idx, child_out, nullptr, s);
  }
  if (rc) return rc;
  // out = v - Z vt (the matvec output of the fused kernel is not needed)
  return do_imv(R.L, R.P, v, nullptr, child_out, out, nullptr, nullptr, nullptr, nullptr,
                nullptr, nullptr, s);
}

}  // extern "C"
