"""FGMRES with the multilevel Krylov (MLK) shift preconditioner, on one B200.

Mirror of reference ``pintmk/solver.py`` (names, arguments, error
behaviour).  The hierarchy is built on the host exactly as the reference
builds it; the solve runs on the device:

* the outer FGMRES (level 0) is driven from Python one iteration at a time
  (one small device->host read per iteration for the stop test,
  solver.py:433-440);
* each iteration is a handful of fused sm_100a kernels (shift+restrict,
  interpolate+subtract+matvec, fused MGS passes, device-side Givens) plus
  the inner recursion, which runs entirely in native code with no host
  synchronisation (solver.py:347-348);
* the coarsest level is a sine-diagonalised or dense direct solve.

Extensions over the reference (default-off): ``SolverConfig.restart``
(FGMRES(m)), the ``"time_space"`` schedule move (reference _space_move with
time_nu = nu, solver.py:127-143).  ``ledger``/``model`` (simulated-parallel
cost accounting, parcost.py) are accepted and ignored: the GPU measures
real time.
"""

from __future__ import annotations

import contextlib
import ctypes
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib
from ._device import SpectralInfo
from .intergrid import (CoarseSystem, MgritPair, TimePair, TimeSpacePair, WeightedSpacePair,
                        agglomerate_partition, perturb_decouple, rediscretized_coarse)
from .spatial import gershgorin_bound
from .stepper import BlockBidiagonalSystem, FineSystem, _to_device


@dataclass
class SolveReport:
    """Outcome of one iterative solve (reference reports.py:8-25)."""

    method: str
    outer_iterations: int = 0
    residual_history: list[float] = field(default_factory=list)
    converged: bool = False
    tol: float = 0.0
    error_vs_oracle: float | None = None
    wall_time: float | None = None
    simulated_elapsed: int | None = None
    level_stats: dict = field(default_factory=dict)
    metadata: dict = field(default_factory=dict)

    @property
    def final_residual(self) -> float:
        return self.residual_history[-1] if self.residual_history else float("inf")


@dataclass
class SolverConfig:
    """Krylov knobs (reference solver.py:37-57) plus ``restart``.

    ``basis_memory_limit``/``basis_dir`` are accepted for compatibility: the
    device keeps the basis in HBM (no disk spill); ``restart`` bounds it.
    """

    mu: float = 1.0
    tol: float = 1e-6
    max_outer: int = 200
    inner_iters: int | list[int] | None = None
    coarsest_n_cgs: int = 0
    basis_memory_limit: int = 2 * 1024**3
    basis_dir: str | None = None
    restart: int | None = None

    def __post_init__(self):
        if self.mu == 0:
            raise ValueError("mu must be nonzero")
        if self.restart is not None and self.restart < 1:
            raise ValueError("restart must be >= 1")


@dataclass(eq=False)
class Level:
    """One rung of the hierarchy (reference solver.py:60-81)."""

    system: BlockBidiagonalSystem
    spatial_matrix: sp.csr_matrix
    dt: float
    implicit_weight: float
    n_steps: int
    grid: tuple[int, int]
    dim: int
    kind: str
    pair: object | None = None
    budget: int = 0
    laplace_factor: float | None = None  # set while spatial_matrix is the pristine Laplacian

    @property
    def state_dim(self) -> int:
        return self.spatial_matrix.shape[0]

    @property
    def total_dim(self) -> int:
        return (self.n_steps + 1) * self.state_dim


_SOLVER_STREAMS: dict = {}


def _solver_stream(device: int):
    import torch

    st = _SOLVER_STREAMS.get(device)
    if st is None:
        st = _SOLVER_STREAMS[device] = torch.cuda.Stream(device=device)
    return st


class LevelHierarchy:
    """Levels, fine system, config, and the native solver state."""

    def __init__(self, levels: list[Level], fine: FineSystem, config: SolverConfig):
        self.levels = levels
        self.fine = fine
        self.config = config
        self.moves: list[str] = []
        self._native = None
        self._buffers: list = []
        self._stream = None

    @contextlib.contextmanager
    def on_stream(self):
        """Run on the solver stream of the device (the inner recursion is
        replayed as CUDA graphs, which cannot be captured on the legacy
        default stream); ordered after / before the caller's stream.  One
        stream per device for every hierarchy: torch's caching allocator
        reuses a freed block only on the stream that freed it, so a stream
        per hierarchy would strand every previous solve's memory."""
        import torch

        if self._stream is None:
            self._stream = _solver_stream(torch.cuda.current_device())
        caller = torch.cuda.current_stream()
        if caller == self._stream:
            yield
            return
        self._stream.wait_stream(caller)
        with torch.cuda.stream(self._stream):
            yield
        caller.wait_stream(self._stream)

    @property
    def n_levels(self) -> int:
        return len(self.levels)

    def describe(self) -> list[dict]:
        return [{"kind": lv.kind, "n_steps": lv.n_steps, "grid": lv.grid, "dt": lv.dt,
                 "implicit_weight": lv.implicit_weight, "budget": lv.budget}
                for lv in self.levels]

    def __del__(self):
        if self._native:
            try:
                _lib.load().pmk_hier_destroy(self._native)
            except Exception:
                pass
            self._native = None


# ------------------------------------------------------------- construction
def _coarse_system_from(spatial_matrix, implicit_weight, dt, n_steps, grid, dim,
                        laplace_factor) -> CoarseSystem:
    """D = I - a dt A, B = I + (1-a) dt A (reference solver.py:105-110)."""
    def diag():
        eye = sp.identity(spatial_matrix.shape[0], format="csr")
        return (eye - implicit_weight * dt * spatial_matrix).tocsr()

    def sub():
        eye = sp.identity(spatial_matrix.shape[0], format="csr")
        return (eye + (1.0 - implicit_weight) * dt * spatial_matrix).tocsr()

    spectral = None
    if laplace_factor is not None:
        # pristine level: the device takes the closed-form stencils; the
        # scipy blocks are assembled only if a caller asks for them
        spectral = SpectralInfo(laplace_factor, implicit_weight * dt,
                                (1.0 - implicit_weight) * dt)
    else:
        diag, sub = diag(), sub()
    return CoarseSystem(diag=diag, sub=sub, n_steps=n_steps, provenance="closed_form",
                        grid=grid, dim=dim, spectral=spectral)


def _time_move(level: Level, nu: int) -> Level:
    """Time coarsening by nu (reference solver.py:113-124)."""
    if level.n_steps % nu != 0:
        raise ValueError(f"time move needs nu | n_steps, got {level.n_steps} / {nu}")
    level.pair = TimePair(level.state_dim, nu, level.n_steps // nu)
    a = 1.0 - (1.0 - level.implicit_weight) / nu
    dt = nu * level.dt
    n_steps = level.n_steps // nu
    system = _coarse_system_from(level.spatial_matrix, a, dt, n_steps, level.grid, level.dim,
                                 level.laplace_factor)
    return Level(system=system, spatial_matrix=level.spatial_matrix, dt=dt, implicit_weight=a,
                 n_steps=n_steps, grid=level.grid, dim=level.dim, kind="time",
                 laplace_factor=level.laplace_factor)


def _space_move(level: Level, time_nu: int = 1) -> Level:
    """Agglomeration in space, optionally with time coarsening (reference
    solver.py:127-143)."""
    gx, gy = level.grid
    groups, (mx, my) = agglomerate_partition(gx, gy if level.dim == 2 else 1)
    if level.n_steps % time_nu != 0:
        raise ValueError("time factor must divide n_steps")
    n_steps = level.n_steps // time_nu
    pair = TimeSpacePair(nu=time_nu, n_T=n_steps, partition=groups, n=level.state_dim)
    level.pair = pair
    coarse_a = (pair.y_space.T @ level.spatial_matrix @ pair.z_space).tocsr()
    a = 1.0 - (1.0 - level.implicit_weight) / time_nu
    dt = time_nu * level.dt
    system = _coarse_system_from(coarse_a, a, dt, n_steps, (mx, my), level.dim, None)
    return Level(system=system, spatial_matrix=coarse_a, dt=dt, implicit_weight=a,
                 n_steps=n_steps, grid=(mx, my), dim=level.dim,
                 kind="space" if time_nu == 1 else "time_space")


def _space_move_fw(level: Level, time_nu: int = 1) -> Level:
    """Space coarsening by full weighting / (bi)linear interpolation onto the
    grid with doubled spacing, optionally with time coarsening: BASELINE
    config 4's transfers.  EXTENSION without a reference counterpart (the
    reference's space move agglomerates, solver.py:127-143).  The coarse
    operator is the Laplacian rediscretised on the coarse grid (the Galerkin
    product of these transfers is a 9-point operator); it needs a level whose
    spatial operator is build_laplacian's and odd grid sizes."""
    from .spatial import laplacian_stencil, stencil_csr

    if level.laplace_factor is None:
        raise ValueError("full-weighting space moves need build_laplacian's operator")
    if level.n_steps % time_nu != 0:
        raise ValueError("time factor must divide n_steps")
    n_steps = level.n_steps // time_nu
    pair = WeightedSpacePair(time_nu, n_steps, level.grid, level.dim)
    level.pair = pair
    mx, my = pair.coarse_grid
    factor = level.laplace_factor / 4.0          # tau / (2 dx)^2, exact
    coarse_a = stencil_csr(mx, my, laplacian_stencil(level.dim, factor))
    a = 1.0 - (1.0 - level.implicit_weight) / time_nu
    dt = time_nu * level.dt
    system = _coarse_system_from(coarse_a, a, dt, n_steps, (mx, my), level.dim, factor)
    return Level(system=system, spatial_matrix=coarse_a, dt=dt, implicit_weight=a,
                 n_steps=n_steps, grid=(mx, my), dim=level.dim,
                 kind="space_fw" if time_nu == 1 else "time_space_fw", laplace_factor=factor)


def _fine_level(fine: FineSystem) -> Level:
    ops = fine.ops
    sp_op = ops.spatial
    pristine = ops.spectral_info is not None
    return Level(system=fine, spatial_matrix=sp_op.matrix, dt=ops.config.delta_t,
                 implicit_weight=ops.config.theta, n_steps=fine.n_t,
                 grid=(sp_op.n_x, sp_op.n_y), dim=sp_op.dim, kind="fine",
                 laplace_factor=sp_op.tau / sp_op.delta_x**2 if pristine else None)


def time_move_is_stable(level: Level, nu: int = 2) -> bool:
    """Stability screen of a prospective time move (reference solver.py:154-163)."""
    explicit = (1.0 - level.implicit_weight) / nu
    lam = gershgorin_bound(level.spatial_matrix) / level.dim
    return (1.0 - 2.0 * explicit) * (nu * level.dt) * lam <= 2.0


def auto_moves_step(level: Level, alternating: bool, next_is_space: bool, nu: int = 2):
    """Next automatic move (reference solver.py:166-175)."""
    if not alternating:
        if level.n_steps % nu == 0 and time_move_is_stable(level, nu):
            return "time", False, False
        alternating = True
        next_is_space = True
    return ("space" if next_is_space else "time"), True, not next_is_space


def _assign_budgets(levels: list[Level], inner_iters) -> None:
    """Inner FGMRES budgets (reference solver.py:219-235)."""
    inter = levels[1:-1]
    if not inter:
        return
    if inner_iters is None:
        budgets = [2] * len(inter)
        if len(budgets) > 1:
            budgets[-1] = 1
    elif isinstance(inner_iters, int):
        budgets = [inner_iters] * len(inter)
    else:
        budgets = list(inner_iters)
        if len(budgets) != len(inter):
            raise ValueError("need one inner budget per intermediate level")
    for lvl, b in zip(inter, budgets):
        if b < 1:
            raise ValueError("budgets must be >= 1")
        lvl.budget = b


def build_hierarchy(fine: FineSystem, n_levels: int, schedule: str | list[str] = "auto",
                    cfg: SolverConfig | None = None, nu: int = 2) -> LevelHierarchy:
    """Level stack by repeated coarsening (reference solver.py:178-216).

    Moves: "time", "space" (reference), "time_space" (agglomeration plus
    time coarsening by nu in one move), and the extensions "space_fw" /
    "time_space_fw" (full-weighting restriction, (bi)linear interpolation,
    rediscretised coarse Laplacian: BASELINE config 4's transfers, which the
    reference does not have).
    """
    cfg = cfg or SolverConfig()
    if n_levels < 2:
        raise ValueError("need at least two levels")
    levels = [_fine_level(fine)]
    moves: list[str] = []
    alternating = False
    next_is_space = False
    for i in range(n_levels - 1):
        cur = levels[-1]
        if schedule == "auto":
            move, alternating, next_is_space = auto_moves_step(cur, alternating, next_is_space,
                                                               nu)
        else:
            move = schedule[i]
        if move == "time":
            levels.append(_time_move(cur, nu))
        elif move == "space":
            levels.append(_space_move(cur))
        elif move == "time_space":
            levels.append(_space_move(cur, time_nu=nu))
        elif move == "space_fw":
            levels.append(_space_move_fw(cur))
        elif move == "time_space_fw":
            levels.append(_space_move_fw(cur, time_nu=nu))
        else:
            raise ValueError(f"unknown move {move!r}")
        moves.append(move)
    _assign_budgets(levels, cfg.inner_iters)
    if cfg.coarsest_n_cgs >= 1:
        levels[-1].system = perturb_decouple(levels[-1].system, cfg.coarsest_n_cgs)
    hier = LevelHierarchy(levels=levels, fine=fine, config=cfg)
    hier.moves = moves
    _setup_native(hier)
    return hier


def build_two_level(fine: FineSystem, family: str, nu: int,
                    cfg: SolverConfig | None = None) -> LevelHierarchy:
    """Two-level hierarchy for the T, TS or MGRIT family (reference
    solver.py:238-265)."""
    cfg = cfg or SolverConfig()
    top = _fine_level(fine)
    if family == "T":
        coarse = _time_move(top, nu)
    elif family == "TS":
        coarse = _space_move(top, time_nu=nu)
    elif family == "MGRIT":
        if fine.n_t % nu != 0:
            raise ValueError("nu must divide n_t")
        n_T = fine.n_t // nu
        top.pair = MgritPair(fine.ops, nu, n_T)
        coarse = Level(system=rediscretized_coarse(fine.ops, nu, n_T),
                       spatial_matrix=fine.ops.spatial.matrix, dt=nu * fine.ops.config.delta_t,
                       implicit_weight=fine.ops.config.theta, n_steps=n_T, grid=top.grid,
                       dim=top.dim, kind="mgrit", laplace_factor=top.laplace_factor)
    else:
        raise ValueError(f"unknown family {family!r}")
    if cfg.coarsest_n_cgs >= 1:
        coarse.system = perturb_decouple(coarse.system, cfg.coarsest_n_cgs)
    hier = LevelHierarchy(levels=[top, coarse], fine=fine, config=cfg)
    hier.moves = [family]
    _setup_native(hier)
    return hier


def _child_size(lvl: Level, nxt: Level) -> int:
    """Per-iteration child buffer: the coarse solution, or for MGRIT pairs its
    interpolation to the fine level (ideal interpolation is not a repeat)."""
    if isinstance(lvl.pair, WeightedSpacePair):  # the solution interpolated in space
        return lvl.pair.child_size()
    return lvl.total_dim if isinstance(lvl.pair, MgritPair) else nxt.total_dim


def _empty(n):
    import torch

    return torch.empty(n, dtype=torch.float64, device="cuda")


def _setup_native(hier: LevelHierarchy) -> None:
    """Register levels, pairs, budgets, the coarsest solver and the inner
    workspaces with the native runtime (prefactor, solver.py:213)."""
    _lib.require_cuda()
    lib = _lib.load()
    L = hier.n_levels
    H = lib.pmk_hier_create(L, float(hier.config.mu))
    if not H:
        raise RuntimeError("pmk_hier_create failed")
    hier._native = H
    keep = hier._buffers
    for idx in range(L - 1):
        lvl = hier.levels[idx]
        pdesc = lvl.pair._pair_desc()
        _lib.check(lib.pmk_hier_set_level(H, idx, ctypes.byref(lvl.system.level_desc()),
                                          ctypes.byref(pdesc), int(lvl.budget)), "set_level")
    coarse = hier.levels[-1].system.diag_factorization
    keep.append(coarse)
    _lib.check(lib.pmk_hier_set_coarse(H, ctypes.byref(coarse.desc)), "set_coarse")
    for idx in range(L - 1):
        lvl = hier.levels[idx]
        nxt = hier.levels[idx + 1]
        ts = None
        if isinstance(lvl.pair, (TimeSpacePair, WeightedSpacePair)):
            ts = _empty((lvl.pair.n_T + 1) * lvl.pair.n)
        if idx == 0:
            rhs = hier.fine.rhs.reshape(-1)
            vs, cos, wb = [], [], None
        else:
            rhs = _empty(lvl.total_dim)
            vs = [_empty(lvl.total_dim) for _ in range(lvl.budget)]
            cos = [_empty(_child_size(lvl, nxt)) for _ in range(lvl.budget)]
            wb = _empty(lvl.total_dim)
        keep += [rhs, vs, cos, wb, ts]
        n = len(vs)
        arr_v = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in vs])
        arr_c = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in cos])
        _lib.check(lib.pmk_hier_set_buffers(H, idx, _lib.ptr(rhs), arr_v, arr_c, n,
                                            _lib.ptr(wb), _lib.ptr(ts)), "set_buffers")
    crhs = _empty(hier.levels[-1].total_dim)
    keep.append(crhs)
    _lib.check(lib.pmk_hier_set_buffers(H, L - 1, _lib.ptr(crhs), None, None, 0, None, None),
               "set_buffers")


# --------------------------------------------------------------------- solve
def apply_preconditioner(hier: LevelHierarchy, level_idx: int, v, ledger=None, model=None):
    """v - Z A_H^{-1} Y^T (A v - mu v) at one level (reference solver.py:323-359)."""
    with hier.on_stream():
        return _apply_preconditioner(hier, level_idx, v)


def _apply_preconditioner(hier: LevelHierarchy, level_idx: int, v):
    if not 0 <= level_idx < hier.n_levels - 1:
        raise ValueError("level_idx must index a non-coarsest level")
    shape = tuple(v.shape) if hasattr(v, "shape") else np.shape(v)
    dv, was_np = _to_device(v)
    lvl, nxt = hier.levels[level_idx], hier.levels[level_idx + 1]
    if dv.numel() != lvl.total_dim:
        raise ValueError("vector size does not match the level")
    out = _empty(lvl.total_dim)
    child = _empty(_child_size(lvl, nxt))
    lib = _lib.load()
    _lib.check(lib.pmk_apply_preconditioner(hier._native, level_idx, _lib.ptr(dv),
                                            _lib.ptr(child), _lib.ptr(out), _lib.stream_ptr()),
               "apply_preconditioner")
    return out.cpu().numpy().reshape(shape) if was_np else out.reshape(shape)


def _state(hier, level_idx, want_arrays=False):
    lib = _lib.load()
    sc = (ctypes.c_double * 4)()
    cap = ctypes.c_int32(0)
    _lib.check(lib.pmk_fgmres_state(hier._native, level_idx, sc, None, None, None,
                                    ctypes.byref(cap), _lib.stream_ptr()), "state")
    out = {"beta": sc[0], "rel": sc[1], "n_iter": int(sc[2]), "breakdown": bool(sc[3]),
           "cap": cap.value}
    if want_arrays:
        c = cap.value
        hist = (ctypes.c_double * c)()
        hraw = (ctypes.c_double * ((c + 1) * c))()
        y = (ctypes.c_double * c)()
        _lib.check(lib.pmk_fgmres_state(hier._native, level_idx, sc, hist, hraw, y, None,
                                        _lib.stream_ptr()), "state")
        out["hist"] = np.frombuffer(hist, dtype=np.float64).copy()
        out["hraw"] = np.frombuffer(hraw, dtype=np.float64).copy().reshape(c + 1, c)
        out["y"] = np.frombuffer(y, dtype=np.float64).copy()
    return out


class _MemoryBudget:
    """Device bytes still available for Krylov vectors (one cudaMemGetInfo
    per fgmres call; per-iteration checks are host arithmetic only)."""

    def __init__(self):
        import torch

        free, _total = torch.cuda.mem_get_info()
        cached = torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
        self.left = free + cached - (512 << 20)

    def take(self, nbytes: int) -> None:
        self.left -= nbytes
        if self.left < 0:
            raise MemoryError(
                "FGMRES basis exceeds free device memory; set SolverConfig.restart to bound it")


def fgmres(hier: LevelHierarchy, level_idx: int, rhs, tol: float | None, max_iter: int,
           ledger=None, model=None, keep_basis: bool = False):
    """Right-preconditioned FGMRES, MGS + Givens, zero initial guess, no
    restarts (reference solver.py:362-456).  tol=None runs exactly max_iter
    iterations (inner solves) unless the basis breaks down."""
    with hier.on_stream():
        x, report = _fgmres(hier, level_idx, rhs, tol, max_iter, keep_basis)
    if not hasattr(rhs, "data_ptr"):  # numpy in -> numpy out, like the reference
        return x.cpu().numpy(), report
    return x, report


def _fgmres(hier: LevelHierarchy, level_idx: int, rhs, tol: float | None, max_iter: int,
            keep_basis: bool = False, copier=None):
    import torch

    if not 0 <= level_idx < hier.n_levels - 1:
        raise ValueError("fgmres runs on a non-coarsest level")
    lib = _lib.load()
    lvl, nxt = hier.levels[level_idx], hier.levels[level_idx + 1]
    b, _ = _to_device(rhs)
    b = b.reshape(-1)
    if b.numel() != lvl.total_dim:
        raise ValueError("rhs size does not match the level")
    report = SolveReport(method=f"fgmres[level {level_idx}]",
                         tol=tol if tol is not None else 0.0)
    s = _lib.stream_ptr()
    H = hier._native
    _lib.check(lib.pmk_fgmres_begin(H, level_idx, _lib.ptr(b), int(max_iter),
                                    float(tol) if tol is not None else 0.0, s), "fgmres_begin")
    st = _state(hier, level_idx)
    if st["beta"] == 0.0:
        return torch.zeros_like(b), report
    vs, cos = [], []
    csize = _child_size(lvl, nxt)
    per_iter = 8 * (lvl.total_dim + csize)
    budget = _MemoryBudget()
    budget.take(8 * lvl.total_dim)
    lazy = _lib.lazy_basis()
    # lazy basis (pmk_lazy_basis): vs[l] holds raw basis vector l -- the rhs,
    # then each step's w (a fresh buffer per step); otherwise the normalised
    # v_l, with one w buffer reused every iteration
    if lazy:
        vs.append(b)
    else:
        w = _empty(lvl.total_dim)
    # Stop test one step behind: step j is enqueued before the host looks at
    # the snapshot taken after step j-1 (pmk_fgmres_snapshot), so the GPU
    # never idles on the host round trip; once an iteration has converged the
    # device turns the already enqueued next step into no-ops.
    snaps = {}
    sc = (ctypes.c_double * 4)()
    for j in range(max_iter):
        budget.take(per_iter)
        co = _empty(csize)
        cos.append(co)
        if lazy:
            v = None
            w = _empty(lvl.total_dim)
        else:
            v = _empty(lvl.total_dim)
            vs.append(v)
        _lib.check(lib.pmk_fgmres_step(H, level_idx, j, _lib.ptr(v), _lib.ptr(w), _lib.ptr(co),
                                       s), "fgmres_step")
        if lazy:
            vs.append(w)
        if tol is not None:
            _lib.check(lib.pmk_fgmres_snapshot(H, level_idx, j % 4, s), "snapshot")
            ev = torch.cuda.Event()
            ev.record()
            snaps[j] = ev
            if j >= 1:
                snaps.pop(j - 1).synchronize()
                _lib.check(lib.pmk_fgmres_snapshot_read(H, level_idx, (j - 1) % 4, sc),
                           "snapshot_read")
                if sc[3] or sc[1] <= tol:  # breakdown / converged at step j-1
                    break
    x = _empty(lvl.total_dim)
    if copier is None:
        _lib.check(lib.pmk_fgmres_finish(H, level_idx, _lib.ptr(x), s), "fgmres_finish")
    else:  # assemble x in slabs of time slices, each copied out while the next is built
        for r0, r1 in _slabs(lvl.n_steps + 1, _nu_of(lvl), _RESULT_SLABS):
            _lib.check(lib.pmk_fgmres_finish_rows(H, level_idx, _lib.ptr(x), r0, r1, s),
                       "fgmres_finish_rows")
            copier.start(x, r0 * lvl.state_dim, r1 * lvl.state_dim)
        copier.src = x
    st = _state(hier, level_idx, want_arrays=True)
    n_iter = st["n_iter"]
    report.outer_iterations = n_iter
    report.residual_history = [float(r) for r in st["hist"][:n_iter]]
    if st["breakdown"] or (tol is not None and n_iter and report.residual_history[-1] <= tol):
        report.converged = True
    if keep_basis:
        if lazy:  # v_l = RN(raw_l * RN(1 / scale_l)), the values the kernels use
            scales = [st["beta"]] + [st["hraw"][l, l - 1] for l in range(1, n_iter)]
            vn = [vs[l].reshape(-1) * (1.0 / scales[l]) for l in range(n_iter)]
            last = vs[n_iter] if len(vs) > n_iter else None
        else:
            vn = vs[:n_iter]
            last = w
        basis = [vn[l].cpu().numpy() for l in range(n_iter)]
        if not st["breakdown"] and last is not None:
            basis.append(last.cpu().numpy() / st["hraw"][n_iter, n_iter - 1])  # IEEE division
        mg = isinstance(lvl.pair, MgritPair)  # cos already hold the interpolated vectors
        expand = getattr(lvl.pair, "expand_child", lvl.pair.interpolate)
        pre = [(vn[l] - (cos[l] if mg else expand(cos[l]))).cpu().numpy()
               for l in range(n_iter)]
        report.metadata["basis"] = basis
        report.metadata["preconditioned"] = pre
        report.metadata["hessenberg"] = st["hraw"][:n_iter + 1, :n_iter].copy()
    del vs, cos, w
    return x, report


_RESULT_SLABS = 8


def _nu_of(lvl) -> int:
    pair = lvl.pair
    return 1 if isinstance(pair, MgritPair) else int(getattr(pair, "nu", 1))


def _slabs(rows: int, nu: int, n: int):
    """[r0, r1) ranges covering rows, every r0 a multiple of nu."""
    step = max(nu, ((rows + n - 1) // n + nu - 1) // nu * nu)
    return [(r0, min(rows, r0 + step)) for r0 in range(0, rows, step)]


class _ResultCopy:
    """Device -> host copy of the solution on a side stream, started as soon
    as a candidate x exists, so that it overlaps the true-residual check
    (stepper.py:191-193) that follows; a further restart cycle first waits
    for the copy to finish reading x."""

    def __init__(self, out):
        import torch

        self.out = out
        self.stream = _copy_stream(torch.cuda.current_device())
        self.src = None

    def start(self, x, lo: int = 0, hi: int | None = None):
        """Copy x[lo:hi] (all of x by default) once the current stream has
        produced it."""
        import torch

        self.stream.wait_stream(torch.cuda.current_stream())
        xf, of = x.reshape(-1), self.out.reshape(-1)
        hi = xf.numel() if hi is None else hi
        with torch.cuda.stream(self.stream):
            of[lo:hi].copy_(xf[lo:hi], non_blocking=True)
        self.src = x

    def fence(self):
        """x is about to change on the current stream."""
        import torch

        if self.src is not None:
            torch.cuda.current_stream().wait_stream(self.stream)
            self.src = None

    def done(self, x) -> bool:
        """Wait for the copy; True when it holds x."""
        self.stream.synchronize()
        return self.src is x


_COPY_STREAMS: dict = {}


def _copy_stream(device: int):
    import torch

    st = _COPY_STREAMS.get(device)
    if st is None:
        st = _COPY_STREAMS[device] = torch.cuda.Stream(device=device)
    return st


def _restarted_fgmres(hier: LevelHierarchy, tol: float, max_outer: int, restart: int,
                      copier: _ResultCopy | None = None):
    """FGMRES(m): cycles of the reference fgmres on the current residual
    (SURVEY.md section 8(c) restart oracle)."""
    import torch

    fine = hier.fine
    lib = _lib.load()
    b = fine.rhs.reshape(-1)
    beta0 = _nrm2(b)
    rn_dev = _empty(1)
    x = None          # x = 0 until the first cycle returns
    r = b
    rn = beta0
    hist: list[float] = []
    total = 0
    cycles = 0
    converged = False
    final_rel = None
    while total < max_outer:
        if rn == 0.0:
            converged = True
            final_rel = 0.0
            break
        m = min(restart, max_outer - total)
        first = x is None
        dx, rep = _fgmres(hier, 0, r, tol=tol * beta0 / rn, max_iter=m,
                          copier=copier if first else None)
        if first:
            x = dx  # (copied out slab by slab as it was assembled)
        else:
            if copier is not None:
                copier.fence()
            _lib.check(lib.pmk_axpy(1.0, _lib.ptr(dx), _lib.ptr(x), x.numel(),
                                    _lib.stream_ptr()), "axpy")     # x = x + dx
            if copier is not None:
                copier.start(x)
        del dx
        total += rep.outer_iterations
        cycles += 1
        hist += [h * rn / beta0 for h in rep.residual_history]
        if r is b:
            r = _empty(b.numel())
        _lib.check(lib.pmk_residual(ctypes.byref(fine.level_desc()), _lib.ptr(x), _lib.ptr(b),
                                    _lib.ptr(r), _lib.ptr(rn_dev), _lib.stream_ptr()),
                   "residual")          # r = b - A x, ||r||
        rn = float(rn_dev.item())
        final_rel = rn / beta0     # ||b - A x|| / ||b|| (stepper.py:191-193)
        if final_rel <= tol:
            converged = True
            break
        if rep.outer_iterations == 0:
            break
    if x is None:
        x = torch.zeros_like(b)
    report = SolveReport(method="fgmres[level 0]", tol=tol)
    report.outer_iterations = total
    report.residual_history = hist
    report.converged = converged
    report.metadata["restart_cycles"] = cycles
    if final_rel is not None:
        report.metadata["final_relative_residual"] = final_rel
    return x, report


def _nrm2(t) -> float:
    import torch

    lib = _lib.load()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.check(lib.pmk_nrm2(_lib.ptr(t), t.numel(), _lib.ptr(out), _lib.stream_ptr()), "nrm2")
    return float(out.item())


def _solve(hier: LevelHierarchy, ledger, model, method_name: str, output: str | None = None,
           out=None):
    import torch

    cfg = hier.config
    rhs = hier.fine.rhs.reshape(-1)
    torch.cuda.synchronize()
    if ledger is not None:  # real-time phase ledger (ledger.py): every launch timed
        _lib.profile_begin(True)
    if output is None:
        output = "host" if hier.fine.host_io else "device"
    if out is None and output == "host":
        # pinned (torch's caching host allocator): a fast D2H that can overlap
        out = torch.empty(hier.fine.rhs.numel(), dtype=torch.float64, pin_memory=True)
        host_out = True
    else:
        host_out = False
    copier = _ResultCopy(out) if out is not None and out.device.type == "cpu" else None
    t0 = time.perf_counter()
    try:
        with hier.on_stream():
            if cfg.restart is None:
                x, report = _fgmres(hier, 0, rhs, tol=cfg.tol, max_iter=cfg.max_outer,
                                    copier=copier)
            else:
                x, report = _restarted_fgmres(hier, cfg.tol, cfg.max_outer, cfg.restart,
                                              copier)
        torch.cuda.current_stream().synchronize()  # (not the result copy's stream)
        report.method = method_name
        report.wall_time = time.perf_counter() - t0
        report.tol = cfg.tol
        true_res = report.metadata.pop("final_relative_residual", None)
        if true_res is None:
            true_res = hier.fine.relative_residual(x)
    finally:
        records = _lib.profile_end_levels() if ledger is not None else None
    if ledger is not None:
        from .ledger import charge_records, phase_of

        charge_records(ledger, records)
        report.simulated_elapsed = ledger.elapsed  # measured GPU microseconds
        phase_ms: dict = {}
        for r in records:
            ph = "coarse_solve" if r["level"] >= 1 else phase_of(r)
            phase_ms[ph] = phase_ms.get(ph, 0.0) + r["ms"]
        report.metadata["gpu_phase_ms"] = phase_ms
    report.metadata["true_relative_residual"] = true_res
    report.converged = true_res <= cfg.tol
    report.level_stats = {"levels": hier.describe(), "moves": hier.moves}
    if out is not None:
        if copier is None or not copier.done(x):
            out.copy_(x.reshape(out.shape))  # e.g. into a pinned host buffer
        if host_out:
            return out.numpy(), report
        return out, report
    return x, report


def two_level_solve(hier: LevelHierarchy, ledger=None, model=None, output: str | None = None,
                    out=None):
    if hier.n_levels != 2:
        raise ValueError("two_level_solve expects a 2-level hierarchy")
    return _solve(hier, ledger, model, "two_level", output, out)


def multilevel_solve(hier: LevelHierarchy, ledger=None, model=None, output: str | None = None,
                     out=None):
    """Outer FGMRES to cfg.tol (reference solver.py:459-488).  Returns x as
    numpy when the fine system was built from a numpy u0, else as a device
    tensor (``output`` = "host" / "device" overrides; ``out`` = a tensor,
    e.g. pinned host memory, that receives x)."""
    return _solve(hier, ledger, model, f"multilevel[{hier.n_levels}]", output, out)
