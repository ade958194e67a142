"""CPU oracle for the MLK space-time solve -- TEST INFRASTRUCTURE ONLY.

A restatement, in plain numpy/scipy, of the reference package `pintmk`
(arXiv 2401.00228) along the hot path solver.multilevel_solve -> fgmres ->
apply_preconditioner -> {matvec, restrict, forward_solve, interpolate}.
Every function cites the reference file:line it follows (paths relative to
/root/reference/pkg/src/pintmk/).  It performs the same floating-point
operations in the same order as the reference, so on this image's
numpy 2.3 / scipy 1.18 it reproduces the reference bitwise; that is checked
against the live reference and the committed golden fixtures by
tests/test_oracle.py (the oracle is "pinned").

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module, and only as the checker.  The product package
(paper_2401_00228_b200) never imports it and has no CPU fallback.

Extensions (not in the reference): `restarted_solve` = FGMRES(m) built from
the reference's own fgmres cycles; and the
"space_fw" / "time_space_fw" moves (`make_fw_pair`, `_space_rung_fw`):
full-weighting restriction, (bi)linear interpolation and a rediscretised
coarse Laplacian, the transfers BASELINE config 4 names and the reference
does not have.  PARITY UNPINNED for that extension: there is no reference
output to pin it to; everything around it (matvec, fgmres, coarsest solve)
is the pinned code above.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from scipy.linalg import solve_banded

# ---------------------------------------------------------------- operators


def laplacian(dim: int, nx: int, ny: int = 1, tau: float = 1.0, length: float = 1.0):
    """spatial.py:37-72.  Returns (A, dx)."""
    dx = length / (nx + 1)
    c = tau / dx**2
    d1 = sp.diags([np.ones(nx - 1), -2.0 * np.ones(nx), np.ones(nx - 1)], offsets=[-1, 0, 1],
                  format="csr")
    if dim == 1:
        return (c * d1).tocsr(), dx
    d2 = sp.diags([np.ones(ny - 1), -2.0 * np.ones(ny), np.ones(ny - 1)], offsets=[-1, 0, 1],
                  format="csr")
    a = c * (sp.kron(sp.identity(ny), d1) + sp.kron(d2, sp.identity(nx)))
    return a.tocsr(), dx


def bump(dim: int, nx: int, ny: int, dx: float) -> np.ndarray:
    """spatial.py:106-114."""
    gx = np.sin(np.pi * (np.arange(1, nx + 1) * dx) / (dx * (nx + 1)))
    if dim == 1:
        return gx
    gy = np.sin(np.pi * (np.arange(1, ny + 1) * dx) / (dx * (ny + 1)))
    return np.outer(gy, gx).ravel()


def blocks_from(a: sp.csr_matrix, weight: float, dt: float):
    """(D, B) = (I - w dt A, I + (1-w) dt A): stepper.py:56-63 / solver.py:105-110."""
    eye = sp.identity(a.shape[0], format="csr")
    return (eye - weight * dt * a).tocsr(), (eye + (1.0 - weight) * dt * a).tocsr()


def is_tridiagonal(m: sp.spmatrix) -> bool:
    """linalg.py:30-32."""
    c = m.tocoo()
    return bool(np.all(np.abs(c.row - c.col) <= 1))


def tridiag_bands(m: sp.spmatrix):
    """linalg.py:17-27: (lower, diag, upper) with lower[i] = M[i, i-1]."""
    c = m.tocoo()
    n = m.shape[0]
    bands = {-1: np.zeros(n), 0: np.zeros(n), 1: np.zeros(n)}
    off = c.col - c.row
    for k, dest in bands.items():
        sel = off == k
        dest[c.row[sel]] = c.data[sel]
    return bands[-1], bands[0], bands[1]


class DiagSolver:
    """One factorisation of D reused for all slices (linalg.py:35-68):
    banded LAPACK for tridiagonal D, SuperLU otherwise."""

    def __init__(self, d: sp.csr_matrix):
        n = d.shape[0]
        self.tri = is_tridiagonal(d)
        if self.tri:
            lo, di, up = tridiag_bands(d)
            self.ab = np.zeros((3, n))
            self.ab[0, 1:] = up[:-1]
            self.ab[1, :] = di
            self.ab[2, :-1] = lo[1:]
        else:
            self.lu = spla.splu(d.tocsc())

    def __call__(self, rhs):
        if self.tri:
            return solve_banded((1, 1), self.ab, rhs, check_finite=False)
        return self.lu.solve(rhs)


@dataclass(eq=False)
class System:
    """Block lower-bidiagonal system [I; -B, D; ...] (stepper.py:66-91)."""

    diag: sp.csr_matrix
    sub: sp.csr_matrix
    n_steps: int
    dropped: tuple = ()
    _solver: DiagSolver | None = None

    @property
    def n(self) -> int:
        return self.diag.shape[0]

    @property
    def size(self) -> int:
        return (self.n_steps + 1) * self.n

    def solver(self) -> DiagSolver:
        if self._solver is None:
            self._solver = DiagSolver(self.diag)
        return self._solver


def matvec(s: System, v: np.ndarray) -> np.ndarray:
    """stepper.py:96-105 (right products, i.e. D^T and B^T)."""
    blk = np.ascontiguousarray(v).reshape(s.n_steps + 1, s.n)
    out = np.empty_like(blk)
    out[0] = blk[0]
    out[1:] = blk[1:] @ s.diag - blk[:-1] @ s.sub
    for k in s.dropped:
        out[k] += blk[k - 1] @ s.sub
    return out.reshape(np.shape(v))


def segments(s: System):
    """stepper.py:107-112."""
    cuts = [c for c in s.dropped if c > 1]
    return list(zip([1] + cuts, cuts + [s.n_steps + 1]))


def _march(ab, bl, bd, bu, u0, f, steps):
    """Chain u_k = D^{-1}(B u_{k-1} + f_k) (_chain_py.py:16-27, the
    reference's fallback backend, bitwise equal to _chain.pyx:37-82)."""
    out = np.empty((steps + 1, u0.shape[0]))
    out[0] = u0
    for k in range(steps):
        r = bd * out[k]
        r[1:] += bl[1:] * out[k, :-1]
        r[:-1] += bu[:-1] * out[k, 1:]
        if f is not None:
            r += f[k]
        out[k + 1] = solve_banded((1, 1), ab, r, check_finite=False)
    return out


def forward_solve(s: System, rhs: np.ndarray) -> np.ndarray:
    """Block forward substitution honouring dropped couplings
    (stepper.py:114-146)."""
    blk = np.ascontiguousarray(rhs).reshape(s.n_steps + 1, s.n)
    out = np.empty_like(blk)
    out[0] = blk[0]
    solve = s.solver()
    cut = set(s.dropped)
    if solve.tri:
        bl, bd, bu = tridiag_bands(s.sub)
        for a, b in segments(s):
            start = a
            if a in cut:
                out[a] = solve(blk[a])
                start = a + 1
            if b - start > 0:
                traj = _march(solve.ab, bl, bd, bu, np.ascontiguousarray(out[start - 1]),
                              np.ascontiguousarray(blk[start:b]), b - start)
                out[start:b] = traj[1:]
    else:
        for k in range(1, s.n_steps + 1):
            r = blk[k].copy()
            if k not in cut:
                r += out[k - 1] @ s.sub
            out[k] = solve(r)
    return out.reshape(np.shape(rhs))


def sequential(diag, sub, u0, n_t) -> np.ndarray:
    """theta-scheme march (stepper.py:201-225), the convergence oracle."""
    s = System(diag, sub, n_t)
    rhs = np.zeros((n_t + 1, diag.shape[0]))
    rhs[0] = u0
    return forward_solve(s, rhs)


# ---------------------------------------------------------------- intergrid


def agglomerate(nx: int, ny: int = 1):
    """intergrid.py:202-227."""
    def cuts(cnt):
        half = cnt // 2
        if half == 0:
            raise ValueError("grid too small to agglomerate")
        e = [[2 * i, 2 * i + 2] for i in range(half)]
        e[-1][1] = cnt
        return e

    ex = cuts(nx)
    if ny == 1:
        return [np.arange(a, b) for a, b in ex], (len(ex), 1)
    ey = cuts(ny)
    groups = [np.array([y * nx + x for y in range(ya, yb) for x in range(xa, xb)])
              for ya, yb in ey for xa, xb in ex]
    return groups, (len(ex), len(ey))


@dataclass(eq=False)
class Pair:
    """TimePair (intergrid.py:37-63) when groups is None, TimeSpacePair
    (intergrid.py:79-120) with groups, MgritPair (intergrid.py:134-167) when
    `phi` is set (coarse-point injection, ideal interpolation)."""

    nu: int
    n_T: int
    n: int
    groups: list | None = None
    y: sp.csr_matrix | None = None
    z: sp.csr_matrix | None = None
    phi: sp.csr_matrix | None = None     # MGRIT: fine phi
    psi_solve: object | None = None      # MGRIT: fine psi factorisation

    @property
    def m(self) -> int:
        if self.groups is None:
            return self.n if self.y is None else self.y.shape[1]
        return len(self.groups)


def make_ts_pair(nu, n_T, groups, n) -> Pair:
    sizes = np.array([len(g) for g in groups])
    rows = np.concatenate(groups)
    cols = np.repeat(np.arange(len(groups)), sizes)
    z = sp.csr_matrix((np.ones(n), (rows, cols)), shape=(n, len(groups)))
    y = sp.csr_matrix((np.repeat(1.0 / sizes, sizes), (rows, cols)), shape=(n, len(groups)))
    return Pair(nu, n_T, n, groups, y, z)


def fw_1d(count: int):
    """EXTENSION (no reference counterpart): 1-D full weighting R (n_c x n,
    rows 1/4 1/2 1/4 centred on fine point 2 c + 1) and linear interpolation
    P = 2 R^T between n and n_c = (n - 1) / 2 interior points."""
    if count < 3 or count % 2 == 0:
        raise ValueError("full weighting needs an odd number (>= 3) of interior points")
    nc = (count - 1) // 2
    r = sp.lil_matrix((nc, count))
    for c in range(nc):
        r[c, 2 * c], r[c, 2 * c + 1], r[c, 2 * c + 2] = 0.25, 0.5, 0.25
    r = r.tocsr()
    return r, (2.0 * r.T).tocsr()


def make_fw_pair(nu, n_T, nx, ny, dim) -> Pair:
    """EXTENSION: full-weighting / (bi)linear pair; y (n x m) restricts as
    `summed @ y`, z (n x m) interpolates as `w @ z.T`, like make_ts_pair."""
    rx, px = fw_1d(nx)
    if dim == 2:
        ry, py = fw_1d(ny)
        r, pz = sp.kron(ry, rx, format="csr"), sp.kron(py, px, format="csr")
    else:
        r, pz = rx, px
    return Pair(nu, n_T, nx * (ny if dim == 2 else 1), None, sp.csr_matrix(r.T),
                sp.csr_matrix(pz))


def restrict(p: Pair, v: np.ndarray) -> np.ndarray:
    """intergrid.py:51-56 / 106-112 / 152-155 (MGRIT injection)."""
    blk = np.ascontiguousarray(v).reshape(p.nu * p.n_T + 1, -1)
    if p.phi is not None:
        out = blk[::p.nu].copy()
        return out.reshape(-1) if v.ndim == 1 else out
    summed = blk[1:].reshape(p.n_T, p.nu, p.n).sum(axis=1)
    out = np.empty((p.n_T + 1, p.m))
    if p.y is None:
        out[0] = blk[0]
        out[1:] = summed
    else:
        out[0] = blk[0] @ p.y
        out[1:] = summed @ p.y
    return out.reshape(-1) if v.ndim == 1 else out


def interpolate(p: Pair, w: np.ndarray) -> np.ndarray:
    """intergrid.py:58-63 / 114-120 / 157-167 (MGRIT: propagate each coarse
    row through the nu - 1 fine steps with zero forcing)."""
    blk = np.ascontiguousarray(w).reshape(p.n_T + 1, -1)
    if p.phi is not None:
        out = np.zeros((p.nu * p.n_T + 1, p.n))
        out[::p.nu] = blk
        cur = blk[:-1]
        for j in range(1, p.nu):
            cur = np.ascontiguousarray(p.psi_solve((cur @ p.phi).T).T)
            out[j::p.nu] = cur
        return out.reshape(-1) if w.ndim == 1 else out
    if p.z is not None:
        blk = blk @ p.z.T
    out = np.empty((p.nu * p.n_T + 1, p.n))
    out[0] = blk[0]
    out[1:] = np.repeat(blk[1:], p.nu, axis=0)
    return out.reshape(-1) if w.ndim == 1 else out


def decouple(n_steps: int, n_cgs: int) -> tuple:
    """Dropped rows of perturb_decouple (intergrid.py:299-311)."""
    if not 1 <= n_cgs <= n_steps + 1:
        raise ValueError(f"n_cgs must be in [1, {n_steps + 1}]")
    parts = np.array_split(np.arange(1, n_steps + 1), min(n_cgs, n_steps))
    return tuple(int(c[0]) for c in parts if len(c))


# ---------------------------------------------------------------- hierarchy


@dataclass(eq=False)
class Rung:
    """Level (solver.py:60-81)."""

    system: System
    a: sp.csr_matrix
    dt: float
    weight: float
    n_steps: int
    grid: tuple
    dim: int
    kind: str
    pair: Pair | None = None
    budget: int = 0


@dataclass
class Config:
    """SolverConfig (solver.py:37-57) plus `restart`."""

    mu: float = 1.0
    tol: float = 1e-6
    max_outer: int = 200
    inner_iters: object = None
    coarsest_n_cgs: int = 0
    restart: int | None = None


@dataclass(eq=False)
class Hierarchy:
    rungs: list
    rhs: np.ndarray
    fine: System
    cfg: Config
    moves: list = field(default_factory=list)


def _time_rung(r: Rung, nu: int) -> Rung:
    """solver.py:113-124."""
    if r.n_steps % nu:
        raise ValueError(f"time move needs nu | n_steps, got {r.n_steps} / {nu}")
    r.pair = Pair(nu, r.n_steps // nu, r.a.shape[0])
    w = 1.0 - (1.0 - r.weight) / nu
    dt = nu * r.dt
    d, b = blocks_from(r.a, w, dt)
    return Rung(System(d, b, r.n_steps // nu), r.a, dt, w, r.n_steps // nu, r.grid, r.dim,
                "time")


def _space_rung(r: Rung, time_nu: int = 1) -> Rung:
    """solver.py:127-143."""
    gx, gy = r.grid
    groups, (mx, my) = agglomerate(gx, gy if r.dim == 2 else 1)
    if r.n_steps % time_nu:
        raise ValueError("time factor must divide n_steps")
    nT = r.n_steps // time_nu
    r.pair = make_ts_pair(time_nu, nT, groups, r.a.shape[0])
    ac = (r.pair.y.T @ r.a @ r.pair.z).tocsr()
    w = 1.0 - (1.0 - r.weight) / time_nu
    dt = time_nu * r.dt
    d, b = blocks_from(ac, w, dt)
    return Rung(System(d, b, nT), ac, dt, w, nT, (mx, my), r.dim,
                "space" if time_nu == 1 else "time_space")


def _space_rung_fw(r: Rung, time_nu: int = 1) -> Rung:
    """EXTENSION (no reference counterpart): full-weighting space move onto
    the grid with doubled spacing, coarse operator = the Laplacian
    rediscretised there: (factor / 4) * unit second differences, factor =
    tau / dx^2 of this rung (read off its pristine matrix)."""
    gx, gy = r.grid
    if r.n_steps % time_nu:
        raise ValueError("time factor must divide n_steps")
    nT = r.n_steps // time_nu
    r.pair = make_fw_pair(time_nu, nT, gx, gy, r.dim)
    mx, my = (gx - 1) // 2, ((gy - 1) // 2 if r.dim == 2 else 1)
    factor = float(r.a[0, 1]) / 4.0
    unit, _ = laplacian(r.dim, mx, my, 1.0, float(mx + 1))
    if r.dim == 2 and my != mx:
        raise ValueError("oracle fw move: square grids only")
    ac = (factor * unit).tocsr()
    w = 1.0 - (1.0 - r.weight) / time_nu
    dt = time_nu * r.dt
    d, b = blocks_from(ac, w, dt)
    return Rung(System(d, b, nT), ac, dt, w, nT, (mx, my), r.dim,
                "space_fw" if time_nu == 1 else "time_space_fw")


def _stable(r: Rung, nu: int) -> bool:
    """solver.py:154-163."""
    expl = (1.0 - r.weight) / nu
    lam = float(np.abs(r.a).sum(axis=1).max()) / r.dim
    return (1.0 - 2.0 * expl) * (nu * r.dt) * lam <= 2.0


def budgets_for(n_inter: int, inner_iters) -> list:
    """solver.py:219-235."""
    if n_inter == 0:
        return []
    if inner_iters is None:
        out = [2] * n_inter
        if n_inter > 1:
            out[-1] = 1
        return out
    if isinstance(inner_iters, int):
        return [inner_iters] * n_inter
    out = list(inner_iters)
    if len(out) != n_inter:
        raise ValueError("need one inner budget per intermediate level")
    return out


def build_mgrit(dim, nx, ny, theta, dt, n_t, u0, cfg: Config, nu=2, tau=1.0,
                length=1.0) -> Hierarchy:
    """build_two_level(fine, "MGRIT", nu, cfg) (solver.py:248-265): MgritPair
    (intergrid.py:134-167) + rediscretized coarse system (intergrid.py:270-280)."""
    a, _dx = laplacian(dim, nx, ny, tau, length)
    d, b = blocks_from(a, theta, dt)
    fine = System(d, b, n_t)
    rhs = np.zeros((n_t + 1, a.shape[0]))
    rhs[0] = u0
    if n_t % nu:
        raise ValueError("nu must divide n_t")
    n_T = n_t // nu
    top = Rung(fine, a, dt, theta, n_t, (nx, ny if dim == 2 else 1), dim, "fine")
    top.pair = Pair(nu, n_T, a.shape[0], phi=b, psi_solve=fine.solver())
    dc, bc = blocks_from(a, theta, nu * dt)
    coarse = Rung(System(dc, bc, n_T), a, nu * dt, theta, n_T, top.grid, dim, "mgrit")
    if cfg.coarsest_n_cgs >= 1:
        coarse.system = System(dc, bc, n_T, decouple(n_T, cfg.coarsest_n_cgs))
    return Hierarchy([top, coarse], rhs, fine, cfg, ["MGRIT"])


def build(dim, nx, ny, theta, dt, n_t, u0, n_levels, schedule, cfg: Config, nu=2,
          tau=1.0, length=1.0, forcing=None, a=None) -> Hierarchy:
    """FineSystem (stepper.py:168-185) + build_hierarchy (solver.py:178-216).
    `a`: a caller's spatial matrix instead of build_laplacian's (the
    reference accepts any SpatialOperator, spatial.py:17-34)."""
    if a is None:
        a, _dx = laplacian(dim, nx, ny, tau, length)
    d, b = blocks_from(a, theta, dt)
    fine = System(d, b, n_t)
    rhs = np.zeros((n_t + 1, a.shape[0]))
    rhs[0] = u0
    if forcing is not None:
        rhs[1:] = dt * forcing
    rungs = [Rung(fine, a, dt, theta, n_t, (nx, ny if dim == 2 else 1), dim, "fine")]
    moves = []
    alternating, next_space = False, False
    for i in range(n_levels - 1):
        cur = rungs[-1]
        if schedule == "auto":
            if not alternating and cur.n_steps % nu == 0 and _stable(cur, nu):
                move = "time"
            else:
                if not alternating:
                    alternating, next_space = True, True
                move = "space" if next_space else "time"
                next_space = not next_space
        else:
            move = schedule[i]
        if move == "time":
            rungs.append(_time_rung(cur, nu))
        elif move == "space":
            rungs.append(_space_rung(cur))
        elif move == "time_space":
            rungs.append(_space_rung(cur, nu))
        elif move == "space_fw":
            rungs.append(_space_rung_fw(cur))
        elif move == "time_space_fw":
            rungs.append(_space_rung_fw(cur, nu))
        else:
            raise ValueError(f"unknown move {move!r}")
        moves.append(move)
    for r, bgt in zip(rungs[1:-1], budgets_for(len(rungs) - 2, cfg.inner_iters)):
        if bgt < 1:
            raise ValueError("budgets must be >= 1")
        r.budget = bgt
    if cfg.coarsest_n_cgs >= 1:
        c = rungs[-1].system
        rungs[-1].system = System(c.diag, c.sub, c.n_steps,
                                  decouple(c.n_steps, cfg.coarsest_n_cgs))
    return Hierarchy(rungs, rhs, fine, cfg, moves)


# ---------------------------------------------------------------- solve


def precondition(h: Hierarchy, lvl: int, v: np.ndarray) -> np.ndarray:
    """apply_preconditioner, solver.py:323-359."""
    cur, nxt = h.rungs[lvl], h.rungs[lvl + 1]
    s = matvec(cur.system, v)
    s -= h.cfg.mu * v
    vh = restrict(cur.pair, s)
    if lvl + 2 == len(h.rungs):
        vt = forward_solve(nxt.system, vh)
    else:
        vt, _ = fgmres(h, lvl + 1, vh, None, nxt.budget)
    return v - interpolate(cur.pair, vt)


def fgmres(h: Hierarchy, lvl: int, rhs: np.ndarray, tol, max_iter: int, keep_basis=False):
    """Right-preconditioned FGMRES, MGS + progressive Givens, zero initial
    guess, no restart (solver.py:362-456).  Returns (x, info dict)."""
    sysl = h.rungs[lvl].system
    b = np.asarray(rhs, dtype=np.float64).ravel()
    info = {"iterations": 0, "history": [], "converged": False, "breakdown": False}
    beta = float(np.linalg.norm(b))
    if beta == 0.0:
        return np.zeros_like(b), info
    V = [b / beta]
    X = []
    H = np.zeros((max_iter + 1, max_iter))
    Hraw = np.zeros_like(H)
    cs = np.zeros(max_iter)
    sn = np.zeros(max_iter)
    g = np.zeros(max_iter + 1)
    g[0] = beta
    n_iter = 0
    for j in range(max_iter):
        xj = precondition(h, lvl, V[j])
        X.append(np.array(xj, copy=True))
        w = matvec(sysl, xj)
        for i in range(j + 1):
            H[i, j] = float(np.dot(w, V[i]))
            w -= H[i, j] * V[i]
        H[j + 1, j] = float(np.linalg.norm(w))
        Hraw[:, j] = H[:, j]
        n_iter = j + 1
        cnorm = float(np.linalg.norm(H[:j + 2, j]))
        broke = H[j + 1, j] <= 1e-14 * max(cnorm, 1e-300)
        if not broke:
            V.append(w / H[j + 1, j])
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        r = math.hypot(H[j, j], H[j + 1, j])
        cs[j] = H[j, j] / r
        sn[j] = H[j + 1, j] / r
        H[j, j] = r
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        rel = abs(g[j + 1]) / beta
        info["history"].append(rel)
        if broke:
            info["converged"] = True
            info["breakdown"] = True
            break
        if tol is not None and rel <= tol:
            info["converged"] = True
            break
    info["iterations"] = n_iter
    y = np.zeros(n_iter)
    for i in range(n_iter - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1:n_iter] @ y[i + 1:n_iter]) / H[i, i]
    x = np.zeros(b.shape[0])
    for i in range(n_iter):
        x += y[i] * X[i]
    if keep_basis:
        info["basis"] = [np.array(v) for v in V[:n_iter if info["breakdown"] else n_iter + 1]]
        info["preconditioned"] = X
        info["hessenberg"] = Hraw[:n_iter + 1, :n_iter].copy()
    return x, info


def relative_residual(h: Hierarchy, x: np.ndarray) -> float:
    """stepper.py:191-193."""
    r = h.rhs - matvec(h.fine, x).reshape(h.rhs.shape)
    return float(np.linalg.norm(r.ravel()) / np.linalg.norm(h.rhs.ravel()))


def solve(h: Hierarchy):
    """multilevel_solve -> _solve (solver.py:459-488)."""
    t0 = time.perf_counter()
    if h.cfg.restart is None:
        x, info = fgmres(h, 0, h.rhs.ravel(), h.cfg.tol, h.cfg.max_outer)
    else:
        x, info = restarted_solve(h)
    info["wall_time"] = time.perf_counter() - t0
    info["true_relative_residual"] = relative_residual(h, x)
    info["converged"] = info["true_relative_residual"] <= h.cfg.tol
    return x, info


def restarted_solve(h: Hierarchy):
    """FGMRES(m): cycles of fgmres on the current residual with the tolerance
    rescaled to the initial residual; stops when the TRUE residual reaches
    tol or after max_outer iterations in total (new knob)."""
    cfg = h.cfg
    b = h.rhs.ravel()
    beta0 = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    r = b.copy()
    hist, total, cycles, conv = [], 0, 0, False
    while total < cfg.max_outer:
        rn = float(np.linalg.norm(r))
        if rn == 0.0:
            conv = True
            break
        m = min(cfg.restart, cfg.max_outer - total)
        dx, inf = fgmres(h, 0, r, cfg.tol * beta0 / rn, m)
        x = x + dx
        total += inf["iterations"]
        cycles += 1
        hist += [v * rn / beta0 for v in inf["history"]]
        r = b - matvec(h.fine, x)
        if float(np.linalg.norm(r)) / beta0 <= cfg.tol:
            conv = True
            break
        if inf["iterations"] == 0:
            break
    return x, {"iterations": total, "history": hist, "converged": conv, "breakdown": False,
               "restart_cycles": cycles}
