"""theta-scheme operators and the all-at-once block-bidiagonal system, on the GPU.

Mirror of reference ``pintmk/stepper.py``.  The step operators phi/psi are
assembled on the host exactly like the reference's (setup); everything that
touches a space-time vector -- matvec, forward substitution, the residual --
runs in the sm_100a kernels of libpmk_b200.so.

Space-time vectors are CUDA float64 tensors laid out (n_steps+1, n) row-major
(flat views accepted), the reference's layout (stepper.py:93-94).  numpy
inputs are accepted too and give numpy outputs (host<->device copies
included), so code written against the reference keeps working.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib
from ._device import CoarseSolver, SpectralInfo, StencilTable, dropped_mask
from .spatial import SpatialOperator, laplacian_stencil, stencil_csr


@dataclass
class ThetaSchemeConfig:
    """theta, step size and step count (reference stepper.py:20-38)."""

    theta: float
    delta_t: float
    n_t: int

    def __post_init__(self):
        if not 0.0 <= self.theta <= 1.0:
            raise ValueError("theta must lie in [0, 1]")
        if self.delta_t <= 0:
            raise ValueError("delta_t must be positive")
        if self.n_t < 1:
            raise ValueError("n_t must be at least 1")

    @property
    def final_time(self) -> float:
        return self.n_t * self.delta_t


class _LazyDiagSolve:
    """psi^{-1} applied slice-wise on the device (the reference prefactors psi
    with LAPACK/SuperLU, linalg.py:35-68)."""

    def __init__(self, ops: "StepOperators"):
        self._ops = ops
        self._sys = None

    def solve(self, rhs):
        """Solve psi x = rhs for one vector or a (k, n) block of row vectors."""
        if self._sys is None:
            o = self._ops
            self._sys = BlockBidiagonalSystem(o.psi, o.phi, 0, grid=o.spatial.grid,
                                              dim=o.spatial.dim, spectral=o.spectral_info)
        return self._sys.diag_solve(rhs)


@dataclass(eq=False)
class StepOperators:
    """psi u_k = phi u_{k-1} + dt g_k (reference stepper.py:41-53)."""

    phi: sp.csr_matrix
    psi: sp.csr_matrix
    psi_factorization: object
    spatial: SpatialOperator
    config: ThetaSchemeConfig
    _spectral: object = field(default=None, init=False, repr=False)
    _spectral_known: bool = field(default=False, init=False, repr=False)

    @property
    def n(self) -> int:
        return self.phi.shape[0]

    @property
    def spectral_info(self) -> SpectralInfo | None:
        """SpectralInfo when psi/phi are the theta-scheme blocks of
        build_laplacian's operator (the device then takes closed-form stencils
        and the sine-basis coarse solve), else None: the kernels read the
        actual matrices (checked once, O(nnz) compares)."""
        if not self._spectral_known:
            spec = None
            op, cfg = self.spatial, self.config
            if _is_pristine(op):
                cand = SpectralInfo(op.tau / op.delta_x**2, cfg.theta * cfg.delta_t,
                                    (1.0 - cfg.theta) * cfg.delta_t)
                d, b = cand.stencils(op.dim)
                if _csr_equal(self.psi, stencil_csr(op.n_x, op.n_y, d)) and \
                        _csr_equal(self.phi, stencil_csr(op.n_x, op.n_y, b)):
                    spec = cand
            self._spectral = spec
            self._spectral_known = True
        return self._spectral


def _csr_equal(a, b) -> bool:
    a = sp.csr_matrix(a)
    a.sort_indices()
    return (a.shape == b.shape and a.nnz == b.nnz and np.array_equal(a.indptr, b.indptr)
            and np.array_equal(a.indices, b.indices) and np.array_equal(a.data, b.data))


def build_step_operators(op: SpatialOperator, cfg: ThetaSchemeConfig) -> StepOperators:
    """phi = I + (1-theta) dt A, psi = I - theta dt A (reference stepper.py:56-63)."""
    spec = None
    if _is_pristine(op):
        # closed form, entry for entry scipy's eye -/+ s * A
        # (tests/test_host.py::test_direct_csr_assembly_bitwise)
        spec = SpectralInfo(op.tau / op.delta_x**2, cfg.theta * cfg.delta_t,
                            (1.0 - cfg.theta) * cfg.delta_t)
        d, b = spec.stencils(op.dim)
        psi = stencil_csr(op.n_x, op.n_y, d)
        phi = stencil_csr(op.n_x, op.n_y, b)
    else:
        eye = sp.identity(op.n, format="csr")
        phi = (eye + (1.0 - cfg.theta) * cfg.delta_t * op.matrix).tocsr()
        psi = (eye - cfg.theta * cfg.delta_t * op.matrix).tocsr()
    ops = StepOperators(phi=phi, psi=psi, psi_factorization=None, spatial=op, config=cfg)
    ops._spectral = spec   # (known: built right here)
    ops._spectral_known = True
    ops.psi_factorization = _LazyDiagSolve(ops)
    return ops


def _is_pristine(op: SpatialOperator) -> bool:
    """op.matrix is build_laplacian's operator (checked on the entries of the
    cached pattern: O(nnz) compares, no sparse arithmetic)."""
    a = op.matrix
    if not (sp.isspmatrix_csr(a) and a.shape == (op.n, op.n) and a.has_sorted_indices):
        return False
    _, _, slots, _, _, _, typed = StencilTable._full_pattern(op.n_x, op.n_y)
    ip, ix = typed.get(a.indices.dtype, typed[np.dtype(np.int64)])
    vals = laplacian_stencil(op.dim, op.tau / op.delta_x**2)
    return (a.nnz == ix.size and np.array_equal(a.indptr, ip) and np.array_equal(a.indices, ix)
            and np.array_equal(a.data, vals[slots]))


def _to_device(v):
    """(tensor on cuda, was_numpy)."""
    torch = _lib.require_cuda()
    if isinstance(v, torch.Tensor):
        if not v.is_cuda:
            return v.to(device="cuda", dtype=torch.float64).contiguous(), False
        return v.to(dtype=torch.float64).contiguous(), False
    arr = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    return torch.from_numpy(arr).cuda(), True


def _back(t, was_numpy: bool, shape):
    if was_numpy:
        return t.cpu().numpy().reshape(shape)
    return t.reshape(shape)


class BlockBidiagonalSystem:
    """Block lower-bidiagonal [I; -B, D; ...; -B, D] with constant blocks
    (reference stepper.py:66-159), applied by fused sm_100a stencil kernels.

    Beyond the reference's arguments the device needs the grid geometry
    (``grid=(n_x, n_y)``, ``dim``); a tridiagonal operator without it is taken
    as a 1-D grid.  ``spectral`` marks pristine-Laplacian blocks (D = I - a dt
    A, B = I + b dt A) whose forward substitution runs in the sine basis.
    """

    def __init__(self, diag: sp.csr_matrix, sub: sp.csr_matrix, n_steps: int,
                 dropped: tuple[int, ...] = (), grid: tuple[int, int] | None = None,
                 dim: int | None = None, spectral: SpectralInfo | None = None):
        # diag / sub may also be zero-argument callables (internal: the
        # closed-form blocks of pristine levels are assembled only when a
        # caller asks for the matrices; the device path uses `spectral`)
        self._diag_src, self._sub_src = diag, sub
        self._diag = None if callable(diag) else sp.csr_matrix(diag)
        self._sub = None if callable(sub) else sp.csr_matrix(sub)
        if self._diag is None and (grid is None or spectral is None):
            raise ValueError("lazily built blocks need the grid and spectral info")
        self.n_steps = n_steps
        self.n = self._diag.shape[0] if self._diag is not None else grid[0] * grid[1]
        self.dropped = tuple(sorted(dropped))
        if grid is None:
            grid = (self.n, 1)
            dim = 1
        if dim is None:
            dim = 1 if grid[1] == 1 else 2
        if grid[0] * grid[1] != self.n:
            raise ValueError(f"grid {grid} does not match operator size {self.n}")
        self.grid = tuple(grid)
        self.dim = dim
        self.spectral = spectral
        self._desc = None
        self._solver = None
        self._keep = []

    @property
    def diag(self) -> sp.csr_matrix:
        if self._diag is None:
            self._diag = sp.csr_matrix(self._diag_src())
        return self._diag

    @property
    def sub(self) -> sp.csr_matrix:
        if self._sub is None:
            self._sub = sp.csr_matrix(self._sub_src())
        return self._sub

    def block_sources(self):
        """(diag, sub) as given: matrices or their lazy builders."""
        return (self._diag if self._diag is not None else self._diag_src,
                self._sub if self._sub is not None else self._sub_src)

    # ---------------------------------------------------------- bookkeeping
    @property
    def total_dim(self) -> int:
        return (self.n_steps + 1) * self.n

    def segment_rows(self) -> list[tuple[int, int]]:
        """Half-open row ranges of independently solvable chains
        (reference stepper.py:107-112)."""
        cuts = [c for c in self.dropped if c > 1]
        return list(zip([1] + cuts, cuts + [self.n_steps + 1]))

    def to_dense(self) -> np.ndarray:
        """Desk-scale dense assembly (tests only; reference stepper.py:148-159)."""
        n, ns = self.n, self.n_steps
        out = np.zeros(((ns + 1) * n, (ns + 1) * n))
        out[:n, :n] = np.eye(n)
        dd, ss = self.diag.toarray(), self.sub.toarray()
        for k in range(1, ns + 1):
            out[k * n:(k + 1) * n, k * n:(k + 1) * n] = dd
            if k not in self.dropped:
                out[k * n:(k + 1) * n, (k - 1) * n:k * n] = -ss
        return out

    # --------------------------------------------------------------- device
    def level_desc(self) -> _lib.LevelDesc:
        if self._desc is None:
            torch = _lib.require_cuda()
            nx, ny = self.grid
            if self.spectral is not None:  # closed form, bitwise the matrices' entries
                cp, cq = self.spectral.stencils(self.dim)
                p = StencilTable.from_constants(cp, nx, ny)
                q = StencilTable.from_constants(cq, nx, ny)
            else:
                p = StencilTable(self.diag.T, nx, ny)   # right-product: v @ D = D^T v
                q = StencilTable(self.sub.T, nx, ny)
            d = _lib.LevelDesc()
            d.dim, d.nx, d.ny, d.n_steps = self.dim, nx, ny, self.n_steps
            d.diag_t = p.desc()
            d.sub_t = q.desc()
            mask = dropped_mask(self.n_steps, self.dropped)
            if mask is not None:
                mt = torch.from_numpy(mask).cuda()
                self._keep.append(mt)
                d.dropped = mt.data_ptr()
            self._keep += [p, q]
            self._desc = d
        return self._desc

    @property
    def diag_factorization(self) -> CoarseSolver:
        """Device forward-substitution tables (the reference prefactors D,
        stepper.py:87-91)."""
        if self._solver is None:
            self._solver = CoarseSolver(self.diag, self.sub, self.n_steps, self.dropped,
                                        self.dim, self.grid[0], self.grid[1], self.spectral)
        return self._solver

    def matvec_into(self, v, out) -> None:
        lib = _lib.load()
        _lib.check(lib.pmk_stmv(ctypes.byref(self.level_desc()), _lib.ptr(v), _lib.ptr(out),
                                _lib.stream_ptr()), "matvec")

    def matvec(self, v):
        """Apply the block matrix; preserves the input's shape and kind
        (reference stepper.py:96-105)."""
        shape = np.shape(v) if not hasattr(v, "shape") else tuple(v.shape)
        dv, was_np = _to_device(v)
        if dv.numel() != self.total_dim:
            raise ValueError(f"vector of size {dv.numel()} does not match system {self.total_dim}")
        out = torch_empty_like(dv)
        self.matvec_into(dv, out)
        return _back(out, was_np, shape)

    def forward_solve(self, rhs):
        """Direct solve by block forward substitution honouring dropped
        couplings (reference stepper.py:114-146)."""
        shape = tuple(rhs.shape) if hasattr(rhs, "shape") else np.shape(rhs)
        dr, was_np = _to_device(rhs)
        if dr.numel() != self.total_dim:
            raise ValueError("rhs size does not match system")
        out = torch_empty_like(dr)
        self.diag_factorization.solve_into(dr, out)
        return _back(out, was_np, shape)

    def diag_solve(self, rhs):
        """D^{-1} applied to each row of a (k, n) block (or one vector)."""
        shape = tuple(rhs.shape) if hasattr(rhs, "shape") else np.shape(rhs)
        dr, was_np = _to_device(rhs)
        rows = dr.numel() // self.n
        # A forward substitution whose every coupling is dropped applies D^{-1}
        # to each row; its row 0 is the identity, so prepend a zero row.
        sys = BlockBidiagonalSystem(*self.block_sources(), rows,
                                    dropped=tuple(range(1, rows + 1)), grid=self.grid,
                                    dim=self.dim, spectral=self.spectral)
        torch = _lib.require_cuda()
        padded = torch.cat([torch.zeros(self.n, dtype=torch.float64, device="cuda"),
                            dr.reshape(-1)])
        out = torch.empty_like(padded)
        sys.diag_factorization.solve_into(padded, out)
        return _back(out[self.n:], was_np, shape)


def torch_empty_like(t):
    import torch

    return torch.empty_like(t)


class FineSystem(BlockBidiagonalSystem):
    """All-at-once system of the fine theta-scheme with its right-hand side
    (reference stepper.py:168-193).  ``rhs`` is a device tensor (n_t+1, n)."""

    def __init__(self, ops: StepOperators, u0, forcing=None):
        if tuple(np.shape(u0) if not hasattr(u0, "shape") else u0.shape) != (ops.n,):
            raise ValueError(f"u0 must have shape ({ops.n},)")
        if forcing is not None and tuple(forcing.shape) != (ops.config.n_t, ops.n):
            raise ValueError("forcing must have shape (n_t, n)")
        sp_op = ops.spatial
        # spectral only for build_laplacian's operator (otherwise the kernels
        # read psi/phi themselves and the coarse solve takes the general path)
        super().__init__(diag=ops.psi, sub=ops.phi, n_steps=ops.config.n_t,
                         grid=sp_op.grid, dim=sp_op.dim, spectral=ops.spectral_info)
        torch = _lib.require_cuda()
        self.ops = ops
        self.host_io = not isinstance(u0, torch.Tensor)
        u0_d, _ = _to_device(u0)
        self.u0 = u0_d
        self.forcing = forcing
        rhs = torch.zeros((ops.config.n_t + 1, ops.n), dtype=torch.float64, device="cuda")
        rhs[0] = u0_d
        if forcing is not None:
            f_d, _ = _to_device(forcing)
            rhs[1:] = ops.config.delta_t * f_d.reshape(ops.config.n_t, ops.n)
        self.rhs = rhs

    @property
    def n_t(self) -> int:
        return self.n_steps

    def relative_residual(self, u) -> float:
        """||rhs - A u|| / ||rhs|| (reference stepper.py:191-193)."""
        torch = _lib.require_cuda()
        lib = _lib.load()
        du, _ = _to_device(u)
        tmp = torch.empty_like(self.rhs).reshape(-1)
        num = torch.empty(1, dtype=torch.float64, device="cuda")
        den = torch.empty(1, dtype=torch.float64, device="cuda")
        s = _lib.stream_ptr()
        _lib.check(lib.pmk_residual_nrm2(ctypes.byref(self.level_desc()), _lib.ptr(du),
                                         _lib.ptr(self.rhs), _lib.ptr(tmp), _lib.ptr(num), s),
                   "residual")
        _lib.check(lib.pmk_nrm2(_lib.ptr(self.rhs), self.total_dim, _lib.ptr(den), s), "nrm2")
        return float(num.item() / den.item())


def assemble_fine_system(ops: StepOperators, u0, forcing=None) -> FineSystem:
    return FineSystem(ops, u0, forcing)


def sequential_solve(ops: StepOperators, u0, forcing=None):
    """theta-scheme march u_k = psi^{-1}(phi u_{k-1} + dt g_k) (reference
    stepper.py:201-225), done as the fine system's forward substitution on the
    device (sine-diagonalised per-mode recurrence)."""
    if tuple(np.shape(u0) if not hasattr(u0, "shape") else u0.shape) != (ops.n,):
        raise ValueError(f"u0 must have shape ({ops.n},)")
    fine = FineSystem(ops, u0, forcing)
    out = fine.forward_solve(fine.rhs)
    if fine.host_io:
        return out.cpu().numpy()
    return out


def relative_residual(system: FineSystem, u) -> float:
    return system.relative_residual(u)
