"""Intergrid pairs and coarse systems on the GPU.

Mirror of reference ``pintmk/intergrid.py``: pure time coarsening (TimePair,
Y = Z = nu-fold identity stacks), simultaneous time-space coarsening by
agglomeration (TimeSpacePair, Z piecewise-constant injection, Y agglomerate
averaging), the MGRIT reduction pair (MgritPair: injection and ideal
interpolation) with its rediscretized coarse system, and the perturbed
decoupling of the coarsest level.
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp

from . import _lib
from .stepper import BlockBidiagonalSystem, StepOperators, _back, _to_device


class CoarseSystem(BlockBidiagonalSystem):
    """Block bidiagonal coarse matrix tagged with its provenance (reference
    intergrid.py:24-30)."""

    def __init__(self, diag, sub, n_steps, provenance: str, dropped: tuple[int, ...] = (),
                 grid=None, dim=None, spectral=None):
        super().__init__(diag, sub, n_steps, dropped=dropped, grid=grid, dim=dim,
                         spectral=spectral)
        self.provenance = provenance


class _PairBase:
    fine_rows: int
    n_T: int
    nu: int

    def _pair_desc(self) -> _lib.PairDesc:
        raise NotImplementedError

    def restrict(self, v):
        """Y^T v (sum over each slab's nu rows; averaging for space pairs)."""
        torch = _lib.require_cuda()
        shape = tuple(v.shape) if hasattr(v, "shape") else np.shape(v)
        dv, was_np = _to_device(v)
        if dv.numel() != self.fine_rows * self.n:
            raise ValueError("vector size does not match the fine level")
        out = torch.empty((self.n_T + 1) * self.m, dtype=torch.float64, device="cuda")
        scratch = None
        if self.m != self.n or getattr(self, "partition", None) is not None:  # space pairs
            scratch = torch.empty((self.n_T + 1) * self.n, dtype=torch.float64, device="cuda")
        lib = _lib.load()
        _lib.check(lib.pmk_restrict(ctypes.byref(self._pair_desc()), _lib.ptr(dv), _lib.ptr(out),
                                    _lib.ptr(scratch), _lib.stream_ptr()), "restrict")
        return _back(out, was_np, (-1,) if len(shape) == 1 else (self.n_T + 1, self.m))

    def interpolate(self, w):
        """Z w (repeat each coarse row nu times; injection for space pairs)."""
        torch = _lib.require_cuda()
        shape = tuple(w.shape) if hasattr(w, "shape") else np.shape(w)
        dw, was_np = _to_device(w)
        if dw.numel() != (self.n_T + 1) * self.m:
            raise ValueError("vector size does not match the coarse level")
        out = torch.empty(self.fine_rows * self.n, dtype=torch.float64, device="cuda")
        lib = _lib.load()
        _lib.check(lib.pmk_interpolate(ctypes.byref(self._pair_desc()), _lib.ptr(dw),
                                       _lib.ptr(out), _lib.stream_ptr()), "interpolate")
        return _back(out, was_np, (-1,) if len(shape) == 1 else (self.fine_rows, self.n))


class TimePair(_PairBase):
    """Pure time coarsening (reference intergrid.py:37-76)."""

    kind = "T"
    partition = None

    def __init__(self, n: int, nu: int, n_T: int):
        if nu < 1:
            raise ValueError("nu must be positive")
        self.n = n
        self.m = n
        self.nu = nu
        self.n_T = n_T
        self.fine_rows = nu * n_T + 1
        self._desc = None

    def _pair_desc(self) -> _lib.PairDesc:
        if self._desc is None:
            d = _lib.PairDesc()
            d.nu, d.n_T, d.m_fine, d.m_coarse = self.nu, self.n_T, self.n, self.n
            d.group_of = d.y_ptr = d.y_idx = d.y_val = None
            self._desc = d
        return self._desc

    def block_matrices(self, k: int):
        """(Y_k, Z_k) for one slab (identical here)."""
        eye = sp.identity(self.n, format="csr")
        z = eye if k == 0 else sp.vstack([eye] * self.nu, format="csr")
        return z, z

    def materialize(self):
        z = sp.block_diag([self.block_matrices(k)[1] for k in range(self.n_T + 1)], format="csr")
        return z, z


class TimeSpacePair(_PairBase):
    """Time and space coarsening by agglomeration (reference
    intergrid.py:79-131); nu = 1 gives the pure space move."""

    kind = "TS"

    def __init__(self, nu: int, n_T: int, partition: list[np.ndarray], n: int):
        if nu < 1:
            raise ValueError("nu must be positive")
        sizes = np.array([len(g) for g in partition])
        if sizes.min() == 0:
            raise ValueError("empty agglomerate")
        flat = np.concatenate(partition)
        if len(np.unique(flat)) != n or len(flat) != n:
            raise ValueError("partition must cover all indices exactly once")
        self.nu = nu
        self.n_T = n_T
        self.n = n
        self.m = len(partition)
        self.partition = partition
        self.fine_rows = nu * n_T + 1
        cols = np.repeat(np.arange(self.m), sizes)
        self.z_space = sp.csr_matrix((np.ones(n), (flat, cols)), shape=(n, self.m))
        self.y_space = sp.csr_matrix((np.repeat(1.0 / sizes, sizes), (flat, cols)),
                                     shape=(n, self.m))
        self._desc = None
        self._keep = []

    def _pair_desc(self) -> _lib.PairDesc:
        if self._desc is None:
            torch = _lib.require_cuda()
            group_of = np.empty(self.n, dtype=np.int32)
            for c, g in enumerate(self.partition):
                group_of[np.asarray(g)] = c
            yt = sp.csr_matrix(self.y_space.T)
            yt.sort_indices()
            tabs = [torch.from_numpy(group_of).cuda(),
                    torch.from_numpy(yt.indptr.astype(np.int32)).cuda(),
                    torch.from_numpy(yt.indices.astype(np.int32)).cuda(),
                    torch.from_numpy(yt.data.astype(np.float64)).cuda()]
            self._keep = tabs
            d = _lib.PairDesc()
            d.nu, d.n_T, d.m_fine, d.m_coarse = self.nu, self.n_T, self.n, self.m
            d.group_of, d.y_ptr, d.y_idx, d.y_val = (t.data_ptr() for t in tabs)
            self._desc = d
        return self._desc

    def block_matrices(self, k: int):
        if k == 0:
            return self.y_space, self.z_space
        return (sp.vstack([self.y_space] * self.nu, format="csr"),
                sp.vstack([self.z_space] * self.nu, format="csr"))

    def materialize(self):
        ys, zs = zip(*(self.block_matrices(k) for k in range(self.n_T + 1)))
        return sp.block_diag(ys, format="csr"), sp.block_diag(zs, format="csr")


def full_weighting_1d(count: int):
    """1-D full-weighting restriction R (n_c x n) and linear interpolation
    P (n x n_c) between n interior points and the n_c = (n - 1) / 2 interior
    points of the grid with doubled spacing (coarse point c sits on fine point
    2 c + 1): R rows (1/4, 1/2, 1/4), P = 2 R^T."""
    if count < 3 or count % 2 == 0:
        raise ValueError("full weighting needs an odd number (>= 3) of interior points")
    nc = (count - 1) // 2
    c = np.arange(nc)
    rows = np.repeat(c, 3)
    cols = (2 * c[:, None] + np.arange(3)[None, :]).ravel()
    vals = np.tile([0.25, 0.5, 0.25], nc)
    r = sp.csr_matrix((vals, (rows, cols)), shape=(nc, count))
    return r, (2.0 * r.T).tocsr()


class WeightedSpacePair(_PairBase):
    """Space coarsening by full-weighting restriction and (bi)linear
    interpolation, optionally with time coarsening by nu -- BASELINE config
    4's transfer operators.  An EXTENSION: the reference only agglomerates
    (intergrid.py:79-131), so this pair has no reference counterpart and its
    parity is pinned to the oracle's restatement of the same formulas only.
    Same conventions as TimeSpacePair: restrict sums each slab's nu rows and
    applies y_space^T (rows of weights summing to 1, like agglomerate
    averaging); interpolate applies z_space (weights 1, 1/2, 1/4) and
    repeats each coarse row nu times."""

    kind = "TS_FW"
    partition = None

    def __init__(self, nu: int, n_T: int, grid: tuple[int, int], dim: int):
        if nu < 1:
            raise ValueError("nu must be positive")
        nx, ny = grid[0], (grid[1] if dim == 2 else 1)
        rx, px = full_weighting_1d(nx)
        if dim == 2:
            ry, py = full_weighting_1d(ny)
            r, pz = sp.kron(ry, rx, format="csr"), sp.kron(py, px, format="csr")
            self.coarse_grid = (rx.shape[0], ry.shape[0])
        else:
            r, pz = rx, px
            self.coarse_grid = (rx.shape[0], 1)
        self.nu, self.n_T = nu, n_T
        self.n, self.m = nx * ny, r.shape[0]
        self.fine_rows = nu * n_T + 1
        self.y_space = sp.csr_matrix(r.T)   # (n, m): restrict = v @ y_space
        self.z_space = sp.csr_matrix(pz)    # (n, m): interpolate = w @ z_space^T
        self._desc = None
        self._keep = []

    def _pair_desc(self) -> _lib.PairDesc:
        if self._desc is None:
            torch = _lib.require_cuda()
            yt = sp.csr_matrix(self.y_space.T)
            yt.sort_indices()
            z = sp.csr_matrix(self.z_space)
            z.sort_indices()
            i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()  # noqa: E731
            f64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()  # noqa: E731
            tabs = [i32(yt.indptr), i32(yt.indices), f64(yt.data),
                    i32(z.indptr), i32(z.indices), f64(z.data),
                    torch.empty((self.n_T + 1) * self.m, dtype=torch.float64, device="cuda")]
            self._keep = tabs
            d = _lib.PairDesc()
            d.nu, d.n_T, d.m_fine, d.m_coarse = self.nu, self.n_T, self.n, self.m
            d.group_of = None
            d.y_ptr, d.y_idx, d.y_val, d.z_ptr, d.z_idx, d.z_val, d.coarse_out = \
                (t.data_ptr() for t in tabs)
            self._desc = d
        return self._desc

    def child_size(self) -> int:
        """The solver's per-iteration child vector: the coarse solution
        interpolated in space ((n_T + 1) x n), repeated in time by K-IMV."""
        return (self.n_T + 1) * self.n

    def expand_child(self, child):
        """Z w from a stored child vector (time repeat only)."""
        return TimePair(self.n, self.nu, self.n_T).interpolate(child)

    def block_matrices(self, k: int):
        if k == 0:
            return self.y_space, self.z_space
        return (sp.vstack([self.y_space] * self.nu, format="csr"),
                sp.vstack([self.z_space] * self.nu, format="csr"))

    def materialize(self):
        ys, zs = zip(*(self.block_matrices(k) for k in range(self.n_T + 1)))
        return sp.block_diag(ys, format="csr"), sp.block_diag(zs, format="csr")


class MgritPair(_PairBase):
    """Coarse-point injection with ideal interpolation (reference
    intergrid.py:134-187): restrict keeps rows 0, nu, 2 nu, ...; interpolate
    fills each slab by propagating its left coarse row through nu - 1 fine
    steps, (psi^{-1} phi)^j, which the device applies in the sine basis of
    the fine grid (diagonal there: ratio beta/delta per mode)."""

    kind = "MGRIT"
    partition = None

    def __init__(self, ops: StepOperators, nu: int, n_T: int):
        self.ops = ops
        self.n = ops.n
        self.m = ops.n
        self.nu = nu
        self.n_T = n_T
        self.fine_rows = nu * n_T + 1
        self._desc = None
        self._keep = []

    def _pair_desc(self) -> _lib.PairDesc:
        if self._desc is None:
            torch = _lib.require_cuda()
            from .spatial import dst_eigenvalues_1d, dst_matrix, fft_dst_tables

            sp_op, cfg = self.ops.spatial, self.ops.config
            if self.ops.spectral_info is None:
                # ideal interpolation runs in the sine basis of the fine grid
                raise NotImplementedError(
                    "MGRIT ideal interpolation needs build_laplacian's operator")
            nx, ny = sp_op.n_x, (sp_op.n_y if sp_op.dim == 2 else 1)
            ex = dst_eigenvalues_1d(nx)
            lam = ex[None, :] if ny == 1 else (dst_eigenvalues_1d(ny)[:, None] + ex[None, :])
            lam = (sp_op.tau / sp_op.delta_x**2) * lam.ravel()
            delta = 1.0 - cfg.theta * cfg.delta_t * lam
            beta = 1.0 + (1.0 - cfg.theta) * cfg.delta_t * lam
            d = _lib.PairDesc()
            d.nu, d.n_T, d.m_fine, d.m_coarse = self.nu, self.n_T, self.n, self.n
            d.mgrit, d.dim, d.nx, d.ny = 1, sp_op.dim, nx, ny
            keep = [torch.from_numpy(beta / delta).cuda()]
            d.ratio = keep[0].data_ptr()
            tabx = fft_dst_tables(nx)
            taby = fft_dst_tables(ny) if ny > 1 else None
            if tabx is not None and nx + 1 <= 1024 and (ny == 1 or (taby is not None
                                                                     and ny + 1 <= 512)):
                keep.append(torch.from_numpy(tabx).cuda())
                d.fft_x = keep[-1].data_ptr()
                d.fft_scale = 2.0 / (nx + 1)
                if ny > 1:
                    keep.append(torch.from_numpy(taby).cuda())
                    d.fft_y = keep[-1].data_ptr()
                    d.fft_scale *= 2.0 / (ny + 1)
            else:
                keep.append(torch.from_numpy(dst_matrix(nx)).cuda())
                d.sx = keep[-1].data_ptr()
                if ny > 1:
                    keep.append(torch.from_numpy(dst_matrix(ny)).cuda())
                    d.sy = keep[-1].data_ptr()
                d.fft_scale = 1.0
            nw = max(self.n_T, 1) * self.n
            for name in ("work0", "work1", "work2"):
                keep.append(torch.empty(nw, dtype=torch.float64, device="cuda"))
                setattr(d, name, keep[-1].data_ptr())
            keep.append(torch.empty((self.n_T + 1) * self.n, dtype=torch.float64, device="cuda"))
            d.coarse_out = keep[-1].data_ptr()
            self._keep = keep
            self._desc = d
        return self._desc


def build_mgrit_pair(part) -> MgritPair:
    return MgritPair(ops=part.fine.ops, nu=part.nu, n_T=part.n_T)


def rediscretized_coarse(ops: StepOperators, nu: int, n_T: int) -> CoarseSystem:
    """theta-scheme with step nu dt (reference intergrid.py:270-280): the
    parareal coarse propagator, used with the reduction pair."""
    from ._device import SpectralInfo

    cfg = ops.config
    big_dt = nu * cfg.delta_t
    eye = sp.identity(ops.n, format="csr")
    diag = (eye - cfg.theta * big_dt * ops.spatial.matrix).tocsr()
    sub = (eye + (1 - cfg.theta) * big_dt * ops.spatial.matrix).tocsr()
    sp_op = ops.spatial
    spectral = None
    if ops.spectral_info is not None:  # build_laplacian's operator
        spectral = SpectralInfo(sp_op.tau / sp_op.delta_x**2, cfg.theta * big_dt,
                                (1 - cfg.theta) * big_dt)
    return CoarseSystem(diag=diag, sub=sub, n_steps=n_T, provenance="rediscretized",
                        grid=sp_op.grid, dim=sp_op.dim, spectral=spectral)


def build_t_pair(n: int, nu: int, n_T: int) -> TimePair:
    return TimePair(n, nu, n_T)


def build_ts_pair(n: int, nu: int, n_T: int, partition) -> TimeSpacePair:
    return TimeSpacePair(nu=nu, n_T=n_T, partition=list(partition), n=n)


def agglomerate_partition(n_x: int, n_y: int = 1):
    """Factor-2 agglomeration per direction, leftovers joining the last group
    (reference intergrid.py:202-227).  Returns (groups, (m_x, m_y)) with the
    groups in row-major coarse order."""
    def spans(count: int):
        half = count // 2
        if half == 0:
            raise ValueError("grid too small to agglomerate")
        bounds = [(2 * i, 2 * i + 2) for i in range(half)]
        bounds[-1] = (bounds[-1][0], count)
        return bounds

    xs = spans(n_x)
    if n_y == 1:
        return [np.arange(a, b) for a, b in xs], (len(xs), 1)
    ys = spans(n_y)
    groups = []
    for ya, yb in ys:
        for xa, xb in xs:
            iy, ix = np.meshgrid(np.arange(ya, yb), np.arange(xa, xb), indexing="ij")
            groups.append((iy * n_x + ix).ravel())
    return groups, (len(xs), len(ys))


def closed_form_t_coarse(ops: StepOperators, nu: int, n_T: int) -> CoarseSystem:
    """Time-coarsened Galerkin system in closed form (reference
    intergrid.py:243-255)."""
    cfg = ops.config
    eye = sp.identity(ops.n, format="csr")
    diag = (eye - (nu - 1 + cfg.theta) * cfg.delta_t * ops.spatial.matrix).tocsr()
    sub = (eye + (1 - cfg.theta) * cfg.delta_t * ops.spatial.matrix).tocsr()
    return CoarseSystem(diag=diag, sub=sub, n_steps=n_T, provenance="closed_form",
                        grid=ops.spatial.grid, dim=ops.spatial.dim)


def perturb_decouple(cs: CoarseSystem, n_cgs: int) -> CoarseSystem:
    """Drop the couplings at balanced chunk starts (reference
    intergrid.py:299-311); n_cgs >= n_T makes the system block diagonal."""
    if not 1 <= n_cgs <= cs.n_steps + 1:
        raise ValueError(f"n_cgs must be in [1, {cs.n_steps + 1}]")
    chunks = np.array_split(np.arange(1, cs.n_steps + 1), min(n_cgs, cs.n_steps))
    dropped = tuple(int(c[0]) for c in chunks if len(c))
    d_src, s_src = cs.block_sources()
    return CoarseSystem(diag=d_src, sub=s_src, n_steps=cs.n_steps, provenance="perturbed",
                        dropped=dropped, grid=cs.grid, dim=cs.dim, spectral=cs.spectral)
