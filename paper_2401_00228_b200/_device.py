"""Device descriptors: stencil extraction, level / coarse-solve tables.

Turns the host-side scipy operators of a level (built exactly like the
reference's, solver.py:105-110) into the flat tables the kernels read:

* a 5-slot stencil (S, W, C, E, N) per operator, either constant (the
  pristine Laplacian levels) or per point (agglomerated levels);
* the coarsest-level forward-substitution tables: orthonormal sine
  transforms plus per-mode eigenvalues (DST), or an explicit inverse
  (DENSE) for small non-Toeplitz levels.
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp

from . import _lib
from .spatial import dst_eigenvalues_1d, dst_matrix, fft_dst_tables

# Largest spatial size for which the DENSE coarsest solve is allowed
# (explicit inverse of m*m doubles: 8192^2 * 8 B = 512 MB).
DENSE_MAX_M = 8192


class StencilTable:
    """Row-form 5-slot stencil of a sparse matrix X: out_i = sum_s c[s, i] *
    in[i + off_s], offsets (-nx, -1, 0, +1, +nx).  Raises NotImplementedError
    when X has entries outside the 5-point pattern of the grid."""

    def __init__(self, matrix: sp.spmatrix, nx: int, ny: int):
        m = nx * ny
        if matrix.shape != (m, m):
            raise ValueError(f"operator shape {matrix.shape} does not match grid {nx}x{ny}")
        self.nx, self.ny, self.m = nx, ny, m
        self._dev = None
        self._coef = None
        self._lazy = None
        if sp.issparse(matrix) and matrix.format in ("csr", "csc") and \
                self._from_full_pattern(matrix):
            return
        x = sp.csr_matrix(matrix)
        coo = x.tocoo()
        rows, cols, vals = coo.row.astype(np.int64), coo.col.astype(np.int64), coo.data
        off = cols - rows
        ry, rx = np.divmod(rows, nx)
        cy, cx = np.divmod(cols, nx)
        slot = np.full(rows.shape, -1)
        slot[(off == 0)] = 2
        same_row = ry == cy
        slot[(off == -1) & same_row] = 1
        slot[(off == 1) & same_row] = 3
        if ny > 1:
            same_col = rx == cx
            slot[(off == -nx) & same_col & (slot < 0)] = 0
            slot[(off == nx) & same_col & (slot < 0)] = 4
        if np.any(slot < 0):
            raise NotImplementedError("operator is not a 5-point stencil on the grid")
        coef = np.zeros((5, m))
        coef[slot, rows] = vals
        present = np.zeros((5, m), dtype=bool)
        present[slot, rows] = True
        exists = self._full_pattern(nx, ny)[4]
        self._coef = coef
        constant = bool(np.all(present == exists))
        consts = np.zeros(5)
        if constant:
            for s in range(5):
                v = coef[s][exists[s]]
                if v.size and not np.all(v == v[0]):
                    constant = False
                    break
                consts[s] = v[0] if v.size else 0.0
        self.constant = constant
        self.consts = consts

    @classmethod
    def from_constants(cls, consts, nx: int, ny: int) -> "StencilTable":
        """Constant stencil (S, W, C, E, N) on an nx x ny grid, without a
        matrix (the closed-form operators of pristine levels)."""
        t = cls.__new__(cls)
        t.nx, t.ny, t.m = nx, ny, nx * ny
        t._dev = None
        t._coef = None
        t._lazy = None
        t.constant = True
        t.consts = np.asarray(consts, dtype=np.float64)
        exists = t._full_pattern(nx, ny)[4]
        t._exists = exists
        return t

    @property
    def coef(self) -> np.ndarray:
        """(5, m) per-point coefficients (zeros where a neighbour is absent)."""
        if self._coef is None and self._lazy is None:
            self._coef = np.where(self._exists, self.consts[:, None], 0.0)
        if self._coef is None:
            self._coef = self._build_coef(*self._lazy)
        return self._coef

    # Fast path: the matrix (CSR, or CSC = the transpose of a CSR) has exactly
    # the full 5-point pattern of the grid in canonical order (every pristine
    # and time-coarsened level).  Its index arrays are compared with a cached
    # pattern whose slot map is then reused; coefficients and constants are
    # read from the matrix entries themselves.
    _patterns: dict = {}
    _OPP = (4, 3, 2, 1, 0)  # slot of the transposed entry: S<->N, W<->E

    @classmethod
    def _full_pattern(cls, nx: int, ny: int):
        key = (nx, ny)
        if key not in cls._patterns:
            m = nx * ny
            iy, ix = np.divmod(np.arange(m, dtype=np.int64), nx)
            exists = np.stack([iy > 0, ix > 0, np.ones(m, bool), ix < nx - 1, iy < ny - 1])
            if ny == 1:
                exists[0] = False
                exists[4] = False
            offs = np.array([-nx, -1, 0, 1, nx], dtype=np.int64)
            cols = np.arange(m, dtype=np.int64)[None, :] + offs[:, None]
            # entries in row-major order, ascending column within a row
            # (slots S < W < C < E < N)
            mask_t = exists.T
            indices = cols.T[mask_t]
            slots = np.broadcast_to(np.arange(5), (m, 5))[mask_t]
            rows = np.broadcast_to(np.arange(m, dtype=np.int64)[:, None], (m, 5))[mask_t]
            indptr = np.concatenate([[0], np.cumsum(mask_t.sum(axis=1))])
            by_slot = [np.flatnonzero(slots == s_) for s_ in range(5)]
            cls._patterns[key] = (indptr, indices, slots, rows, exists, by_slot,
                                  {np.dtype(np.int64): (indptr, indices),
                                   np.dtype(np.int32): (indptr.astype(np.int32),
                                                        indices.astype(np.int32))})
        return cls._patterns[key]

    def _from_full_pattern(self, x) -> bool:
        nx, ny = self.nx, self.ny
        if not x.has_sorted_indices:
            return False
        pat = self._full_pattern(nx, ny)
        by_slot, typed = pat[5], pat[6]
        ip, ix = typed.get(x.indices.dtype, typed[np.dtype(np.int64)])
        if x.nnz != ix.size or not (np.array_equal(x.indptr, ip) and np.array_equal(x.indices, ix)):
            return False
        transposed = x.format == "csc"   # x = C^T, C the CSR with these arrays
        data = x.data
        # constant iff every entry equals the first entry of its slot
        first = np.array([data[b[0]] if b.size else 0.0 for b in by_slot])
        constant = bool(np.array_equal(data, first[pat[2]]))
        consts = np.zeros(5)
        if constant:
            for s_ in range(5):
                consts[self._OPP[s_] if transposed else s_] = first[s_]
        self.constant = constant
        self.consts = consts
        self._lazy = (data.copy(), transposed)
        return True

    def _build_coef(self, data: np.ndarray, transposed: bool) -> np.ndarray:
        nx, ny, m = self.nx, self.ny, self.m
        _, _, slots, rows, exists = self._full_pattern(nx, ny)[:5]
        c = np.zeros((5, m))
        c[slots, rows] = data            # row form of C
        if not transposed:
            return c
        # X = C^T: X[i, i + off_s] = C[i + off_s, i] = c[opp(s), i + off_s]
        offs = (-nx, -1, 0, 1, nx)
        out = np.zeros((5, m))
        for s_ in range(5):
            src = c[self._OPP[s_]]
            o = offs[s_]
            if o >= 0:
                out[s_, :m - o] = src[o:]
            else:
                out[s_, -o:] = src[:m + o]
            out[s_][~exists[s_]] = 0.0
        return out

    def desc(self) -> _lib.Stencil:
        st = _lib.Stencil()
        if self.constant:
            st.var = 0
            for s in range(5):
                st.c[s] = float(self.consts[s])
            st.coef = None
        else:
            import torch

            if self._dev is None:
                self._dev = torch.from_numpy(np.ascontiguousarray(self.coef)).cuda()
            st.var = 1
            st.coef = self._dev.data_ptr()
        return st


def dropped_mask(n_steps: int, dropped) -> np.ndarray | None:
    if not dropped:
        return None
    mask = np.zeros(n_steps + 1, dtype=np.uint8)
    mask[list(dropped)] = 1
    return mask


class SpectralInfo:
    """diag = I - a_dt * A and sub = I + b_dt * A with A = factor * (pristine
    Dirichlet second-difference operator on an nx x ny grid)."""

    def __init__(self, factor: float, a_dt: float, b_dt: float):
        self.factor = float(factor)
        self.a_dt = float(a_dt)
        self.b_dt = float(b_dt)

    def stencils(self, dim: int) -> tuple[np.ndarray, np.ndarray]:
        """(S, W, C, E, N) constants of diag and sub, equal bit for bit to the
        entries scipy produces for ``eye - a_dt * A`` and ``eye + b_dt * A``
        (spatial.py build_laplacian, solver.py _coarse_system_from): A's
        off-diagonal entries are factor * 1, its diagonal factor * (-2 per
        direction); a_dt * A rounds each entry once, the identity update once
        more on the diagonal only.  Both blocks are symmetric, so these are
        also the right-product (transposed) stencils."""
        f = self.factor
        ac = f * (-4.0 if dim == 2 else -2.0)
        d_off, s_off = -(self.a_dt * f), self.b_dt * f
        d_c, s_c = 1.0 - self.a_dt * ac, 1.0 + self.b_dt * ac
        if dim == 2:
            return (np.array([d_off, d_off, d_c, d_off, d_off]),
                    np.array([s_off, s_off, s_c, s_off, s_off]))
        return (np.array([0.0, d_off, d_c, d_off, 0.0]),
                np.array([0.0, s_off, s_c, s_off, 0.0]))


def _tridiag_eig(lower: np.ndarray, diag: np.ndarray, upper: np.ndarray):
    """Eigen-decomposition K = V diag(lam) V^{-1} of a real tridiagonal K
    (lower[i] = K[i, i-1], upper[i] = K[i, i+1]) whose off-diagonal products
    are positive: K = Dl T Dl^{-1} with T symmetric (Dl diagonal), so
    V = Dl Q and V^{-1} = Q^T Dl^{-1}.  None when some product is <= 0."""
    from scipy.linalg import eigh_tridiagonal

    n = diag.size
    if n == 1:
        return np.ones((1, 1)), np.ones((1, 1)), diag.copy()
    prod = lower[1:] * upper[:-1]
    if np.any(prod <= 0.0):
        return None
    # Dl[i+1] / Dl[i] = sqrt(lower[i+1] / upper[i]); log-space for range
    ratio = 0.5 * (np.log(np.abs(lower[1:])) - np.log(np.abs(upper[:-1])))
    logd = np.concatenate([[0.0], np.cumsum(ratio)])
    logd -= 0.5 * (logd.max() + logd.min())
    dl = np.exp(logd)
    off = np.sign(upper[:-1]) * np.sqrt(prod)
    lam, q = eigh_tridiagonal(diag, off)
    v = dl[:, None] * q
    vinv = q.T / dl[None, :]
    return v, vinv, lam


class SeparableFactors:
    """D = I - K, B = I + b K with K = I (x) Kx + Ky (x) I (x fastest) and
    tridiagonal Kx, Ky: true for every level this package builds (pristine
    Laplacian levels, and agglomerated ones, since agglomerate_partition is
    a tensor product of 1-D groupings, intergrid.py:202-227) and checked
    here on the matrices themselves.  K's eigenvectors V = Vy (x) Vx
    diagonalise D and B together; in 2-D the reference couples slices with
    B^T (stepper.py:144), which differs from B by b N, N = K^T - K, when
    agglomeration left K non-symmetric (odd grids: the 3-wide last group).
    N is a handful of entries next to the odd group, so in the mode basis it
    is a low-rank correction: per direction, `points` physical indices c with
    h_c = row c of V (the physical value at c of a mode row) and
    u_c = sum over N's entries (r, c, val) of val * column r of V^{-1}."""

    MAX_POINTS = 8

    def __init__(self, vx, vxi, lx, vy, vyi, ly, b, corr_x, corr_y):
        self.vx, self.vxi, self.lx = vx, vxi, lx
        self.vy, self.vyi, self.ly = vy, vyi, ly
        self.b = b
        self.corr_x, self.corr_y = corr_x, corr_y  # (h [P][n], u [P][n]) or None

    @staticmethod
    def _correction(lower, upper, v, vinv):
        s = lower[1:] - upper[:-1]          # N[i, i+1] = K[i+1, i] - K[i, i+1]
        idx = np.flatnonzero(s != 0.0)
        if idx.size == 0:
            return None
        cols: dict = {}
        for i in idx:                        # entries (i, i+1, s_i), (i+1, i, -s_i)
            cols.setdefault(i + 1, []).append((i, s[i]))
            cols.setdefault(i, []).append((i + 1, -s[i]))
        if len(cols) > SeparableFactors.MAX_POINTS:
            return False
        pts = sorted(cols)
        h = np.stack([v[c, :] for c in pts])
        u = np.stack([sum(val * vinv[:, r] for r, val in cols[c]) for c in pts])
        return np.ascontiguousarray(h), np.ascontiguousarray(u)

    @classmethod
    def detect(cls, diag, sub, nx: int, ny: int, dim: int, tol: float = 1e-12):
        m = nx * ny
        d = sp.csr_matrix(diag)
        b = sp.csr_matrix(sub)
        eye = sp.identity(m, format="csr")
        try:
            kt = StencilTable(eye - d, nx, ny).coef
            et = StencilTable(b - eye, nx, ny).coef
        except NotImplementedError:
            return None
        kk = float(np.sum(kt * kt))
        if kk == 0.0:
            return None
        bfac = float(np.sum(kt * et)) / kk
        scale = max(float(np.abs(et).max()), float(np.abs(kt).max()) * abs(bfac), 1e-300)
        if float(np.abs(et - bfac * kt).max()) > tol * scale:
            return None                      # B is not I + b K
        S, W, C, E, N = (kt[s].reshape(ny, nx) for s in range(5))
        kscale = float(np.abs(kt).max())
        close = lambda a, ref: float(np.abs(a - ref).max()) <= tol * kscale  # noqa: E731
        if not (close(W, W[:1]) and close(E, E[:1]) and close(S, S[:, :1]) and
                close(N, N[:, :1])):
            return None
        c0 = C[0, 0]
        if not close(C, C[:1, :] + C[:, :1] - c0):
            return None
        if dim == 1 or ny == 1:
            fx = _tridiag_eig(W[0], C[0], E[0])
            if fx is None:
                return None
            vy = vyi = np.ones((1, 1))
            ly = np.zeros(1)
            vx, vxi, lx = fx
            corr_x = corr_y = None           # 1-D couples with B itself (_chain.pyx:64-71)
        else:
            fx = _tridiag_eig(W[0], C[0] - 0.5 * c0, E[0])
            fy = _tridiag_eig(S[:, 0], C[:, 0] - 0.5 * c0, N[:, 0])
            if fx is None or fy is None:
                return None
            vx, vxi, lx = fx
            vy, vyi, ly = fy
            corr_x = cls._correction(W[0], E[0], vx, vxi)
            corr_y = cls._correction(S[:, 0], N[:, 0], vy, vyi)
            if corr_x is False or corr_y is False:
                return None
        return cls(vx, vxi, lx, vy, vyi, ly, bfac, corr_x, corr_y)

    def mode_tables(self):
        """(delta, beta) per mode, y-mode slow: eigenvalues of D and B."""
        lam = (self.ly[:, None] + self.lx[None, :]).ravel()
        return 1.0 - lam, 1.0 + self.b * lam


def pcr_tables(lower: np.ndarray, diag: np.ndarray, upper: np.ndarray):
    """Matrix part of parallel cyclic reduction for the tridiagonal system
    lower[i] x[i-1] + diag[i] x[i] + upper[i] x[i+1] = r[i] (the reference
    factors the same matrix once with factor_tridiag, _chain.pyx:15-34).
    Level l (stride s = 2^l) replaces row i by itself plus alpha[l, i] times
    row i - s plus gamma[l, i] times row i + s, which removes its couplings
    at distance s and leaves couplings at distance 2 s; after ceil(log2 m)
    levels every row is diagonal.  Returns (alpha, gamma) of shape
    (levels, m) and inv = 1 / final pivots: a right-hand side is solved by
    r <- r + alpha[l] * r[. - s] + gamma[l] * r[. + s] per level, x = r * inv.
    No pivoting: D = I - a dt A is strictly diagonally dominant for the
    levels this package builds; a zero pivot raises LinAlgError as the
    reference's factorisation does (_chain.pyx:29-31)."""
    m = diag.size
    levels = int(np.ceil(np.log2(m))) if m > 1 else 0
    a = np.array(lower, dtype=np.float64)
    b = np.array(diag, dtype=np.float64)
    c = np.array(upper, dtype=np.float64)
    a[0] = 0.0
    c[-1] = 0.0
    alpha = np.zeros((levels, m))
    gamma = np.zeros((levels, m))
    for lv in range(levels):
        s = 1 << lv
        if np.any(b == 0.0):
            raise np.linalg.LinAlgError("factorization failed: zero pivot in cyclic reduction")
        al = np.zeros(m)
        ga = np.zeros(m)
        al[s:] = -a[s:] / b[:-s]
        ga[:-s] = -c[:-s] / b[s:]
        nb = b.copy()
        nb[s:] += al[s:] * c[:-s]
        nb[:-s] += ga[:-s] * a[s:]
        na = np.zeros(m)
        nc = np.zeros(m)
        na[s:] = al[s:] * a[:-s]
        nc[:-s] = ga[:-s] * c[s:]
        alpha[lv], gamma[lv] = al, ga
        a, b, c = na, nb, nc
    if np.any(b == 0.0) or not np.all(np.isfinite(b)):
        raise np.linalg.LinAlgError("factorization failed: zero pivot in cyclic reduction")
    return alpha, gamma, 1.0 / b


def line_tables(coef: np.ndarray, nx: int, ny: int):
    """Block-Thomas tables of a 5-point operator D given in row form
    (coef[s, i], slots S W C E N): D is block tridiagonal over grid lines,
    with tridiagonal T_j on the diagonal and diagonal couplings
    L_j = diag(coef[0]) / U_j = diag(coef[4]) to the lines below / above.
    G_j = (T_j - L_j G_{j-1} U_{j-1})^{-1}, dense nx x nx (the role of the
    reference's sparse LU, linalg.py:42-55).  Returns G of shape
    (ny, nx, nx)."""
    g = np.empty((ny, nx, nx))
    for j in range(ny):
        sl = slice(j * nx, (j + 1) * nx)
        t = np.diag(coef[2, sl])
        if nx > 1:
            t += np.diag(coef[1, sl][1:], -1) + np.diag(coef[3, sl][:-1], 1)
        if j > 0:
            up_prev = coef[4, (j - 1) * nx:j * nx]
            t -= coef[0, sl][:, None] * g[j - 1] * up_prev[None, :]
        try:
            g[j] = np.linalg.inv(t)
        except np.linalg.LinAlgError as exc:
            raise np.linalg.LinAlgError(f"factorization failed: {exc}") from exc
    return g


def line_cluster_size(n_chains: int) -> int:
    """CTAs per chain of the LINE kernel: the largest power of two <= 8 that
    still leaves every chain's cluster resident at once (148 SMs)."""
    cs = 8
    while cs > 1 and cs * n_chains > 148:
        cs //= 2
    return cs


def line_chunks(g: np.ndarray, cs: int) -> np.ndarray:
    """G (ny, nx, nx) re-laid for a cluster of cs CTAs per chain: CTA q owns
    rows [q R, q R + R), R = ceil(nx / cs), stored [j][q][r][c] (row-major
    chunks, zero rows past nx)."""
    ny, nx, _ = g.shape
    r = -(-nx // cs)
    pad = np.zeros((ny, cs * r, nx))
    pad[:, :nx, :] = g
    return np.ascontiguousarray(pad.reshape(ny, cs, r, nx))


# 1-D levels take PCR (a CTA per chain, (log2 m + 3) block barriers per slice)
# when the longest chain is at most this many slices: against the FFT sine
# transforms + per-mode recurrence on pristine levels, against the
# eigen-transform GEMMs on other tridiagonal levels
# (profiles/r2_coarse_kinds.md).
PCR_MAX_CHAIN_VS_DST = 8
PCR_MAX_CHAIN_VS_EIG = 40
PCR_MAX_M = 9000      # three shared-memory rows of m doubles per CTA
LINE_MAX_NX = 1536    # a line is staged by 512 threads x 3 elements
LINE_MAX_TABLE_BYTES = 16 << 30   # ny nx^2 doubles of inverted Schur blocks (host and device)


def forced_coarse_kind() -> str:
    """PMK_COARSE_KIND = pcr | line | eig | dense | dst: take that coarsest kind
    wherever it applies (tests and A/B runs); empty = the default choice."""
    import os

    return os.environ.get("PMK_COARSE_KIND", "").strip().lower()


class CoarseSolver:
    """Device tables of the block forward substitution of one level
    (reference stepper.py:114-146)."""

    def __init__(self, diag, sub, n_steps, dropped, dim, nx, ny, spectral: SpectralInfo | None):
        import torch

        _lib.require_cuda()
        self.dim, self.nx, self.ny = dim, nx, (ny if dim == 2 else 1)
        self.m = self.nx * self.ny
        self.n_steps = n_steps
        self.N = (n_steps + 1) * self.m
        mask = dropped_mask(n_steps, dropped)
        self._dropped = tuple(dropped)
        self._mask = None if mask is None else torch.from_numpy(mask).cuda()
        self._keep = []
        d = _lib.CoarseDesc()
        d.dim, d.nx, d.ny, d.n_steps = dim, self.nx, self.ny, n_steps
        d.dropped = None if self._mask is None else self._mask.data_ptr()
        forced = forced_coarse_kind()
        cuts = sorted(int(c) for c in self._dropped if c > 1)
        longest = max(b - a for a, b in zip([1] + cuts, cuts + [n_steps + 1])) if n_steps else 0
        one_d = self.ny == 1
        pcr_fits = one_d and self.nx <= PCR_MAX_M and forced not in ("eig", "dense", "dst")
        if forced == "pcr" and one_d and self.nx <= PCR_MAX_M:
            self._setup_pcr(d, diag, sub, torch)
        elif forced == "line" and not one_d and self.nx <= LINE_MAX_NX:
            self._setup_line(d, diag, sub, torch)
        elif spectral is not None and pcr_fits and 0 < longest <= PCR_MAX_CHAIN_VS_DST \
                and forced != "dst":
            self._setup_pcr(d, diag, sub, torch)
        elif spectral is not None and forced not in ("eig", "dense"):
            d.kind = _lib.PMK_COARSE_DST
            ex = dst_eigenvalues_1d(self.nx)
            tabx = fft_dst_tables(self.nx)
            taby = fft_dst_tables(self.ny) if self.ny > 1 else None
            use_fft = (tabx is not None and self.nx + 1 <= 1024
                       and (self.ny == 1 or (taby is not None and self.ny + 1 <= 512)))
            if self.ny > 1:
                ey = dst_eigenvalues_1d(self.ny)
                lam = spectral.factor * (ey[:, None] + ex[None, :])  # y-mode slow
            else:
                lam = spectral.factor * ex[None, :]
            lam = lam.ravel()
            self.kind_detail = "dst-fft" if use_fft else "dst-gemm"
            if use_fft:
                fx = torch.from_numpy(tabx).cuda()
                self._keep.append(fx)
                d.fft_x = fx.data_ptr()
                scale = 2.0 / (self.nx + 1)
                if self.ny > 1:
                    fy = torch.from_numpy(taby).cuda()
                    self._keep.append(fy)
                    d.fft_y = fy.data_ptr()
                    scale *= 2.0 / (self.ny + 1)
                d.fft_scale = scale
            delta = 1.0 - spectral.a_dt * lam
            beta = 1.0 + spectral.b_dt * lam
            tabs = [torch.from_numpy(delta).cuda(), torch.from_numpy(beta).cuda()]
            d.delta = tabs[0].data_ptr()
            d.beta = tabs[1].data_ptr()
            if not use_fft:  # dense sine matrices only for the GEMM transforms
                sx = torch.from_numpy(dst_matrix(self.nx)).cuda()
                tabs.append(sx)
                d.sx = sx.data_ptr()
                if self.ny > 1:
                    sy = torch.from_numpy(dst_matrix(self.ny)).cuda()
                    tabs.append(sy)
                    d.sy = sy.data_ptr()
            self._keep += tabs
            self.work0 = torch.empty(self.N, dtype=torch.float64, device="cuda")
            # 2-D: second transform buffer; 1-D: chunked-recurrence scratch
            self.work1 = torch.empty(self.N, dtype=torch.float64, device="cuda")
            self.kind = "dst"
        elif pcr_fits and 0 < longest <= PCR_MAX_CHAIN_VS_EIG:
            # short independent chains (perturb_decouple): a CTA per chain
            self._setup_pcr(d, diag, sub, torch)
        elif forced != "dense" \
                and (fac := SeparableFactors.detect(diag, sub, self.nx, self.ny, dim)) is not None \
                and (self.nx <= 8192 if one_d else (self.nx <= 256 and self.ny <= 512)):
            self._setup_eig(d, fac, torch)
        elif pcr_fits:
            self._setup_pcr(d, diag, sub, torch)
        elif not one_d and self.m > DENSE_MAX_M and self.nx <= LINE_MAX_NX:
            self._setup_line(d, diag, sub, torch)
        else:
            if self.m > DENSE_MAX_M:
                raise NotImplementedError(
                    f"coarsest level with {self.m} unknowns per slice whose operator is neither "
                    f"separable nor a sine-diagonal Laplacian exceeds the dense-inverse limit "
                    f"({DENSE_MAX_M})")
            d.kind = _lib.PMK_COARSE_DENSE
            dd = np.asarray(sp.csr_matrix(diag).toarray())
            try:
                dinv = np.linalg.inv(dd)
            except np.linalg.LinAlgError as exc:
                raise np.linalg.LinAlgError(f"factorization failed: {exc}") from exc
            dinv_t = torch.from_numpy(np.ascontiguousarray(dinv)).cuda()
            # coupling: B in 1-D (chain march, _chain.pyx:64-71), B^T in 2-D
            # (stepper.py:144, `out[k-1] @ sub`)
            cmat = sub if dim == 1 else sp.csr_matrix(sub).T
            self._coupling = StencilTable(cmat, self.nx, self.ny)
            d.dinv = dinv_t.data_ptr()
            d.coupling = self._coupling.desc()
            self._keep.append(dinv_t)
            self._set_chains(d, torch)
            # one work row per chain (cooperative chain kernel)
            self.work0 = torch.empty(max(d.n_seg, 1) * self.m, dtype=torch.float64,
                                     device="cuda")
            self.work1 = None
            self.kind = "dense"
        d.work0 = self.work0.data_ptr()
        d.work1 = None if self.work1 is None else self.work1.data_ptr()
        self.desc = d

    def _setup_eig(self, d, fac: "SeparableFactors", torch) -> None:
        """EIG tables: dense eigen-transforms (GEMM operands), per-mode
        eigenvalues of D and B, the 2-D low-rank B^T correction and the chain
        starts (reference segment_rows, stepper.py:107-112)."""
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()  # noqa: E731
        d.kind = _lib.PMK_COARSE_EIG
        keep = []

        def put(name, arr):
            t = dev(arr)
            keep.append(t)
            setattr(d, name, t.data_ptr())

        put("sx", fac.vxi.T)   # forward x: rows times Vx^{-T}
        put("ix", fac.vx.T)    # inverse x: rows times Vx^T
        if self.ny > 1:
            put("sy", fac.vyi)  # forward y: Vy^{-1} times the slice
            put("iy", fac.vy)
        delta, beta = fac.mode_tables()
        put("delta", delta)
        put("beta", beta)
        d.coupling_b = fac.b
        d.n_cx = d.n_cy = 0
        if self.ny > 1 and fac.corr_x is not None:
            d.n_cx = fac.corr_x[0].shape[0]
            put("cx_h", fac.corr_x[0])
            put("cx_u", fac.corr_x[1])
        if self.ny > 1 and fac.corr_y is not None:
            d.n_cy = fac.corr_y[0].shape[0]
            put("cy_h", fac.corr_y[0])
            put("cy_u", fac.corr_y[1])
        self._set_chains(d, torch)
        self._keep += keep
        self.factors = fac
        self.work0 = torch.empty(self.N, dtype=torch.float64, device="cuda")
        self.work1 = torch.empty(self.N, dtype=torch.float64, device="cuda")
        self.kind = "eig"
        self.kind_detail = "eig-chain" if (d.n_cx or d.n_cy) else "eig"

    def _coupling_table(self, d, sub) -> None:
        """C of out_k = D^{-1} (rhs_k + C out_{k-1}) as a row-form stencil:
        B in 1-D (chain march, _chain.pyx:64-71), B^T in 2-D (stepper.py:144,
        `out[k-1] @ sub`)."""
        cmat = sub if self.dim == 1 else sp.csr_matrix(sub).T
        self._coupling = StencilTable(cmat, self.nx, self.ny)
        d.coupling = self._coupling.desc()

    def _setup_pcr(self, d, diag, sub, torch) -> None:
        """PCR tables of a 1-D level (any tridiagonal D)."""
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()  # noqa: E731
        coef = StencilTable(diag, self.nx, 1).coef
        alpha, gamma, inv = pcr_tables(coef[1], coef[2], coef[3])
        d.kind = _lib.PMK_COARSE_PCR
        d.pcr_levels = int(alpha.shape[0])
        tabs = [dev(alpha if alpha.size else np.zeros(1)),
                dev(gamma if gamma.size else np.zeros(1)), dev(inv)]
        d.pcr_alpha, d.pcr_gamma, d.pcr_inv = (t.data_ptr() for t in tabs)
        self._keep += tabs
        self._coupling_table(d, sub)
        self._set_chains(d, torch)
        self.work0 = torch.empty(1, dtype=torch.float64, device="cuda")
        self.work1 = None
        self.kind = self.kind_detail = "pcr"

    def _setup_line(self, d, diag, sub, torch) -> None:
        """Block-Thomas tables of a 2-D 5-point level of any size."""
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()  # noqa: E731
        table_bytes = 8 * self.ny * self.nx * self.nx
        if table_bytes > LINE_MAX_TABLE_BYTES:
            raise NotImplementedError(
                f"coarsest level {self.nx}x{self.ny}: the block-Thomas tables of a non-separable "
                f"operator would take {table_bytes / 2**30:.1f} GiB "
                f"(limit {LINE_MAX_TABLE_BYTES / 2**30:.0f} GiB); coarsen in space first")
        coef = StencilTable(diag, self.nx, self.ny).coef
        g = line_tables(coef, self.nx, self.ny)
        d.kind = _lib.PMK_COARSE_LINE
        n_chains = 1 + sum(1 for c in self._dropped if c > 1)
        d.line_cs = line_cluster_size(n_chains)
        tabs = [dev(line_chunks(g, d.line_cs)), dev(coef[0]), dev(coef[4])]
        d.line_g, d.line_l, d.line_u = (t.data_ptr() for t in tabs)
        self._keep += tabs
        self._coupling_table(d, sub)
        self._set_chains(d, torch)
        # the y lines of every chain (line_chain_kernel)
        self.work0 = torch.empty(max(d.n_seg, 1) * 2 * self.m, dtype=torch.float64,
                                 device="cuda")
        self.work1 = None
        self.kind = self.kind_detail = "line"

    def _set_chains(self, d, torch) -> None:
        """First row of every independent chain (reference segment_rows,
        stepper.py:107-112): 1 and each dropped row > 1."""
        cuts = sorted(int(c) for c in self._dropped if c > 1)
        starts = np.array([1] + cuts, dtype=np.int32)
        st = torch.from_numpy(starts).cuda()
        self._keep.append(st)
        d.seg_start = st.data_ptr()
        d.n_seg = int(starts.size) if self.n_steps >= 1 else 0

    def solve_into(self, rhs, out) -> None:
        lib = _lib.load()
        _lib.check(lib.pmk_coarsest_solve(ctypes.byref(self.desc), _lib.ptr(rhs), _lib.ptr(out),
                                          _lib.stream_ptr()), "coarsest solve")
