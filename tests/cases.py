"""Seeded workload definitions shared by the golden-fixture generator, the
oracle tests, the GPU parity tests and bench.py.

u0 recipes follow BASELINE.json:
  * "bump":  initial_bump + 0.1 * N(0,1) noise, rng = default_rng(seed)
  * "modes": sum of 8 sine modes, indices rng.integers(1, 17, (8, 2)) drawn
             first, then amplitudes rng.standard_normal(8)
The literal BASELINE configs run at Courant numbers 24-512, where the
reference MLK stagnates; the "_c" companions keep
the shapes and pick T so that C matches the paper (0.64 in 1-D, 0.16 in
2-D), as SURVEY.md section 8(d) recommends.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Case:
    name: str
    dim: int
    nx: int
    n_t: int
    theta: float
    n_levels: int
    schedule: tuple
    nu: int = 2
    T: float | None = None          # final time (dt = T / n_t) ...
    courant: float | None = None    # ... or dt from the Courant number
    u0: str = "bump"
    seed: int = 0
    mu: float = 1.0
    tol: float = 1e-8
    max_outer: int = 200
    inner_iters: object = None
    n_cgs: int = 0
    restart: int | None = None
    two_level_family: str | None = None   # use build_two_level(family) instead
    perturb: str | None = None   # "rowscale": A -> diag(w) A (not build_laplacian's)
    forcing: str | None = None   # "seeded": g(t, x) = N(0, 1) draws (rng seed + 1)

    @property
    def ny(self) -> int:
        return self.nx if self.dim == 2 else 1

    @property
    def m(self) -> int:
        return self.nx * self.ny

    @property
    def N(self) -> int:
        return (self.n_t + 1) * self.m

    def dx(self) -> float:
        return 1.0 / (self.nx + 1)

    def dt(self) -> float:
        if self.T is not None:
            return self.T / self.n_t
        factor = 2.0 if self.dim == 1 else 3.0
        return self.courant * self.dx() ** 2 / factor

    def u0_vector(self) -> np.ndarray:
        rng = np.random.default_rng(self.seed)
        nx, ny, h = self.nx, self.ny, self.dx()
        x = np.arange(1, nx + 1) * h
        if self.u0 == "bump":
            gx = np.sin(np.pi * x / (h * (nx + 1)))
            if self.dim == 1:
                base = gx
            else:
                y = np.arange(1, ny + 1) * h
                gy = np.sin(np.pi * y / (h * (ny + 1)))
                base = np.outer(gy, gx).ravel()
            return base + 0.1 * rng.standard_normal(self.m)
        if self.u0 == "modes":
            idx = rng.integers(1, 17, size=(8, 2))
            amp = rng.standard_normal(8)
            y = np.arange(1, ny + 1) * h
            u = np.zeros((ny, nx))
            for (p, q), a in zip(idx, amp):
                if self.dim == 1:
                    u[0] += a * np.sin(p * np.pi * x)
                else:
                    u += a * np.outer(np.sin(q * np.pi * y), np.sin(p * np.pi * x))
            return u.ravel()
        raise ValueError(self.u0)

    def forcing_array(self):
        """The source term g (n_t, m) of FineSystem (stepper.py:171-185), or None."""
        if self.forcing is None:
            return None
        if self.forcing == "seeded":
            return np.random.default_rng(self.seed + 1).standard_normal((self.n_t, self.m))
        raise ValueError(self.forcing)

    def spatial_matrix(self, a):
        """The case's spatial operator from build_laplacian's matrix `a`:
        unchanged, or row-scaled by w_i = 1 + 0.3 sin(2 pi i / n) (a
        variable-diffusivity operator: non-symmetric, not separable in 2-D)."""
        if self.perturb is None:
            return a
        if self.perturb == "rowscale":
            import scipy.sparse as sp

            n = a.shape[0]
            w = 1.0 + 0.3 * np.sin(2.0 * np.pi * np.arange(n) / n)
            return (sp.diags(w) @ a).tocsr()
        raise ValueError(self.perturb)

    def schedule_arg(self):
        """The build_hierarchy schedule argument: "auto" or a list of moves."""
        return "auto" if self.schedule == "auto" else list(self.schedule)

    def scaled(self, **kw) -> "Case":
        d = dict(self.__dict__)
        d.update(kw)
        return Case(**d)


# Small cases: the CPU oracle finishes each in well under a second.
SMALL = {
    # config-1 shape, shrunk: 1-D theta=1, 2-level T, exact coarsest
    "c1_small": Case("c1_small", 1, 15, 32, 1.0, 2, ("time",), T=0.02),
    # config-1 literal regime (C=32 at n=63): fixed budget, decoupled coarsest
    "c1_lit_small": Case("c1_lit_small", 1, 15, 32, 1.0, 2, ("time",), T=1.0, n_cgs=4,
                         max_outer=12),
    # config-2 shape, shrunk: 1-D CN, 4 levels
    "c2_small": Case("c2_small", 1, 31, 64, 0.5, 4, ("time",) * 3, courant=0.64),
    # config-3 shape, shrunk: 2-D CN, 3 levels
    "c3_small": Case("c3_small", 2, 7, 32, 0.5, 3, ("time",) * 2, courant=0.16),
    # config-4 shape, shrunk: 2-D theta=1, TS x TS nu=4 (agglomeration), odd grid
    "c4_small": Case("c4_small", 2, 15, 64, 1.0, 3, ("time_space",) * 2, nu=4, courant=0.16,
                     u0="modes", max_outer=40),
    # config-5 shape, shrunk: 2-D CN, 5 levels, perturbed decoupled coarsest
    "c5_small": Case("c5_small", 2, 15, 64, 0.5, 5, ("time",) * 4, courant=0.16, n_cgs=4),
    # same with the exact coarsest chain and FGMRES(restart)
    "c5_small_restart": Case("c5_small_restart", 2, 15, 64, 0.5, 5, ("time",) * 4,
                             courant=0.16, restart=4),
    # [time, space] schedule (space move on an odd grid: transpose semantics)
    "space_small": Case("space_small", 2, 15, 16, 1.0, 3, ("time", "space"), courant=0.16,
                        max_outer=30),
    # 2-level TS family (build_two_level)
    "ts2_small": Case("ts2_small", 1, 31, 32, 0.5, 2, ("TS",), courant=0.64,
                      two_level_family="TS", max_outer=40),
    # long 1-D horizon: the coarsest recurrence takes the chunked-scan path
    # (>= 64 coarse slices, few modes); exact and decoupled (segment cuts)
    "long1_small": Case("long1_small", 1, 31, 512, 0.5, 2, ("time",), courant=0.64,
                        max_outer=40),
    "long1_dec_small": Case("long1_dec_small", 1, 31, 512, 0.5, 2, ("time",), courant=0.64,
                            n_cgs=6, max_outer=40),
    # 2-level MGRIT family (build_two_level; injection + ideal interpolation)
    "mgrit1_small": Case("mgrit1_small", 1, 31, 32, 0.5, 2, ("MGRIT",), nu=4, courant=0.64,
                         two_level_family="MGRIT", max_outer=40),
    "mgrit2_small": Case("mgrit2_small", 2, 15, 32, 0.5, 2, ("MGRIT",), nu=2, courant=0.16,
                         two_level_family="MGRIT", max_outer=40),
    "mgrit2_dec_small": Case("mgrit2_dec_small", 2, 15, 48, 1.0, 2, ("MGRIT",), nu=3,
                             courant=0.16, two_level_family="MGRIT", n_cgs=4, max_outer=40),
}

# Round-2 coverage (golden from the live reference): the default "auto"
# schedule where the stability screen fires (space moves), grids whose n + 1
# is not a power of two (dense sine-transform GEMMs; MGRIT's GEMM path), and
# agglomerated coarsest levels (EIG: separable eigen-transforms, 2-D B^T
# coupling correction on odd grids; even grids need none).
SMALL.update({
    "auto_small": Case("auto_small", 2, 15, 32, 0.5, 4, "auto", courant=3.0, max_outer=40),
    "np2_1d_small": Case("np2_1d_small", 1, 20, 32, 0.5, 3, ("time", "time"), courant=0.64,
                         max_outer=40),
    "np2_2d_small": Case("np2_2d_small", 2, 12, 16, 1.0, 3, ("time", "time"), courant=0.16,
                         max_outer=40),
    "np2_mgrit_small": Case("np2_mgrit_small", 2, 12, 16, 0.5, 2, ("MGRIT",), nu=2,
                            courant=0.16, two_level_family="MGRIT", max_outer=40),
    "even_space_small": Case("even_space_small", 2, 12, 16, 0.5, 3, ("space", "time"),
                             courant=0.16, max_outer=40),
    "rowscale_small": Case("rowscale_small", 2, 15, 32, 0.5, 3, ("time", "time"),
                           courant=0.16, perturb="rowscale", max_outer=40),
    # forcing g != 0 and a shift mu != 1 (SolverConfig.mu, solver.py:47)
    "forced_small": Case("forced_small", 2, 15, 32, 0.5, 3, ("time", "time"), courant=0.16,
                         forcing="seeded", mu=2.5, max_outer=40),
    "forced_1d_small": Case("forced_1d_small", 1, 31, 64, 1.0, 3, ("time", "time"),
                            courant=0.64, forcing="seeded", mu=0.5, n_cgs=3, max_outer=40),
    "rowscale_dec_small": Case("rowscale_dec_small", 2, 15, 32, 1.0, 2, ("time",),
                               courant=0.16, perturb="rowscale", n_cgs=5, max_outer=40),
    "rowscale_1d_small": Case("rowscale_1d_small", 1, 31, 32, 0.5, 2, ("time",),
                              courant=0.64, perturb="rowscale", max_outer=40),
    "space_dec_small": Case("space_dec_small", 2, 15, 24, 0.5, 3, ("time", "space"),
                            courant=0.16, n_cgs=3, max_outer=40),
})

# Mid-size cases (fingerprints, not full vectors: tests/golden/make_golden.py
# --mid): realistic agglomerated coarsest levels.
MID = {
    # 1-D: coarsest 511 points x 129 slices, tridiagonal non-symmetric (3-wide group)
    "agg1_mid": Case("agg1_mid", 1, 1023, 256, 0.5, 3, ("time", "space"), courant=0.64,
                     max_outer=60),
    # the spatial-coarsening switch at the end of a time hierarchy: 127^2 -> 63^2
    "ttts_mid": Case("ttts_mid", 2, 127, 256, 0.5, 5, ("time", "time", "time", "space"),
                     courant=0.16, max_outer=60),
    # the default schedule at a Courant number where time moves fail the screen
    "auto_mid": Case("auto_mid", 2, 63, 128, 0.5, 4, "auto", courant=3.0, max_outer=60),
    # the headline grid with the switch: 255^2 x 512, coarsest 127^2 x 64 slices
    "ttts_255": Case("ttts_255", 2, 255, 512, 0.5, 5, ("time", "time", "time", "space"),
                     courant=0.16, max_outer=60),
    # a caller's own (row-scaled, non-separable) operator whose coarsest level
    # has 127^2 = 16129 unknowns per slice: past the dense-inverse limit, the
    # LINE (block Thomas) coarsest solve; exact chain and 4 decoupled chains
    "line_mid": Case("line_mid", 2, 127, 32, 0.5, 2, ("time",), courant=0.16,
                     perturb="rowscale", max_outer=60),
    "line_dec_mid": Case("line_dec_mid", 2, 127, 32, 1.0, 2, ("time",), courant=0.16,
                         perturb="rowscale", n_cgs=4, max_outer=30),
    # the headline grid: 255^2 = 65025 unknowns per coarsest slice (two rows
    # of G_j per warp, 133 MB of Schur-block inverses)
    "line_255_mid": Case("line_255_mid", 2, 255, 16, 0.5, 2, ("time",), courant=0.16,
                         perturb="rowscale", max_outer=60),
    # 1-D, 32 decoupled chains (16 slices each) of a non-Toeplitz tridiagonal
    # level: PCR, a CTA per chain
    "pcr_dec_mid": Case("pcr_dec_mid", 1, 1023, 1024, 0.5, 2, ("time",), courant=0.64,
                        perturb="rowscale", n_cgs=32, max_outer=60),
}

# EXTENSION cases (no reference counterpart, checked against the oracle's
# restatement only): full-weighting restriction / (bi)linear interpolation
# space moves with a rediscretised coarse Laplacian -- the transfers BASELINE
# config 4 names; the reference agglomerates instead.
FW = {
    # config-4 shape, shrunk: theta = 1, two time_space_fw moves, nu = 4 (15 -> 7 -> 3)
    "fw_c4_small": Case("fw_c4_small", 2, 15, 64, 1.0, 3, ("time_space_fw",) * 2, nu=4,
                        courant=0.16, u0="modes", max_outer=40),
    "fw_space_small": Case("fw_space_small", 2, 15, 16, 0.5, 3, ("time", "space_fw"),
                           courant=0.16, max_outer=40),
    "fw_1d_small": Case("fw_1d_small", 1, 31, 32, 0.5, 3, ("space_fw", "time"), courant=0.64,
                        max_outer=40),
    "fw_dec_small": Case("fw_dec_small", 2, 31, 32, 0.5, 4, ("time", "space_fw", "time"),
                         courant=0.16, n_cgs=3, max_outer=40),
}

# BASELINE.json configs (literal) and their regime-adjusted companions.
BASELINE = {
    "c1": Case("c1", 1, 63, 256, 1.0, 2, ("time",), T=1.0, n_cgs=128),
    "c2": Case("c2", 1, 1023, 4096, 0.5, 4, ("time",) * 3, T=1.0),
    "c3": Case("c3", 2, 63, 512, 0.5, 3, ("time",) * 2, T=1.0),
    "c4": Case("c4", 2, 127, 1024, 1.0, 3, ("time_space",) * 2, nu=4, T=1.0, u0="modes"),
    "c5": Case("c5", 2, 255, 4096, 0.5, 5, ("time",) * 4, T=1.0, n_cgs=256, restart=30),
    "c1_c": Case("c1_c", 1, 63, 256, 1.0, 2, ("time",), courant=0.64),
    "c2_c": Case("c2_c", 1, 1023, 4096, 0.5, 4, ("time",) * 3, courant=0.64),
    "c3_c": Case("c3_c", 2, 63, 512, 0.5, 3, ("time",) * 2, courant=0.16),
    "c4_c": Case("c4_c", 2, 127, 1024, 1.0, 3, ("time_space",) * 2, nu=4, courant=0.16,
                 u0="modes"),
    # config 4 with the transfers it names (full weighting / bilinear): extension
    "c4_fw": Case("c4_fw", 2, 127, 1024, 1.0, 3, ("time_space_fw",) * 2, nu=4, T=1.0,
                  u0="modes"),
    "c4_fw_c": Case("c4_fw_c", 2, 127, 1024, 1.0, 3, ("time_space_fw",) * 2, nu=4,
                    courant=0.16, u0="modes"),
    # headline workload: config-5 shape at the paper's Courant number, exact
    # coarsest chain (grid-independent ~19 iterations), FGMRES(30)
    "c5_c": Case("c5_c", 2, 255, 4096, 0.5, 5, ("time",) * 4, courant=0.16, restart=30),
    # decoupled variant (one independent solve per coarse slice)
    "c5_c_dec": Case("c5_c_dec", 2, 255, 4096, 0.5, 5, ("time",) * 4, courant=0.16,
                     n_cgs=256, restart=30),
    # mid-size companions the CPU oracle solves in seconds
    "mid_2d": Case("mid_2d", 2, 63, 256, 0.5, 5, ("time",) * 4, courant=0.16),
}


MID_STRIDE = 97


def mid_stride(n: int) -> int:
    """Fingerprint stride for a vector of n entries: a multiple of 97 that
    keeps about 40k samples."""
    return MID_STRIDE * max(1, -(-n // (MID_STRIDE * 40000)))


def fingerprint(v, rows):
    """A vector at a fixed stride plus the l2 norm of every time slice (the
    mid-size fixtures; the vectors themselves are too large to commit)."""
    v = np.asarray(v).ravel()
    return {"sub": np.ascontiguousarray(v[::mid_stride(v.size)]),
            "norms": np.linalg.norm(v.reshape(rows, -1), axis=1)}


def mid_inputs(case, hier_sizes):
    """Seeded (coarsest rhs, fine vector) of the mid-size records."""
    rng = np.random.default_rng(4321)
    return rng.standard_normal(hier_sizes[0]), rng.standard_normal(hier_sizes[1])


def oracle_hierarchy(case: Case):
    """Build the CPU oracle hierarchy for a case (test infrastructure)."""
    from oracle import pintmk_oracle as O

    cfg = O.Config(mu=case.mu, tol=case.tol, max_outer=case.max_outer,
                   inner_iters=case.inner_iters, coarsest_n_cgs=case.n_cgs,
                   restart=case.restart)
    if case.two_level_family == "MGRIT":
        return O.build_mgrit(case.dim, case.nx, case.ny, case.theta, case.dt(), case.n_t,
                             case.u0_vector(), cfg, nu=case.nu)
    a = None
    if case.perturb is not None:
        a = case.spatial_matrix(O.laplacian(case.dim, case.nx, case.ny)[0])
    if case.two_level_family is not None:
        fam = {"T": ["time"], "TS": ["time_space"]}[case.two_level_family]
        return O.build(case.dim, case.nx, case.ny, case.theta, case.dt(), case.n_t,
                       case.u0_vector(), 2, fam, cfg, nu=case.nu, a=a,
                       forcing=case.forcing_array())
    return O.build(case.dim, case.nx, case.ny, case.theta, case.dt(), case.n_t,
                   case.u0_vector(), case.n_levels, case.schedule_arg(), cfg, nu=case.nu, a=a,
                   forcing=case.forcing_array())


def gpu_hierarchy(case: Case, u0=None):
    """Build the device hierarchy through the product's public API."""
    import paper_2401_00228_b200 as P

    op = P.build_laplacian(case.dim, case.nx, case.ny if case.dim == 2 else 1)
    if case.perturb is not None:
        op = P.SpatialOperator(op.dim, op.n_x, op.n_y, op.delta_x, op.tau,
                               case.spatial_matrix(op.matrix))
    ops = P.build_step_operators(op, P.ThetaSchemeConfig(case.theta, case.dt(), case.n_t))
    fine = P.FineSystem(ops, case.u0_vector() if u0 is None else u0,
                        forcing=case.forcing_array())
    cfg = P.SolverConfig(mu=case.mu, tol=case.tol, max_outer=case.max_outer,
                         inner_iters=case.inner_iters, coarsest_n_cgs=case.n_cgs,
                         restart=case.restart)
    if case.two_level_family is not None:
        return P.build_two_level(fine, case.two_level_family, case.nu, cfg)
    return P.build_hierarchy(fine, case.n_levels, case.schedule_arg(), cfg, nu=case.nu)
