"""Real-time phase ledger: the reference's cost-ledger phases filled with
measured GPU kernel time.

The reference's ``CostLedger`` (parcost.py:63-122) accumulates *simulated*
work units per phase -- matvec, restriction, interpolation, coarse_solve,
orthogonalization, theta_scheme -- and attributes every charge issued from a
level >= 1 to ``coarse_solve`` (parcost.py:86-93), which is how the paper's
Table 3 "CGS fraction" is formed.  Here every kernel launch of a solve is
bracketed by CUDA events and tagged with the hierarchy level that issued it
(``_lib.profile_end_levels``); the measured microseconds are charged into the
caller's ledger through the same ``charge(phase, task_costs, parallel, level)``
interface, so a reference ``CostLedger`` works unchanged (its unit becomes
GPU microseconds), and so does ``PhaseLedger`` below.

Category -> phase at the issuing level:
  K-MV / K-MVR / K-IMV (stencil passes; restriction, shift and interpolation
  are fused into them, the reference's default weight for those is 0)
                                  -> matvec
  one-reduce MGS passes           -> orthogonalization
  MGRIT ideal interpolation       -> interpolation
  space-pair gathers / transfers  -> restriction
  sine transforms / recurrence    -> coarse_solve
  norms, Givens, back substitution, solution assembly
                                  -> krylov_other (not charged by the reference)
Stand-alone calls (the true residual, the restart wrapper's norms) are
charged at level 0.
"""

from __future__ import annotations

from . import _lib

PHASES = ("matvec", "restriction", "interpolation", "coarse_solve", "orthogonalization",
          "theta_scheme")

_CATEGORY_PHASE = {
    "march_mv": "matvec", "march_mvr": "matvec", "march_imv": "matvec",
    "mgs_pass": "orthogonalization",
    "transfer": "restriction",
    "coarse_gemm": "coarse_solve", "coarse_recurrence": "coarse_solve",
    "coarse_misc": "coarse_solve", "coarse_dst": "coarse_solve",
    "coarse_chain": "coarse_solve",
    "reduce": "krylov_other", "fgmres_small": "krylov_other", "assemble": "krylov_other",
}


def phase_of(record: dict) -> str:
    if record.get("hint"):
        return record["hint"]
    return _CATEGORY_PHASE.get(record["category"], "krylov_other")


class PhaseLedger:
    """Ledger with the reference CostLedger's interface (PHASES, charge,
    total_work, cgs_fraction, rows, elapsed, phase_elapsed, proc_work) whose
    unit is a microsecond of measured GPU kernel time.  ``records`` keeps the
    raw per-(level, category) measurements."""

    PHASES = PHASES

    def __init__(self, n_proc: int = 1, n_cgs: int = 1):
        if n_proc < 1 or n_cgs < 1:
            raise ValueError("processor counts must be positive")
        self.n_proc = n_proc
        self.n_cgs = n_cgs
        self.proc_work: dict[str, list[int]] = {}
        self.phase_elapsed: dict[str, int] = {}
        self.elapsed = 0
        self.records: list[dict] = []

    def charge(self, phase: str, task_costs, parallel: bool = True, level: int = 0) -> None:
        costs = [int(c) for c in task_costs]
        if not costs:
            return
        if min(costs) < 0:
            raise ValueError("task costs must be nonnegative")
        # work issued below the finest level is the coarse-grid solve of the
        # finest level (parcost.py:86-93)
        if level >= 1:
            phase = "coarse_solve"
        lanes = (self.n_cgs if phase == "coarse_solve" else self.n_proc) if parallel else 1
        per_lane = [sum(costs[i::lanes]) for i in range(lanes)]
        work = self.proc_work.setdefault(phase, [])
        work.extend([0] * (lanes - len(work)))
        for i, c in enumerate(per_lane):
            work[i] += c
        step = max(per_lane)
        self.phase_elapsed[phase] = self.phase_elapsed.get(phase, 0) + step
        self.elapsed += step

    def total_work(self, phase: str | None = None) -> int:
        if phase is None:
            return sum(sum(w) for w in self.proc_work.values())
        return sum(self.proc_work.get(phase, []))

    def cgs_fraction(self) -> float:
        return self.phase_elapsed.get("coarse_solve", 0) / self.elapsed if self.elapsed else 0.0

    def rows(self):
        for phase in sorted(self.proc_work):
            for p, c in enumerate(self.proc_work[phase]):
                yield phase, p, c

    # ------------------------------------------------------------- GPU extras
    def phase_ms(self) -> dict[str, float]:
        return {p: us / 1000.0 for p, us in self.phase_elapsed.items()}

    def level_ms(self) -> dict[int, dict[str, float]]:
        """{level: {kernel category: ms}} of the charged records."""
        out: dict[int, dict[str, float]] = {}
        for r in self.records:
            lv = out.setdefault(max(r["level"], 0), {})
            lv[r["category"]] = lv.get(r["category"], 0.0) + r["ms"]
        return out


def charge_records(ledger, records: list[dict]) -> None:
    """Charge measured launches (``_lib.profile_end_levels``) into any ledger
    with the CostLedger ``charge`` interface, in microseconds."""
    for r in records:
        ledger.charge(phase_of(r), [round(1000.0 * r["ms"])], parallel=False,
                      level=max(r["level"], 0))
    if isinstance(ledger, PhaseLedger):
        ledger.records.extend(records)


def measured_theta_scheme_ledger(ops, u0, forcing=None) -> PhaseLedger:
    """GPU counterpart of parcost.theta_scheme_ledger (parcost.py:141-148):
    the sequential theta-scheme march, timed on the device."""
    from .stepper import sequential_solve

    ledger = PhaseLedger()
    _lib.profile_begin(True)
    try:
        sequential_solve(ops, u0, forcing)
    finally:
        records = _lib.profile_end_levels()
    for r in records:
        ledger.charge("theta_scheme", [round(1000.0 * r["ms"])], parallel=False, level=0)
    ledger.records.extend(records)
    return ledger


def report_relative(ledger, theta_ledger) -> dict[str, float]:
    """Solve time relative to the sequential stepper and the CGS share
    (parcost.py report_relative), from measured ledgers."""
    if theta_ledger.elapsed == 0:
        raise ValueError("reference ledger is empty")
    return {"relative_total": ledger.elapsed / theta_ledger.elapsed,
            "cgs_fraction": ledger.cgs_fraction()}
