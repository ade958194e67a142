"""Re-export of the solve record (reference module name kept for imports)."""

from .solver import SolveReport  # noqa: F401
