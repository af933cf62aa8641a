"""Exception classes of the drop-in, named after the reference taxonomy
(reference errors.py:4-105) so callers catching `skipm` errors keep working.

Device status words from libskb map onto these (include/skb.h SKB_ST_*):
breakdown -> Breakdown, Cholesky pivot loss -> RankDeficient, nonpositive
scaling -> NonpositiveScaling.
"""

from __future__ import annotations


class SkipmError(Exception):
    """Root of every solver error."""


def _make(name: str, doc: str, base=SkipmError):
    return type(name, (base,), {"__doc__": doc, "__module__": __name__})


DimensionMismatch = _make("DimensionMismatch", "Operand shapes disagree with the problem.")
InvalidDensity = _make("InvalidDensity", "Fill density outside (0, 1].")
EmptyDataset = _make("EmptyDataset", "Dataset without samples or features.")
ParseError = _make("ParseError", "Malformed problem or dataset file.")
InvalidDims = _make("InvalidDims", "Sketch dimensions violate 1 <= s <= w <= n*s.")
NonpositiveScaling = _make("NonpositiveScaling", "Column scaling d must be strictly positive.")
TooLargeForDiagnostic = _make("TooLargeForDiagnostic", "Dense diagnostic refused by its size cap.")
RankDeficient = _make("RankDeficient", "ADW lost row rank (sigma ratio below tolerance).")
Breakdown = _make("Breakdown", "CG met nonpositive curvature or a negative r'z.")
InvalidZeta = _make("InvalidZeta", "zeta outside (0, 1].")
NotPositiveDefinite = _make("NotPositiveDefinite", "Cholesky of the normal matrix failed.")
TooLarge = _make("TooLarge", "Dense fallback requested beyond its cap.")
NonpositivePoint = _make("NonpositivePoint", "x or s not strictly positive.")
StaleFactor = _make("StaleFactor", "Factor built from a different sketch.")
NeighborhoodViolated = _make("NeighborhoodViolated", "Iterate outside the central-path neighborhood.")
InvariantViolated = _make("InvariantViolated", "A runtime algebraic identity failed its tolerance.")
Infeasible = _make("Infeasible", "The LP has no feasible point.")
Unbounded = _make("Unbounded", "The LP objective is unbounded below.")
Singular = _make("Singular", "Smallest singular value numerically zero.")


class ZeroRow(SkipmError):
    """A constraint row is identically zero."""

    def __init__(self, row: int):
        self.row = row
        super().__init__(f"constraint row {row} is identically zero")


class DegenerateRow(SkipmError):
    """b_i == 0 leaves phase 1 no interior slack."""

    def __init__(self, row: int):
        self.row = row
        super().__init__(f"b[{row}] == 0: row admits no interior slack")


class MaxIterations(SkipmError):
    """Outer budget exhausted; .report holds the partial SolveReport."""

    def __init__(self, message: str, report=None):
        self.report = report
        super().__init__(message)
