"""Exception taxonomy of the drop-in (reference errors.py:4-105).

When the reference package `skipm` is importable (the deployment this build
drops into), every class here IS the reference's class object: `except
skipm.errors.RankDeficient` catches the device path's RankDeficient and the
reference CLI's `except SkipmError` (cli.py:531) maps device failures to its
exit codes (cli.py:49-52). Without `skipm`, classes of the same names and
hierarchy are defined here (`_compat.py`; `SKB_STANDALONE=1` forces the
standalone definitions, and the tests exercise both).

Device status words from libskb map onto these (include/skb.h SKB_ST_*):
breakdown -> Breakdown, Cholesky pivot loss -> RankDeficient, nonpositive
scaling -> NonpositiveScaling. Raw libskb failures (negative SKB_ERR_* codes)
raise `DeviceError`, a SkipmError that is also a RuntimeError; a multi-GPU
exchange whose peer never arrived raises `CollectiveTimeout`.
"""

from __future__ import annotations

from ._compat import reference_module

_NAMES = ("SkipmError", "DimensionMismatch", "ZeroRow", "InvalidDensity", "EmptyDataset",
          "DegenerateRow", "ParseError", "InvalidDims", "NonpositiveScaling",
          "TooLargeForDiagnostic", "RankDeficient", "Breakdown", "InvalidZeta",
          "NotPositiveDefinite", "TooLarge", "NonpositivePoint", "StaleFactor",
          "NeighborhoodViolated", "InvariantViolated", "MaxIterations", "Infeasible",
          "Unbounded", "Singular")


def _reference_errors():
    ref = reference_module("errors")  # the package this build drops into
    if ref is None or not all(hasattr(ref, n) for n in _NAMES):
        return None
    return ref


_ref = _reference_errors()
REFERENCE_TAXONOMY = _ref is not None

if _ref is not None:
    globals().update({n: getattr(_ref, n) for n in _NAMES})
else:
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
    TooLargeForDiagnostic = _make("TooLargeForDiagnostic", "Dense diagnostic refused by its cap.")
    RankDeficient = _make("RankDeficient", "ADW lost row rank (sigma ratio below tolerance).")
    Breakdown = _make("Breakdown", "CG met nonpositive curvature or a negative r'z.")
    InvalidZeta = _make("InvalidZeta", "zeta outside (0, 1].")
    NotPositiveDefinite = _make("NotPositiveDefinite", "Cholesky of the normal matrix failed.")
    TooLarge = _make("TooLarge", "Dense fallback requested beyond its cap.")
    NonpositivePoint = _make("NonpositivePoint", "x or s not strictly positive.")
    StaleFactor = _make("StaleFactor", "Factor built from a different sketch.")
    NeighborhoodViolated = _make("NeighborhoodViolated",
                                 "Iterate outside the central-path neighborhood.")
    InvariantViolated = _make("InvariantViolated",
                              "A runtime algebraic identity failed its tolerance.")
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


class DeviceError(SkipmError, RuntimeError):  # type: ignore[misc,valid-type]
    """A libskb call failed (CUDA error, bad workspace, unsupported shape): a
    device-side failure with no counterpart in the CPU reference."""


class CollectiveTimeout(SkipmError):  # type: ignore[misc,valid-type]
    """A peer rank never joined an NVLink all-reduce (csrc/skb_p2p.cu); the
    result of that exchange was poisoned with NaN and the solve stops."""
