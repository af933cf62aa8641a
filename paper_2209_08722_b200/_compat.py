"""The reference package this build drops into, when it is importable.

`skipm` (the reference, pure Python) owns the public data classes of the
solver API: the exception taxonomy (errors.py), IpmParams, StepRecord and
SolveReport (ipm_core.py:131-173, 343-376, 588-658). When it is installed
next to this package, the drop-in uses those very class objects, so code
written against `skipm` (its CLI's JSON emitters, `except skipm.errors.X`,
`isinstance(report, skipm.SolveReport)`) works unchanged on the device path.
Only classes are taken from it; no reference function is ever called on the
product path. `SKB_STANDALONE=1` ignores an installed `skipm`.
"""

from __future__ import annotations

import os


def reference_module(name: str):
    """skipm.<name> if the reference package is importable, else None."""
    if os.environ.get("SKB_STANDALONE", "0") == "1":
        return None
    try:
        import importlib
        return importlib.import_module(f"skipm.{name}")
    except Exception:
        return None
