"""Drop-in boundary on the CPU: the device path's public classes are the
reference's own when `skipm` is installed (errors.py:4-105, ipm_core.py:131-173,
343-376, 588-658), and a standalone taxonomy of the same shape otherwise."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_taxonomy_is_the_reference_classes():
    skipm = pytest.importorskip("skipm")
    import skipm.errors as RE

    from paper_2209_08722_b200 import _lib, errors
    for name in errors._NAMES:
        assert getattr(errors, name) is getattr(RE, name), name
    assert errors.REFERENCE_TAXONOMY
    # raw libskb failures and collective timeouts are SkipmErrors too: the
    # reference CLI's `except SkipmError` (cli.py:531) maps them to exit code 2
    assert issubclass(_lib.SkbError, RE.SkipmError)
    assert issubclass(_lib.SkbError, RuntimeError)
    assert issubclass(errors.CollectiveTimeout, RE.SkipmError)
    try:
        raise errors.RankDeficient("x")
    except skipm.errors.RankDeficient:
        pass
    e = errors.MaxIterations("budget", report="r")
    assert isinstance(e, skipm.MaxIterations) and e.report == "r"


def test_public_dataclasses_are_the_reference_classes():
    skipm = pytest.importorskip("skipm")
    import paper_2209_08722_b200 as skb
    assert skb.IpmParams is skipm.IpmParams
    assert skb.SolveReport is skipm.SolveReport
    assert skb.StepRecord is skipm.ipm_core.StepRecord
    from paper_2209_08722_b200.ipm_core import _as_params
    p = skipm.IpmParams(mode="feasible", gamma=0.7, w=64, s=4)
    assert _as_params(p) is p


def test_standalone_taxonomy_without_the_reference():
    code = (
        "import paper_2209_08722_b200 as skb\n"
        "from paper_2209_08722_b200 import errors, _lib\n"
        "from paper_2209_08722_b200.ipm_core import _as_params\n"
        "import sys\n"
        "assert not errors.REFERENCE_TAXONOMY\n"
        "assert errors.SkipmError.__module__ == 'paper_2209_08722_b200.errors'\n"
        "for n in errors._NAMES:\n"
        "    c = getattr(errors, n)\n"
        "    assert c is errors.SkipmError or issubclass(c, errors.SkipmError), n\n"
        "assert issubclass(_lib.SkbError, errors.SkipmError)\n"
        "e = errors.MaxIterations('m', report=3); assert e.report == 3\n"
        "assert errors.ZeroRow(4).row == 4\n"
        "assert skb.IpmParams.__module__ == 'paper_2209_08722_b200.ipm_core'\n"
        "try:\n"
        "    import skipm\n"
        "    q = _as_params(skipm.IpmParams(mode='feasible', gamma=0.6, w=32))\n"
        "    assert isinstance(q, skb.IpmParams) and q.gamma == 0.6 and q.w == 32\n"
        "except ImportError:\n"
        "    pass\n"
        "print('ok')\n")
    env = dict(os.environ, SKB_STANDALONE="1",
               PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "baseline", "_ref")]))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=ROOT, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr
