"""Concurrent solves from a thread pool, as the reference's run_comparison does
(oracle_bench.py:217-238): per-thread scratch and PCG buffers keep the solves
independent, so each concurrent result equals the same solve run alone."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_thread_pool_solves_match_sequential():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_08722_b200 import ipm_core as IC
    from paper_2209_08722_b200.lp_model import LinearProgram
    from paper_2209_08722_b200.problems import wide_dense_lp
    lpd = wide_dense_lp(40, 3000, 5)
    lp = LinearProgram(lpd.A, lpd.b, lpd.c)
    base = dict(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, tol_outer=1e-6)
    configs = [dict(base, solver="pcg", w=160, s=4, seed=1),
               dict(base, solver="chebyshev", w=1200, s=12, seed=2),
               dict(base, solver="pcg", w=320, s=2, seed=3),
               dict(base, solver="direct", w=160, s=4, seed=4)]

    def run(kw):
        st = IC.make_iterate(IC._to_device_lp(lp, None), lpd.x0, lpd.y0, lpd.s0)
        rep = IC.solve(lp, st, IC.IpmParams(**kw))
        torch.cuda.synchronize()
        return rep.outer, rep.mu_trace, rep.x

    alone = [run(kw) for kw in configs]
    with ThreadPoolExecutor(max_workers=len(configs)) as pool:
        together = list(pool.map(run, configs))
    for (o1, mu1, x1), (o2, mu2, x2) in zip(alone, together):
        assert o1 == o2 and mu1 == mu2 and np.array_equal(x1, x2)
