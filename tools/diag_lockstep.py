"""Lock-step c1 s=1: print per-step device vs oracle PCG traces (diagnostic)."""
import copy, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp
from oracle import ipm_oracle as O
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
from paper_2209_08722_b200.problems import wide_dense_lp
lpd = wide_dense_lp(100, 10_000, 0); A = sp.csr_matrix(lpd.A)
dlp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c))
g = lpd.gamma_run(0.1)
prm = IC.IpmParams(mode="feasible", gamma=g, sigma=0.5, w=400, s=1, tol_outer=1e-6)
oprm = O.Params(mode="feasible", gamma=g, sigma=0.5, w=400, s=1, tol_outer=1e-6)
it = IC.make_iterate(dlp, lpd.x0, lpd.y0, lpd.s0)
rng = np.random.Generator(np.random.Philox(0)); mu0, r0 = it.mu, it.residual_norm
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 24):
    st = copy.deepcopy(rng.bit_generator.state)
    x, y, s = it.x.cpu().numpy(), it.y.cpu().numpy(), it.s.cpu().numpy()
    new, rec = IC.ipm_step(dlp, it, prm, rng, r0, mu0)
    orng = np.random.Generator(np.random.Philox(0)); orng.bit_generator.state = st
    traces = []
    oit = O.make_iterate(A, lpd.b, lpd.c, x, y, s, k)
    onew, orec = O.ipm_step(A, lpd.b, lpd.c, oit, oprm, orng, r0, mu0,
                            trace_hook=lambda W, f, dy, norms: traces.append(norms))
    f0 = orec["f_norm0"]
    print(k, "inner", rec.inner_iterations, orec["inner_iterations"], "tot", rec.inner_iterations_total,
          orec["inner_iterations_total"], "vret", rec.v_retries, orec["v_retries"],
          f"mu {abs(rec.mu_after-orec['mu_after'])/orec['mu_after']:.2e}", flush=True)
    if rec.inner_iterations != orec["inner_iterations"]:
        a = np.array(rec.inner_residual_norms) / f0; b = np.array(orec["inner_residual_norms"]) / f0
        print("   dev", np.array2string(a[:len(b)] - b[:len(a)], precision=2, max_line_width=200))
        print("   dev tail", a[-5:], b[-5:])
    it = new
