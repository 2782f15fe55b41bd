"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): precompute
on d = 1, 2, 3 (cubic and linear, with probe streams, both slice scatters), K_G apply, the
persistent EFCG, the probe-batched EFLA log-likelihood.  Sizes are tiny (sanitizers run ~100×
slower)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_11751_b200 as G  # noqa: E402

rng = np.random.default_rng(0)
for d, sizes, n, scheme in [(1, (60,), 40_000, G.InterpScheme.Cubic), (2, (40, 30), 60_000, G.InterpScheme.Cubic),
                            (2, (300, 300), 40_000, G.InterpScheme.Cubic), (3, (12, 10, 9), 60_000, G.InterpScheme.Cubic),
                            (3, (10, 9, 8), 30_000, G.InterpScheme.Linear)]:
    x = rng.random((n, d)).astype(np.float32 if d == 3 else np.float64)
    y = (np.cos(3 * x).sum(axis=1) + 0.1 * rng.standard_normal(n)).astype(x.dtype)
    g = G.fit_grid_to_data(np.zeros(d), np.ones(d), sizes, scheme)
    acc = G.SufficientStatsAccumulator(g, scheme)
    acc.enable_probes(5, seed=1)
    acc.add(x[: n // 2], y[: n // 2])
    acc.add(x[n // 2:], y[n // 2:])
    st = acc.finalize()
    print(d, sizes, "n", st.n(), "probes", st.probe_images().shape, flush=True)
    if scheme == G.InterpScheme.Cubic and g.num_points() < 5000:
        spec = G.KernelSpec(G.Hyperparams(0.3, [0.2] * d, 1.0))
        kg = G.ToeplitzOperator(g, spec)
        v = kg.apply(st.wty())
        m = G.posterior_mean_gsgp(st, kg, spec, scheme, 0.3, 1e-6, 20000)
        r = G.log_likelihood_gsgp(st, kg, 0.3, G.LoglikOptions(solve_tol=1e-6, probes=5, slq=G.SlqOptions(10, 0.0),
                                                                seed=1, maxiter=20000, route=G.LogdetRoute.SkiOperator))
        print("  cg iters", m.solve_iterations, "loglik", r.loglik, flush=True)
print("sanitize case done")
