"""Oracle log-likelihood on a 1e6-row prefix of BASELINE config 5 (tests/golden/loglik_config5.json).

The oracle's factorized CG at solve_tol 1e-8 (~7.7e3 iterations on a 64³ grid through the
restated circulant FFT) plus 30 probes × 50 EFLA steps takes ~25 min on 16 host threads, too long
to run inside the GPU test suite, so its result is computed once here (on the CPU, from the
numpy rows synthetic.generate(5, 1e6), which are the same on every machine) and committed;
tests/test_gpu_solve_parity.py recomputes the GPU side live and compares.

    python tests/golden/make_loglik5_golden.py      (CPU only; ~1 h on 8 threads)

The committed file was generated on the GPU box's 16 host threads (stats 105 s, log-likelihood
1367 s; log in profiles/r2u_loglik5_golden_generation.log), round 2.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

N = 1_000_000
OPTS = dict(solve_tol=1e-8, probes=30, max_depth=50, quad_tol=0.0, seed=0, route="ski-operator", maxiter=20000)


def main():
    O.set_threads(os.cpu_count() or 8)
    cfg = S.CONFIGS[5]
    x, y = S.generate(5, N)
    mins, maxs, sizes = [], [], list(cfg.sizes)
    for k in range(3):  # fit_grid_to_data(0, 1) as synthetic.grid_for
        s = 1.0 / (sizes[k] - 5)
        mins.append(0.0 - 2 * s)
        maxs.append(1.0 + 2 * s)
    og = O.fit_grid_to_data(np.zeros(3), np.ones(3), sizes)
    t0 = time.time()
    ost = O.sufficient_stats(og, x, y, nthreads=os.cpu_count() or 8)
    t1 = time.time()
    okg = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
    r = O.log_likelihood_gsgp(ost, okg, cfg.noise_std, grid=og, x=x, **OPTS)
    t2 = time.time()
    wty = ost.csr()[3]
    out = {"config": 5, "n": N, "rows": "paper_2101_11751_b200.synthetic.generate(5, 1_000_000)", "options": OPTS,
           "oracle": {k: (float(v) if isinstance(v, (float, np.floating)) else v) for k, v in r.items()},
           "stats_check": {"n": int(ost.n), "yty": float(ost.yty), "wty_sum": float(wty.sum()),
                           "wty_abs_sum": float(np.abs(wty).sum())},
           "seconds": {"stats": t1 - t0, "loglik": t2 - t1}, "threads": O.lib().orc_get_threads()}
    json.dump(out, open(os.path.join(HERE, "loglik_config5.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
