"""Generate the golden fixtures under tests/golden/ (committed; rerun to refresh).

The reference's own tests are empty stubs (proj/tests/*_test.cpp hold only
`#include <doctest.h>`) and the reference cannot be built here, so the fixtures pin the
oracle and the GPU path against values computed INDEPENDENTLY of both:

* keys_kat.json     — SPEC.md:185-187 known answers (Keys weights at offset 0.25, on-grid
                      identity, linear midpoint), evaluated here from the Keys formula.
* small_{1,2,3}d.npz — dense-algebra restatements in numpy: dense W from a separate Python
                      implementation of interp_weights (tests/helpers.dense_W), W^T W,
                      W^T y, y^T y, dense K_G from the SE kernel, K_G v, the posterior mean
                      coefficients  K_G W^T (W K_G W^T + σ²I)^{-1} y  (Fact 1 / Theorem 1),
                      and the exact log-likelihood terms.
* mt19937_64.json   — the first draws of the reference probe generator (std::seed_seq +
                      std::mt19937_64, gp.cpp:16-25) from a pure-Python implementation of
                      the published algorithms (C++ [rand.util.seedseq], [rand.eng.mers]).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from helpers import dense_W  # noqa: E402

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF


def seed_seq_generate(seeds, n):
    """std::seed_seq::generate for 32-bit outputs."""
    s = len(seeds)
    b = [0x8B8B8B8B] * n
    t = 11 if n >= 623 else (7 if n >= 68 else (5 if n >= 39 else (3 if n >= 7 else (n - 1) // 2)))
    p = (n - t) // 2
    q = p + t
    m = max(s + 1, n)

    def T(x):
        return (x ^ (x >> 27)) & M32

    for k in range(m):
        r1 = (1664525 * T(b[k % n] ^ b[(k + p) % n] ^ b[(k - 1) % n])) & M32
        if k == 0:
            r2 = (r1 + s) & M32
        elif k <= s:
            r2 = (r1 + (k % n) + seeds[k - 1]) & M32
        else:
            r2 = (r1 + (k % n)) & M32
        b[(k + p) % n] = (b[(k + p) % n] + r1) & M32
        b[(k + q) % n] = (b[(k + q) % n] + r2) & M32
        b[k % n] = r2
    for k in range(m, m + n):
        r3 = (1566083941 * T((b[k % n] + b[(k + p) % n] + b[(k - 1) % n]) & M32)) & M32
        r4 = (r3 - (k % n)) & M32
        b[(k + p) % n] ^= r3
        b[(k + q) % n] ^= r4
        b[k % n] = r4
    return b


class MT19937_64:
    n, m = 312, 156
    A = 0xB5026F5AA96619E9
    U, D = 29, 0x5555555555555555
    S, B = 17, 0x71D67FFFEDA60000
    T_, C = 37, 0xFFF7EEE000000000
    L = 43
    F = 6364136223846793005

    def __init__(self, seq_words):
        # seed(SeedSeq&): generate n*2 32-bit words, pair them into 64-bit state words
        w = seed_seq_generate(seq_words, self.n * 2)
        self.mt = [(w[2 * i] | (w[2 * i + 1] << 32)) & M64 for i in range(self.n)]
        # [rand.eng.mers]: if the top w-r bits of x_0 and the rest are zero, set x_0 = 2^(w-1)
        if (self.mt[0] >> 31) == 0 and all(v == 0 for v in self.mt[1:]):
            self.mt[0] = 1 << 63
        self.idx = self.n

    def _twist(self):
        mt = self.mt
        upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
        for i in range(self.n):
            y = (mt[i] & upper) | (mt[(i + 1) % self.n] & lower)
            v = mt[(i + self.m) % self.n] ^ (y >> 1)
            if y & 1:
                v ^= self.A
            mt[i] = v
        self.idx = 0

    def __call__(self):
        if self.idx >= self.n:
            self._twist()
        z = self.mt[self.idx]
        self.idx += 1
        z ^= (z >> self.U) & self.D
        z ^= (z << self.S) & self.B & M64
        z ^= (z << self.T_) & self.C & M64
        z ^= z >> self.L
        return z & M64


def probe_draws(seed, p, count):
    words = [seed & M32, (seed >> 32) & M32, p & M32, (p >> 32) & M32]
    g = MT19937_64(words)
    return [g() for _ in range(count)]


def keys(t):
    a = abs(t)
    if a <= 1.0:
        return (1.5 * a - 2.5) * a * a + 1.0
    if a < 2.0:
        return ((-0.5 * a + 2.5) * a - 4.0) * a + 2.0
    return 0.0


def se_kernel(x, x2, ls, s):
    q = 0.0
    for i in range(len(x)):
        dd = (x[i] - x2[i]) / ls[i]
        q += dd * dd
    return s * np.exp(-0.5 * q)


def small_case(d, seed):
    rng = np.random.default_rng(seed)
    sizes = {1: (24,), 2: (12, 10), 3: (8, 7, 6)}[d]
    r = 2
    mins, maxs = [], []
    for k in range(d):
        s = 1.0 / (sizes[k] - 1 - 2 * r)
        mins.append(0.0 - r * s)
        maxs.append(1.0 + r * s)
    n = {1: 150, 2: 300, 3: 400}[d]
    x = rng.random((n, d))
    x[:3] = 0.0   # boundary points (snap / zero-weight drop paths)
    x[3:5] = 1.0
    y = np.sin(3 * x).sum(axis=1) + 0.1 * rng.standard_normal(n)
    Wm = dense_W(mins, maxs, sizes, x, 4)
    m = int(np.prod(sizes))
    ls = [0.3, 0.25, 0.4][:d]
    outputscale, noise_std = 1.3, 0.2
    sp = [(maxs[k] - mins[k]) / (sizes[k] - 1) for k in range(d)]
    pts = np.array([[mins[k] + i[k] * sp[k] for k in range(d)] for i in np.ndindex(*sizes)])
    K = np.array([[se_kernel(pts[a], pts[b], ls, outputscale) for b in range(m)] for a in range(m)])
    v = rng.standard_normal(m)
    s2 = noise_std * noise_std
    A = Wm @ K @ Wm.T + s2 * np.eye(n)
    alpha = np.linalg.solve(A, y)
    mean_coeffs = K @ (Wm.T @ alpha)
    sign, logdet_n = np.linalg.slogdet(A)
    loglik = -0.5 * (logdet_n + y @ alpha + n * np.log(2 * np.pi))
    # m-system decomposition (gp.cpp:236-238): logdet_term = logdet(K WtW + s2 I)
    sign_m, logdet_m = np.linalg.slogdet(K @ (Wm.T @ Wm) + s2 * np.eye(m))
    test_pts = rng.random((20, d))
    pred = dense_W(mins, maxs, sizes, test_pts, 4) @ mean_coeffs
    return dict(mins=np.array(mins), maxs=np.array(maxs), sizes=np.array(sizes), x=x, y=y, wtw=Wm.T @ Wm,
                wty=Wm.T @ y, yty=np.array(y @ y), K=K, v=v, Kv=K @ v, lengthscales=np.array(ls),
                outputscale=np.array(outputscale), noise_std=np.array(noise_std), mean_coeffs=mean_coeffs,
                test_pts=test_pts, pred=pred, loglik=np.array(loglik), logdet_m=np.array(logdet_m),
                logdet_n=np.array(logdet_n), quad=np.array(y @ alpha))


def main():
    kat = {
        "source": "SPEC.md:185-187 (interp_weights examples)",
        "cubic_offset_0.25": {"t": 0.25, "weights": [keys(1.25), keys(0.25), keys(0.75), keys(1.75)],
                              "expected": [-0.0703125, 0.8671875, 0.2265625, -0.0234375]},
        "cubic_on_grid": {"t": 0.0, "weights": [keys(1.0), keys(0.0), keys(1.0), keys(2.0)],
                          "expected": [0.0, 1.0, 0.0, 0.0]},
        "linear_midpoint": {"t": 0.5, "expected": [0.5, 0.5]},
    }
    with open(os.path.join(HERE, "keys_kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    for d, seed in ((1, 11), (2, 12), (3, 13)):
        np.savez_compressed(os.path.join(HERE, f"small_{d}d.npz"), **small_case(d, seed))
    mt = {"source": "std::seed_seq{seed_lo, seed_hi, p_lo, p_hi} + std::mt19937_64 (gp.cpp:16-25)",
          "draws": {f"seed{s}_p{p}": [str(v) for v in probe_draws(s, p, 640)]
                    for s, p in ((0, 0), (0, 1), (0, 29), (12345678901, 3))}}
    with open(os.path.join(HERE, "mt19937_64.json"), "w") as f:
        json.dump(mt, f)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
