"""MT19937-64 jump-ahead of the probe streams (csrc/mt_jump.cu), checked on the host against
the oracle's sequential rademacher_probe (gp.cpp:16-25: std::seed_seq + std::mt19937_64, bit 0
of each draw).  The device kernel computes the same correlation; tests/test_gpu_probes.py
checks it through the precompute."""
import numpy as np
import pytest

import oracle as O
import paper_2101_11751_b200 as G

OFFSETS = [0, 1, 155, 311, 312, 313, 624, 1000, 65_537, 1_048_320, 1_048_321, 2_096_639, 5_000_000]


@pytest.mark.parametrize("seed,p", [(0, 0), (0, 29), (12345678901, 7)])
def test_jumped_stream_matches_sequential_draws(seed, p):
    n = 400
    full = O.rademacher_probe(max(OFFSETS) + n, seed, p) > 0
    for off in OFFSETS:
        got = G.probe_stream_bits(seed, p, off, n)
        assert np.array_equal(got.astype(bool), full[off: off + n]), off


def test_substream_boundaries():
    """Substreams start every 1,048,320 draws (16 per 16.7M-row slab): the draws just before and
    after each start, reached by jump, continue the one sequential stream."""
    L = 312 * 3360
    full = O.rademacher_probe(3 * L + 64, 0, 5) > 0
    for k in (1, 2, 3):
        got = G.probe_stream_bits(0, 5, k * L - 32, 64)
        assert np.array_equal(got.astype(bool), full[k * L - 32: k * L + 32])


def test_next_fast_fft_size_matches_oracle():
    """grid.cpp:73-82 through the C ABI (host only) against the oracle's restatement."""
    for x in list(range(-2, 400)) + [1999, 2047, 4095, 5999, 19999, 123457]:
        assert G.next_fast_fft_size(x) == O.next_fast_fft_size(x), x
