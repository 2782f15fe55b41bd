"""GSGPDAT1 ingest on the GPU: sufficient_stats(grid, scheme,
BinaryRowStream(path)) — the reference's CLI path (gsgp_main.cpp:229 over io.cpp:103-122 and
interp.cpp:244-263) — against the oracle and against the in-memory path, plus the
reference's error texts and their order (a bad row before a truncation point wins) and the
transactional guarantee (a failing file leaves the accumulator unchanged)."""
import numpy as np
import pytest

import oracle as O
import paper_2101_11751_b200 as G
from test_gpu_parity import compare_stats, ogrid

pytestmark = pytest.mark.gpu


def _data(n, d, seed):
    rng = np.random.default_rng(seed)
    x = rng.random((n, d)) * 0.9 + 0.05
    y = np.sin(3 * x).sum(axis=1) + 0.1 * rng.standard_normal(n)
    return x, y


@pytest.mark.parametrize("d,sizes,n", [(1, (40,), 20000), (2, (23, 17), 30000), (3, (11, 9, 8), 20000)])
def test_file_matches_oracle_and_memory(tmp_path, d, sizes, n):
    x, y = _data(n, d, 7 + d)
    path = tmp_path / "data.bin"
    G.write_dataset_binary(path, x, y)
    g = G.fit_grid_to_data(np.zeros(d), np.ones(d), sizes)
    stream = G.BinaryRowStream(path)
    assert stream.rows() == n and stream.dim() == d
    gs = G.sufficient_stats(g, G.InterpScheme.Cubic, stream)
    os_ = O.sufficient_stats(ogrid(g), x, y, nthreads=4)
    compare_stats(gs, os_, 4, sizes)
    gm = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    assert gm.n() == gs.n() and gm.yty() == gs.yty()
    np.testing.assert_allclose(gs.wty(), gm.wty(), rtol=0, atol=1e-12 * np.abs(gm.wty()).max())


def test_multi_chunk_file_and_append(tmp_path):
    """> 4 Mi rows: several reader chunks (pinned double buffers); appending a file to an
    accumulator that already holds rows equals one pass over all rows."""
    n = (1 << 22) + 123457
    x, y = _data(n, 1, 3)
    path = tmp_path / "big.bin"
    G.write_dataset_binary(path, x, y)
    g = G.fit_grid_to_data([0.0], [1.0], [300])
    acc = G.SufficientStatsAccumulator(g, G.InterpScheme.Cubic)
    acc.add(x[:1000], y[:1000])
    assert acc.add_file(path) == n
    st = acc.finalize()
    ref = G.sufficient_stats(g, G.InterpScheme.Cubic, np.concatenate([x[:1000], x]), np.concatenate([y[:1000], y]))
    assert st.n() == n + 1000
    assert abs(st.yty() - ref.yty()) <= 1e-12 * ref.yty()
    np.testing.assert_allclose(st.wty(), ref.wty(), rtol=1e-12, atol=1e-12 * np.abs(ref.wty()).max())
    a, _ = st.stencil()
    b, _ = ref.stencil()
    np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-11 * np.abs(b[0]).max())


def _raw(path, data: bytes):
    with open(path, "wb") as f:
        f.write(data)


def test_file_errors_match_reference_texts(tmp_path):
    g = G.Grid([G.GridDim(0.0, 10.0, 11)])
    hdr = lambda n, d: b"GSGPDAT1" + np.array([n, d], "<u8").tobytes()  # noqa: E731
    rows = np.array([[2.0, 1.0], [3.0, 2.0], [4.0, 3.0]])
    p = tmp_path / "f.bin"
    acc = G.SufficientStatsAccumulator(g, G.InterpScheme.Cubic)

    def err(data):
        _raw(p, data)
        with pytest.raises(G.InvalidArgument) as e:
            acc.add_file(p)
        return e.value

    assert "bad magic in binary dataset" in str(err(b"GSGPDAT2" + hdr(3, 1)[8:]))
    assert "truncated file while reading row count" in str(err(b"GSGPDAT1\x01"))
    assert "truncated file while reading dimension" in str(err(hdr(3, 1)[:20]))
    assert "binary dataset: bad dimension" in str(err(hdr(3, 0)))
    assert "stream/grid dimension mismatch" in str(err(hdr(3, 2)))
    # truncated inside row 3: coordinate vs response
    assert "truncated file while reading coordinate" in str(err(hdr(3, 1) + rows[:2].tobytes()))
    assert "truncated file while reading response" in str(err(hdr(3, 1) + rows.tobytes()[:-8]))
    # a bad row before the truncation point is reported first (stream order)
    bad = rows.copy()
    bad[1, 0] = 11.5
    e = err(hdr(3, 1) + bad.tobytes()[:-8])
    assert e.row == 2 and "stream row 2" in str(e) and "outside grid" in str(e)
    with pytest.raises(G.InvalidArgument, match="cannot open binary dataset"):
        acc.add_file(tmp_path / "missing.bin")
    # nothing was committed by any failed file
    _raw(p, hdr(3, 1) + rows.tobytes())
    assert acc.add_file(p) == 3
    st = acc.finalize()
    assert st.n() == 3 and st.yty() == 14.0


def test_failing_later_chunk_leaves_accumulator_unchanged(tmp_path):
    n = (1 << 22) + 5000
    x, y = _data(n, 1, 5)
    x[n - 10, 0] = 2.0  # outside [0, 1] in the second reader chunk
    path = tmp_path / "bad.bin"
    G.write_dataset_binary(path, x, y)
    g = G.fit_grid_to_data([0.0], [1.0], [64])
    acc = G.SufficientStatsAccumulator(g, G.InterpScheme.Cubic)
    acc.add(x[:100], y[:100])
    before = acc.finalize()
    wty0, yty0 = before.wty().copy(), before.yty()
    with pytest.raises(G.InvalidArgument) as e:
        acc.add_file(path)
    assert e.value.row == n - 9
    st = acc.finalize()
    assert st.n() == 100 and st.yty() == yty0
    assert np.array_equal(st.wty(), wty0)
