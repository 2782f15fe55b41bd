"""GSGPDAT1 host-side handling (no GPU): the writer's byte layout (io.cpp:139-186) and the
BinaryRowStream header checks (io.cpp:103-113), compared with the oracle's reader."""
import numpy as np
import pytest

import paper_2101_11751_b200 as G


def test_writer_layout_and_header(tmp_path):
    rng = np.random.default_rng(0)
    x, y = rng.random((17, 3)), rng.random(17)
    p = tmp_path / "d.bin"
    G.write_dataset_binary(p, x, y)
    raw = p.read_bytes()
    assert raw[:8] == b"GSGPDAT1"
    n, d = np.frombuffer(raw[8:24], "<u8")
    assert (n, d) == (17, 3)
    rows = np.frombuffer(raw[24:], "<f8").reshape(17, 4)
    assert np.array_equal(rows[:, :3], x) and np.array_equal(rows[:, 3], y)
    s = G.BinaryRowStream(p)
    assert s.rows() == 17 and s.dim() == 3


def test_header_errors(tmp_path):
    p = tmp_path / "e.bin"
    with pytest.raises(G.InvalidArgument, match="cannot open binary dataset"):
        G.BinaryRowStream(tmp_path / "nope.bin")
    p.write_bytes(b"NOTMAGIC" + bytes(16))
    with pytest.raises(G.InvalidArgument, match="bad magic"):
        G.BinaryRowStream(p)
    p.write_bytes(b"GSGPDAT1" + bytes(4))
    with pytest.raises(G.InvalidArgument, match="row count"):
        G.BinaryRowStream(p)
    p.write_bytes(b"GSGPDAT1" + np.array([1], "<u8").tobytes())
    with pytest.raises(G.InvalidArgument, match="dimension"):
        G.BinaryRowStream(p)
    p.write_bytes(b"GSGPDAT1" + np.array([1, 65], "<u8").tobytes())
    with pytest.raises(G.InvalidArgument, match="bad dimension"):
        G.BinaryRowStream(p)
    with pytest.raises(G.InvalidArgument, match="size mismatch"):
        G.write_dataset_binary(p, np.zeros((3, 1)), np.zeros(2))
