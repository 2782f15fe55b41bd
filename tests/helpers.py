"""Shared helpers for the parity tests (oracle ↔ GPU layouts)."""
import numpy as np


def half_offsets(d, W):
    E = 2 * W - 1
    S = E ** d
    c0 = (S - 1) // 2
    offs = []
    for q in range(c0, S):
        dig = []
        r = q
        for _ in range(d):
            dig.append(r % E - (W - 1))
            r //= E
        offs.append(dig[::-1])
    return np.array(offs, dtype=np.int64)


def csr_to_half_stencil(rp, col, val, sizes, W):
    """Reference CSR (SufficientStats::wtw) → half-stencil values [S_min, m]."""
    sizes = list(sizes)
    d = len(sizes)
    m = int(np.prod(sizes))
    offs = half_offsets(d, W)
    E = 2 * W - 1
    key = {tuple(o): i for i, o in enumerate(offs)}
    st = np.zeros((len(offs), m))
    rows = np.repeat(np.arange(m), np.diff(rp))
    rc = np.array(np.unravel_index(rows, sizes)).T
    cc = np.array(np.unravel_index(col, sizes)).T
    dl = cc - rc
    assert np.all(np.abs(dl) <= W - 1), "W^T W entry outside the stencil"
    for r, dd, v in zip(rows, map(tuple, dl), val):
        if dd in key:
            st[key[dd], r] = v
    return st


def rel_err(a, b, floor=0.0):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = max(np.abs(b).max(initial=0.0), floor)
    if den == 0.0:
        return float(np.abs(a - b).max(initial=0.0))
    return float(np.abs(a - b).max(initial=0.0) / den)


def dense_W(grid_mins, grid_maxs, sizes, x, W=4):
    """Independent numpy restatement of interp_weights → dense W (n × m); used for
    golden values and to cross-check the oracle."""
    sizes = list(sizes)
    d = len(sizes)
    m = int(np.prod(sizes))
    x = np.asarray(x, dtype=np.float64).reshape(-1, d)
    n = x.shape[0]
    Wm = np.zeros((n, m))

    def cubic(t):
        a = abs(t)
        if a <= 1.0:
            return (1.5 * a - 2.5) * a * a + 1.0
        if a < 2.0:
            return ((-0.5 * a + 2.5) * a - 4.0) * a + 2.0
        return 0.0

    def lin(t):
        a = abs(t)
        return 1.0 - a if a <= 1.0 else 0.0

    for i in range(n):
        starts, ws = [], []
        for k in range(d):
            sp = (grid_maxs[k] - grid_mins[k]) / (sizes[k] - 1)
            u = (x[i, k] - grid_mins[k]) / sp
            r = np.round(u)
            if abs(u - r) < 1e-9:
                u = r
            i0 = min(int(np.floor(u)), sizes[k] - 2)
            t = u - i0
            if W == 4:
                starts.append(i0 - 1)
                ws.append([cubic(t + 1.0), cubic(t), cubic(1.0 - t), cubic(2.0 - t)])
            else:
                starts.append(i0)
                ws.append([lin(t), lin(1.0 - t)])
        for combo in np.ndindex(*([W] * d)):
            w = 1.0
            idx = []
            for k, o in enumerate(combo):
                w *= ws[k][o]
                idx.append(starts[k] + o)
            if w != 0.0:
                Wm[i, np.ravel_multi_index(idx, sizes)] += w
    return Wm


def write_gsgpsst1(path, sizes_mins_maxs, scheme, rp, col, val, wty, yty, n):
    """Write statistics in the reference's save_stats layout (io.cpp:192-221): magic
    "GSGPSST1", u64 d, per dimension (f64 min, f64 max, u64 size), u64 scheme, u64 m, u64 n,
    u64 nnz, f64 yty, m × f64 W^T y, nnz × (u64 row, u64 col, f64 value) in CSR row order.
    Used to hand the ORACLE's statistics to the GPU (gsgpc_stats_load), so both solvers run on
    identical statistics."""
    mins, maxs, sizes = sizes_mins_maxs
    d = len(sizes)
    m = int(np.prod(sizes))
    with open(path, "wb") as f:
        f.write(b"GSGPSST1")
        f.write(np.array([d], np.uint64).tobytes())
        for k in range(d):
            f.write(np.array([mins[k], maxs[k]], np.float64).tobytes())
            f.write(np.array([sizes[k]], np.uint64).tobytes())
        f.write(np.array([int(scheme), m, int(n), len(val)], np.uint64).tobytes())
        f.write(np.array([yty], np.float64).tobytes())
        f.write(np.ascontiguousarray(wty, np.float64).tobytes())
        rows = np.repeat(np.arange(m), np.diff(rp))
        trip = np.zeros(len(val), dtype=[("r", "<u8"), ("c", "<u8"), ("v", "<f8")])
        trip["r"], trip["c"], trip["v"] = rows, col, val
        f.write(trip.tobytes())


def oracle_stats_from_gpu(gs):
    """The GPU's statistics as an oracle SufficientStats (CSR export → orc_stats_from_csr):
    the other direction of the identical-statistics handoff, for prefixes where the oracle's
    own hash-map precompute would take minutes."""
    import oracle as O

    rp, col, val = gs.csr()
    return O.SufficientStats.from_csr(gs.grid_size(), rp, col, val, gs.wty(), gs.yty(), gs.n())
