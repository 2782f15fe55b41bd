"""Python mirror of the reference's ``gsgp`` C++ API (proj/include/gsgp/*.hpp) on libgsgpc.

Same names, argument meaning and error behaviour as the reference for the hot path:

* ``Grid`` / ``GridDim`` / ``fit_grid_to_data``            grid.hpp:15-44, interp.hpp:168-172
* ``interp_weights``                                        interp.hpp:38-41
* ``SufficientStatsAccumulator`` / ``SufficientStats`` /
  ``sufficient_stats``                                      interp.hpp:87-160
* ``ToeplitzOperator``                                      grid.hpp:58-90
* ``factorized_cg_grid_rhs`` / ``GridRhsTolerance``         solvers.hpp:127-151
* ``posterior_mean_gsgp`` / ``PosteriorModel``              gp.hpp:101-122
* ``factorized_lanczos_fused`` (probe-batched)              solvers.hpp:178-183
* ``log_likelihood_gsgp`` / ``LoglikOptions``               gp.hpp:62-90
* ``save_stats`` / ``load_stats``                           io.hpp:82-97

Errors: ``InvalidArgument`` (a ``ValueError``; the reference's ``std::invalid_argument``,
with ``.row`` = 1-based stream row for out-of-grid points), ``SolverBreakdown``,
``SolverNonConvergence`` (``.residual_sq``, ``.iterations``), ``RuntimeError``.

Arrays: numpy arrays and CPU torch tensors are host memory; CUDA torch tensors are passed
to the library as device pointers (zero copy).  All compute runs in libgsgpc.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as _L

try:  # torch is optional for the API, required for device-resident inputs
    import torch
except Exception:  # noqa: BLE001
    torch = None


# ---------------------------------------------------------------- errors
class InvalidArgument(ValueError):
    def __init__(self, msg, row=0):
        super().__init__(msg)
        self.row = row


class SolverBreakdown(RuntimeError):
    pass


class SolverNonConvergence(RuntimeError):
    def __init__(self, msg, residual_sq=float("nan"), iterations=0):
        super().__init__(msg)
        self.residual_sq = residual_sq
        self.iterations = iterations


class GsgpcCudaError(RuntimeError):
    pass


def _raise(ctx, code, info=None):
    lib = _L.load()
    msg = lib.gsgpc_last_error(ctx).decode() if ctx else f"gsgpc error {code}"
    row = int(lib.gsgpc_last_error_row(ctx)) if ctx else 0
    if code in (_L.INVALID_ARGUMENT, _L.OUT_OF_GRID):
        raise InvalidArgument(msg, row)
    if code == _L.BREAKDOWN:
        raise SolverBreakdown(msg)
    if code == _L.NONCONVERGENCE:
        raise SolverNonConvergence(msg, info.residual_sq if info else float("nan"), info.iterations if info else 0)
    if code == _L.UNSUPPORTED:
        raise NotImplementedError(msg)
    if code == _L.CUDA_ERROR:
        raise GsgpcCudaError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------- context
class Context:
    """One device + one CUDA stream (gsgpc_ctx)."""

    def __init__(self, device: int = 0):
        lib = _L.load()
        h = C.c_void_p()
        code = lib.gsgpc_ctx_create(int(device), C.byref(h))
        if code != _L.OK:
            raise GsgpcCudaError(f"gsgpc_ctx_create(device={device}) failed with status {code}")
        self._h = h
        self.device = int(device)

    @property
    def handle(self):
        return self._h

    def check(self, code, info=None):
        if code != _L.OK:
            _raise(self._h, code, info)

    def synchronize(self):
        self.check(_L.load().gsgpc_ctx_synchronize(self._h))

    def set_stream(self, stream_ptr: int):
        self.check(_L.load().gsgpc_ctx_set_stream(self._h, C.c_void_p(stream_ptr)))

    @property
    def stream(self) -> int:
        return int(_L.load().gsgpc_ctx_stream(self._h) or 0)

    @property
    def launch_count(self) -> int:
        return int(_L.load().gsgpc_ctx_launch_count(self._h))

    def enable_phase_timing(self, on=True):
        self.check(_L.load().gsgpc_ctx_enable_phase_timing(self._h, 1 if on else 0))

    def phase_times(self):
        ms = (C.c_double * 10)()
        calls = (C.c_int64 * 10)()
        self.check(_L.load().gsgpc_ctx_phase_times(self._h, ms, calls))
        names = ["classify", "scan", "scatter", "moments", "finalize", "h2d", "split_fix", "probe_moments",
                 "probe_rng", "p9"]
        return {names[i]: (ms[i], calls[i]) for i in range(10) if calls[i]}

    def fp64_peak_tflops(self) -> float:
        v = C.c_double()
        self.check(_L.load().gsgpc_diag_fp64_peak(self._h, C.byref(v)))
        return v.value

    def fp64_tensor_tflops(self):
        """(DMMA alone, DMMA + DFMA interleaved) TFLOP/s."""
        a, b = C.c_double(), C.c_double()
        self.check(_L.load().gsgpc_diag_fp64_tensor(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def reset_phase_times(self):
        self.check(_L.load().gsgpc_ctx_reset_phase_times(self._h))

    @classmethod
    def _borrowed(cls, handle, device: int, owner):
        """A context owned by someone else (a DeviceGroup): never destroyed here."""
        c = cls.__new__(cls)
        c._h = handle
        c.device = int(device)
        c._owner = owner
        return c

    def close(self):
        if getattr(self, "_owner", None) is not None:
            self._h = None
            return
        if getattr(self, "_h", None):
            _L.load().gsgpc_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


_default_ctx = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def version() -> str:
    return _L.load().gsgpc_version().decode()


# ---------------------------------------------------------------- array plumbing
class _Arr:
    """A pointer into host or device memory plus a keep-alive reference."""

    def __init__(self, obj, dtype, writable=False):
        if torch is not None and isinstance(obj, torch.Tensor):
            want = torch.float32 if dtype == np.float32 else (torch.float64 if dtype == np.float64 else None)
            t = obj
            if want is not None and t.dtype != want:
                if writable:
                    raise InvalidArgument(f"output tensor must be {want}")
                t = t.to(want)
            if not t.is_contiguous():
                if writable:
                    raise InvalidArgument("output tensor must be contiguous")
                t = t.contiguous()
            if t.is_cuda:
                # the library runs on its own stream: the work torch queued for this tensor
                # (its producer, or the conversion above) must be complete before it reads it
                torch.cuda.current_stream(t.device).synchronize()
            self.keep = t
            self.ptr = t.data_ptr()
            self.device = t.is_cuda
            self.shape = tuple(t.shape)
        else:
            a = np.asarray(obj)
            if writable:
                if a.dtype != dtype or not a.flags.c_contiguous:
                    raise InvalidArgument("output array must be C-contiguous " + str(np.dtype(dtype)))
            else:
                a = np.ascontiguousarray(a, dtype=dtype)
            self.keep = a
            self.ptr = a.ctypes.data
            self.device = False
            self.shape = a.shape

    @property
    def vp(self):
        return C.c_void_p(self.ptr)


def _dtype_code(obj):
    if torch is not None and isinstance(obj, torch.Tensor):
        return _L.F32 if obj.dtype == torch.float32 else _L.F64
    a = np.asarray(obj)
    return _L.F32 if a.dtype == np.float32 else _L.F64


def _points(x, y, d):
    """gsgpc_points for coordinates x (n×d) and responses y (n), or packed rows x (n×(d+1)) with y=None."""
    dt = _L.F32 if (_dtype_code(x) == _L.F32 and (y is None or _dtype_code(y) == _L.F32)) else _L.F64
    npdt = np.float32 if dt == _L.F32 else np.float64
    xa = _Arr(x, npdt)
    shp = xa.shape if len(xa.shape) > 1 else (xa.shape[0], 1)
    n = shp[0]
    p = _L.Points_t()
    p.dtype = dt
    p.x = xa.ptr
    keep = [xa]
    if y is None:
        if shp[1] != d + 1:
            raise InvalidArgument(f"packed rows need d+1 = {d + 1} columns, got {shp[1]}")
        p.x_row_stride = d + 1
        for k in range(d):
            p.x_col_offset[k] = k
        p.y = xa.ptr + (d) * (4 if dt == _L.F32 else 8)
        p.y_stride = d + 1
    else:
        if shp[1] != d:
            raise InvalidArgument(f"sufficient_stats: stream/grid dimension mismatch ({shp[1]} vs {d})")
        p.x_row_stride = d
        for k in range(d):
            p.x_col_offset[k] = k
        ya = _Arr(y, npdt)
        if ya.shape[0] != n:
            raise InvalidArgument("x and y row counts differ")
        keep.append(ya)
        p.y = ya.ptr
        p.y_stride = 1
    return p, n, keep


def _coords(x, d):
    dt = _dtype_code(x)
    npdt = np.float32 if dt == _L.F32 else np.float64
    xa = _Arr(x, npdt)
    shp = xa.shape if len(xa.shape) > 1 else (xa.shape[0], 1)
    if shp[1] != d:
        raise InvalidArgument(f"interp_weights: dimension mismatch ({shp[1]} vs {d})")
    p = _L.Points_t()
    p.dtype = dt
    p.x = xa.ptr
    p.x_row_stride = d
    for k in range(d):
        p.x_col_offset[k] = k
    p.y = xa.ptr
    p.y_stride = 0
    return p, shp[0], [xa]


def _out_like(n, device_like=None):
    if device_like is not None and torch is not None and isinstance(device_like, torch.Tensor) and device_like.is_cuda:
        return torch.empty(n, dtype=torch.float64, device=device_like.device)
    return np.zeros(n, dtype=np.float64)


# ---------------------------------------------------------------- grid
class InterpScheme(enum.IntEnum):
    Linear = 0
    Cubic = 1


def stencil_radius(scheme) -> int:
    return 1 if int(scheme) == InterpScheme.Linear else 2


@dataclass
class GridDim:
    min: float = 0.0
    max: float = 1.0
    size: int = 2


class Grid:
    """Regular lattice, row-major flattening with the last dimension fastest (grid.hpp:20-44)."""

    def __init__(self, dims: Sequence[GridDim]):
        dims = list(dims)
        if not dims:
            raise InvalidArgument("Grid: need at least one dimension")
        for d in dims:
            if d.size < 2:
                raise InvalidArgument("Grid: size must be >= 2 per dimension")
            if not d.max > d.min:
                raise InvalidArgument("Grid: max must exceed min")
        self._dims = [GridDim(float(d.min), float(d.max), int(d.size)) for d in dims]

    def dim(self) -> int:
        return len(self._dims)

    def size(self, k) -> int:
        return self._dims[k].size

    def min(self, k) -> float:
        return self._dims[k].min

    def max(self, k) -> float:
        return self._dims[k].max

    def spacing(self, k) -> float:
        d = self._dims[k]
        return (d.max - d.min) / float(d.size - 1)

    def num_points(self) -> int:
        return int(np.prod([d.size for d in self._dims]))

    def dims(self) -> List[GridDim]:
        return list(self._dims)

    def flat_index(self, multi) -> int:
        f = 0
        for k, i in enumerate(multi):
            f = f * self._dims[k].size + int(i)
        return f

    def point(self, flat) -> np.ndarray:
        x = np.zeros(self.dim())
        for k in range(self.dim() - 1, -1, -1):
            i = flat % self._dims[k].size
            flat //= self._dims[k].size
            x[k] = self._dims[k].min + float(i) * self.spacing(k)
        return x

    def _c(self) -> _L.Grid_t:
        g = _L.Grid_t()
        g.dim = self.dim()
        for k, d in enumerate(self._dims):
            if k < _L.MAX_DIM:
                g.min[k], g.max[k], g.size[k] = d.min, d.max, d.size
        return g

    def __eq__(self, other):
        return isinstance(other, Grid) and self._dims == other._dims

    def __repr__(self):
        return "Grid(" + ", ".join(f"[{d.min}:{d.max}:{d.size}]" for d in self._dims) + ")"


def fit_grid_to_data(lo, hi, sizes, scheme=InterpScheme.Cubic) -> Grid:
    """interp.cpp:286-306: pad the data box by stencil_radius(scheme) cells per side."""
    lo = np.asarray(lo, dtype=np.float64).reshape(-1)
    hi = np.asarray(hi, dtype=np.float64).reshape(-1)
    sizes = [int(s) for s in sizes]
    if lo.size != hi.size or lo.size != len(sizes):
        raise InvalidArgument("fit_grid_to_data: dimension mismatch")
    r = stencil_radius(scheme)
    dims = []
    for k, m in enumerate(sizes):
        if m < 2 * r + 2:
            raise InvalidArgument(f"fit_grid_to_data: need at least {2 * r + 2} points per dimension")
        if not hi[k] > lo[k]:
            raise InvalidArgument("fit_grid_to_data: empty data range")
        s = (hi[k] - lo[k]) / float(m - 1 - 2 * r)
        dims.append(GridDim(lo[k] - r * s, hi[k] + r * s, m))
    return Grid(dims)


# ---------------------------------------------------------------- kernels
@dataclass
class Hyperparams:
    noise_std: float = 1.0
    lengthscales: Sequence[float] = field(default_factory=lambda: [1.0])
    outputscale: float = 1.0

    def __post_init__(self):
        if not self.noise_std > 0.0:
            raise InvalidArgument("Hyperparams: noise_std must be positive")
        if len(self.lengthscales) == 0:
            raise InvalidArgument("Hyperparams: need at least one lengthscale")
        if any(not float(v) > 0.0 for v in self.lengthscales):
            raise InvalidArgument("Hyperparams: lengthscales must be positive")
        if not self.outputscale > 0.0:
            raise InvalidArgument("Hyperparams: outputscale must be positive")

    def dim(self) -> int:
        return len(self.lengthscales)

    def noise_variance(self) -> float:
        return self.noise_std * self.noise_std


@dataclass
class KernelSpec:
    hyper: Hyperparams


# ---------------------------------------------------------------- interpolation weights
def interp_weights(grid: Grid, x, scheme=InterpScheme.Cubic, ctx: Optional[Context] = None):
    """Weights of one point: (indices, values), exact zeros dropped (interp.cpp:79-134)."""
    idx, w, nnz, st = interp_weights_batch(grid, np.asarray(x, dtype=np.float64).reshape(1, -1), scheme, ctx)
    if st[0] == 1:
        raise InvalidArgument("interp_weights: point outside grid")
    if st[0] == 2:
        raise InvalidArgument("interp_weights: stencil leaves the grid (point too close to the boundary for the "
                              "requested scheme)")
    return idx[0, : nnz[0]].copy(), w[0, : nnz[0]].copy()


def interp_weights_batch(grid: Grid, x, scheme=InterpScheme.Cubic, ctx: Optional[Context] = None):
    """Weights of n points on the GPU: idx (n×(2r)^d), w, nnz, status (0 ok, 1 outside, 2 leaves)."""
    ctx = ctx or default_context()
    d = grid.dim()
    p, n, keep = _coords(x, d)
    width = (2 * stencil_radius(scheme)) ** d
    idx = np.zeros((n, width), np.int64)
    w = np.zeros((n, width), np.float64)
    nnz = np.zeros(n, np.int32)
    st = np.zeros(n, np.int32)
    g = grid._c()
    ctx.check(_L.load().gsgpc_interp_weights(ctx.handle, C.byref(g), int(scheme), C.byref(p), n,
                                             idx.ctypes.data, w.ctypes.data, nnz.ctypes.data, st.ctypes.data))
    return idx, w, nnz, st


# ---------------------------------------------------------------- sufficient statistics
class SufficientStats:
    """Device-resident W^T W (symmetric 7^d-offset stencil), W^T y, y^T y, n."""

    def __init__(self, handle, grid: Grid, scheme, ctx: Context, owner=None):
        self._h = handle
        self._grid = grid
        self._scheme = InterpScheme(int(scheme))
        self._ctx = ctx
        self._owner = owner  # the accumulator that owns the handle, if any
        self._wtw_count = 0

    @property
    def handle(self):
        return self._h

    @property
    def context(self):
        return self._ctx

    def _info(self):
        m, n, yty, so = C.c_int64(), C.c_int64(), C.c_double(), C.c_int64()
        pr = C.c_int32()
        self._ctx.check(_L.load().gsgpc_stats_info(self._ctx.handle, self._h, C.byref(m), C.byref(n), C.byref(yty),
                                                   C.byref(so), C.byref(pr)))
        return m.value, n.value, yty.value, so.value, pr.value

    def grid(self) -> Grid:
        return self._grid

    def scheme(self) -> InterpScheme:
        return self._scheme

    def grid_size(self) -> int:
        return self._grid.num_points()

    def n(self) -> int:
        return self._info()[1]

    def yty(self) -> float:
        return self._info()[2]

    def n_offsets(self) -> int:
        return self._info()[3]

    def probes(self) -> int:
        return self._info()[4]

    def wty(self, out=None):
        out = np.zeros(self.grid_size()) if out is None else out
        oa = _Arr(out, np.float64, writable=True)
        self._ctx.check(_L.load().gsgpc_stats_copy_wty(self._ctx.handle, self._h, oa.vp))
        if oa.device:  # results on the library stream: complete before torch uses them
            self._ctx.synchronize()
        return out

    def stencil(self):
        """(values (n_offsets × m), offsets (n_offsets × d)) of the symmetric half stencil."""
        so = self.n_offsets()
        vals = np.zeros((so, self.grid_size()))
        offs = np.zeros((so, self._grid.dim()), np.int32)
        self._ctx.check(_L.load().gsgpc_stats_copy_stencil(self._ctx.handle, self._h, vals.ctypes.data,
                                                           offs.ctypes.data))
        return vals, offs

    def probe_images(self):
        p = self.probes()
        out = np.zeros((p, self.grid_size()))
        self._ctx.check(_L.load().gsgpc_stats_copy_probe_images(self._ctx.handle, self._h, out.ctypes.data))
        return out

    def csr(self):
        lib = _L.load()
        nnz, mx = C.c_int64(), C.c_int64()
        self._ctx.check(lib.gsgpc_stats_csr_nnz(self._ctx.handle, self._h, C.byref(nnz), C.byref(mx)))
        m = self.grid_size()
        rp = np.zeros(m + 1, np.int64)
        col = np.zeros(nnz.value, np.int64)
        val = np.zeros(nnz.value, np.float64)
        self._ctx.check(lib.gsgpc_stats_export_csr(self._ctx.handle, self._h, rp.ctypes.data, col.ctypes.data,
                                                   val.ctypes.data))
        return rp, col, val

    def wtw(self):
        """SufficientStats::wtw() as a scipy CSR matrix (interp.hpp:129)."""
        import scipy.sparse as sp

        rp, col, val = self.csr()
        m = self.grid_size()
        return sp.csr_matrix((val, col, rp), shape=(m, m))

    def max_row_nnz(self) -> int:
        nnz, mx = C.c_int64(), C.c_int64()
        self._ctx.check(_L.load().gsgpc_stats_csr_nnz(self._ctx.handle, self._h, C.byref(nnz), C.byref(mx)))
        return mx.value

    def apply_wtw(self, v, out=None):
        m = self.grid_size()
        va = _Arr(v, np.float64)
        if va.shape[0] != m:
            raise InvalidArgument("SufficientStats::apply_wtw: length mismatch")
        out = _out_like(m, v) if out is None else out
        oa = _Arr(out, np.float64, writable=True)
        self._ctx.check(_L.load().gsgpc_stats_apply_wtw(self._ctx.handle, self._h, va.vp, oa.vp))
        self._wtw_count += 1
        if oa.device:  # results on the library stream: complete before torch uses them
            self._ctx.synchronize()
        return out

    def matvec_count(self) -> int:
        return self._wtw_count

    def reduce_buffer(self):
        """(device pointer, count) of the finalized [stencil|W^T y|probe images|yty|n] buffer."""
        p, c = C.c_void_p(), C.c_int64()
        self._ctx.check(_L.load().gsgpc_stats_reduce_buffer(self._ctx.handle, self._h, C.byref(p), C.byref(c)))
        return int(p.value), int(c.value)

    def pattern_buffer(self):
        """(device pointer, count) of the per-cell zero-weight pattern bytes (W^T W structure)."""
        p, c = C.c_void_p(), C.c_int64()
        self._ctx.check(_L.load().gsgpc_stats_pattern_buffer(self._ctx.handle, self._h, C.byref(p), C.byref(c)))
        return int(p.value), int(c.value)

    def reduce_tensor(self):
        """torch view (no copy) of reduce_buffer() on the context's device."""
        from .distributed import stats_buffer_tensor

        return stats_buffer_tensor(self)

    def pattern_tensor(self):
        """torch view (no copy) of pattern_buffer() on the context's device."""
        from .distributed import stats_pattern_tensor

        return stats_pattern_tensor(self)

    def mark_reduced(self):
        self._ctx.check(_L.load().gsgpc_stats_mark_reduced(self._ctx.handle, self._h))

    def save(self, path: str):
        self._ctx.check(_L.load().gsgpc_stats_save(self._ctx.handle, self._h, path.encode()))

    def __del__(self):
        if self._owner is None and getattr(self, "_h", None):
            try:
                _L.load().gsgpc_stats_destroy(self._h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None


def memory_footprint(stats: SufficientStats) -> int:
    """interp.cpp:277-284 (GSGP mode): nnz(W^T W) + 2m."""
    rp, _, _ = stats.csr()
    return int(rp[-1]) + 2 * stats.grid_size()


class SufficientStatsAccumulator:
    """interp.hpp:87-105: one-pass accumulation; ``add`` takes a batch of rows."""

    def __init__(self, grid: Grid, scheme=InterpScheme.Cubic, ctx: Optional[Context] = None):
        self._ctx = ctx or default_context()
        self._grid = grid
        self._scheme = InterpScheme(int(scheme))
        h = C.c_void_p()
        g = grid._c()
        self._ctx.check(_L.load().gsgpc_stats_create(self._ctx.handle, C.byref(g), int(scheme), C.byref(h)))
        self._h = h
        self._rows = 0

    def add(self, x, y=None, probe_words=None, probes: int = 0):
        """Add rows: x (n×d) + y (n), or packed rows x (n×(d+1)) with y None."""
        p, n, keep = _points(x, y, self._grid.dim())
        pw = None
        if probes:
            pw = _Arr(probe_words, None) if (torch is not None and isinstance(probe_words, torch.Tensor)) else \
                _Arr(np.asarray(probe_words, dtype=np.uint64), np.uint64)
        self._ctx.check(_L.load().gsgpc_stats_add(self._ctx.handle, self._h, C.byref(p), n,
                                                  pw.vp if pw else None, int(probes)))
        self._rows += n

    def add_file(self, path) -> int:
        """Add every row of a GSGPDAT1 file (BinaryRowStream, io.cpp:103-122); returns the
        rows added.  Reading, host-to-device copies and the precompute overlap."""
        rows = C.c_int64(0)
        self._ctx.check(_L.load().gsgpc_stats_add_file(self._ctx.handle, self._h, os.fsencode(path),
                                                       C.byref(rows)))
        self._rows += rows.value
        return rows.value

    def enable_probes(self, probes: int = 30, seed: int = 0, first_row: int = 0):
        """Accumulate W^T v_p for the reference's Rademacher probes p < probes (gp.cpp:16-25),
        generated in stream order by the library; call before adding rows.  first_row: the
        global index of this accumulator's first row (a shard of one stream: the probe streams
        start there, by jump-ahead, so shard images sum to the single-pass images)."""
        self._ctx.check(_L.load().gsgpc_stats_enable_probes_at(self._ctx.handle, self._h, int(probes), int(seed),
                                                               int(first_row)))

    def reset(self):
        """Back to the freshly constructed state (buffers kept)."""
        self._ctx.check(_L.load().gsgpc_stats_reset(self._ctx.handle, self._h))
        self._rows = 0

    def merge(self, other: "SufficientStatsAccumulator"):
        self._ctx.check(_L.load().gsgpc_stats_merge(self._ctx.handle, self._h, other._h))
        self._rows += other._rows

    def finalize(self) -> SufficientStats:
        self._ctx.check(_L.load().gsgpc_stats_finalize(self._ctx.handle, self._h))
        return SufficientStats(self._h, self._grid, self._scheme, self._ctx, owner=self)

    def rows_seen(self) -> int:
        return self._rows

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                _L.load().gsgpc_stats_destroy(self._h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None


class _OwnedStats(SufficientStats):
    pass


class BinaryRowStream:
    """GSGPDAT1 dataset (io.hpp:31-45): 8-byte magic, u64 n, u64 d, n rows of (d+1) f64.
    The constructor validates the header like io.cpp:103-113; the rows are read by the
    library (gsgpc_stats_add_file) when the stream is handed to sufficient_stats."""

    def __init__(self, path):
        self.path = os.fspath(path)
        try:
            f = open(self.path, "rb")
        except OSError:
            raise InvalidArgument("cannot open binary dataset: " + self.path) from None
        with f:
            magic = f.read(8)
            if magic != DATA_MAGIC:
                raise InvalidArgument("bad magic in binary dataset: " + self.path)
            hdr = f.read(8)
            if len(hdr) < 8:
                raise InvalidArgument("truncated file while reading row count")
            self._n = int(np.frombuffer(hdr, "<u8")[0])
            hdr = f.read(8)
            if len(hdr) < 8:
                raise InvalidArgument("truncated file while reading dimension")
            self._d = int(np.frombuffer(hdr, "<u8")[0])
        if self._d < 1 or self._d > 64:
            raise InvalidArgument("binary dataset: bad dimension")

    def dim(self) -> int:
        return self._d

    def rows(self) -> int:
        return self._n


DATA_MAGIC = b"GSGPDAT1"


def next_fast_fft_size(x: int) -> int:
    """grid.cpp:73-82: the smallest 5-smooth integer >= x (the circulant embedding size)."""
    return int(_L.load().gsgpc_next_fast_fft_size(int(x)))


def probe_stream_bits(seed: int, p: int, offset: int, n: int) -> np.ndarray:
    """Bit 0 of draws [offset, offset + n) of rademacher_probe's (seed, p) stream (gp.cpp:16-25)
    reached by the library's GF(2) jump-ahead (host only; 1 = +1)."""
    out = np.zeros(max(int(n), 0), np.uint8)
    code = _L.load().gsgpc_probe_stream_bits(int(seed), int(p), int(offset), int(n), out.ctypes.data)
    if code != 0:
        raise InvalidArgument(f"gsgpc_probe_stream_bits failed ({code})")
    return out


def write_dataset_binary(path, x, y):
    """write_dataset_binary / BinaryDatasetWriter (io.cpp:139-186): GSGPDAT1, f64 AoS rows."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    y = np.asarray(y, dtype=np.float64).reshape(-1)
    if x.shape[0] != y.size:
        raise InvalidArgument("write_dataset_binary: size mismatch")
    rows = np.empty((x.shape[0], x.shape[1] + 1), dtype="<f8")
    rows[:, :-1] = x
    rows[:, -1] = y
    with open(path, "wb") as f:
        f.write(DATA_MAGIC)
        f.write(np.array([x.shape[0], x.shape[1]], dtype="<u8").tobytes())
        f.write(rows.tobytes())


def sufficient_stats(grid: Grid, scheme, x, y=None, ctx: Optional[Context] = None) -> SufficientStats:
    """interp.cpp:244-263: single pass over the rows — an in-memory stream (x, y arrays or
    packed rows) or a BinaryRowStream (GSGPDAT1 file, streamed by the library)."""
    ctx = ctx or default_context()
    if isinstance(x, BinaryRowStream):
        if x.dim() != grid.dim():
            raise InvalidArgument("sufficient_stats: stream/grid dimension mismatch")
        acc = SufficientStatsAccumulator(grid, scheme, ctx=ctx)
        acc.add_file(x.path)
        return acc.finalize()
    p, n, keep = _points(x, y, grid.dim())
    h = C.c_void_p()
    g = grid._c()
    ctx.check(_L.load().gsgpc_sufficient_stats(ctx.handle, C.byref(g), int(scheme), C.byref(p), n, C.byref(h)))
    return SufficientStats(h, grid, scheme, ctx)


class DeviceGroup:
    """Several GPUs driven from one process (gsgpc_group: SURVEY §8(b)'s
    gsgpc_ctx_create(device_ids[], ngpu)).  One context per device; `sufficient_stats` shards
    the rows over the devices and combines the per-device statistics with one all-reduce
    (NCCL for distinct devices) — the reference's merge() (interp.cpp:202-210) — so every
    device holds the full statistics for a replicated solve."""

    def __init__(self, devices):
        lib = _L.load()
        devs = [int(d) for d in devices]
        if not devs:
            raise InvalidArgument("DeviceGroup: need at least one device")
        arr = (C.c_int * len(devs))(*devs)
        h = C.c_void_p()
        code = lib.gsgpc_group_create(arr, len(devs), C.byref(h))
        if code != _L.OK:
            raise GsgpcCudaError(f"gsgpc_group_create({devs}) failed with status {code}")
        self._h = h
        self.devices = devs
        self._ctx = [Context._borrowed(lib.gsgpc_group_ctx(h, r), d, self) for r, d in enumerate(devs)]

    def __len__(self):
        return len(self.devices)

    def context(self, rank: int) -> Context:
        return self._ctx[rank]

    @property
    def uses_nccl(self) -> bool:
        n, u = C.c_int(), C.c_int()
        _L.load().gsgpc_group_info(self._h, C.byref(n), C.byref(u))
        return bool(u.value)

    def _check(self, code):
        if code != _L.OK:
            lib = _L.load()
            msg = lib.gsgpc_group_last_error(self._h).decode()
            row = int(lib.gsgpc_group_last_error_row(self._h))
            if code in (_L.INVALID_ARGUMENT, _L.OUT_OF_GRID):
                raise InvalidArgument(msg, row)
            if code == _L.UNSUPPORTED:
                raise NotImplementedError(msg)
            if code == _L.CUDA_ERROR:
                raise GsgpcCudaError(msg)
            raise RuntimeError(msg)

    def sufficient_stats(self, grid: Grid, scheme, x, y=None, probes: int = 0, seed: int = 0):
        """interp.cpp:244-263 over the group: device r takes rows [r·n/G, (r+1)·n/G); returns one
        SufficientStats per device, each the merged statistics of all rows."""
        p, n, keep = _points(x, y, grid.dim())
        g = grid._c()
        out = (C.c_void_p * len(self.devices))()
        self._check(_L.load().gsgpc_group_sufficient_stats(self._h, C.byref(g), int(scheme), C.byref(p), n,
                                                           int(probes), int(seed), out))
        del keep
        return [SufficientStats(C.c_void_p(out[r]), grid, scheme, self._ctx[r]) for r in range(len(self.devices))]

    def allreduce(self, stats):
        """The exchange step alone: per-device finalized statistics become their sum."""
        if len(stats) != len(self.devices):
            raise InvalidArgument("DeviceGroup.allreduce: one stats object per device")
        arr = (C.c_void_p * len(stats))(*[s.handle.value if hasattr(s.handle, "value") else s.handle for s in stats])
        self._check(_L.load().gsgpc_group_allreduce_stats(self._h, arr))

    def close(self):
        if getattr(self, "_h", None):
            for c in self._ctx:
                c._h = None
            _L.load().gsgpc_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def save_stats(path: str, stats: SufficientStats, grid: Grid = None, scheme=None):
    if grid is not None and grid.num_points() != stats.grid_size():
        raise InvalidArgument("save_stats: grid does not match the statistics")
    stats.save(path)


@dataclass
class StatsFile:
    grid: Grid
    scheme: InterpScheme
    stats: SufficientStats


def load_stats(path: str, ctx: Optional[Context] = None) -> StatsFile:
    ctx = ctx or default_context()
    h = C.c_void_p()
    ctx.check(_L.load().gsgpc_stats_load(ctx.handle, path.encode(), C.byref(h)))
    g = _L.Grid_t()
    sch = C.c_int()
    _L.load().gsgpc_stats_grid(h, C.byref(g), C.byref(sch))
    grid = Grid([GridDim(g.min[k], g.max[k], g.size[k]) for k in range(g.dim)])
    st = SufficientStats(h, grid, sch.value, ctx)
    return StatsFile(grid, InterpScheme(sch.value), st)


# ---------------------------------------------------------------- K_G
class ToeplitzOperator:
    """K_G on the grid for the SE-ARD kernel (grid.hpp:58-90)."""

    def __init__(self, grid: Grid, spec: KernelSpec, ctx: Optional[Context] = None, fft_min_nodes: int = 0):
        """fft_min_nodes: dimensions with at least this many nodes apply T_k by the reference's
        circulant embedding + FFT (0: the default, dimensions above 2040 nodes)."""
        self._ctx = ctx or default_context()
        if spec.hyper.dim() != grid.dim():
            raise InvalidArgument("build_toeplitz_operator: kernel/grid dimension mismatch")
        self._grid = grid
        self._spec = spec
        ls = np.asarray(spec.hyper.lengthscales, dtype=np.float64)
        h = C.c_void_p()
        g = grid._c()
        self._ctx.check(_L.load().gsgpc_kg_create_ex(self._ctx.handle, C.byref(g), ls.ctypes.data,
                                                     float(spec.hyper.outputscale), float(spec.hyper.noise_std),
                                                     int(fft_min_nodes), C.byref(h)))
        self._h = h
        self._count = 0

    @property
    def handle(self):
        return self._h

    def dim(self) -> int:
        return self._grid.num_points()

    def noise_variance(self) -> float:
        return self._spec.hyper.noise_variance()

    def grid(self) -> Grid:
        return self._grid

    def apply(self, v, out=None):
        m = self.dim()
        va = _Arr(v, np.float64)
        if va.shape[0] != m:
            raise InvalidArgument("ToeplitzOperator::apply: length mismatch")
        out = _out_like(m, v) if out is None else out
        oa = _Arr(out, np.float64, writable=True)
        self._ctx.check(_L.load().gsgpc_kg_apply(self._ctx.handle, self._h, va.vp, oa.vp))
        self._count += 1
        if oa.device:  # results on the library stream: complete before torch uses them
            self._ctx.synchronize()
        return out

    def matvec_count(self) -> int:
        return self._count

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                _L.load().gsgpc_kg_destroy(self._h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None


def build_toeplitz_operator(grid: Grid, spec: KernelSpec, ctx: Optional[Context] = None) -> ToeplitzOperator:
    return ToeplitzOperator(grid, spec, ctx)


# ---------------------------------------------------------------- solvers
kDefaultMaxIter = 1000


@dataclass
class GridRhsTolerance:
    eps_abs: float = -1.0
    rel_tol: float = -1.0


@dataclass
class GridSolveResult:
    xhat_d: np.ndarray
    iterations: int = 0
    converged: bool = False
    residual_sq: float = 0.0
    residual_trace: np.ndarray = None
    alphas: np.ndarray = None
    betas: np.ndarray = None
    loop_seconds: float = 0.0


def factorized_cg_grid_rhs(kg: ToeplitzOperator, stats: SufficientStats, rhat0, sigma: float,
                           tol: GridRhsTolerance, maxiter: int = kDefaultMaxIter) -> GridSolveResult:
    """solvers.cpp:271-336 on the GPU (device-resident α, β, ρ; CUDA-graph replay)."""
    ctx = stats.context
    m = kg.dim()
    ra = _Arr(rhat0, np.float64)
    if ra.shape[0] != m:
        raise InvalidArgument("factorized_cg_grid_rhs: dimension mismatch")
    x = np.zeros(m)
    tr = np.zeros(maxiter + 1)
    al = np.zeros(max(maxiter, 1))
    be = np.zeros(max(maxiter, 1))
    info = _L.SolveInfo_t()
    ctx.check(_L.load().gsgpc_factorized_cg_grid_rhs(ctx.handle, kg.handle, stats.handle, ra.vp, float(sigma),
                                                     float(tol.eps_abs), float(tol.rel_tol), int(maxiter),
                                                     x.ctypes.data, C.byref(info), tr.ctypes.data, al.ctypes.data,
                                                     be.ctypes.data), info)
    k = info.iterations
    nb = k - 1 if info.converged else k
    return GridSolveResult(x, k, bool(info.converged), info.residual_sq, tr[: k + 1].copy(), al[:k].copy(),
                           be[: max(nb, 0)].copy(), info.loop_seconds)


@dataclass
class PosteriorModel:
    spec: KernelSpec
    scheme: InterpScheme
    sigma: float
    mean_coeffs: np.ndarray
    kg: ToeplitzOperator
    stats: SufficientStats
    solve_iterations: int = 0
    solve_residual_sq: float = 0.0
    fit_path: str = "gsgp"
    loop_seconds: float = 0.0

    def grid(self) -> Grid:
        return self.kg.grid()

    def predict_mean(self, points, ctx: Optional[Context] = None):
        """PosteriorModel::predict_mean (gp.cpp:309-324) for one point or a batch."""
        ctx = ctx or self.stats.context
        pts = np.asarray(points, dtype=np.float64) if not (torch is not None and isinstance(points, torch.Tensor)) \
            else points
        single = getattr(pts, "ndim", 2) == 1
        if single:
            pts = pts.reshape(1, -1)
        d = self.grid().dim()
        p, n, keep = _coords(pts, d)
        out = np.zeros(n)
        mc = _Arr(self.mean_coeffs, np.float64)
        g = self.grid()._c()
        ctx.check(_L.load().gsgpc_predict_mean(ctx.handle, C.byref(g), int(self.scheme), mc.vp, C.byref(p), n,
                                               out.ctypes.data))
        return float(out[0]) if single else out


@dataclass
class CovResult:
    """gp.hpp:132-136."""
    cov: np.ndarray
    max_asymmetry: float = 0.0
    total_iterations: int = 0


def _test_points(model, points):
    pts = np.asarray(points, dtype=np.float64) if not (torch is not None and isinstance(points, torch.Tensor)) \
        else points
    if getattr(pts, "ndim", 2) == 1:
        pts = pts.reshape(1, -1)
    return _coords(pts, model.grid().dim())


def posterior_cov_exact(model: "PosteriorModel", points, tol: float, maxiter: int = kDefaultMaxIter) -> CovResult:
    """gp.cpp:381-427: exact posterior covariance between test points (one grid-rhs solve per
    point; the solves run batched on the device)."""
    ctx = model.stats.context
    p, n, keep = _test_points(model, points)
    cov = np.zeros((n, n))
    asym = C.c_double(0.0)
    iters = C.c_int32(0)
    ctx.check(_L.load().gsgpc_posterior_cov_exact(ctx.handle, model.stats.handle, model.kg.handle, float(model.sigma),
                                                  C.byref(p), n, float(tol), int(maxiter), cov.ctypes.data,
                                                  C.byref(asym), C.byref(iters)))
    return CovResult(cov, asym.value, iters.value)


class LowRankCov:
    """gp.hpp:148-167: rank-k posterior covariance from one factorized Lanczos run."""

    def __init__(self, h, model, ctx):
        self._h = h
        self._model = model
        self._ctx = ctx

    def __del__(self):
        try:
            if self._h:
                _L.load().gsgpc_lowrank_destroy(self._h)
        except Exception:
            pass

    def rank(self) -> int:
        r = C.c_int64(0)
        _L.load().gsgpc_lowrank_rank(self._h, C.byref(r))
        return r.value

    def query(self, x, x2) -> float:
        a = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        b = np.ascontiguousarray(x2, dtype=np.float64).reshape(-1)
        out = C.c_double(0.0)
        self._ctx.check(_L.load().gsgpc_lowrank_query(self._ctx.handle, self._h, a.ctypes.data, b.ctypes.data,
                                                      C.byref(out)))
        return out.value

    def cov_matrix(self, points) -> np.ndarray:
        p, n, keep = _test_points(self._model, points)
        cov = np.zeros((n, n))
        self._ctx.check(_L.load().gsgpc_lowrank_cov_matrix(self._ctx.handle, self._h, C.byref(p), n,
                                                           cov.ctypes.data))
        return cov


def posterior_cov_lowrank(model: "PosteriorModel", rank: int) -> LowRankCov:
    """gp.cpp:429-475."""
    ctx = model.stats.context
    h = C.c_void_p()
    ctx.check(_L.load().gsgpc_posterior_cov_lowrank(ctx.handle, model.stats.handle, model.kg.handle,
                                                    float(model.sigma), int(rank), C.byref(h)))
    return LowRankCov(h, model, ctx)


def posterior_mean_gsgp(stats: SufficientStats, kg: ToeplitzOperator, spec: KernelSpec, scheme, sigma: float,
                        tol: float, maxiter: int = kDefaultMaxIter) -> PosteriorModel:
    """gp.cpp:326-352."""
    ctx = stats.context
    m = kg.dim()
    out = np.zeros(m)
    info = _L.SolveInfo_t()
    ctx.check(_L.load().gsgpc_posterior_mean_gsgp(ctx.handle, stats.handle, kg.handle, float(sigma), float(tol),
                                                  int(maxiter), out.ctypes.data, C.byref(info)), info)
    return PosteriorModel(spec, InterpScheme(int(scheme)), float(sigma), out, kg, stats, info.iterations,
                          info.residual_sq, "gsgp", info.loop_seconds)


# ---------------------------------------------------------------- Lanczos / log-likelihood
@dataclass
class SlqOptions:
    max_depth: int = 100
    quad_tol: float = 0.01


class LogdetRoute(enum.IntEnum):
    """gp.hpp:55-60."""
    Auto = 0
    SymmetricGrid = 1
    SkiOperator = 2
    Dense = 3


ROUTE_NAMES = {1: "symmetric-grid-slq", 2: "ski-operator-slq", 3: "dense"}


@dataclass
class LoglikOptions:
    solve_tol: float = 0.01
    probes: int = 30
    slq: SlqOptions = field(default_factory=SlqOptions)
    seed: int = 0
    maxiter: int = kDefaultMaxIter
    route: LogdetRoute = LogdetRoute.Auto
    dense_cap: int = 2048
    probe_begin: int = 0   # SLQ probe shard [probe_begin, probe_end); (0, 0) = all probes
    probe_end: int = 0


@dataclass
class LoglikResult:
    loglik: float = 0.0
    logdet_term: float = 0.0
    quad_term: float = 0.0
    const_term: float = 0.0
    probes_used: int = 0
    solver_iterations: int = 0
    logdet_route: str = "ski-operator-slq"
    max_depth_used: int = 0
    slq_sum: float = 0.0      # probe-shard combine: logdet = Σ slq_sum / Σ slq_count + logdet_shift
    slq_count: int = 0
    logdet_shift: float = 0.0


def factorized_lanczos_fused(kg: ToeplitzOperator, stats: SufficientStats, kgwt_z0, wt_z0, z0_sq, sigma_sq: float,
                             k: int):
    """Probe-batched EFLA (solvers.cpp:464-538): kgwt_z0 / wt_z0 are P×m, z0_sq P.
    Returns (alpha P×k, beta P×k, order P)."""
    ctx = stats.context
    kw = np.ascontiguousarray(np.atleast_2d(kgwt_z0), dtype=np.float64)
    w0 = np.ascontiguousarray(np.atleast_2d(wt_z0), dtype=np.float64)
    zs = np.ascontiguousarray(np.atleast_1d(z0_sq), dtype=np.float64)
    P = kw.shape[0]
    alpha = np.zeros((P, k))
    beta = np.zeros((P, k))
    order = np.zeros(P, np.int32)
    ctx.check(_L.load().gsgpc_factorized_lanczos_fused(ctx.handle, kg.handle, stats.handle, P, kw.ctypes.data,
                                                       w0.ctypes.data, zs.ctypes.data, float(sigma_sq), int(k),
                                                       alpha.ctypes.data, beta.ctypes.data, order.ctypes.data))
    return alpha, beta, order


def log_likelihood_gsgp(stats: SufficientStats, kg: ToeplitzOperator, sigma: float,
                        opts: LoglikOptions = None) -> LoglikResult:
    """gp.cpp:158-240.  Routes (opts.route): SkiOperator over the probe images accumulated in the
    precompute (enable_probes), SymmetricGrid, Dense, or Auto (as the reference chooses)."""
    opts = opts or LoglikOptions()
    ctx = stats.context
    o = _L.LoglikOptions_t()
    o.solve_tol = opts.solve_tol
    o.probes = opts.probes
    o.max_depth = opts.slq.max_depth
    o.quad_tol = opts.slq.quad_tol
    o.seed = opts.seed
    o.maxiter = opts.maxiter
    o.route = int(opts.route)
    o.dense_cap = int(opts.dense_cap)
    o.probe_begin = int(opts.probe_begin)
    o.probe_end = int(opts.probe_end)
    r = _L.LoglikResult_t()
    ctx.check(_L.load().gsgpc_log_likelihood_gsgp(ctx.handle, stats.handle, kg.handle, float(sigma), C.byref(o),
                                                  C.byref(r)))
    return LoglikResult(r.loglik, r.logdet_term, r.quad_term, r.const_term, r.probes_used, r.solver_iterations,
                        ROUTE_NAMES.get(r.logdet_route, "?"), r.max_depth_used, r.slq_sum, r.slq_count,
                        r.logdet_shift)
