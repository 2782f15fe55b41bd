"""TEST INFRASTRUCTURE ONLY — ctypes front-end of the CPU oracle (gsgp_oracle.cpp).

The oracle restates the reference hot path (arXiv 2101.11751 C++ reference,
/root/reference/proj) on the CPU.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this module,
and only as the checker / CPU baseline.  The product path never routes through it.

Parity status: the reference's own build cannot run in this image (Eigen3, FFTW3 and
nlohmann-json are absent), and its own tests are empty stubs.  The restatement is pinned
(1) against the reference's OWN SOURCES compiled where they lie against self-written stand-ins
for those headers (``oracle/refshim``, ``oracle/ref.py``, ``tests/test_ref_pin.py``: grids,
weights, statistics, probes bit-exact; solves to round-off) and (2) against the SPEC.md
known-answer examples and independent numpy fixtures (``tests/golden``).  What stays unpinned
is the bit pattern of real Eigen's / FFTW's internal reductions.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libgsgp_oracle.so")

OK, INVALID_ARGUMENT, OUT_OF_GRID, BREAKDOWN, NONCONVERGENCE = 0, 1, 2, 3, 4
RUNTIME_ERROR = 7
LINEAR, CUBIC = 0, 1


class OracleError(RuntimeError):
    def __init__(self, code, msg, row=0):
        super().__init__(msg)
        self.code = code
        self.row = row


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (idempotent)."""
    src = os.path.join(_HERE, "gsgp_oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE], check=True, stdout=subprocess.DEVNULL)
    return _LIB_PATH


_lib = None

_P = C.POINTER
_d = C.c_double
_i64 = C.c_int64
_pd = _P(C.c_double)
_pi64 = _P(C.c_int64)
_pi = _P(C.c_int)
_vp = C.c_void_p


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    L = C.CDLL(_LIB_PATH)
    sig = {
        "orc_last_error": (C.c_char_p, []),
        "orc_last_error_row": (_i64, []),
        "orc_fit_grid_to_data": (C.c_int, [C.c_int, _pd, _pd, _pi64, C.c_int, _pd, _pd]),
        "orc_interp_weights": (C.c_int, [C.c_int, _pd, _pd, _pi64, C.c_int, _pd, _pi64, _pd, _pi]),
        "orc_sufficient_stats": (C.c_int, [C.c_int, _pd, _pd, _pi64, C.c_int, _vp, _vp, _i64, C.c_int, _P(_vp)]),
        "orc_sufficient_stats_f32": (C.c_int, [C.c_int, _pd, _pd, _pi64, C.c_int, _vp, _vp, _i64, C.c_int, _P(_vp)]),
        "orc_stats_destroy": (None, [_vp]),
        "orc_stats_info": (None, [_vp, _pi64, _pi64, _pi64, _pd]),
        "orc_stats_export": (None, [_vp, _vp, _vp, _vp, _vp]),
        "orc_stats_from_csr": (C.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _d, _i64, _P(_vp)]),
        "orc_stats_apply_wtw": (C.c_int, [_vp, _vp, _vp]),
        "orc_stats_max_row_nnz": (_i64, [_vp]),
        "orc_kg_create": (C.c_int, [C.c_int, _pd, _pd, _pi64, _pd, _d, _d, _P(_vp)]),
        "orc_kg_destroy": (None, [_vp]),
        "orc_kg_dim": (_i64, [_vp]),
        "orc_kg_embed_shape": (None, [_vp, _pi64]),
        "orc_kg_apply": (C.c_int, [_vp, _vp, _vp]),
        "orc_kernel_generator": (C.c_int, [_vp, _vp]),
        "orc_kg_dense": (C.c_int, [_vp, _vp, _i64]),
        "orc_next_fast_fft_size": (_i64, [_i64]),
        "orc_kg_set_direct": (None, [_vp, C.c_int]),
        "orc_set_threads": (None, [C.c_int]),
        "orc_get_threads": (C.c_int, []),
        "orc_factorized_cg_grid_rhs": (C.c_int, [_vp, _vp, _vp, _d, _d, _d, C.c_int, _vp, _pi, _pi, _pd, _vp, _vp, _vp, _pd]),
        "orc_posterior_mean_gsgp": (C.c_int, [_vp, _vp, _d, _d, C.c_int, _vp, _pi, _pd]),
        "orc_predict_mean": (C.c_int, [C.c_int, _pd, _pd, _pi64, C.c_int, _vp, _vp, _i64, _vp]),
        "orc_rademacher_probe": (None, [_i64, C.c_uint64, C.c_uint64, _vp]),
        "orc_rademacher_bits": (None, [_i64, C.c_uint64, C.c_int, _vp, C.c_int]),
        "orc_wt_apply": (C.c_int, [C.c_int, _pd, _pd, _pi64, C.c_int, _vp, _i64, _vp, _vp]),
        "orc_factorized_lanczos_fused": (C.c_int, [_vp, _vp, _vp, _vp, _d, _d, C.c_int, _vp, _vp, _vp, _vp, _pi]),
        "orc_quadrature_logdet": (C.c_int, [_vp, _vp, C.c_int, _d, _d, _pd, _pi]),
        "orc_tridiag_eig": (C.c_int, [C.c_int, _vp, _vp, _vp, _vp]),
        "orc_slq_logdet_ski_factorized": (C.c_int, [_vp, _vp, C.c_int, _pd, _pd, _pi64, C.c_int, _vp, _i64, _d, C.c_int, C.c_int, _d, C.c_uint64, _pd, _pi]),
        "orc_posterior_cov_exact": (C.c_int, [_vp, _vp, C.c_int, _d, _vp, _i64, _d, C.c_int, _vp, _pd, _pi]),
        "orc_posterior_cov_lowrank": (C.c_int, [_vp, _vp, C.c_int, _d, _i64, _vp, _i64, _vp, _vp, _vp, _pd, _pi]),
        "orc_log_likelihood_gsgp": (C.c_int, [_vp, _vp, _d, _d, C.c_int, C.c_int, _d, C.c_uint64, C.c_int, _i64, C.c_int, C.c_int, _pd, _pd, _pi64, C.c_int, _vp, _i64, _vp, _vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(code):
    if code != OK:
        L = lib()
        raise OracleError(code, L.orc_last_error().decode(), int(L.orc_last_error_row()))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _dp(a):
    return a.ctypes.data_as(_pd)


def _ip(a):
    return a.ctypes.data_as(_pi64)


@dataclass
class Grid:
    """gsgp::Grid (grid.hpp:15-44): per-dimension min, max, size."""

    mins: np.ndarray
    maxs: np.ndarray
    sizes: np.ndarray

    def __post_init__(self):
        self.mins = _f64(self.mins).reshape(-1)
        self.maxs = _f64(self.maxs).reshape(-1)
        self.sizes = np.ascontiguousarray(self.sizes, dtype=np.int64).reshape(-1)

    @property
    def dim(self):
        return int(self.mins.size)

    @property
    def m(self):
        return int(np.prod(self.sizes))

    def args(self):
        return (self.dim, _dp(self.mins), _dp(self.maxs), _ip(self.sizes))


def fit_grid_to_data(lo, hi, sizes, scheme=CUBIC) -> Grid:
    lo, hi = _f64(lo).reshape(-1), _f64(hi).reshape(-1)
    sizes = np.ascontiguousarray(sizes, dtype=np.int64).reshape(-1)
    mn, mx = np.zeros_like(lo), np.zeros_like(lo)
    _check(lib().orc_fit_grid_to_data(lo.size, _dp(lo), _dp(hi), _ip(sizes), scheme, _dp(mn), _dp(mx)))
    return Grid(mn, mx, sizes)


def interp_weights(grid: Grid, x, scheme=CUBIC):
    x = _f64(x).reshape(-1)
    cap = 4 ** grid.dim
    idx = np.zeros(cap, np.int64)
    w = np.zeros(cap, np.float64)
    nnz = C.c_int(0)
    _check(lib().orc_interp_weights(*grid.args(), scheme, _dp(x), _ip(idx), _dp(w), C.byref(nnz)))
    return idx[: nnz.value].copy(), w[: nnz.value].copy()


class SufficientStats:
    """gsgp::SufficientStats (interp.hpp:107-146) held by the oracle."""

    def __init__(self, handle):
        self._h = handle
        m, n, nnz, yty = _i64(), _i64(), _i64(), _d()
        lib().orc_stats_info(self._h, C.byref(m), C.byref(n), C.byref(nnz), C.byref(yty))
        self.m, self.n, self.nnz, self.yty = m.value, n.value, nnz.value, yty.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_stats_destroy(self._h)
            self._h = None

    def csr(self):
        rp = np.zeros(self.m + 1, np.int64)
        col = np.zeros(self.nnz, np.int64)
        val = np.zeros(self.nnz, np.float64)
        wty = np.zeros(self.m, np.float64)
        lib().orc_stats_export(self._h, _ptr(rp), _ptr(col), _ptr(val), _ptr(wty))
        return rp, col, val, wty

    @property
    def wty(self):
        return self.csr()[3]

    def apply_wtw(self, v):
        v = _f64(v)
        out = np.zeros(self.m)
        _check(lib().orc_stats_apply_wtw(self._h, _ptr(v), _ptr(out)))
        return out

    def max_row_nnz(self):
        return int(lib().orc_stats_max_row_nnz(self._h))

    def dense_wtw(self):
        rp, col, val, _ = self.csr()
        a = np.zeros((self.m, self.m))
        for i in range(self.m):
            a[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
        return a

    @classmethod
    def from_csr(cls, m, row_ptr, col, val, wty, yty, n):
        h = C.c_void_p()
        rp = np.ascontiguousarray(row_ptr, np.int64)
        cl = np.ascontiguousarray(col, np.int64)
        vl, wy = _f64(val), _f64(wty)
        _check(lib().orc_stats_from_csr(m, cl.size, _ptr(rp), _ptr(cl), _ptr(vl), _ptr(wy), yty, n, C.byref(h)))
        return cls(h)


def sufficient_stats(grid: Grid, x, y, scheme=CUBIC, nthreads=1) -> SufficientStats:
    """gsgp::sufficient_stats (interp.cpp:244-263) over in-memory rows (stream order)."""
    x = np.asarray(x)
    n = int(np.asarray(y).shape[0])
    x = x.reshape(n, grid.dim)
    h = C.c_void_p()
    if x.dtype == np.float32:
        xs = np.ascontiguousarray(x, np.float32)
        ys = np.ascontiguousarray(y, np.float32)
        code = lib().orc_sufficient_stats_f32(*grid.args(), scheme, _ptr(xs), _ptr(ys), n, nthreads, C.byref(h))
    else:
        xs = _f64(x)
        ys = _f64(y)
        code = lib().orc_sufficient_stats(*grid.args(), scheme, _ptr(xs), _ptr(ys), n, nthreads, C.byref(h))
    _check(code)
    return SufficientStats(h)


class ToeplitzOperator:
    """gsgp::ToeplitzOperator (grid.hpp:58-90) with the SE kernel."""

    def __init__(self, grid: Grid, lengthscales, outputscale, noise_std):
        self.grid = grid
        ls = _f64(lengthscales).reshape(-1)
        h = C.c_void_p()
        _check(lib().orc_kg_create(*grid.args(), _dp(ls), float(outputscale), float(noise_std), C.byref(h)))
        self._h = h
        self.noise_variance = float(noise_std) * float(noise_std)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_kg_destroy(self._h)
            self._h = None

    @property
    def dim(self):
        return int(lib().orc_kg_dim(self._h))

    def embed_shape(self):
        s = np.zeros(self.grid.dim, np.int64)
        lib().orc_kg_embed_shape(self._h, _ip(s))
        return s

    def apply(self, v):
        v = _f64(v)
        out = np.zeros(self.dim)
        _check(lib().orc_kg_apply(self._h, _ptr(v), _ptr(out)))
        return out

    def set_direct(self, on=True):
        """Sensitivity study only: direct separable Toeplitz sums instead of the circulant FFT
        (same operator, different rounding)."""
        lib().orc_kg_set_direct(self._h, 1 if on else 0)

    def generator(self):
        out = np.zeros(self.dim)
        _check(lib().orc_kernel_generator(self._h, _ptr(out)))
        return out

    def dense(self, max_points=8192):
        m = self.dim
        out = np.zeros((m, m))
        _check(lib().orc_kg_dense(self._h, _ptr(out), max_points))
        return out


def set_threads(n: int) -> None:
    """Host threads for independent CSR rows, FFT lines and SLQ probes (results are identical
    for every thread count: each reduction keeps its sequential order)."""
    lib().orc_set_threads(int(n))


def next_fast_fft_size(x):
    return int(lib().orc_next_fast_fft_size(x))


@dataclass
class GridSolveResult:
    xhat_d: np.ndarray
    iterations: int
    converged: bool
    residual_sq: float
    residual_trace: np.ndarray
    alphas: np.ndarray
    betas: np.ndarray
    loop_seconds: float


def factorized_cg_grid_rhs(kg, stats, rhat0, sigma, eps_abs=-1.0, rel_tol=-1.0, maxiter=1000):
    m = kg.dim
    r0 = _f64(rhat0)
    x = np.zeros(m)
    it, conv = C.c_int(0), C.c_int(0)
    rs, ls = _d(), _d()
    tr = np.zeros(maxiter + 1)
    al = np.zeros(maxiter + 1)
    be = np.zeros(maxiter + 1)
    _check(lib().orc_factorized_cg_grid_rhs(kg._h, stats._h, _ptr(r0), sigma, eps_abs, rel_tol, maxiter,
                                            _ptr(x), C.byref(it), C.byref(conv), C.byref(rs),
                                            _ptr(tr), _ptr(al), _ptr(be), C.byref(ls)))
    k = it.value
    nb = k - 1 if conv.value else k
    return GridSolveResult(x, k, bool(conv.value), rs.value, tr[: k + 1].copy(), al[:k].copy(),
                           be[: max(nb, 0)].copy(), ls.value)


def posterior_mean_gsgp(kg, stats, sigma, tol, maxiter=1000):
    out = np.zeros(kg.dim)
    it, rs = C.c_int(0), _d()
    _check(lib().orc_posterior_mean_gsgp(kg._h, stats._h, sigma, tol, maxiter, _ptr(out), C.byref(it), C.byref(rs)))
    return out, it.value, rs.value


def predict_mean(grid, mean_coeffs, pts, scheme=CUBIC):
    pts = _f64(pts).reshape(-1, grid.dim)
    mc = _f64(mean_coeffs)
    out = np.zeros(pts.shape[0])
    _check(lib().orc_predict_mean(*grid.args(), scheme, _ptr(mc), _ptr(pts), pts.shape[0], _ptr(out)))
    return out


def rademacher_probe(n, seed, p):
    out = np.zeros(n)
    lib().orc_rademacher_probe(n, seed, p, _ptr(out))
    return out


def rademacher_bits(n, seed, probes, nthreads=8):
    out = np.zeros(n, np.uint64)
    lib().orc_rademacher_bits(n, seed, probes, _ptr(out), nthreads)
    return out


def wt_apply(grid, x, u, scheme=CUBIC):
    x = _f64(x).reshape(-1, grid.dim)
    u = _f64(u)
    out = np.zeros(grid.m)
    _check(lib().orc_wt_apply(*grid.args(), scheme, _ptr(x), x.shape[0], _ptr(u), _ptr(out)))
    return out


def factorized_lanczos_fused(kg, stats, kgwt_z0, wt_z0, z0_sq, sigma_sq, k, want_basis=False):
    m = kg.dim
    a, b, dv = np.zeros(k), np.zeros(max(k - 1, 1)), np.zeros(k)
    basis = np.zeros((k, m)) if want_basis else None
    order = C.c_int(0)
    kw, w = _f64(kgwt_z0), _f64(wt_z0)
    _check(lib().orc_factorized_lanczos_fused(kg._h, stats._h, _ptr(kw), _ptr(w), z0_sq, sigma_sq, k,
                                              _ptr(a), _ptr(b), _ptr(dv),
                                              _ptr(basis) if want_basis else None, C.byref(order)))
    o = order.value
    res = dict(alpha=a[:o].copy(), beta=b[: max(o - 1, 0)].copy(), d=dv[:o].copy())
    if want_basis:
        res["basis"] = basis[:o].T.copy()
    return res


def quadrature_logdet(alpha, beta, probe_sq, quad_tol):
    a = _f64(alpha)
    b = _f64(beta) if len(beta) else np.zeros(1)
    v, dpt = _d(), C.c_int()
    _check(lib().orc_quadrature_logdet(_ptr(a), _ptr(b), a.size, probe_sq, quad_tol, C.byref(v), C.byref(dpt)))
    return v.value, dpt.value


def tridiag_eig(alpha, beta):
    a = _f64(alpha)
    b = _f64(beta) if len(beta) else np.zeros(1)
    ev, fr = np.zeros(a.size), np.zeros(a.size)
    _check(lib().orc_tridiag_eig(a.size, _ptr(a), _ptr(b), _ptr(ev), _ptr(fr)))
    return ev, fr


def slq_logdet_ski_factorized(kg, stats, grid, x, sigma, num_probes, max_depth, quad_tol, seed, scheme=CUBIC):
    x = _f64(x).reshape(-1, grid.dim)
    v, dpt = _d(), C.c_int()
    _check(lib().orc_slq_logdet_ski_factorized(kg._h, stats._h, *grid.args(), scheme, _ptr(x), x.shape[0], sigma,
                                               num_probes, max_depth, quad_tol, seed, C.byref(v), C.byref(dpt)))
    return v.value, dpt.value


ROUTES = {"auto": 0, "symmetric-grid": 1, "ski-operator": 2, "dense": 3}
ROUTE_NAMES = {1: "symmetric-grid-slq", 2: "ski-operator-slq", 3: "dense"}


def log_likelihood_gsgp(stats, kg, sigma, grid=None, x=None, scheme=CUBIC, solve_tol=0.01, probes=30,
                        max_depth=100, quad_tol=0.01, seed=0, route="auto", dense_cap=2048, maxiter=1000):
    out = np.zeros(4)
    iout = np.zeros(3, np.int32)
    if x is not None:
        x = _f64(x).reshape(-1, grid.dim)
        gargs = grid.args()
        xp, npts = _ptr(x), x.shape[0]
    else:
        g = kg.grid
        gargs = g.args()
        xp, npts = None, 0
    _check(lib().orc_log_likelihood_gsgp(stats._h, kg._h, sigma, solve_tol, probes, max_depth, quad_tol, seed,
                                         ROUTES[route], dense_cap, maxiter, *gargs, scheme, xp, npts,
                                         _ptr(out), _ptr(iout)))
    return dict(loglik=out[0], logdet_term=out[1], quad_term=out[2], const_term=out[3],
                probes_used=int(iout[0]), solver_iterations=int(iout[1]), logdet_route=ROUTE_NAMES[int(iout[2])])


# ---------------------------------------------------------------- covariance (gp.cpp:381-528)
def posterior_cov_exact(kg, stats, sigma, points, tol=1e-8, maxiter=1000, scheme=CUBIC):
    pts = _f64(points).reshape(-1, kg.grid.dim)
    ns = pts.shape[0]
    cov = np.zeros((ns, ns))
    asym, iters = _d(), C.c_int()
    _check(lib().orc_posterior_cov_exact(kg._h, stats._h, scheme, sigma, _ptr(pts), ns, tol, maxiter, _ptr(cov),
                                         C.byref(asym), C.byref(iters)))
    return dict(cov=cov, max_asymmetry=asym.value, total_iterations=iters.value)


def posterior_cov_lowrank(kg, stats, sigma, rank, points=None, query=None, scheme=CUBIC):
    """Returns dict(rank, cov (at points), query (cov between the two query points))."""
    d = kg.grid.dim
    pts = _f64(points).reshape(-1, d) if points is not None else np.zeros((0, d))
    ns = pts.shape[0]
    cov = np.zeros((max(ns, 1), max(ns, 1)))
    rk = C.c_int()
    qo = _d()
    qx = _f64(query[0]) if query is not None else None
    qx2 = _f64(query[1]) if query is not None else None
    _check(lib().orc_posterior_cov_lowrank(kg._h, stats._h, scheme, sigma, int(rank), _ptr(pts) if ns else None, ns,
                                           _ptr(cov), _ptr(qx) if qx is not None else None,
                                           _ptr(qx2) if qx2 is not None else None,
                                           C.byref(qo) if query is not None else None, C.byref(rk)))
    return dict(rank=rk.value, cov=cov[:ns, :ns], query=qo.value if query is not None else None)
