// api.cu — the C ABI (include/gsgpc.h): handles, host/device staging, the precompute
// pipeline, the EFCG driver (CUDA-graph replay with device-resident scalars), posterior
// mean, prediction and the GSGPSST1 stats file.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <random>
#include <thread>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/gsgpc.h"
#include "internal.cuh"
#include "precompute.cuh"

#ifndef GSGPC_GIT
#define GSGPC_GIT "unknown"
#endif

using namespace gsgpc;

namespace gsgpc {
double measure_fp64_peak(cudaStream_t s);
void measure_fp64_tensor(cudaStream_t s, double* dmma_tflops, double* mixed_tflops);
void run_add_div(const Launch& L, int64_t n, const double* x, double sx, const double* y, double b, double* out);
}

namespace {

// ------------------------------------------------------------------ device buffers
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    GSGPC_CUDA(cudaMalloc(&p, std::max<size_t>(b, 256)));
    bytes = std::max<size_t>(b, 256);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    GSGPC_CUDA(cudaMallocHost(&p, std::max<size_t>(b, 256)));
    bytes = std::max<size_t>(b, 256);
  }
};

// Device or host?  A CUDA error already pending when we ask is surfaced (never swallowed:
// clearing it here would hide a fault from an earlier launch and then treat a device pointer
// as host memory).  A device allocation of another GPU than the context's is rejected — its
// kernels would dereference a foreign address.
bool is_device_ptr(const void* p) {
  if (!p) return false;
  const cudaError_t pend = cudaPeekAtLastError();
  if (pend != cudaSuccess) {
    cudaGetLastError();
    throw Error(GSGPC_CUDA_ERROR, std::string("CUDA error pending before the pointer query: ") +
                                      cudaGetErrorString(pend));
  }
  cudaPointerAttributes a{};
  const cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(GSGPC_CUDA_ERROR, std::string("cudaPointerGetAttributes failed: ") + cudaGetErrorString(e));
  }
  if (a.type == cudaMemoryTypeDevice) {
    int dev = 0;
    GSGPC_CUDA(cudaGetDevice(&dev));
    if (a.device != dev)
      invalid("device array lives on device " + std::to_string(a.device) + ", the context is on device " +
              std::to_string(dev));
    return true;
  }
  return a.type == cudaMemoryTypeManaged;
}

}  // namespace

// ------------------------------------------------------------------ handles
struct CgCache;
constexpr int kPhases = 10;  // gsgpc_ctx_phase_times

struct gsgpc_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t err_row = 0;
  uint64_t launches = 0;
  bool timing = false;
  double phase_ms[kPhases] = {0};
  int64_t phase_calls[kPhases] = {0};
  std::map<std::string, std::unique_ptr<DBuf>> bufs;
  PinnedBuf pin;
  std::unique_ptr<CgCache> cg;
  cudaStream_t copy = nullptr;   // H2D staging stream (overlaps the next batch's copy with compute)
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  PinnedBuf file_pin[2];         // GSGPDAT1 ingest: host read buffers (reader thread fills one while
                                 // the other is copied to the device)
  cudaStream_t sort = nullptr;   // slice sort of bucket group j+1 overlaps K1 of group j
  void ensure_sort_stream() {
    if (sort) return;
    int lo = 0, hi = 0;
    GSGPC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GSGPC_CUDA(cudaStreamCreateWithPriority(&sort, cudaStreamNonBlocking, hi));  // memory-bound: dispatch first
  }
  Launch L() { return Launch{stream, &launches}; }
  void ensure_copy_stream() {
    if (copy) return;
    GSGPC_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      GSGPC_CUDA(cudaEventCreateWithFlags(&ev_copied[i], cudaEventDisableTiming));
      GSGPC_CUDA(cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming));
    }
  }
  DBuf& buf(const std::string& name) {
    auto& b = bufs[name];
    if (!b) b.reset(new DBuf());
    return *b;
  }
};

struct gsgpc_stats {
  int device = 0;
  gsgpc_grid grid{};
  int scheme = 1;
  GridDev g{};
  int Q = 0, QY = 0, S_min = 0;
  DBuf mom;      // cells × Q
  int NP = 1;    // zero-weight patterns per cell (3^d)
  DBuf pat;      // cells × NP bytes: W^T W structure (see run_touched)
  std::vector<uint8_t> loaded_touched;  // GSGPSST1-loaded statistics: structure from the file
  DBuf pmom;     // cells × P × QY
  DBuf yty;      // device scalar Σ y²
  DBuf fin;      // [S_min·m | m | P·m | yty | n]
  int probes = 0;
  int64_t n = 0;
  bool finalized = false;
  bool reduced = false;
  // seeded Rademacher probes (gsgpc_stats_enable_probes): one generator per probe
  bool probe_seeded = false;
  uint64_t probe_seed = 0;
  int64_t probe_first_row = 0;  // global row index of this accumulator's first row (stream offset)
  DBuf rng;  // probe_seeded: per probe the MT19937-64 state (312 words) + index, on the device
  int64_t fin_count() const { return static_cast<int64_t>(S_min) * g.m + g.m + static_cast<int64_t>(probes) * g.m + 2; }
  double* stencil() const { return fin.as<double>(); }
  double* wty() const { return fin.as<double>() + static_cast<int64_t>(S_min) * g.m; }
  double* pimg() const { return wty() + g.m; }
  double* tail() const { return pimg() + static_cast<int64_t>(probes) * g.m; }
};

struct gsgpc_kg {
  int device = 0;
  gsgpc_grid grid{};
  int64_t m = 0;
  double noise_std = 1.0;
  DBuf gen[GSGPC_MAX_DIM];
  KgDev dev{};
  std::shared_ptr<KgFft> fft;  // circulant-FFT route of the long dimensions (operators.cu)
};

// LowRankCov (gp.hpp:148-167): R (k × m, row j = column j of the reference's r_), the
// tridiagonal T, and its own copy of the K_G generators (the reference holds a shared_ptr
// to the operator).
struct gsgpc_lowrank {
  int device = 0;
  GridDev g{};
  int scheme = 1;
  int64_t m = 0;
  int k = 0;
  DBuf R;
  std::vector<double> alpha, beta;
  DBuf gen[GSGPC_MAX_DIM];
  KgDev kg{};
  std::shared_ptr<KgFft> fft;
};

struct CgCache {
  // buffers + a captured graph of B iterations for one (stats, kg) pairing
  const gsgpc_stats* stats = nullptr;
  const gsgpc_kg* kg = nullptr;
  int64_t m = 0;
  DBuf r, u, s, z, x, kt0, kt1, pa, pb, tr, al, be, st;
  int trace_cap = 0;
  cudaGraphExec_t exec = nullptr;
  int B = 0;
  ~CgCache() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

namespace {

template <class F>
gsgpc_status guard(gsgpc_ctx* ctx, F&& f) {
  try {
    if (ctx) GSGPC_CUDA(cudaSetDevice(ctx->device));
    f();
    return GSGPC_OK;
  } catch (const Error& e) {
    if (ctx) {
      ctx->err = e.what();
      ctx->err_row = e.row;
    }
    return e.code;
  } catch (const std::bad_alloc& e) {
    if (ctx) ctx->err = std::string("out of host memory: ") + e.what();
    return GSGPC_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return GSGPC_RUNTIME_ERROR;
  }
}

int scheme_width(int scheme) {
  if (scheme == GSGPC_CUBIC) return 4;
  if (scheme == GSGPC_LINEAR) return 2;
  invalid("unknown interpolation scheme");
  return 0;
}

// Grid::Grid validation (grid.cpp:12-23) + the device descriptor.
GridDev make_grid(const gsgpc_grid* gr, int scheme) {
  if (!gr) invalid("grid is NULL");
  if (gr->dim < 1) invalid("Grid: need at least one dimension");
  if (gr->dim > GSGPC_MAX_DIM) {
    throw Error(GSGPC_UNSUPPORTED, "grid dimension " + std::to_string(gr->dim) + " > 3 is not supported by this build");
  }
  GridDev g{};
  g.d = gr->dim;
  g.W = scheme_width(scheme);
  g.m = 1;
  g.cells = 1;
  for (int k = 0; k < g.d; ++k) {
    if (gr->size[k] < 2) invalid("Grid: size must be >= 2 per dimension");
    if (!(gr->max[k] > gr->min[k])) invalid("Grid: max must exceed min");
    g.mn[k] = gr->min[k];
    g.sp[k] = (gr->max[k] - gr->min[k]) / static_cast<double>(gr->size[k] - 1);
    g.isp[k] = 1.0 / g.sp[k];
    g.sz[k] = gr->size[k];
    g.nc[k] = gr->size[k] - 1;
    g.m *= g.sz[k];
    g.cells *= g.nc[k];
  }
  return g;
}

StencilDesc stencil_desc(const gsgpc_stats* s) {
  if (static_cast<double>(s->S_min) * static_cast<double>(s->g.m) >= 2147483647.0) {
    throw Error(GSGPC_UNSUPPORTED, "W^T W stencil larger than 2^31 entries is not supported by this build");
  }
  StencilDesc sd{};
  sd.d = s->g.d;
  sd.W = s->g.W;
  sd.S_min = s->S_min;
  for (int k = 0; k < sd.d; ++k) sd.sz[k] = s->g.sz[k];
  sd.m = s->g.m;
  return sd;
}

// Host/device array staging ----------------------------------------------------------
// Input: returns a device pointer holding `count` doubles of `p` (copied if host memory).
const double* dev_in(gsgpc_ctx* ctx, const double* p, int64_t count, const char* slot) {
  if (!p) invalid(std::string("NULL array argument (") + slot + ")");
  if (is_device_ptr(p)) return p;
  DBuf& b = ctx->buf(slot);
  b.ensure(sizeof(double) * count);
  GSGPC_CUDA(cudaMemcpyAsync(b.p, p, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
  return b.as<double>();
}

// Output: device destination to write `count` doubles into, then finish() copies back.
struct DevOut {
  gsgpc_ctx* ctx;
  double* user;
  double* dev;
  int64_t count;
  bool host;
  DevOut(gsgpc_ctx* c, double* u, int64_t n, const char* slot) : ctx(c), user(u), count(n) {
    if (!u) invalid(std::string("NULL output array (") + slot + ")");
    host = !is_device_ptr(u);
    if (host) {
      DBuf& b = ctx->buf(slot);
      b.ensure(sizeof(double) * n);
      dev = b.as<double>();
    } else {
      dev = u;
    }
  }
  void finish() {
    if (host) {
      GSGPC_CUDA(cudaMemcpyAsync(user, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
      GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  }
};

void copy_out(gsgpc_ctx* ctx, void* user, const void* dev, size_t bytes) {
  GSGPC_CUDA(cudaMemcpyAsync(user, dev, bytes, cudaMemcpyDefault, ctx->stream));
  GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
}

double read_scalar(gsgpc_ctx* ctx, const double* dev) {
  double v = 0.0;
  copy_out(ctx, &v, dev, sizeof(double));
  return v;
}

// Phase timing (events on the context stream) ----------------------------------------
struct PhaseTimer {
  gsgpc_ctx* ctx;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> ev;
  explicit PhaseTimer(gsgpc_ctx* c) : ctx(c) {}
  int begin(int phase) {
    if (!ctx->timing) return -1;
    cudaEvent_t a, b;
    GSGPC_CUDA(cudaEventCreate(&a));
    GSGPC_CUDA(cudaEventCreate(&b));
    GSGPC_CUDA(cudaEventRecord(a, ctx->stream));
    ev.emplace_back(phase, a, b);
    return static_cast<int>(ev.size()) - 1;
  }
  void end(int h) {
    if (h < 0) return;
    GSGPC_CUDA(cudaEventRecord(std::get<2>(ev[h]), ctx->stream));
  }
  ~PhaseTimer() {
    if (ev.empty()) return;
    cudaStreamSynchronize(ctx->stream);
    for (auto& e : ev) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, std::get<1>(e), std::get<2>(e)) == cudaSuccess) {
        ctx->phase_ms[std::get<0>(e)] += ms;
        ctx->phase_calls[std::get<0>(e)] += 1;
      }
      cudaEventDestroy(std::get<1>(e));
      cudaEventDestroy(std::get<2>(e));
    }
  }
};

// Points validation + device descriptor ----------------------------------------------
size_t dtype_size(int dt) {
  if (dt == GSGPC_F32) return 4;
  if (dt == GSGPC_F64) return 8;
  invalid("unknown dtype");
  return 0;
}

PointsDev points_dev(const gsgpc_points* p, int d, int64_t row0) {
  PointsDev q{};
  const size_t es = dtype_size(p->dtype);
  q.x = static_cast<const char*>(p->x) + es * row0 * p->x_row_stride;
  q.y = static_cast<const char*>(p->y) + es * row0 * p->y_stride;
  q.xs = p->x_row_stride;
  for (int k = 0; k < GSGPC_MAX_DIM; ++k) q.xo[k] = k < d ? p->x_col_offset[k] : 0;
  q.ys = p->y_stride;
  return q;
}

void check_points(const gsgpc_points* p, int64_t n, bool need_y) {
  if (!p) invalid("points descriptor is NULL");
  if (n < 0) invalid("negative row count");
  if (n == 0) return;
  if (!p->x) invalid("points: x is NULL");
  if (need_y && !p->y) invalid("points: y is NULL");
  dtype_size(p->dtype);
}

// Stage rows [r0, r1) of a host-resident point set into device memory; returns the device
// descriptor for that chunk (row 0 = r0).
PointsDev stage_points(gsgpc_ctx* ctx, const gsgpc_points* p, int d, int64_t r0, int64_t r1, bool need_y,
                       const char* slot, cudaStream_t strm = nullptr) {
  if (!strm) strm = ctx->stream;
  const size_t es = dtype_size(p->dtype);
  const int64_t rows = r1 - r0;
  PointsDev q{};
  const char* hx = static_cast<const char*>(p->x);
  const char* hy = static_cast<const char*>(p->y);
  int64_t maxo = 0;
  for (int k = 0; k < d; ++k) maxo = std::max(maxo, p->x_col_offset[k]);
  const bool columns = p->x_row_stride == 1 && d > 1;
  const int64_t xelems = columns ? rows * d : rows * p->x_row_stride;
  // y inside the x rows (AoS (x..., y))?
  const int64_t yoff = (hy - hx) / static_cast<int64_t>(es);
  const bool y_in_x = need_y && !columns && p->y_stride == p->x_row_stride && hy >= hx &&
                      (hy - hx) % static_cast<int64_t>(es) == 0 && yoff < p->x_row_stride;
  const int64_t yelems = (!need_y || y_in_x) ? 0 : rows * p->y_stride;
  DBuf& b = ctx->buf(slot);
  b.ensure(es * (xelems + yelems) + 64);
  char* dx = b.as<char>();
  if (columns) {
    for (int k = 0; k < d; ++k) {
      GSGPC_CUDA(cudaMemcpyAsync(dx + es * k * rows, hx + es * (p->x_col_offset[k] + r0), es * rows,
                                 cudaMemcpyHostToDevice, strm));
      q.xo[k] = k * rows;
    }
    q.xs = 1;
  } else {
    if (maxo >= p->x_row_stride && rows > 1) {
      throw Error(GSGPC_UNSUPPORTED, "host points: column offset beyond the row stride");
    }
    const int64_t span = (rows - 1) * p->x_row_stride + std::max(maxo, y_in_x ? yoff : 0) + 1;
    GSGPC_CUDA(cudaMemcpyAsync(dx, hx + es * r0 * p->x_row_stride, es * span, cudaMemcpyHostToDevice, strm));
    q.xs = p->x_row_stride;
    for (int k = 0; k < d; ++k) q.xo[k] = p->x_col_offset[k];
  }
  q.x = dx;
  if (!need_y) {
    q.y = dx;
    q.ys = 0;
  } else if (y_in_x) {
    q.y = dx + es * yoff;
    q.ys = p->y_stride;
  } else {
    char* dy = dx + es * xelems;
    const int64_t span = (rows - 1) * p->y_stride + 1;
    GSGPC_CUDA(cudaMemcpyAsync(dy, hy + es * r0 * p->y_stride, es * span, cudaMemcpyHostToDevice, strm));
    q.y = dy;
    q.ys = p->y_stride;
  }
  return q;
}

void ensure_fin(gsgpc_stats* s) {
  s->fin.ensure(sizeof(double) * s->fin_count());
}

void finalize_stats(gsgpc_ctx* ctx, gsgpc_stats* s) {
  if (s->reduced || s->finalized) return;
  PhaseTimer pt(ctx);
  const int h = pt.begin(4);
  ensure_fin(s);
  const Launch L = ctx->L();
  const int64_t ws = finalize_ws_elems(s->g);
  DBuf& w = ctx->buf("finalize_ws");
  w.ensure(sizeof(double) * ws);
  static const bool poison = [] {  // diagnostics: NaN-fill the workspace (reads of unwritten data show up)
    const char* e = getenv("GSGPC_DEBUG_POISON_WS");
    return e && e[0] == '1';
  }();
  if (poison) GSGPC_CUDA(cudaMemsetAsync(w.p, 0xFF, sizeof(double) * ws, ctx->stream));
  run_finalize(L, s->g, s->mom.as<double>(), s->probes, s->probes ? s->pmom.as<double>() : nullptr, s->stencil(),
               s->wty(), s->pimg(), w.as<double>(), ws);
  // tail: yty, n
  GSGPC_CUDA(cudaMemcpyAsync(s->tail(), s->yty.p, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  const double nd = static_cast<double>(s->n);
  double* pin = static_cast<double*>(ctx->pin.p);
  ctx->pin.ensure(64);
  pin = static_cast<double*>(ctx->pin.p);
  pin[0] = nd;
  GSGPC_CUDA(cudaMemcpyAsync(s->tail() + 1, pin, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
  pt.end(h);
  s->finalized = true;
}

double stats_yty(gsgpc_ctx* ctx, gsgpc_stats* s) {
  if (s->reduced) return read_scalar(ctx, s->tail());
  return read_scalar(ctx, s->yty.as<double>());
}

gsgpc_stats* new_stats(gsgpc_ctx* ctx, const gsgpc_grid* grid, int scheme) {
  std::unique_ptr<gsgpc_stats> s(new gsgpc_stats());
  s->device = ctx->device;
  s->g = make_grid(grid, scheme);
  s->grid = *grid;
  s->scheme = scheme;
  s->Q = moments_per_cell(s->g.d, s->g.W);
  int qy = 1, S = 1;
  for (int k = 0; k < s->g.d; ++k) {
    qy *= s->g.W;
    S *= 2 * s->g.W - 1;
  }
  s->QY = qy;
  s->S_min = (S + 1) / 2;
  // + 2 doubles: finalize's bulk copies of record tiles round their size up to 16 bytes
  s->mom.ensure(sizeof(double) * (s->g.cells * s->Q + 2));
  GSGPC_CUDA(cudaMemsetAsync(s->mom.p, 0, sizeof(double) * (s->g.cells * s->Q + 2), ctx->stream));
  s->yty.ensure(sizeof(double));
  GSGPC_CUDA(cudaMemsetAsync(s->yty.p, 0, sizeof(double), ctx->stream));
  for (int k = 0; k < s->g.d; ++k) s->NP *= 3;
  s->pat.ensure(static_cast<size_t>(s->g.cells) * s->NP);
  GSGPC_CUDA(cudaMemsetAsync(s->pat.p, 0, static_cast<size_t>(s->g.cells) * s->NP, ctx->stream));
  return s.release();
}

// The precompute pipeline on one device-resident chunk.
// Bucket groups for overlapping the slice sort (HBM-bound, high-priority sort stream) with
// K1 (FP64-bound, compute stream).  Buckets are whole cells, so splitting K1 by bucket
// ranges adds no moment flushes (splitting by row ranges re-flushed every cell per part).
// Measured: no gain — K1 needs all its resident warps to hide DMMA latency, and sort blocks
// co-scheduled on its SMs cost more than the overlap saves — so the default is sequential;
// GSGPC_BUCKET_GROUPS = G > 1 enables the overlap.  Phase timing always runs sequentially.
static int bucket_groups(gsgpc_ctx* ctx, int64_t nvalid, int nb) {
  static const int env = [] {
    const char* e = getenv("GSGPC_BUCKET_GROUPS");
    return e ? std::max(1, atoi(e)) : 1;  // B200, config 3: 1 → 9.22, 2 → 9.29, 4 → 9.92, 8 → 10.8 ms
  }();
  if (ctx->timing || nvalid < (int64_t{1} << 22)) return 1;
  return std::min(env, nb);
}

// Device-resident batches of several chunks: the binning of chunk k + 1 (classify … slice sort,
// on the high-priority sort stream) can overlap the moments kernel of chunk k (compute stream).
// Each of the two scratch sets is reused once the K1 that read it has finished; every kernel
// and every order of accumulation is the sequential path's, so the statistics are bitwise the
// same.  Measured on B200 (GSGPC_CHUNK_PIPE=1): config 4, 1e9 rows in 8 chunks 58.7 → 68.9 ms
// (the latency-bound d = 2 K1 and the sorts contend for the same DRAM queues); config 3 in four
// 2^25-row chunks 11.03 → 10.54 ms (one chunk: 9.24 ms).  Off by default.
struct ChunkPipe {
  cudaStream_t bin = nullptr;
  cudaEvent_t binned[2] = {nullptr, nullptr}, k1done[2] = {nullptr, nullptr};
  int set = 0;
  int64_t k = 0;
};

void add_chunk(gsgpc_ctx* ctx, gsgpc_stats* s, int dtype, const PointsDev& P, int64_t n, int64_t row0,
               const uint64_t* pw_dev, int probes, const ChunkPipe* pipe) {
  const Launch LK = ctx->L();
  const Launch L = pipe ? Launch{pipe->bin, &ctx->launches} : LK;  // binning launches
  const GridDev& g = s->g;
  PhaseTimer pt(ctx);
  const std::string sfx = pipe && pipe->set ? "#1" : "";
  auto sbuf = [&](const char* name) -> DBuf& { return ctx->buf(name + sfx); };
  if (pipe && pipe->k >= 2) GSGPC_CUDA(cudaStreamWaitEvent(pipe->bin, pipe->k1done[pipe->set], 0));
  if (n >= (int64_t{1} << 31)) throw Error(GSGPC_INVALID_ARGUMENT, "sufficient_stats: batch too large");
  const BinDesc bd = bin_desc(g.cells);
  const int64_t ntiles = bin_tiles(n);
  DBuf& tcnt = sbuf("bin_tcnt");
  tcnt.ensure(sizeof(int) * ntiles * bd.nb);
  DBuf& gsum = sbuf("bin_gsum");
  gsum.ensure(sizeof(int) * bin_groups(n) * bd.nb);
  DBuf& bbase = sbuf("bin_base");
  bbase.ensure(sizeof(int64_t) * (bd.nb + 1));
  DBuf& sbase = sbuf("bin_sbase");
  sbase.ensure(sizeof(int64_t) * (bd.nb + 1));
  DBuf& off = sbuf("off");
  off.ensure(sizeof(int64_t) * (g.cells + 2));
  DBuf& cellid = sbuf("cellid");
  cellid.ensure(sizeof(int) * n);
  DBuf& err = ctx->buf("err");
  err.ensure(sizeof(unsigned long long) * 2);
  const int nblk = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, sm_count() * 6)));
  DBuf& part = sbuf("yty_part");
  part.ensure(sizeof(double) * nblk);
  DBuf& ychunk = sbuf("yty_chunk");
  ychunk.ensure(sizeof(double));

  // err: reset once per public call (stats_add / add_file), checked by the caller after the
  // whole batch — see BinGate (precompute.cu)
  int h = pt.begin(0);
  GSGPC_CUDA(cudaMemsetAsync(ychunk.p, 0, sizeof(double), L.s));
  run_classify(L, dtype, P, n, row0, g, bd, tcnt.as<int>(), err.as<unsigned long long>(), part.as<double>(), nblk,
               cellid.as<int>());
  run_sum_partials(L, part.as<double>(), nblk, ychunk.as<double>());
  pt.end(h);
  h = pt.begin(1);
  run_bucket_totals(L, bd, n, tcnt.as<int>(), gsum.as<int>(), bbase.as<int64_t>(), sbase.as<int64_t>());
  pt.end(h);
  const unsigned long long* errp = err.as<unsigned long long>();
  run_commit_add(L, errp, ychunk.as<double>(), s->yty.as<double>());
  // binning → moments without a host round trip: sizes are upper bounds (every row valid),
  // the kernels read the true counts from bbase / sbase
  const int64_t nvalid = n, nslices = bin_slices_max(n, bd);
  const int G = pipe ? 1 : bucket_groups(ctx, nvalid, bd.nb);
  std::vector<int64_t> hb, hsl;
  if (G > 1) {  // the optional overlap needs the bucket offsets on the host
    const int64_t NB1 = bd.nb + 1;
    hb.resize(NB1);
    hsl.resize(NB1);
    GSGPC_CUDA(cudaMemcpyAsync(hb.data(), bbase.p, sizeof(int64_t) * NB1, cudaMemcpyDeviceToHost, ctx->stream));
    GSGPC_CUDA(cudaMemcpyAsync(hsl.data(), sbase.p, sizeof(int64_t) * NB1, cudaMemcpyDeviceToHost, ctx->stream));
    GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  {
    // the binning sorts (cell, row) keys; K1 gathers the rows (and probe words) of P through
    // the cell-sorted row indices
    DBuf& idx_s = sbuf("bin_idx_sorted");
    idx_s.ensure(sizeof(int) * nvalid);
    DBuf& cid1 = sbuf("bin_cid");
    cid1.ensure(sizeof(int) * nvalid);
    DBuf& idx1 = sbuf("bin_idx");
    idx1.ensure(sizeof(int) * nvalid);
    DBuf& spv = sbuf("k1_split_v");
    DBuf& spc = sbuf("k1_split_c");
    const int64_t spw = split_rec_warps(nvalid), spr = split_rec_doubles(g, probes);
    spv.ensure(sizeof(double) * spw * spr);
    spc.ensure(sizeof(int64_t) * spw);
    const SplitBuf sb{spv.as<double>(), spc.as<int64_t>(), spw, spr};
    DBuf& scnt = sbuf("bin_scnt");
    scnt.ensure(sizeof(int) * std::max<int64_t>(1, nslices) * (int64_t{1} << bd.bsh));
    h = pt.begin(2);
    run_partition(L, n, bd, cellid.as<int>(), tcnt.as<int>(), cid1.as<int>(), idx1.as<int>(), errp);
    const int64_t* rows_end = bbase.as<int64_t>() + bd.nb;
    if (G == 1) {
      run_slice_sort(L, bd, g.cells, 0, bd.nb, 0, nslices, cid1.as<int>(), idx1.as<int>(), bbase.as<int64_t>(),
                     sbase.as<int64_t>(), scnt.as<int>(), off.as<int64_t>(), idx_s.as<int>(), errp);
      pt.end(h);
      if (pipe) {  // K1 of this chunk waits for its binning; the next chunk's binning starts now
        GSGPC_CUDA(cudaEventRecord(pipe->binned[pipe->set], pipe->bin));
        GSGPC_CUDA(cudaStreamWaitEvent(ctx->stream, pipe->binned[pipe->set], 0));
      }
      int hk = pt.begin(3);
      SplitFixJob fix{};
      run_moments(LK, dtype, P, idx_s.as<int>(), off.as<int64_t>(), 0, nvalid, 0, g.cells, g, s->mom.as<double>(),
                  s->pat.as<uint8_t>(), errp, sb, rows_end, &fix);
      pt.end(hk);
      hk = pt.begin(6);
      run_split_fix(LK, sb, fix);
      pt.end(hk);
      hk = pt.begin(7);
      if (probes > 0) {
        run_probe_moments(LK, dtype, P, idx_s.as<int>(), pw_dev, off.as<int64_t>(), 0, nvalid, 0, g.cells, g, probes,
                          s->pmom.as<double>(), errp, sb, rows_end);
      }
      pt.end(hk);
      if (pipe) GSGPC_CUDA(cudaEventRecord(pipe->k1done[pipe->set], ctx->stream));
    } else {
      // bucket groups of ~equal rows; group j's K1 overlaps group j+1's slice sort
      const int64_t nv = hb[bd.nb];
      std::vector<int> gb(G + 1, bd.nb);
      gb[0] = 0;
      for (int j = 1; j < G; ++j) {
        const int64_t target = nv * j / G;
        gb[j] = static_cast<int>(std::upper_bound(hb.begin(), hb.end(), target) - hb.begin()) - 1;
        gb[j] = std::max(gb[j], gb[j - 1]);
      }
      std::vector<cudaEvent_t> evs;
      struct EvFree {
        std::vector<cudaEvent_t>* v;
        ~EvFree() {
          for (cudaEvent_t e : *v) cudaEventDestroy(e);
        }
      } evf{&evs};
      auto record = [&](cudaStream_t st) {
        cudaEvent_t e;
        GSGPC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs.push_back(e);
        GSGPC_CUDA(cudaEventRecord(e, st));
        return e;
      };
      ctx->ensure_sort_stream();
      const cudaStream_t ss = ctx->sort;
      GSGPC_CUDA(cudaStreamWaitEvent(ss, record(ctx->stream), 0));
      const Launch LS{ss, &ctx->launches};
      for (int j = 0; j < G; ++j) {
        const int b0 = gb[j], b1 = gb[j + 1];
        if (b1 <= b0) continue;
        run_slice_sort(LS, bd, g.cells, b0, b1, hsl[b0], hsl[b1], cid1.as<int>(), idx1.as<int>(),
                       bbase.as<int64_t>(), sbase.as<int64_t>(), scnt.as<int>(), off.as<int64_t>(), idx_s.as<int>(),
                       errp);
        GSGPC_CUDA(cudaStreamWaitEvent(ctx->stream, record(ss), 0));
        const int64_t c_lo = static_cast<int64_t>(b0) << bd.bsh;
        const int64_t c_hi = std::min<int64_t>(static_cast<int64_t>(b1) << bd.bsh, g.cells);
        run_moments(L, dtype, P, idx_s.as<int>(), off.as<int64_t>(), hb[b0], hb[b1], c_lo, c_hi, g,
                    s->mom.as<double>(), s->pat.as<uint8_t>(), errp, sb);
        if (probes > 0) {
          run_probe_moments(L, dtype, P, idx_s.as<int>(), pw_dev, off.as<int64_t>(), hb[b0], hb[b1], c_lo, c_hi, g,
                            probes, s->pmom.as<double>(), errp, sb);
        }
      }
      pt.end(h);
    }
  }
  s->n += n;
  s->finalized = false;
}

// Out-of-grid check of a whole add call: the classify pass records the first bad row
// (atomicMin of (row+1) << 2 | status) and every committing kernel after it is a no-op.
void bin_error_reset(gsgpc_ctx* ctx) {
  DBuf& err = ctx->buf("err");
  err.ensure(sizeof(unsigned long long) * 2);
  GSGPC_CUDA(cudaMemsetAsync(err.p, 0xff, sizeof(unsigned long long), ctx->stream));
}

void bin_error_check(gsgpc_ctx* ctx) {
  ctx->pin.ensure(64);
  GSGPC_CUDA(cudaMemcpyAsync(ctx->pin.p, ctx->buf("err").p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
  unsigned long long e = 0;
  std::memcpy(&e, ctx->pin.p, 8);
  if (e == ~0ull) return;
  const int64_t row = static_cast<int64_t>(e >> 2);
  const int kind = static_cast<int>(e & 3);
  const std::string what =
      kind == PT_OUTSIDE ? "interp_weights: point outside grid"
                         : "interp_weights: stencil leaves the grid (point too close to the boundary for the "
                           "requested scheme)";
  throw Error(GSGPC_OUT_OF_GRID, "sufficient_stats: stream row " + std::to_string(row) + ": " + what, row);
}

// Draw the next `rows` values of every probe stream on the device (probe_rng.cu) and pack
// them into the "probe_stage" buffer (bit p of word i = probe p is +1 at row i).
void gen_probe_words(gsgpc_ctx* ctx, gsgpc_stats* s, int64_t rows) {
  DBuf& st = ctx->buf("probe_stage");
  st.ensure(sizeof(uint64_t) * rows);
  DBuf& planes = ctx->buf("probe_planes");
  planes.ensure(static_cast<size_t>(s->probes) * std::min(rows, probe_rng_slab(s->probes)));
  DBuf& scr = ctx->buf("probe_rng_scratch");
  scr.ensure(sizeof(uint64_t) * probe_rng_scratch_words(s->probes));
  run_probe_rng(ctx->L(), s->rng.as<uint64_t>(), s->probes, rows, planes.as<uint8_t>(), st.as<uint64_t>(),
                scr.as<uint64_t>());
}

// Generator states of rademacher_probe(·, seed, p), p < probes, positioned at draw
// probe_first_row (the accumulator's first global row): a fresh stream for row 0, else the
// seeded state advanced by the GF(2) jump-ahead (mt_jump.cu) — 312·q draws as a block jump,
// the remainder r as the generator's index.
void seed_probe_streams(gsgpc_ctx* ctx, gsgpc_stats* s) {
  std::vector<uint64_t> h(static_cast<size_t>(s->probes) * 313);
  for (int p = 0; p < s->probes; ++p) mt_seed_state(s->probe_seed, static_cast<uint64_t>(p), h.data() + p * 313);
  s->rng.ensure(sizeof(uint64_t) * h.size());
  const uint64_t o = static_cast<uint64_t>(s->probe_first_row);
  if (o == 0) {
    GSGPC_CUDA(cudaMemcpyAsync(s->rng.p, h.data(), sizeof(uint64_t) * h.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
  } else {
    const uint64_t a = 312 + o;  // a seeded generator sits at index 312 (its first draw twists)
    for (int p = 0; p < s->probes; ++p) h[static_cast<size_t>(p) * 313 + 312] = a % 312;
    DBuf& tmp = ctx->buf("probe_seed_tmp");
    tmp.ensure(sizeof(uint64_t) * (h.size() + 312));
    GSGPC_CUDA(cudaMemcpyAsync(tmp.p, h.data(), sizeof(uint64_t) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
    run_mt_jump(ctx->L(), tmp.as<uint64_t>(), s->probes, {a / 312}, tmp.as<uint64_t>() + h.size(),
                s->rng.as<uint64_t>());
  }
  GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* gsgpc_version(void) {
  return "gsgpc sm_100a " GSGPC_GIT " (precompute: cell-sorted polynomial moments; K_G: Kronecker Toeplitz)";
}

gsgpc_status gsgpc_probe_stream_bits(uint64_t seed, uint64_t p, uint64_t offset, int64_t n, uint8_t* out) {
  if (n < 0 || (n > 0 && !out)) return GSGPC_INVALID_ARGUMENT;
  return guard(nullptr, [&] {
    uint64_t st[313];
    mt_seed_state(seed, p, st);
    mt_jump_host(st, offset);
    // sequential draws from the jumped generator (std::mt19937_64 semantics, [rand.eng.mers])
    constexpr uint64_t A = 0xB5026F5AA96619E9ull, UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    uint64_t idx = st[312];
    for (int64_t i = 0; i < n; ++i) {
      if (idx >= 312) {
        for (int k = 0; k < 312; ++k) {
          const uint64_t x = (st[k] & UM) | (st[(k + 1) % 312] & LM);
          st[k] = st[(k + 156) % 312] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
        }
        idx = 0;
      }
      uint64_t y = st[idx++];
      y ^= (y >> 29) & 0x5555555555555555ull;
      y ^= (y << 17) & 0x71D67FFFEDA60000ull;
      y ^= (y << 37) & 0xFFF7EEE000000000ull;
      y ^= y >> 43;
      out[i] = static_cast<uint8_t>(y & 1u);
    }
  });
}

gsgpc_status gsgpc_ctx_create(int device, gsgpc_ctx** out) {
  if (!out) return GSGPC_INVALID_ARGUMENT;
  *out = nullptr;
  std::unique_ptr<gsgpc_ctx> c(new gsgpc_ctx());
  c->device = device;
  const gsgpc_status st = guard(c.get(), [&] {
    int ndev = 0;
    GSGPC_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) invalid("gsgpc_ctx_create: bad device ordinal");
    GSGPC_CUDA(cudaSetDevice(device));
    GSGPC_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->stream = c->own;
  });
  if (st != GSGPC_OK) {
    std::fprintf(stderr, "gsgpc_ctx_create: %s\n", c->err.c_str());
    return st;
  }
  *out = c.release();
  return GSGPC_OK;
}

void gsgpc_ctx_destroy(gsgpc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->sort) {
    cudaStreamSynchronize(ctx->sort);
    cudaStreamDestroy(ctx->sort);
  }
  ctx->cg.reset();
  ctx->bufs.clear();
  if (ctx->copy) {
    cudaStreamSynchronize(ctx->copy);
    cudaStreamDestroy(ctx->copy);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(ctx->ev_copied[i]);
      cudaEventDestroy(ctx->ev_free[i]);
    }
  }
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
}

gsgpc_status gsgpc_ctx_set_stream(gsgpc_ctx* ctx, void* s) {
  if (!ctx) return GSGPC_INVALID_ARGUMENT;
  ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
  ctx->cg.reset();
  return GSGPC_OK;
}

void* gsgpc_ctx_stream(gsgpc_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

gsgpc_status gsgpc_ctx_synchronize(gsgpc_ctx* ctx) {
  return guard(ctx, [&] { GSGPC_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

const char* gsgpc_last_error(const gsgpc_ctx* ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }
int64_t gsgpc_last_error_row(const gsgpc_ctx* ctx) { return ctx ? ctx->err_row : 0; }
uint64_t gsgpc_ctx_launch_count(const gsgpc_ctx* ctx) { return ctx ? ctx->launches : 0; }

gsgpc_status gsgpc_ctx_enable_phase_timing(gsgpc_ctx* ctx, int enable) {
  if (!ctx) return GSGPC_INVALID_ARGUMENT;
  ctx->timing = enable != 0;
  return GSGPC_OK;
}

gsgpc_status gsgpc_ctx_phase_times(gsgpc_ctx* ctx, double* ms_out, int64_t* calls_out) {
  if (!ctx) return GSGPC_INVALID_ARGUMENT;
  for (int i = 0; i < kPhases; ++i) {
    if (ms_out) ms_out[i] = ctx->phase_ms[i];
    if (calls_out) calls_out[i] = ctx->phase_calls[i];
  }
  return GSGPC_OK;
}

gsgpc_status gsgpc_ctx_reset_phase_times(gsgpc_ctx* ctx) {
  if (!ctx) return GSGPC_INVALID_ARGUMENT;
  for (int i = 0; i < kPhases; ++i) {
    ctx->phase_ms[i] = 0;
    ctx->phase_calls[i] = 0;
  }
  return GSGPC_OK;
}

gsgpc_status gsgpc_diag_fp64_peak(gsgpc_ctx* ctx, double* tflops) {
  return guard(ctx, [&] {
    if (!tflops) invalid("tflops is NULL");
    *tflops = gsgpc::measure_fp64_peak(ctx->stream);
  });
}

gsgpc_status gsgpc_diag_fp64_tensor(gsgpc_ctx* ctx, double* dmma, double* mixed) {
  return guard(ctx, [&] {
    if (!dmma || !mixed) invalid("NULL argument");
    gsgpc::measure_fp64_tensor(ctx->stream, dmma, mixed);
  });
}

gsgpc_status gsgpc_fit_grid_to_data(int dim, const double* lo, const double* hi, const int64_t* sizes, int scheme,
                                    gsgpc_grid* out) {
  try {
    if (!out || !lo || !hi || !sizes) return GSGPC_INVALID_ARGUMENT;
    if (dim < 1 || dim > GSGPC_MAX_DIM) return dim < 1 ? GSGPC_INVALID_ARGUMENT : GSGPC_UNSUPPORTED;
    const int r = scheme == GSGPC_LINEAR ? 1 : 2;
    gsgpc_grid g{};
    g.dim = dim;
    for (int k = 0; k < dim; ++k) {
      const int64_t m = sizes[k];
      if (m < 2 * r + 2) return GSGPC_INVALID_ARGUMENT;  // "need at least 2r+2 points per dimension"
      if (!(hi[k] > lo[k])) return GSGPC_INVALID_ARGUMENT;  // "empty data range"
      const double s = (hi[k] - lo[k]) / static_cast<double>(m - 1 - 2 * r);
      g.min[k] = lo[k] - r * s;
      g.max[k] = hi[k] + r * s;
      g.size[k] = m;
    }
    *out = g;
    return GSGPC_OK;
  } catch (...) {
    return GSGPC_RUNTIME_ERROR;
  }
}

gsgpc_status gsgpc_interp_weights(gsgpc_ctx* ctx, const gsgpc_grid* grid, int scheme, const gsgpc_points* pts,
                                  int64_t n, int64_t* idx, double* w, int32_t* nnz, int32_t* status) {
  return guard(ctx, [&] {
    const GridDev g = make_grid(grid, scheme);
    check_points(pts, n, false);
    if (n == 0) return;
    int width = 1;
    for (int k = 0; k < g.d; ++k) width *= g.W;
    const bool dev = is_device_ptr(pts->x);
    const PointsDev P = dev ? points_dev(pts, g.d, 0) : stage_points(ctx, pts, g.d, 0, n, false, "iw_stage");
    DBuf& bi = ctx->buf("iw_idx");
    DBuf& bw = ctx->buf("iw_w");
    DBuf& bn = ctx->buf("iw_nnz");
    DBuf& bs = ctx->buf("iw_st");
    bi.ensure(sizeof(int64_t) * n * width);
    bw.ensure(sizeof(double) * n * width);
    bn.ensure(sizeof(int) * n);
    bs.ensure(sizeof(int) * n);
    run_interp_weights(ctx->L(), pts->dtype, P, n, g, bi.as<int64_t>(), bw.as<double>(), bn.as<int>(), bs.as<int>());
    if (idx) GSGPC_CUDA(cudaMemcpyAsync(idx, bi.p, sizeof(int64_t) * n * width, cudaMemcpyDefault, ctx->stream));
    if (w) GSGPC_CUDA(cudaMemcpyAsync(w, bw.p, sizeof(double) * n * width, cudaMemcpyDefault, ctx->stream));
    if (nnz) GSGPC_CUDA(cudaMemcpyAsync(nnz, bn.p, sizeof(int) * n, cudaMemcpyDefault, ctx->stream));
    if (status) GSGPC_CUDA(cudaMemcpyAsync(status, bs.p, sizeof(int) * n, cudaMemcpyDefault, ctx->stream));
    GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

gsgpc_status gsgpc_stats_create(gsgpc_ctx* ctx, const gsgpc_grid* grid, int scheme, gsgpc_stats** out) {
  return guard(ctx, [&] {
    if (!out) invalid("out is NULL");
    *out = new_stats(ctx, grid, scheme);
  });
}

void gsgpc_stats_destroy(gsgpc_stats* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  cudaDeviceSynchronize();
  delete s;
}

// A batch committed in several chunks snapshots the accumulator first, so a failing later
// chunk leaves it unchanged (the reference's single pass throws before returning any
// statistics).
struct StatsSnapshot {
  gsgpc_ctx* ctx;
  gsgpc_stats* s;
  bool active = false;
  int64_t n_before = 0;
  StatsSnapshot(gsgpc_ctx* c, gsgpc_stats* st, bool take) : ctx(c), s(st), active(take), n_before(st->n) {
    if (s->probe_seeded) {  // probe stream positions (restored on any failure)
      DBuf& br = ctx->buf("bk_rng");
      br.ensure(sizeof(uint64_t) * s->probes * 313);
      GSGPC_CUDA(cudaMemcpyAsync(br.p, s->rng.p, sizeof(uint64_t) * s->probes * 313, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
    }
    if (!active) return;
    DBuf& bm = ctx->buf("bk_mom");
    bm.ensure(sizeof(double) * s->g.cells * s->Q + 8);
    GSGPC_CUDA(cudaMemcpyAsync(bm.p, s->mom.p, sizeof(double) * s->g.cells * s->Q, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    DBuf& bq = ctx->buf("bk_pat");
    bq.ensure(static_cast<size_t>(s->g.cells) * s->NP);
    GSGPC_CUDA(cudaMemcpyAsync(bq.p, s->pat.p, static_cast<size_t>(s->g.cells) * s->NP, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    DBuf& by = ctx->buf("bk_yty");
    by.ensure(sizeof(double));
    GSGPC_CUDA(cudaMemcpyAsync(by.p, s->yty.p, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    if (s->probes) {
      DBuf& bp = ctx->buf("bk_pmom");
      bp.ensure(sizeof(double) * s->g.cells * s->probes * s->QY);
      GSGPC_CUDA(cudaMemcpyAsync(bp.p, s->pmom.p, sizeof(double) * s->g.cells * s->probes * s->QY,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
    }
  }
  void restore() {
    if (s->probe_seeded) {
      cudaStreamSynchronize(ctx->stream);
      cudaMemcpy(s->rng.p, ctx->buf("bk_rng").p, sizeof(uint64_t) * s->probes * 313, cudaMemcpyDeviceToDevice);
    }
    s->n = n_before;  // the failing batch's add_chunk counted its rows before the check
    s->finalized = false;
    if (!active) return;
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpy(s->mom.p, ctx->buf("bk_mom").p, sizeof(double) * s->g.cells * s->Q, cudaMemcpyDeviceToDevice);
    cudaMemcpy(s->yty.p, ctx->buf("bk_yty").p, sizeof(double), cudaMemcpyDeviceToDevice);
    cudaMemcpy(s->pat.p, ctx->buf("bk_pat").p, static_cast<size_t>(s->g.cells) * s->NP, cudaMemcpyDeviceToDevice);
    if (s->probes) {
      cudaMemcpy(s->pmom.p, ctx->buf("bk_pmom").p, sizeof(double) * s->g.cells * s->probes * s->QY,
                 cudaMemcpyDeviceToDevice);
    }
    s->n = n_before;
    s->finalized = false;
  }
};

gsgpc_status gsgpc_stats_add(gsgpc_ctx* ctx, gsgpc_stats* s, const gsgpc_points* pts, int64_t n,
                             const uint64_t* probe_words, int probes) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    if (s->reduced) invalid("SufficientStatsAccumulator::add: statistics were all-reduced; create a new accumulator");
    check_points(pts, n, true);
    if (probes < 0 || probes > 64) throw Error(GSGPC_UNSUPPORTED, "probes must be in [0, 64]");
    if (s->probe_seeded) {
      if (probe_words) invalid("this accumulator generates its probes (gsgpc_stats_enable_probes)");
      probes = s->probes;
    }
    if (probes > 0 && !probe_words && !s->probe_seeded) invalid("probe words are NULL");
    if (probes > 0) {
      if (s->probes == 0) {
        if (s->n > 0) invalid("probes must be supplied from the first row on");
        s->probes = probes;
        s->pmom.ensure(sizeof(double) * s->g.cells * probes * s->QY);
        GSGPC_CUDA(cudaMemsetAsync(s->pmom.p, 0, sizeof(double) * s->g.cells * probes * s->QY, ctx->stream));
      } else if (s->probes != probes) {
        invalid("probe count differs from the earlier batches");
      }
    } else if (s->probes > 0 && n > 0) {
      invalid("this accumulator carries probe images: every batch needs probe words");
    }
    if (n == 0) return;
    const bool dev = is_device_ptr(pts->x);
    const int nw = probes > 0 ? (probes + 63) / 64 : 0;
    const bool pw_dev = nw ? is_device_ptr(probe_words) : true;
    static const int host_chunk_log2 = [] {
      const char* e = getenv("GSGPC_HOST_CHUNK_LOG2");  // diagnostics: host staging chunk (rows)
      return e ? std::max(16, std::min(28, atoi(e))) : 23;  // B200 config 3 e2e: 2^22 37.5, 2^23 36.9, 2^24 37.3 ms
    }();
    static const int dev_chunk_log2 = [] {
      const char* e = getenv("GSGPC_DEV_CHUNK_LOG2");  // diagnostics: device-resident chunk (rows)
      return e ? std::max(16, std::min(30, atoi(e))) : 27;
    }();
    // host rows: equal chunks of at most 2^host_chunk_log2 rows (no short last chunk)
    const int64_t CH0 = dev ? (int64_t{1} << dev_chunk_log2) : (int64_t{1} << host_chunk_log2);
    const int64_t CH = ceil_div(n, ceil_div(n, CH0));
    const int64_t nchunks = ceil_div(n, CH);
    StatsSnapshot snap(ctx, s, nchunks > 1);
    // host rows: double-buffered staging, the copy of chunk k+1 overlaps the compute of chunk k
    static const char* kSlot[2] = {"stage0", "stage1"};
    PointsDev staged[2];
    static const bool trace = [] {
      const char* e = getenv("GSGPC_E2E_TRACE");  // diagnostics: per-chunk copy / compute timeline
      return e && e[0] == '1';
    }();
    std::vector<cudaEvent_t> tev;  // trace: per chunk copy begin/end, compute begin/end
    auto tmark = [&](cudaStream_t st) {
      if (!trace) return;
      cudaEvent_t e;
      GSGPC_CUDA(cudaEventCreate(&e));
      GSGPC_CUDA(cudaEventRecord(e, st));
      tev.push_back(e);
    };
    std::vector<int> tkind;
    auto stage = [&](int64_t k) {
      const int sl = static_cast<int>(k & 1);
      const int64_t a0 = k * CH, a1 = std::min(n, a0 + CH);
      if (k >= 2) GSGPC_CUDA(cudaStreamWaitEvent(ctx->copy, ctx->ev_free[sl], 0));
      tmark(ctx->copy);
      staged[sl] = stage_points(ctx, pts, s->g.d, a0, a1, true, kSlot[sl], ctx->copy);
      tmark(ctx->copy);
      if (trace) tkind.push_back(0);
      GSGPC_CUDA(cudaEventRecord(ctx->ev_copied[sl], ctx->copy));
    };
    // device-resident rows in several chunks: binning of chunk k + 1 under K1 of chunk k (ChunkPipe)
    static const int pipe_env = [] {
      const char* e = getenv("GSGPC_CHUNK_PIPE");  // diagnostics: 1 = on (default off: measured slower at d = 2)
      return e ? atoi(e) : 0;
    }();
    ChunkPipe pipe;
    const bool piped = dev && nchunks > 1 && probes == 0 && !ctx->timing && pipe_env > 0;
    struct PipeEvents {
      ChunkPipe* p;
      ~PipeEvents() {
        for (int i = 0; i < 2; ++i) {
          if (p->binned[i]) cudaEventDestroy(p->binned[i]);
          if (p->k1done[i]) cudaEventDestroy(p->k1done[i]);
        }
      }
    } pipe_events{&pipe};
    try {
      bin_error_reset(ctx);
      if (piped) {
        ctx->ensure_sort_stream();
        pipe.bin = ctx->sort;
        for (int i = 0; i < 2; ++i) {
          GSGPC_CUDA(cudaEventCreateWithFlags(&pipe.binned[i], cudaEventDisableTiming));
          GSGPC_CUDA(cudaEventCreateWithFlags(&pipe.k1done[i], cudaEventDisableTiming));
        }
        // fork: the binning stream starts after everything queued so far (snapshot, error reset)
        GSGPC_CUDA(cudaEventRecord(pipe.binned[0], ctx->stream));
        GSGPC_CUDA(cudaStreamWaitEvent(pipe.bin, pipe.binned[0], 0));
      }
      if (!dev) {
        ctx->ensure_copy_stream();
        // the staging buffers may still be read by earlier work on the compute stream
        GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
        stage(0);
      }
      for (int64_t k = 0; k < nchunks; ++k) {
        const int64_t r0 = k * CH, r1 = std::min(n, r0 + CH);
        PointsDev P;
        if (dev) {
          P = points_dev(pts, s->g.d, r0);
        } else {
          if (k + 1 < nchunks) stage(k + 1);
          GSGPC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[k & 1], 0));
          P = staged[k & 1];
        }
        const uint64_t* pw = nullptr;
        if (s->probe_seeded && !probe_words) {
          PhaseTimer ptr(ctx);
          const int hr = ptr.begin(8);
          gen_probe_words(ctx, s, r1 - r0);
          ptr.end(hr);
          pw = ctx->buf("probe_stage").as<uint64_t>();
        } else if (nw) {
          if (pw_dev) {
            pw = probe_words + r0 * nw;
          } else {
            DBuf& b = ctx->buf("probe_stage");
            b.ensure(sizeof(uint64_t) * nw * (r1 - r0));
            GSGPC_CUDA(cudaMemcpyAsync(b.p, probe_words + r0 * nw, sizeof(uint64_t) * nw * (r1 - r0),
                                       cudaMemcpyHostToDevice, ctx->stream));
            pw = b.as<uint64_t>();
          }
        }
        tmark(ctx->stream);
        pipe.set = static_cast<int>(k & 1);
        pipe.k = k;
        add_chunk(ctx, s, pts->dtype, P, r1 - r0, s->n, pw, probes, piped ? &pipe : nullptr);
        tmark(ctx->stream);
        if (trace) tkind.push_back(1);
        if (!dev) GSGPC_CUDA(cudaEventRecord(ctx->ev_free[k & 1], ctx->stream));
      }
      if (!dev) GSGPC_CUDA(cudaStreamSynchronize(ctx->copy));
      if (trace && !tev.empty()) {
        GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
        for (size_t i = 0; i < tkind.size(); ++i) {
          float a = 0.0f, b = 0.0f;
          GSGPC_CUDA(cudaEventElapsedTime(&a, tev[0], tev[2 * i]));
          GSGPC_CUDA(cudaEventElapsedTime(&b, tev[0], tev[2 * i + 1]));
          std::fprintf(stderr, "[gsgpc e2e trace] %s %8.3f .. %8.3f ms\n", tkind[i] ? "compute" : "copy   ", a, b);
        }
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
      }
      bin_error_check(ctx);
    } catch (...) {
      if (ctx->copy) cudaStreamSynchronize(ctx->copy);
      if (piped && pipe.bin) cudaStreamSynchronize(pipe.bin);
      snap.restore();
      throw;
    }
  });
}

// GSGPDAT1 ingest (BinaryRowStream, io.hpp:31-45 / io.cpp:103-122, driven like
// sufficient_stats, interp.cpp:244-263).  A reader thread fills one pinned buffer while the
// other is copied to the device (copy stream) and binned / accumulated (compute stream).
// Errors keep the reference's texts and order: rows before a truncation point are processed
// first (an out-of-grid row there wins), then "truncated file while reading coordinate /
// response".  Transactional: on any error the accumulator is left unchanged.
gsgpc_status gsgpc_stats_add_file(gsgpc_ctx* ctx, gsgpc_stats* s, const char* path, int64_t* rows_added) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    if (!path) invalid("path is NULL");
    if (s->reduced) invalid("SufficientStatsAccumulator::add: statistics were all-reduced; create a new accumulator");
    if (s->probes > 0 && !s->probe_seeded) {
      invalid("this accumulator carries caller-supplied probe images: add rows with gsgpc_stats_add");
    }
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "rb"), std::fclose);
    if (!f) invalid(std::string("cannot open binary dataset: ") + path);
    char magic[8];
    if (std::fread(magic, 1, 8, f.get()) != 8 || std::memcmp(magic, "GSGPDAT1", 8) != 0) {
      invalid(std::string("bad magic in binary dataset: ") + path);
    }
    uint64_t hdr[2];
    if (std::fread(&hdr[0], 8, 1, f.get()) != 1) invalid("truncated file while reading row count");
    if (std::fread(&hdr[1], 8, 1, f.get()) != 1) invalid("truncated file while reading dimension");
    const int64_t n = static_cast<int64_t>(hdr[0]);
    const int64_t d = static_cast<int64_t>(hdr[1]);
    if (d < 1 || d > 64) invalid("binary dataset: bad dimension");
    if (d != s->g.d) invalid("sufficient_stats: stream/grid dimension mismatch");
    if (n < 0) invalid("binary dataset: bad row count");
    if (std::fseek(f.get(), 0, SEEK_END) != 0) invalid(std::string("cannot seek binary dataset: ") + path);
    const int64_t size = static_cast<int64_t>(ftello(f.get()));
    std::fseek(f.get(), 24, SEEK_SET);
    const int64_t rowb = (d + 1) * 8;
    const int64_t avail = std::min<int64_t>(n, std::max<int64_t>(0, size - 24) / rowb);
    const bool truncated = avail < n;
    const int64_t tail_fields = truncated ? (std::max<int64_t>(0, size - 24) - avail * rowb) / 8 : 0;
    const int64_t CH = int64_t{1} << 22;  // rows per chunk (128 MiB of f64 rows at d = 3)
    const int64_t nchunks = ceil_div(avail, CH);
    StatsSnapshot snap(ctx, s, nchunks > 1 || (truncated && avail > 0));
    ctx->ensure_copy_stream();
    GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));  // staging slots may still be in use
    for (int b = 0; b < 2; ++b) ctx->file_pin[b].ensure(static_cast<size_t>(std::min(CH, std::max<int64_t>(avail, 1)) * rowb));
    cudaEvent_t h2d[2];
    for (int b = 0; b < 2; ++b) GSGPC_CUDA(cudaEventCreateWithFlags(&h2d[b], cudaEventDisableTiming));
    struct EvGuard {
      cudaEvent_t* e;
      ~EvGuard() {
        for (int b = 0; b < 2; ++b) cudaEventDestroy(e[b]);
      }
    } evg{h2d};
    auto read_chunk = [&](int64_t k) -> bool {
      const int64_t rows = std::min(CH, avail - k * CH);
      return std::fread(ctx->file_pin[k & 1].p, static_cast<size_t>(rowb), static_cast<size_t>(rows), f.get()) ==
             static_cast<size_t>(rows);
    };
    static const char* kSlot[2] = {"stage0", "stage1"};
    int64_t done = 0;
    try {
      bin_error_reset(ctx);
      bool ok_next = nchunks > 0 ? read_chunk(0) : true;
      for (int64_t k = 0; k < nchunks; ++k) {
        if (!ok_next) invalid("truncated file while reading coordinate");
        const int64_t rows = std::min(CH, avail - k * CH);
        const int sl = static_cast<int>(k & 1);
        gsgpc_points hp{};
        hp.dtype = GSGPC_F64;
        hp.x = ctx->file_pin[sl].p;
        hp.x_row_stride = d + 1;
        for (int j = 0; j < d; ++j) hp.x_col_offset[j] = j;
        hp.y = static_cast<const double*>(ctx->file_pin[sl].p) + d;
        hp.y_stride = d + 1;
        if (k >= 2) GSGPC_CUDA(cudaStreamWaitEvent(ctx->copy, ctx->ev_free[sl], 0));
        const PointsDev P = stage_points(ctx, &hp, static_cast<int>(d), 0, rows, true, kSlot[sl], ctx->copy);
        GSGPC_CUDA(cudaEventRecord(h2d[sl], ctx->copy));
        // read the next chunk into the other buffer while this one is copied and binned
        std::thread reader;
        bool ok = true;
        if (k + 1 < nchunks) {
          GSGPC_CUDA(cudaEventSynchronize(h2d[sl ^ 1]));  // its previous copy has finished
          reader = std::thread([&] { ok = read_chunk(k + 1); });
        }
        try {
          GSGPC_CUDA(cudaStreamWaitEvent(ctx->stream, h2d[sl], 0));
          const uint64_t* pw = nullptr;
          if (s->probe_seeded) {
            gen_probe_words(ctx, s, rows);
            pw = ctx->buf("probe_stage").as<uint64_t>();
          }
          add_chunk(ctx, s, GSGPC_F64, P, rows, done, pw, s->probes, nullptr);
          GSGPC_CUDA(cudaEventRecord(ctx->ev_free[sl], ctx->stream));
        } catch (...) {
          if (reader.joinable()) reader.join();
          throw;
        }
        if (reader.joinable()) reader.join();
        ok_next = ok;
        done += rows;
      }
      GSGPC_CUDA(cudaStreamSynchronize(ctx->copy));
      bin_error_check(ctx);  // a bad row before the truncation point is reported first
      if (truncated) {
        invalid(std::string("truncated file while reading ") + (tail_fields < d ? "coordinate" : "response"));
      }
    } catch (...) {
      cudaStreamSynchronize(ctx->copy);
      snap.restore();
      throw;
    }
    if (rows_added) *rows_added = done;
  });
}

gsgpc_status gsgpc_stats_enable_probes(gsgpc_ctx* ctx, gsgpc_stats* s, int probes, uint64_t seed) {
  return gsgpc_stats_enable_probes_at(ctx, s, probes, seed, 0);
}

gsgpc_status gsgpc_stats_enable_probes_at(gsgpc_ctx* ctx, gsgpc_stats* s, int probes, uint64_t seed,
                                          int64_t first_row) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    if (probes < 1 || probes > 64) throw Error(GSGPC_UNSUPPORTED, "probes must be in [1, 64]");
    if (first_row < 0) invalid("gsgpc_stats_enable_probes_at: first_row must be >= 0");
    if (s->n > 0 || s->probes > 0) invalid("gsgpc_stats_enable_probes: call before the first row is added");
    s->probes = probes;
    s->probe_seeded = true;
    s->probe_seed = seed;
    s->probe_first_row = first_row;
    seed_probe_streams(ctx, s);  // rademacher_probe (gp.cpp:16-25) streams, generated on the device
    s->pmom.ensure(sizeof(double) * s->g.cells * probes * s->QY);
    GSGPC_CUDA(cudaMemsetAsync(s->pmom.p, 0, sizeof(double) * s->g.cells * probes * s->QY, ctx->stream));
  });
}

gsgpc_status gsgpc_stats_reset(gsgpc_ctx* ctx, gsgpc_stats* s) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    GSGPC_CUDA(cudaMemsetAsync(s->mom.p, 0, sizeof(double) * s->g.cells * s->Q, ctx->stream));
    GSGPC_CUDA(cudaMemsetAsync(s->pat.p, 0, static_cast<size_t>(s->g.cells) * s->NP, ctx->stream));
    s->loaded_touched.clear();
    if (s->probes) {
      GSGPC_CUDA(cudaMemsetAsync(s->pmom.p, 0, sizeof(double) * s->g.cells * s->probes * s->QY, ctx->stream));
    }
    GSGPC_CUDA(cudaMemsetAsync(s->yty.p, 0, sizeof(double), ctx->stream));
    s->n = 0;
    s->finalized = false;
    s->reduced = false;
    if (s->probe_seeded) seed_probe_streams(ctx, s);  // a fresh pass restarts the probe streams
  });
}

gsgpc_status gsgpc_stats_merge(gsgpc_ctx* ctx, gsgpc_stats* dst, const gsgpc_stats* src) {
  return guard(ctx, [&] {
    if (!dst || !src) invalid("stats is NULL");
    if (dst->reduced || src->reduced) invalid("SufficientStatsAccumulator::merge: all-reduced statistics");
    bool same = dst->scheme == src->scheme && dst->g.d == src->g.d && dst->probes == src->probes;
    for (int k = 0; same && k < dst->g.d; ++k) {
      same = dst->grid.size[k] == src->grid.size[k] && dst->grid.min[k] == src->grid.min[k] &&
             dst->grid.max[k] == src->grid.max[k];
    }
    if (!same) invalid("SufficientStatsAccumulator::merge: mismatched shards");
    // seeded probe images are sums over global rows: shards merge only when their rows are
    // adjacent in the one stream order ([first, first + n) intervals touching)
    bool src_after = true;
    if (dst->probe_seeded || src->probe_seeded) {
      if (!(dst->probe_seeded && src->probe_seeded) || dst->probe_seed != src->probe_seed) {
        invalid("SufficientStatsAccumulator::merge: shards carry different probe streams");
      }
      src_after = src->probe_first_row == dst->probe_first_row + dst->n;
      const bool src_before = dst->probe_first_row == src->probe_first_row + src->n;
      if (!src_after && !src_before) {
        invalid("SufficientStatsAccumulator::merge: probe-seeded shards must cover adjacent row ranges "
                "(gsgpc_stats_enable_probes_at first_row)");
      }
    }
    const Launch L = ctx->L();
    const int64_t nm = dst->g.cells * dst->Q;
    run_axpby(L, nm, 1.0, dst->mom.as<double>(), 1.0, src->mom.as<double>(), dst->mom.as<double>());
    run_or_bytes(L, dst->g.cells * dst->NP, dst->pat.as<uint8_t>(), src->pat.as<uint8_t>());
    if (dst->probes) {
      const int64_t np = dst->g.cells * dst->probes * dst->QY;
      run_axpby(L, np, 1.0, dst->pmom.as<double>(), 1.0, src->pmom.as<double>(), dst->pmom.as<double>());
    }
    run_axpby(L, 1, 1.0, dst->yty.as<double>(), 1.0, src->yty.as<double>(), dst->yty.as<double>());
    if (dst->probe_seeded) {
      if (src_after) {  // continue from the end of src's rows
        GSGPC_CUDA(cudaMemcpyAsync(dst->rng.p, src->rng.p, sizeof(uint64_t) * dst->probes * 313,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
      } else {
        dst->probe_first_row = src->probe_first_row;
      }
    }
    dst->n += src->n;
    dst->finalized = false;
    GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

gsgpc_status gsgpc_stats_finalize(gsgpc_ctx* ctx, gsgpc_stats* s) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    finalize_stats(ctx, s);
  });
}

gsgpc_status gsgpc_sufficient_stats(gsgpc_ctx* ctx, const gsgpc_grid* grid, int scheme, const gsgpc_points* pts,
                                    int64_t n, gsgpc_stats** out) {
  if (!out) return GSGPC_INVALID_ARGUMENT;
  *out = nullptr;
  gsgpc_stats* s = nullptr;
  gsgpc_status st = gsgpc_stats_create(ctx, grid, scheme, &s);
  if (st != GSGPC_OK) return st;
  st = gsgpc_stats_add(ctx, s, pts, n, nullptr, 0);
  if (st == GSGPC_OK) st = gsgpc_stats_finalize(ctx, s);
  if (st != GSGPC_OK) {
    gsgpc_stats_destroy(s);
    return st;
  }
  *out = s;
  return GSGPC_OK;
}

gsgpc_status gsgpc_stats_info(gsgpc_ctx* ctx, gsgpc_stats* s, int64_t* m, int64_t* n, double* yty,
                              int64_t* n_offsets, int32_t* probes) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    if (m) *m = s->g.m;
    if (n) *n = s->reduced ? static_cast<int64_t>(read_scalar(ctx, s->tail() + 1)) : s->n;
    if (yty) *yty = stats_yty(ctx, s);
    if (n_offsets) *n_offsets = s->S_min;
    if (probes) *probes = s->probes;
  });
}

gsgpc_status gsgpc_stats_grid(const gsgpc_stats* s, gsgpc_grid* grid, int* scheme) {
  if (!s) return GSGPC_INVALID_ARGUMENT;
  if (grid) *grid = s->grid;
  if (scheme) *scheme = s->scheme;
  return GSGPC_OK;
}

gsgpc_status gsgpc_stats_copy_wty(gsgpc_ctx* ctx, gsgpc_stats* s, double* out) {
  return guard(ctx, [&] {
    if (!s || !out) invalid("NULL argument");
    finalize_stats(ctx, s);
    copy_out(ctx, out, s->wty(), sizeof(double) * s->g.m);
  });
}

gsgpc_status gsgpc_stats_copy_stencil(gsgpc_ctx* ctx, gsgpc_stats* s, double* values, int32_t* offsets) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    finalize_stats(ctx, s);
    if (values) copy_out(ctx, values, s->stencil(), sizeof(double) * s->S_min * s->g.m);
    if (offsets) {
      const int E = 2 * s->g.W - 1, d = s->g.d;
      int S = 1;
      for (int k = 0; k < d; ++k) S *= E;
      const int c0 = (S - 1) / 2;
      for (int i = 0; i < s->S_min; ++i) {
        int q = c0 + i;
        for (int k = d - 1; k >= 0; --k) {
          offsets[i * d + k] = q % E - (s->g.W - 1);
          q /= E;
        }
      }
    }
  });
}

gsgpc_status gsgpc_stats_copy_probe_images(gsgpc_ctx* ctx, gsgpc_stats* s, double* out) {
  return guard(ctx, [&] {
    if (!s || !out) invalid("NULL argument");
    if (s->probes == 0) invalid("no probe images were accumulated");
    finalize_stats(ctx, s);
    copy_out(ctx, out, s->pimg(), sizeof(double) * s->probes * s->g.m);
  });
}

}  // extern "C"

namespace {

// Host CSR view of the stencil (SufficientStats::wtw() layout).
struct HostCsr {
  std::vector<int64_t> rp, col;
  std::vector<double> val;
};

HostCsr build_csr(gsgpc_ctx* ctx, gsgpc_stats* s) {
  finalize_stats(ctx, s);
  const int64_t m = s->g.m;
  const int d = s->g.d, W = s->g.W, E = 2 * W - 1;
  std::vector<double> st(static_cast<size_t>(s->S_min) * m);
  copy_out(ctx, st.data(), s->stencil(), sizeof(double) * st.size());
  // structure: the pairs some row touched (the reference's hash keys), not the nonzero values
  std::vector<uint8_t> tmask;
  const std::vector<uint8_t>* touched = &s->loaded_touched;
  if (s->loaded_touched.empty()) {
    DBuf& tb = ctx->buf("touched");
    tb.ensure(st.size());
    run_touched(ctx->L(), s->g, s->S_min, s->pat.as<uint8_t>(), tb.as<uint8_t>());
    tmask.resize(st.size());
    copy_out(ctx, tmask.data(), tb.p, tmask.size());
    touched = &tmask;
  }
  int S = 1;
  for (int k = 0; k < d; ++k) S *= E;
  const int c0 = (S - 1) / 2;
  // full offset list in lexicographic order
  std::vector<std::array<int, 3>> dl(S);
  std::vector<int64_t> fl(S);
  for (int q = 0; q < S; ++q) {
    int r = q;
    std::array<int, 3> dd{0, 0, 0};
    for (int k = d - 1; k >= 0; --k) {
      dd[k] = r % E - (W - 1);
      r /= E;
    }
    dl[q] = dd;
    int64_t f = 0;
    for (int k = 0; k < d; ++k) f = f * s->g.sz[k] + dd[k];
    fl[q] = f;
  }
  HostCsr c;
  c.rp.assign(m + 1, 0);
  std::vector<std::pair<int64_t, double>> row;
  for (int64_t a = 0; a < m; ++a) {
    int64_t co[3] = {0, 0, 0};
    int64_t r = a;
    for (int k = d - 1; k >= 0; --k) {
      co[k] = r % s->g.sz[k];
      r /= s->g.sz[k];
    }
    row.clear();
    for (int q = 0; q < S; ++q) {
      bool ok = true;
      for (int k = 0; k < d; ++k) {
        const int64_t v = co[k] + dl[q][k];
        ok = ok && v >= 0 && v < s->g.sz[k];
      }
      if (!ok) continue;
      const int64_t b = a + fl[q];
      const size_t h = q >= c0 ? static_cast<size_t>(q - c0) * m + a : static_cast<size_t>((S - 1 - q) - c0) * m + b;
      if ((*touched)[h]) row.emplace_back(b, st[h]);
    }
    std::sort(row.begin(), row.end());
    for (auto& e : row) {
      c.col.push_back(e.first);
      c.val.push_back(e.second);
    }
    c.rp[a + 1] = static_cast<int64_t>(c.col.size());
  }
  return c;
}

}  // namespace

extern "C" {

gsgpc_status gsgpc_stats_csr_nnz(gsgpc_ctx* ctx, gsgpc_stats* s, int64_t* nnz, int64_t* max_row_nnz) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    const HostCsr c = build_csr(ctx, s);
    if (nnz) *nnz = static_cast<int64_t>(c.val.size());
    if (max_row_nnz) {
      int64_t b = 0;
      for (size_t i = 0; i + 1 < c.rp.size(); ++i) b = std::max(b, c.rp[i + 1] - c.rp[i]);
      *max_row_nnz = b;
    }
  });
}

gsgpc_status gsgpc_stats_export_csr(gsgpc_ctx* ctx, gsgpc_stats* s, int64_t* row_ptr, int64_t* col, double* val) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    const HostCsr c = build_csr(ctx, s);
    if (row_ptr) std::memcpy(row_ptr, c.rp.data(), sizeof(int64_t) * c.rp.size());
    if (col) std::memcpy(col, c.col.data(), sizeof(int64_t) * c.col.size());
    if (val) std::memcpy(val, c.val.data(), sizeof(double) * c.val.size());
  });
}

gsgpc_status gsgpc_stats_apply_wtw(gsgpc_ctx* ctx, gsgpc_stats* s, const double* v, double* out) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    finalize_stats(ctx, s);
    const StencilDesc sd = stencil_desc(s);
    const double* dv = dev_in(ctx, v, sd.m, "wtw_in");
    DevOut o(ctx, out, sd.m, "wtw_out");
    DBuf& fl = ctx->buf("wtw_flag");
    fl.ensure(sizeof(int));
    GSGPC_CUDA(cudaMemsetAsync(fl.p, 0, sizeof(int), ctx->stream));
    run_spmv(ctx->L(), sd, s->stencil(), dv, o.dev, fl.as<int>());
    int bad = 0;
    copy_out(ctx, &bad, fl.p, sizeof(int));
    if (bad) {  // non-finite input met: the rows at stake follow the reference's stored pairs
      const size_t nt = static_cast<size_t>(s->S_min) * sd.m;
      DBuf& tb = ctx->buf("touched");
      tb.ensure(nt);
      if (!s->loaded_touched.empty()) {
        GSGPC_CUDA(cudaMemcpyAsync(tb.p, s->loaded_touched.data(), nt, cudaMemcpyHostToDevice, ctx->stream));
      } else {
        run_touched(ctx->L(), s->g, s->S_min, s->pat.as<uint8_t>(), tb.as<uint8_t>());
      }
      run_spmv_touched(ctx->L(), sd, s->stencil(), dv, tb.as<uint8_t>(), o.dev);
    }
    o.finish();
  });
}

gsgpc_status gsgpc_stats_reduce_buffer(gsgpc_ctx* ctx, gsgpc_stats* s, double** dev_ptr, int64_t* count) {
  return guard(ctx, [&] {
    if (!s || !dev_ptr || !count) invalid("NULL argument");
    finalize_stats(ctx, s);
    *dev_ptr = s->fin.as<double>();
    *count = s->fin_count();
  });
}

gsgpc_status gsgpc_stats_pattern_buffer(gsgpc_ctx* ctx, gsgpc_stats* s, uint8_t** dev_ptr, int64_t* count) {
  return guard(ctx, [&] {
    if (!s || !dev_ptr || !count) invalid("NULL argument");
    if (s->reduced) invalid("gsgpc_stats_pattern_buffer: statistics were already all-reduced");
    *dev_ptr = s->pat.as<uint8_t>();
    *count = s->g.cells * s->NP;
  });
}

gsgpc_status gsgpc_stats_mark_reduced(gsgpc_ctx* ctx, gsgpc_stats* s) {
  return guard(ctx, [&] {
    if (!s) invalid("stats is NULL");
    if (!s->finalized && !s->reduced) invalid("gsgpc_stats_mark_reduced: call gsgpc_stats_reduce_buffer first");
    s->reduced = true;
    GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
    s->n = static_cast<int64_t>(read_scalar(ctx, s->tail() + 1));
  });
}

// ---------------------------------------------------------------- GSGPSST1 (io.cpp:192-262)
gsgpc_status gsgpc_stats_save(gsgpc_ctx* ctx, gsgpc_stats* s, const char* path) {
  return guard(ctx, [&] {
    if (!s || !path) invalid("NULL argument");
    const HostCsr c = build_csr(ctx, s);
    std::vector<double> wty(s->g.m);
    copy_out(ctx, wty.data(), s->wty(), sizeof(double) * s->g.m);
    const double yty = stats_yty(ctx, s);
    std::ofstream f(path, std::ios::binary);
    if (!f) invalid(std::string("cannot open for writing: ") + path);
    auto u64 = [&](uint64_t v) { f.write(reinterpret_cast<const char*>(&v), 8); };
    auto f64 = [&](double v) { f.write(reinterpret_cast<const char*>(&v), 8); };
    f.write("GSGPSST1", 8);
    u64(static_cast<uint64_t>(s->grid.dim));
    for (int k = 0; k < s->grid.dim; ++k) {
      f64(s->grid.min[k]);
      f64(s->grid.max[k]);
      u64(static_cast<uint64_t>(s->grid.size[k]));
    }
    u64(s->scheme == GSGPC_LINEAR ? 0 : 1);
    u64(static_cast<uint64_t>(s->g.m));
    u64(static_cast<uint64_t>(s->n));
    u64(static_cast<uint64_t>(c.val.size()));
    f64(yty);
    for (double v : wty) f64(v);
    // triplets in CSR row order
    std::vector<char> blob(24 * c.val.size());
    size_t o = 0;
    for (int64_t r = 0; r + 1 < static_cast<int64_t>(c.rp.size()); ++r) {
      for (int64_t k = c.rp[r]; k < c.rp[r + 1]; ++k) {
        const uint64_t rr = static_cast<uint64_t>(r), cc = static_cast<uint64_t>(c.col[k]);
        std::memcpy(&blob[o], &rr, 8);
        std::memcpy(&blob[o + 8], &cc, 8);
        std::memcpy(&blob[o + 16], &c.val[k], 8);
        o += 24;
      }
    }
    f.write(blob.data(), static_cast<std::streamsize>(blob.size()));
    if (!f) invalid(std::string("write failed: ") + path);
  });
}

gsgpc_status gsgpc_stats_load(gsgpc_ctx* ctx, const char* path, gsgpc_stats** out) {
  return guard(ctx, [&] {
    if (!path || !out) invalid("NULL argument");
    std::ifstream f(path, std::ios::binary);
    if (!f) invalid(std::string("cannot open stats file: ") + path);
    char magic[8];
    if (!f.read(magic, 8) || std::memcmp(magic, "GSGPSST1", 8) != 0) {
      invalid(std::string("bad magic in stats file: ") + path);
    }
    auto u64 = [&](const char* what) {
      uint64_t v;
      if (!f.read(reinterpret_cast<char*>(&v), 8)) invalid(std::string("truncated file while reading ") + what);
      return v;
    };
    auto f64 = [&](const char* what) {
      double v;
      if (!f.read(reinterpret_cast<char*>(&v), 8)) invalid(std::string("truncated file while reading ") + what);
      return v;
    };
    const int d = static_cast<int>(u64("grid dimension"));
    if (d < 1 || d > 64) invalid("stats file: bad grid dimension");
    if (d > GSGPC_MAX_DIM) throw Error(GSGPC_UNSUPPORTED, "stats file: grid dimension > 3 is not supported");
    gsgpc_grid g{};
    g.dim = d;
    for (int k = 0; k < d; ++k) {
      g.min[k] = f64("grid min");
      g.max[k] = f64("grid max");
      g.size[k] = static_cast<int64_t>(u64("grid size"));
    }
    const int scheme = u64("scheme") == 0 ? GSGPC_LINEAR : GSGPC_CUBIC;
    const int64_t m = static_cast<int64_t>(u64("grid size"));
    const int64_t n = static_cast<int64_t>(u64("row count"));
    const int64_t nnz = static_cast<int64_t>(u64("nnz"));
    const double yty = f64("yty");
    std::unique_ptr<gsgpc_stats> s(new_stats(ctx, &g, scheme));
    if (s->g.m != m) invalid("stats file: grid/statistics size mismatch");
    std::vector<double> wty(m);
    for (int64_t i = 0; i < m; ++i) wty[i] = f64("wty");
    const int W = s->g.W, E = 2 * W - 1;
    int S = 1;
    for (int k = 0; k < d; ++k) S *= E;
    const int c0 = (S - 1) / 2;
    std::vector<double> st(static_cast<size_t>(s->S_min) * m, 0.0);
    s->loaded_touched.assign(st.size(), 0);
    for (int64_t i = 0; i < nnz; ++i) {
      const int64_t r = static_cast<int64_t>(u64("triplet row"));
      const int64_t c = static_cast<int64_t>(u64("triplet col"));
      const double v = f64("triplet value");
      if (r < 0 || r >= m || c < 0 || c >= m) invalid("stats file: triplet index out of range");
      // stencil offset of (r, c); stored once, on the row whose offset is non-negative
      int64_t rr = r, cc = c;
      int q = 0;
      bool ok = true;
      int dig[3];
      for (int k = d - 1; k >= 0; --k) {
        const int64_t ar = rr % s->g.sz[k], ac = cc % s->g.sz[k];
        rr /= s->g.sz[k];
        cc /= s->g.sz[k];
        const int64_t dd = ac - ar;
        if (dd < -(W - 1) || dd > W - 1) ok = false;
        dig[k] = static_cast<int>(dd);
      }
      if (!ok) throw Error(GSGPC_UNSUPPORTED, "stats file: W^T W entry outside the grid stencil");
      for (int k = 0; k < d; ++k) q = q * E + dig[k] + (W - 1);
      if (q >= c0) {
        st[static_cast<size_t>(q - c0) * m + r] = v;
        s->loaded_touched[static_cast<size_t>(q - c0) * m + r] = 1;
      }
    }
    s->fin.ensure(sizeof(double) * s->fin_count());
    GSGPC_CUDA(cudaMemcpyAsync(s->stencil(), st.data(), sizeof(double) * st.size(), cudaMemcpyHostToDevice, ctx->stream));
    GSGPC_CUDA(cudaMemcpyAsync(s->wty(), wty.data(), sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
    const double tail[2] = {yty, static_cast<double>(n)};
    GSGPC_CUDA(cudaMemcpyAsync(s->tail(), tail, sizeof(tail), cudaMemcpyHostToDevice, ctx->stream));
    GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
    s->n = n;
    s->finalized = true;
    s->reduced = true;  // loaded statistics carry no moments: no further add()
    *out = s.release();
  });
}

// ---------------------------------------------------------------- K_G
gsgpc_status gsgpc_kg_create(gsgpc_ctx* ctx, const gsgpc_grid* grid, const double* ls, double outputscale,
                             double noise_std, gsgpc_kg** out) {
  return gsgpc_kg_create_ex(ctx, grid, ls, outputscale, noise_std, 0, out);
}

int64_t gsgpc_next_fast_fft_size(int64_t x) { return next_fast_fft_size(x); }

gsgpc_status gsgpc_kg_create_ex(gsgpc_ctx* ctx, const gsgpc_grid* grid, const double* ls, double outputscale,
                                double noise_std, int64_t fft_min_nodes, gsgpc_kg** out) {
  return guard(ctx, [&] {
    if (!out || !ls) invalid("NULL argument");
    const GridDev g = make_grid(grid, GSGPC_CUBIC);
    if (!(noise_std > 0.0)) invalid("Hyperparams: noise_std must be positive");
    if (!(outputscale > 0.0)) invalid("Hyperparams: outputscale must be positive");
    for (int k = 0; k < g.d; ++k) {
      if (!(ls[k] > 0.0)) invalid("Hyperparams: lengthscales must be positive");
    }
    std::unique_ptr<gsgpc_kg> kg(new gsgpc_kg());
    kg->device = ctx->device;
    kg->grid = *grid;
    kg->m = g.m;
    kg->noise_std = noise_std;
    kg->dev.d = g.d;
    kg->dev.m = g.m;
    for (int k = 0; k < g.d; ++k) {
      // 1-D generator: k(g_0, g_j) along dim k (grid.cpp:42-52 / kernels.cpp:43-55 per factor):
      // d = (x[k] - x2[k]) / ℓ_k with x = min, x2 = min + j·spacing (Grid::point).
      std::vector<double> col(g.sz[k]);
      for (int64_t j = 0; j < g.sz[k]; ++j) {
        const double x2 = g.mn[k] + static_cast<double>(j) * g.sp[k];
        const double dd = (g.mn[k] - x2) / ls[k];
        col[j] = std::exp(-0.5 * (dd * dd));
        if (k == 0) col[j] *= outputscale;
      }
      kg->gen[k].ensure(sizeof(double) * g.sz[k]);
      GSGPC_CUDA(cudaMemcpyAsync(kg->gen[k].p, col.data(), sizeof(double) * g.sz[k], cudaMemcpyHostToDevice,
                                 ctx->stream));
      kg->dev.sz[k] = g.sz[k];
      kg->dev.gen[k] = kg->gen[k].as<double>();
    }
    GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
    kg->fft = kg_fft_create(kg->dev, fft_min_nodes > 0 ? fft_min_nodes : kKgFftMinNodes, ctx->stream);
    kg->dev.fft = kg->fft.get();
    *out = kg.release();
  });
}

void gsgpc_kg_destroy(gsgpc_kg* kg) {
  if (!kg) return;
  cudaSetDevice(kg->device);
  cudaDeviceSynchronize();
  delete kg;
}

gsgpc_status gsgpc_kg_info(const gsgpc_kg* kg, int64_t* m, double* noise_variance) {
  if (!kg) return GSGPC_INVALID_ARGUMENT;
  if (m) *m = kg->m;
  if (noise_variance) *noise_variance = kg->noise_std * kg->noise_std;
  return GSGPC_OK;
}

gsgpc_status gsgpc_kg_apply(gsgpc_ctx* ctx, gsgpc_kg* kg, const double* v, double* out) {
  return guard(ctx, [&] {
    if (!kg) invalid("kg is NULL");
    const double* dv = dev_in(ctx, v, kg->m, "kg_in");
    DevOut o(ctx, out, kg->m, "kg_out");
    DBuf& t0 = ctx->buf("kg_t0");
    DBuf& t1 = ctx->buf("kg_t1");
    t0.ensure(sizeof(double) * kg->m);
    t1.ensure(sizeof(double) * kg->m);
    run_kg_apply(ctx->L(), kg->dev, dv, o.dev, t0.as<double>(), t1.as<double>());
    o.finish();
  });
}

}  // extern "C"

// ---------------------------------------------------------------- EFCG driver
namespace {

constexpr int kGraphIters = 16;

CgCache& cg_setup(gsgpc_ctx* ctx, gsgpc_stats* s, gsgpc_kg* kg, int maxiter) {
  const int64_t m = s->g.m;
  if (!ctx->cg || ctx->cg->stats != s || ctx->cg->kg != kg || ctx->cg->m != m || ctx->cg->trace_cap < maxiter + 1) {
    ctx->cg.reset(new CgCache());
    CgCache& c = *ctx->cg;
    c.stats = s;
    c.kg = kg;
    c.m = m;
    for (DBuf* b : {&c.r, &c.u, &c.s, &c.z, &c.x, &c.kt0, &c.kt1}) b->ensure(sizeof(double) * m);
    const int np = cg_partials_needed(m) + 4096;
    c.pa.ensure(sizeof(double) * np);
    c.pb.ensure(sizeof(double) * np * 4);
    c.trace_cap = std::max(maxiter + 1, 1024);
    c.tr.ensure(sizeof(double) * (c.trace_cap + 1));
    c.al.ensure(sizeof(double) * (c.trace_cap + 1));
    c.be.ensure(sizeof(double) * (c.trace_cap + 1));
    c.st.ensure(sizeof(CgState));
  }
  return *ctx->cg;
}

CgBufs cg_bufs(CgCache& c) {
  CgBufs b{};
  b.r = c.r.as<double>();
  b.u = c.u.as<double>();
  b.s = c.s.as<double>();
  b.z = c.z.as<double>();
  b.x = c.x.as<double>();
  b.kt0 = c.kt0.as<double>();
  b.kt1 = c.kt1.as<double>();
  b.part_a = c.pa.as<double>();
  b.part_b = c.pb.as<double>();
  b.trace = c.tr.as<double>();
  b.alphas = c.al.as<double>();
  b.betas = c.be.as<double>();
  b.st = c.st.as<CgState>();
  return b;
}

struct CgOutcome {
  int iterations = 0;
  bool converged = false;
  bool breakdown = false;
  double residual_sq = 0.0;
  double loop_ms = 0.0;
};

// factorized_cg_grid_rhs on device buffers; rhat0_dev and xhat_out_dev are device arrays.
CgOutcome run_efcg(gsgpc_ctx* ctx, gsgpc_stats* s, gsgpc_kg* kg, const double* rhat0_dev, double sigma,
                   double eps_abs, double rel_tol, int maxiter, double* xhat_out_dev, double* trace_out,
                   double* alphas_out, double* betas_out) {
  if (kg->m != s->g.m) invalid("factorized_cg_grid_rhs: dimension mismatch");
  if (eps_abs < 0.0 && rel_tol < 0.0) invalid("factorized_cg_grid_rhs: set eps_abs or rel_tol");
  if (maxiter < 0) invalid("factorized_cg_grid_rhs: maxiter must be >= 0");
  finalize_stats(ctx, s);
  const int64_t m = s->g.m;
  CgCache& c = cg_setup(ctx, s, kg, maxiter);
  const CgBufs b = cg_bufs(c);
  const StencilDesc sd = stencil_desc(s);
  const Launch L = ctx->L();
  CgState st0{};
  st0.eps_abs = eps_abs;
  st0.rel_tol = rel_tol;
  st0.sigma_sq = sigma * sigma;
  st0.maxiter = maxiter;
  ctx->pin.ensure(sizeof(CgState) + 64);
  std::memcpy(ctx->pin.p, &st0, sizeof(CgState));
  GSGPC_CUDA(cudaMemcpyAsync(b.st, ctx->pin.p, sizeof(CgState), cudaMemcpyHostToDevice, ctx->stream));
  GSGPC_CUDA(cudaMemcpyAsync(b.r, rhat0_dev, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
  GSGPC_CUDA(cudaMemsetAsync(b.s, 0, sizeof(double) * m, ctx->stream));
  GSGPC_CUDA(cudaMemsetAsync(b.z, 0, sizeof(double) * m, ctx->stream));
  GSGPC_CUDA(cudaMemsetAsync(b.x, 0, sizeof(double) * m, ctx->stream));
  static const bool use_graph = [] {
    const char* e = getenv("GSGPC_CG_GRAPH");
    return e && e[0] == '1';
  }();
  const int per_iter = 2 + s->g.d;
  cudaEvent_t e0, e1;
  GSGPC_CUDA(cudaEventCreate(&e0));
  GSGPC_CUDA(cudaEventCreate(&e1));
  CgState h{};
  // the persistent kernel runs the tensor-core mode products only: an FFT-route K_G (a grid
  // dimension > 2040 nodes) takes the per-phase kernels + cuFFT, graph-replayed
  if (!use_graph && !kg->dev.fft) {
    // one cooperative launch runs the whole solve (efcg_persistent.cu)
    static const bool trace = [] {
      const char* e = getenv("GSGPC_CG_TRACE");
      return e && e[0] == '1';
    }();
    DBuf& tb = ctx->buf("cg_trace");
    if (trace) {
      tb.ensure(sizeof(unsigned long long) * 64 * 8);
      GSGPC_CUDA(cudaMemsetAsync(tb.p, 0, sizeof(unsigned long long) * 64 * 8, ctx->stream));
    }
    GSGPC_CUDA(cudaEventRecord(e0, ctx->stream));
    run_efcg_persistent(L, sd, s->stencil(), kg->dev, b, 1, trace ? tb.as<unsigned long long>() : nullptr);
    GSGPC_CUDA(cudaEventRecord(e1, ctx->stream));
    if (trace) {  // diagnostics: mean per-phase time over iterations 2..63
      std::vector<unsigned long long> t(64 * 8);
      GSGPC_CUDA(cudaMemcpyAsync(t.data(), tb.p, sizeof(unsigned long long) * 64 * 8, cudaMemcpyDeviceToHost,
                                 ctx->stream));
      GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
      double acc[8] = {0};
      int cnt = 0;
      for (int it = 2; it < 63; ++it) {
        const unsigned long long* r = &t[it * 8];
        if (!r[0] || !r[6] || !t[(it + 1) * 8]) continue;
        acc[0] += r[1] - r[0];              // update + sync
        acc[1] += r[2] - r[1];              // SpMV + sync
        unsigned long long prev = r[2];
        for (int ph = 3; ph <= 5; ++ph) {
          if (r[ph]) {
            acc[ph - 1] += r[ph] - prev;    // Toeplitz modes
            prev = r[ph];
          }
        }
        acc[5] += r[6] - prev;              // last mode + epilogue + sync
        acc[6] += t[(it + 1) * 8] - r[6];   // reduce, scalars
        ++cnt;
      }
      if (cnt) {
        std::fprintf(stderr, "[gsgpc cg trace] us/iter: update %.1f spmv %.1f mode2 %.1f mode1 %.1f mode0+epi %.1f "
                     "tail %.1f (n=%d)\n", acc[0] / cnt / 1e3, acc[1] / cnt / 1e3, acc[2] / cnt / 1e3,
                     acc[3] / cnt / 1e3, acc[5] / cnt / 1e3, acc[6] / cnt / 1e3, cnt);
      }
    }
    GSGPC_CUDA(cudaMemcpyAsync(ctx->pin.p, b.st, sizeof(CgState), cudaMemcpyDeviceToHost, ctx->stream));
    GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(&h, ctx->pin.p, sizeof(CgState));
  } else {
    run_cg_init(L, sd, s->stencil(), kg->dev, b, m);
    // capture (once per cache) a graph of kGraphIters iterations
    if (!c.exec) {
      cudaGraph_t graph;
      uint64_t dummy = 0;
      const Launch Lc{ctx->stream, &dummy};
      GSGPC_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < kGraphIters; ++i) run_cg_iter(Lc, sd, s->stencil(), kg->dev, b, m);
      GSGPC_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
      GSGPC_CUDA(cudaGraphInstantiate(&c.exec, graph, 0));
      GSGPC_CUDA(cudaGraphDestroy(graph));
      c.B = kGraphIters;
    }
    GSGPC_CUDA(cudaEventRecord(e0, ctx->stream));
    for (;;) {
      GSGPC_CUDA(cudaMemcpyAsync(ctx->pin.p, b.st, sizeof(CgState), cudaMemcpyDeviceToHost, ctx->stream));
      GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
      std::memcpy(&h, ctx->pin.p, sizeof(CgState));
      if (h.done) break;
      GSGPC_CUDA(cudaGraphLaunch(c.exec, ctx->stream));
      ctx->launches += static_cast<uint64_t>(per_iter) * c.B;
    }
    GSGPC_CUDA(cudaEventRecord(e1, ctx->stream));
  }
  GSGPC_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  GSGPC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CgOutcome o;
  o.iterations = h.iter;
  o.converged = h.converged != 0;
  o.breakdown = h.breakdown != 0;
  o.residual_sq = h.rho;
  o.loop_ms = ms;
  if (xhat_out_dev) {
    GSGPC_CUDA(cudaMemcpyAsync(xhat_out_dev, b.x, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (trace_out) {
    GSGPC_CUDA(cudaMemcpyAsync(trace_out, b.trace, sizeof(double) * (o.iterations + 1), cudaMemcpyDefault, ctx->stream));
  }
  if (alphas_out && o.iterations > 0) {
    GSGPC_CUDA(cudaMemcpyAsync(alphas_out, b.alphas, sizeof(double) * o.iterations, cudaMemcpyDefault, ctx->stream));
  }
  const int nb = o.converged ? std::max(0, o.iterations - 1) : o.iterations;
  if (betas_out && nb > 0) {
    GSGPC_CUDA(cudaMemcpyAsync(betas_out, b.betas, sizeof(double) * nb, cudaMemcpyDefault, ctx->stream));
  }
  GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (o.breakdown) {
    throw Error(GSGPC_BREAKDOWN, "factorized_cg_grid_rhs: p^T A p <= 0, operator is not positive definite");
  }
  return o;
}

}  // namespace

extern "C" {

gsgpc_status gsgpc_factorized_cg_grid_rhs(gsgpc_ctx* ctx, gsgpc_kg* kg, gsgpc_stats* s, const double* rhat0,
                                          double sigma, double eps_abs, double rel_tol, int maxiter,
                                          double* xhat_d, gsgpc_solve_info* info, double* residual_trace,
                                          double* alphas, double* betas) {
  return guard(ctx, [&] {
    if (!kg || !s) invalid("NULL handle");
    const double* r0 = dev_in(ctx, rhat0, s->g.m, "cg_r0");
    DevOut o(ctx, xhat_d, s->g.m, "cg_x");
    const CgOutcome r = run_efcg(ctx, s, kg, r0, sigma, eps_abs, rel_tol, maxiter, o.dev, residual_trace, alphas, betas);
    o.finish();
    if (info) {
      info->iterations = r.iterations;
      info->converged = r.converged ? 1 : 0;
      info->residual_sq = r.residual_sq;
      info->loop_seconds = r.loop_ms * 1e-3;
    }
  });
}

gsgpc_status gsgpc_posterior_mean_gsgp(gsgpc_ctx* ctx, gsgpc_stats* s, gsgpc_kg* kg, double sigma, double tol,
                                       int maxiter, double* mean_coeffs, gsgpc_solve_info* info) {
  gsgpc_status nonconv = GSGPC_OK;
  const gsgpc_status st = guard(ctx, [&] {
    if (!kg || !s) invalid("posterior_mean_gsgp: null inputs");
    finalize_stats(ctx, s);
    const int64_t m = s->g.m;
    if (kg->m != m) invalid("posterior_mean_gsgp: kernel/grid size mismatch");
    const double sigma_sq = sigma * sigma;
    const Launch L = ctx->L();
    DBuf& t0 = ctx->buf("pm_t0");
    DBuf& t1 = ctx->buf("pm_t1");
    DBuf& kw = ctx->buf("pm_kw");
    DBuf& r0 = ctx->buf("pm_r0");
    DBuf& xd = ctx->buf("pm_x");
    for (DBuf* b : {&t0, &t1, &kw, &r0, &xd}) b->ensure(sizeof(double) * m);
    // rhat0 = -K_G W^T y / σ²  (gp.cpp:331)
    run_kg_apply(L, kg->dev, s->wty(), kw.as<double>(), t0.as<double>(), t1.as<double>());
    run_add_div(L, m, nullptr, 0.0, kw.as<double>(), -sigma_sq, r0.as<double>());
    const double yty = stats_yty(ctx, s);
    const double eps_abs = tol * tol * yty;  // gp.cpp:333
    const CgOutcome r = run_efcg(ctx, s, kg, r0.as<double>(), sigma, eps_abs, -1.0, maxiter, xd.as<double>(),
                                 nullptr, nullptr, nullptr);
    if (info) {
      info->iterations = r.iterations;
      info->converged = r.converged ? 1 : 0;
      info->residual_sq = r.residual_sq;
      info->loop_seconds = r.loop_ms * 1e-3;
    }
    if (!r.converged) {
      nonconv = GSGPC_NONCONVERGENCE;
      throw Error(GSGPC_NONCONVERGENCE, "posterior_mean_gsgp: solver hit maxiter");
    }
    // mean_coeffs = K_G (x̂_d + W^T y / σ²)  (gp.cpp:345)
    run_add_div(L, m, xd.as<double>(), 1.0, s->wty(), sigma_sq, r0.as<double>());
    DevOut o(ctx, mean_coeffs, m, "pm_out");
    run_kg_apply(L, kg->dev, r0.as<double>(), o.dev, t0.as<double>(), t1.as<double>());
    o.finish();
  });
  (void)nonconv;
  return st;
}

gsgpc_status gsgpc_predict_mean(gsgpc_ctx* ctx, const gsgpc_grid* grid, int scheme, const double* mean_coeffs,
                                const gsgpc_points* pts, int64_t n, double* out) {
  return guard(ctx, [&] {
    const GridDev g = make_grid(grid, scheme);
    check_points(pts, n, false);
    if (n == 0) return;
    const double* c = dev_in(ctx, mean_coeffs, g.m, "pred_coeffs");
    const bool dev = is_device_ptr(pts->x);
    const PointsDev P = dev ? points_dev(pts, g.d, 0) : stage_points(ctx, pts, g.d, 0, n, false, "pred_stage");
    DevOut o(ctx, out, n, "pred_out");
    DBuf& st = ctx->buf("pred_status");
    st.ensure(sizeof(int) * n);
    run_predict(ctx->L(), pts->dtype, P, n, g, c, o.dev, st.as<int>());
    o.finish();
    std::vector<int> hs(n);
    copy_out(ctx, hs.data(), st.p, sizeof(int) * n);
    for (int64_t i = 0; i < n; ++i) {
      if (hs[i] == PT_OUTSIDE) throw Error(GSGPC_OUT_OF_GRID, "interp_weights: point outside grid", i + 1);
      if (hs[i] == PT_LEAVES) {
        throw Error(GSGPC_OUT_OF_GRID,
                    "interp_weights: stencil leaves the grid (point too close to the boundary for the requested "
                    "scheme)",
                    i + 1);
      }
    }
  });
}

}  // extern "C"

// ---------------------------------------------------------------- EFLA / log-likelihood
extern "C" {

gsgpc_status gsgpc_factorized_lanczos_fused(gsgpc_ctx* ctx, gsgpc_kg* kg, gsgpc_stats* s, int probes,
                                            const double* kgwt_z0, const double* wt_z0, const double* z0_sq,
                                            double sigma_sq, int k, double* alpha, double* beta, int32_t* order) {
  return guard(ctx, [&] {
    if (!kg || !s || !alpha || !beta || !order || !z0_sq) invalid("NULL argument");
    if (probes < 1) invalid("factorized_lanczos_fused: need at least one start vector");
    if (k < 1) invalid("factorized_lanczos_fused: bad k");
    finalize_stats(ctx, s);
    const int64_t m = s->g.m;
    if (kg->m != m) invalid("factorized_lanczos_fused: dimension mismatch");
    std::vector<double> zs(probes);
    copy_out(ctx, zs.data(), z0_sq, sizeof(double) * probes);
    for (double v : zs) {
      if (!(v > 0.0)) invalid("factorized_lanczos_fused: start vector is zero");
    }
    const double* kw = dev_in(ctx, kgwt_z0, static_cast<int64_t>(probes) * m, "efla_kw");
    const double* w0 = dev_in(ctx, wt_z0, static_cast<int64_t>(probes) * m, "efla_w0");
    DBuf& zd = ctx->buf("efla_z0");
    zd.ensure(sizeof(double) * probes);
    GSGPC_CUDA(cudaMemcpyAsync(zd.p, zs.data(), sizeof(double) * probes, cudaMemcpyHostToDevice, ctx->stream));
    const StencilDesc sd = stencil_desc(s);
    for (int p0 = 0; p0 < probes; p0 += 32) {
      const int P = std::min(32, probes - p0);
      const EflaOut o = efla_run(ctx->L(), sd, s->stencil(), kg->dev, P, kw + static_cast<int64_t>(p0) * m,
                                 w0 + static_cast<int64_t>(p0) * m, zd.as<double>() + p0, sigma_sq, k);
      std::vector<double> ha(o.alpha), hb(o.beta);
      std::vector<int32_t> ho(o.order.begin(), o.order.end());
      copy_out(ctx, alpha + static_cast<int64_t>(p0) * k, ha.data(), sizeof(double) * P * k);
      copy_out(ctx, beta + static_cast<int64_t>(p0) * k, hb.data(), sizeof(double) * P * k);
      copy_out(ctx, order + p0, ho.data(), sizeof(int32_t) * P);
    }
  });
}

gsgpc_status gsgpc_log_likelihood_gsgp(gsgpc_ctx* ctx, gsgpc_stats* s, gsgpc_kg* kg, double sigma,
                                       const gsgpc_loglik_options* opts, gsgpc_loglik_result* out) {
  return guard(ctx, [&] {
    if (!s || !kg || !opts || !out) invalid("NULL argument");
    finalize_stats(ctx, s);
    const int64_t m = s->g.m;
    if (kg->m != m) invalid("log_likelihood_gsgp: kernel/grid size mismatch");
    const int P = opts->probes;
    const int64_t dense_cap = opts->dense_cap > 0 ? opts->dense_cap : 2048;
    const bool all_probes = opts->probe_begin == 0 && opts->probe_end == 0;
    const int pb = all_probes ? 0 : opts->probe_begin, pe = all_probes ? P : opts->probe_end;
    if (pb < 0 || pe < pb || pe > P) invalid("log_likelihood_gsgp: bad probe range");
    if (opts->route < GSGPC_ROUTE_AUTO || opts->route > GSGPC_ROUTE_DENSE) invalid("log_likelihood_gsgp: bad route");
    const Launch L = ctx->L();
    const double n = static_cast<double>(s->reduced ? static_cast<int64_t>(read_scalar(ctx, s->tail() + 1)) : s->n);
    const double sigma_sq = sigma * sigma;
    const double yty = stats_yty(ctx, s);
    // quadratic term (gp.cpp:166-178)
    DBuf& t0 = ctx->buf("ll_t0");
    DBuf& t1 = ctx->buf("ll_t1");
    DBuf& kw = ctx->buf("ll_kw");
    DBuf& r0 = ctx->buf("ll_r0");
    DBuf& xd = ctx->buf("ll_x");
    for (DBuf* b : {&t0, &t1, &kw, &r0, &xd}) b->ensure(sizeof(double) * m);
    run_kg_apply(L, kg->dev, s->wty(), kw.as<double>(), t0.as<double>(), t1.as<double>());
    run_add_div(L, m, nullptr, 0.0, kw.as<double>(), -sigma_sq, r0.as<double>());
    const double eps_abs = opts->solve_tol * opts->solve_tol * yty;
    const CgOutcome cg = run_efcg(ctx, s, kg, r0.as<double>(), sigma, eps_abs, -1.0, opts->maxiter, xd.as<double>(),
                                  nullptr, nullptr, nullptr);
    if (!cg.converged) throw Error(GSGPC_NONCONVERGENCE, "log_likelihood_gsgp: mean solve did not converge");
    run_add_div(L, m, xd.as<double>(), 1.0, s->wty(), sigma_sq, r0.as<double>());
    run_kg_apply(L, kg->dev, r0.as<double>(), kw.as<double>(), t0.as<double>(), t1.as<double>());
    std::vector<double> hw(m), hz(m);
    copy_out(ctx, hw.data(), s->wty(), sizeof(double) * m);
    copy_out(ctx, hz.data(), kw.p, sizeof(double) * m);
    double wz = 0.0;
    for (int64_t i = 0; i < m; ++i) wz += hw[i] * hz[i];
    const double quad = (yty - wz) / sigma_sq;
    // route (gp.cpp:181-232)
    int route = opts->route;
    if (route == GSGPC_ROUTE_AUTO) {
      if (s->probes > 0) {
        route = GSGPC_ROUTE_SKI_OPERATOR;
      } else if (kg_condition_estimate(L, kg->dev) > 1e8 && m <= dense_cap) {
        route = GSGPC_ROUTE_DENSE;
      } else {
        route = GSGPC_ROUTE_SYMMETRIC_GRID;
      }
    }
    const StencilDesc sd = stencil_desc(s);
    double logdet = 0.0, slq_sum = 0.0, logdet_shift = 0.0;
    int probes_used = 0, max_used = 0, slq_count = 0;
    if (route == GSGPC_ROUTE_SKI_OPERATOR) {
      // SLQ over the probe images (gp.cpp:85-111)
      if (P < 1) invalid("slq_logdet_ski_factorized: need at least one probe");
      if (s->probes < P) {
        invalid("log_likelihood_gsgp: the SkiOperator logdet route needs probe images W^T v_p accumulated in the "
                "precompute (gsgpc_stats_enable_probes)");
      }
      if (s->probe_seeded && s->probe_seed != opts->seed) {
        invalid("log_likelihood_gsgp: probe images were accumulated with seed " + std::to_string(s->probe_seed));
      }
      const int depth = static_cast<int>(std::min<double>(opts->max_depth, n));
      if (depth < 1) invalid("slq: need at least one Lanczos step");
      DBuf& kwt = ctx->buf("ll_kwt");
      DBuf& kt0 = ctx->buf("ll_kt0");
      DBuf& kt1 = ctx->buf("ll_kt1");
      kwt.ensure(sizeof(double) * P * m);
      kt0.ensure(sizeof(double) * P * m);
      kt1.ensure(sizeof(double) * P * m);
      run_kg_batched(L, kg->dev, P, s->pimg(), kwt.as<double>(), kt0.as<double>(), kt1.as<double>());
      DBuf& zd = ctx->buf("ll_z0");
      zd.ensure(sizeof(double) * P);
      std::vector<double> zs(P, n);  // v·v = n for ±1 probes
      GSGPC_CUDA(cudaMemcpyAsync(zd.p, zs.data(), sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
      double total = 0.0;
      for (int p0 = pb; p0 < pe; p0 += 32) {
        const int Pb = std::min(32, pe - p0);
        const EflaOut o = efla_run(L, sd, s->stencil(), kg->dev, Pb, kwt.as<double>() + static_cast<int64_t>(p0) * m,
                                   s->pimg() + static_cast<int64_t>(p0) * m, zd.as<double>() + p0, sigma_sq, depth);
        for (int p = 0; p < Pb; ++p) {
          const auto q = quadrature_logdet_host(o.alpha.data() + static_cast<size_t>(p) * depth,
                                                o.beta.data() + static_cast<size_t>(p) * depth, o.order[p], n,
                                                opts->quad_tol);
          total += q.first;
          max_used = std::max(max_used, q.second);
        }
      }
      slq_sum = total;
      slq_count = pe - pb;
      logdet_shift = -(n - static_cast<double>(m)) * std::log(sigma_sq);
      logdet = (slq_count > 0 ? total / slq_count : 0.0) + logdet_shift;
      probes_used = slq_count;
    } else if (route == GSGPC_ROUTE_SYMMETRIC_GRID) {
      // slq_logdet(K WᵀW K + σ²K) − slq_logdet(K), shared probes, quad_tol 0 (gp.cpp:206-219)
      if (P < 1) invalid("slq_logdet: need at least one probe");
      const int Pb = std::min(P, 32);
      DBuf& ku = ctx->buf("ll_sym_ku");
      DBuf& wku = ctx->buf("ll_sym_wku");
      DBuf& kt0 = ctx->buf("ll_kt0");
      DBuf& kt1 = ctx->buf("ll_kt1");
      for (DBuf* b : {&ku, &wku, &kt0, &kt1}) b->ensure(sizeof(double) * Pb * m);
      const double s1 = slq_logdet_sum(L, m, pb, pe, opts->max_depth, 0.0, opts->seed, [&](int np) {
        return sym_op(L, sd, s->stencil(), kg->dev, np, sigma_sq, ku.as<double>(), wku.as<double>(),
                      kt0.as<double>(), kt1.as<double>());
      });
      const double s2 = slq_logdet_sum(L, m, pb, pe, opts->max_depth, 0.0, opts->seed, [&](int np) {
        return kg_op(L, kg->dev, np, kt0.as<double>(), kt1.as<double>());
      });
      slq_sum = s1 - s2;
      slq_count = pe - pb;
      logdet = slq_count > 0 ? slq_sum / slq_count : 0.0;
      probes_used = 2 * slq_count;
      max_used = static_cast<int>(std::min<int64_t>(opts->max_depth, m));
    } else {
      if (m > dense_cap) invalid("log_likelihood_gsgp: grid too large for the dense logdet route");
      logdet = dense_logdet_grid_system(L, sd, s->stencil(), kg->dev, sigma_sq);
      slq_sum = logdet;
    }
    const double kLog2Pi = 1.8378770664093453;
    out->logdet_term = logdet;
    out->quad_term = quad;
    out->const_term = n * kLog2Pi + (n - static_cast<double>(m)) * std::log(sigma_sq);
    out->loglik = -0.5 * (out->logdet_term + out->quad_term + out->const_term);
    out->probes_used = probes_used;
    out->solver_iterations = cg.iterations;
    out->max_depth_used = max_used;
    out->logdet_route = route;
    out->slq_sum = slq_sum;
    out->slq_count = slq_count;
    out->logdet_shift = logdet_shift;
  });
}


// ---------------------------------------------------------------- covariance (gp.cpp:381-528)
namespace {

struct TestWeights {
  int cap = 0;
  DBuf *idx = nullptr, *w = nullptr, *nnz = nullptr;
};

// interp_weights of the test points on the device (errors as the reference's interp_weights)
TestWeights test_weights(gsgpc_ctx* ctx, const GridDev& g, const gsgpc_points* pts, int64_t ns, const char* tag) {
  TestWeights t;
  t.cap = 1;
  for (int k = 0; k < g.d; ++k) t.cap *= g.W;
  const std::string p(tag);
  const bool dev = is_device_ptr(pts->x);
  const PointsDev P = dev ? points_dev(pts, g.d, 0) : stage_points(ctx, pts, g.d, 0, ns, false, (p + "_stage").c_str());
  t.idx = &ctx->buf(p + "_idx");
  t.w = &ctx->buf(p + "_w");
  t.nnz = &ctx->buf(p + "_nnz");
  DBuf& st = ctx->buf(p + "_status");
  t.idx->ensure(sizeof(int64_t) * ns * t.cap);
  t.w->ensure(sizeof(double) * ns * t.cap);
  t.nnz->ensure(sizeof(int) * ns);
  st.ensure(sizeof(int) * ns);
  run_interp_weights(ctx->L(), pts->dtype, P, ns, g, t.idx->as<int64_t>(), t.w->as<double>(), t.nnz->as<int>(),
                     st.as<int>());
  std::vector<int> hs(ns);
  copy_out(ctx, hs.data(), st.p, sizeof(int) * ns);
  for (int64_t i = 0; i < ns; ++i) {
    if (hs[i] == PT_OUTSIDE) throw Error(GSGPC_OUT_OF_GRID, "interp_weights: point outside grid", i + 1);
    if (hs[i] == PT_LEAVES) {
      throw Error(GSGPC_OUT_OF_GRID,
                  "interp_weights: stencil leaves the grid (point too close to the boundary for the requested scheme)",
                  i + 1);
    }
  }
  return t;
}

// H = K_G W_xᵀ rows (ns × m) and prior(i, j) = w_iᵀ h_j (ns × ns), both on the device
void prior_and_h(gsgpc_ctx* ctx, const KgDev& kg, int64_t m, const TestWeights& t, int64_t ns, DBuf& H,
                 DBuf& prior) {
  const Launch L = ctx->L();
  DBuf& wx = ctx->buf("cov_wx");
  DBuf& t0 = ctx->buf("cov_t0");
  DBuf& t1 = ctx->buf("cov_t1");
  for (DBuf* b : {&wx, &H, &t0, &t1}) b->ensure(sizeof(double) * ns * m);
  prior.ensure(sizeof(double) * ns * ns);
  cov_scatter_w(L, ns, m, t.cap, t.idx->as<int64_t>(), t.w->as<double>(), t.nnz->as<int>(), wx.as<double>());
  run_kg_apply_batched(L, kg, ns, wx.as<double>(), H.as<double>(), t0.as<double>(), t1.as<double>());
  cov_gather(L, ns, ns, m, t.cap, t.idx->as<int64_t>(), t.w->as<double>(), t.nnz->as<int>(), H.as<double>(),
             prior.as<double>());
}

// T y = b for the symmetric positive definite tridiagonal T (LDLᵀ, k small, on the host)
void tridiag_solve_host(const std::vector<double>& a, const std::vector<double>& b, double* z) {
  const int k = static_cast<int>(a.size());
  std::vector<double> dd(k), l(k > 1 ? k - 1 : 0);
  dd[0] = a[0];
  for (int i = 1; i < k; ++i) {
    l[i - 1] = b[i - 1] / dd[i - 1];
    dd[i] = a[i] - l[i - 1] * b[i - 1];
  }
  for (int i = 1; i < k; ++i) z[i] -= l[i - 1] * z[i - 1];
  for (int i = 0; i < k; ++i) z[i] /= dd[i];
  for (int i = k - 2; i >= 0; --i) z[i] -= l[i] * z[i + 1];
}

// unsymmetrised low-rank covariance prior − φᵀ T⁻¹ φ at ns points (host out, ns × ns)
std::vector<double> lowrank_cov_raw(gsgpc_ctx* ctx, gsgpc_lowrank* lr, const gsgpc_points* pts, int64_t ns) {
  const Launch L = ctx->L();
  const TestWeights t = test_weights(ctx, lr->g, pts, ns, "lr");
  DBuf& H = ctx->buf("cov_h");
  DBuf& prior = ctx->buf("cov_prior");
  prior_and_h(ctx, lr->kg, lr->m, t, ns, H, prior);
  if (lr->k > 0) {
    DBuf& phi = ctx->buf("lr_phi");
    DBuf& y = ctx->buf("lr_y");
    phi.ensure(sizeof(double) * ns * lr->k);
    y.ensure(sizeof(double) * ns * lr->k);
    cov_gather(L, ns, lr->k, lr->m, t.cap, t.idx->as<int64_t>(), t.w->as<double>(), t.nnz->as<int>(),
               lr->R.as<double>(), phi.as<double>());
    std::vector<double> hp(static_cast<size_t>(ns) * lr->k);
    copy_out(ctx, hp.data(), phi.p, sizeof(double) * hp.size());
    for (int64_t i = 0; i < ns; ++i) tridiag_solve_host(lr->alpha, lr->beta, hp.data() + i * lr->k);
    GSGPC_CUDA(cudaMemcpyAsync(y.p, hp.data(), sizeof(double) * hp.size(), cudaMemcpyHostToDevice, ctx->stream));
    cov_sub_abt(L, static_cast<int>(ns), lr->k, phi.as<double>(), y.as<double>(), prior.as<double>());
  }
  std::vector<double> c(static_cast<size_t>(ns) * ns);
  copy_out(ctx, c.data(), prior.p, sizeof(double) * c.size());
  return c;
}

}  // namespace

gsgpc_status gsgpc_posterior_cov_exact(gsgpc_ctx* ctx, gsgpc_stats* s, gsgpc_kg* kg, double sigma,
                                       const gsgpc_points* pts, int64_t ns, double tol, int maxiter, double* cov,
                                       double* max_asymmetry, int32_t* total_iterations) {
  return guard(ctx, [&] {
    if (!s || !kg || !cov) invalid("NULL argument");
    check_points(pts, ns, false);
    finalize_stats(ctx, s);
    const int64_t m = s->g.m;
    if (kg->m != m) invalid("posterior_cov_exact: kernel/grid size mismatch");
    if (ns == 0) return;
    const Launch L = ctx->L();
    const TestWeights t = test_weights(ctx, s->g, pts, ns, "cov");
    DBuf& H = ctx->buf("cov_h");
    DBuf& C = ctx->buf("cov_prior");
    prior_and_h(ctx, kg->dev, m, t, ns, H, C);
    DBuf& X = ctx->buf("cov_x");
    X.ensure(sizeof(double) * ns * m);
    const StencilDesc sd = stencil_desc(s);
    int64_t total = 0;
    for (int64_t j0 = 0; j0 < ns; j0 += 32) {
      const int P = static_cast<int>(std::min<int64_t>(32, ns - j0));
      const BcgOut o = bcg_run(L, sd, s->stencil(), kg->dev, P, H.as<double>() + j0 * m, sigma, -1.0, tol, maxiter,
                               X.as<double>() + j0 * m);
      if (o.breakdown) {
        throw Error(GSGPC_BREAKDOWN, "factorized_cg_grid_rhs: p^T A p <= 0, operator is not positive definite");
      }
      for (int p = 0; p < P; ++p) {
        if (!o.converged[p]) {
          ctx->err_row = o.iterations[p];
          throw Error(GSGPC_NONCONVERGENCE, "posterior_cov_exact: solver hit maxiter");
        }
        total += o.iterations[p];
      }
    }
    cov_sub_abt(L, static_cast<int>(ns), m, H.as<double>(), X.as<double>(), C.as<double>());
    std::vector<double> c(static_cast<size_t>(ns) * ns);
    copy_out(ctx, c.data(), C.p, sizeof(double) * c.size());
    double asym = 0.0;
    for (int64_t i = 0; i < ns; ++i)
      for (int64_t j = 0; j < ns; ++j) {
        asym = std::max(asym, std::fabs(c[i * ns + j] - c[j * ns + i]));
        cov[i * ns + j] = 0.5 * (c[i * ns + j] + c[j * ns + i]);
      }
    if (max_asymmetry) *max_asymmetry = asym;
    if (total_iterations) *total_iterations = static_cast<int32_t>(total);
  });
}

gsgpc_status gsgpc_posterior_cov_lowrank(gsgpc_ctx* ctx, gsgpc_stats* s, gsgpc_kg* kg, double sigma, int64_t rank,
                                         gsgpc_lowrank** out) {
  return guard(ctx, [&] {
    if (!s || !kg || !out) invalid("NULL argument");
    finalize_stats(ctx, s);
    const int64_t m = s->g.m;
    if (kg->m != m) invalid("posterior_cov_lowrank: kernel/grid size mismatch");
    if (rank < 0 || rank > m) invalid("posterior_cov_lowrank: need 0 <= rank <= grid size");
    std::unique_ptr<gsgpc_lowrank> lr(new gsgpc_lowrank());
    lr->device = ctx->device;
    lr->g = s->g;
    lr->scheme = s->scheme;
    lr->m = m;
    lr->kg = kg->dev;
    lr->fft = kg->fft;  // the spectra do not depend on the generator copies below
    for (int k = 0; k < kg->dev.d; ++k) {
      const size_t b = sizeof(double) * kg->dev.sz[k];
      lr->gen[k].ensure(b);
      GSGPC_CUDA(cudaMemcpyAsync(lr->gen[k].p, kg->dev.gen[k], b, cudaMemcpyDeviceToDevice, ctx->stream));
      lr->kg.gen[k] = lr->gen[k].as<double>();
    }
    const double n = static_cast<double>(s->reduced ? static_cast<int64_t>(read_scalar(ctx, s->tail() + 1)) : s->n);
    const Launch L = ctx->L();
    if (rank > 0 && n > 0) {
      // start direction ĝ = WᵀW 1 / ‖WᵀW 1‖ (gp.cpp:446-452)
      const StencilDesc sd = stencil_desc(s);
      DBuf& a = ctx->buf("lr_a");
      DBuf& b = ctx->buf("lr_b");
      DBuf& c = ctx->buf("lr_c");
      DBuf& t0 = ctx->buf("lr_t0");
      DBuf& t1 = ctx->buf("lr_t1");
      for (DBuf* q : {&a, &b, &c, &t0, &t1}) q->ensure(sizeof(double) * m);
      std::vector<double> h(m, 1.0);
      GSGPC_CUDA(cudaMemcpyAsync(a.p, h.data(), sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
      run_spmv(L, sd, s->stencil(), a.as<double>(), b.as<double>());
      copy_out(ctx, h.data(), b.p, sizeof(double) * m);
      double gn = 0.0;
      for (double v : h) gn += v * v;
      gn = std::sqrt(gn);
      if (gn != 0.0) {
        for (double& v : h) v /= gn;
        GSGPC_CUDA(cudaMemcpyAsync(a.p, h.data(), sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
        run_spmv(L, sd, s->stencil(), a.as<double>(), b.as<double>());        // wt_z0 = WᵀW ĝ
        run_kg_apply(L, kg->dev, b.as<double>(), c.as<double>(), t0.as<double>(), t1.as<double>());  // K wt_z0
        std::vector<double> wt(m);
        copy_out(ctx, wt.data(), b.p, sizeof(double) * m);
        double z0 = 0.0;
        for (int64_t i = 0; i < m; ++i) z0 += h[i] * wt[i];
        if (z0 > 0.0) {
          DBuf& zd = ctx->buf("lr_z0");
          zd.ensure(sizeof(double));
          GSGPC_CUDA(cudaMemcpyAsync(zd.p, &z0, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
          DBuf& Q = ctx->buf("lr_basis");
          Q.ensure(sizeof(double) * rank * m);
          const EflaOut o = efla_run(L, sd, s->stencil(), kg->dev, 1, c.as<double>(), b.as<double>(), zd.as<double>(),
                                     sigma * sigma, static_cast<int>(rank), Q.as<double>());
          const int k = o.order[0];
          lr->k = k;
          lr->alpha.assign(o.alpha.begin(), o.alpha.begin() + k);
          lr->beta.assign(o.beta.begin(), o.beta.begin() + (k > 1 ? k - 1 : 0));
          // R[j] = K_G (WᵀW q̂_j + d_j · wt_z0 / √z0)   (gp.cpp:466-470)
          DBuf& U = ctx->buf("lr_u");
          DBuf& T0 = ctx->buf("lr_bt0");
          DBuf& T1 = ctx->buf("lr_bt1");
          for (DBuf* q : {&U, &T0, &T1}) q->ensure(sizeof(double) * k * m);
          lr->R.ensure(sizeof(double) * k * m);
          spmm_batched(L, sd, s->stencil(), Q.as<double>(), U.as<double>(), k);
          const double bn = std::sqrt(z0);
          for (int j = 0; j < k; ++j) {
            run_axpby(L, m, 1.0, U.as<double>() + static_cast<int64_t>(j) * m, o.d[j] / bn, b.as<double>(),
                      U.as<double>() + static_cast<int64_t>(j) * m);
          }
          run_kg_apply_batched(L, lr->kg, k, U.as<double>(), lr->R.as<double>(), T0.as<double>(), T1.as<double>());
        }
      }
    }
    GSGPC_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = lr.release();
  });
}

void gsgpc_lowrank_destroy(gsgpc_lowrank* lr) { delete lr; }

gsgpc_status gsgpc_lowrank_rank(const gsgpc_lowrank* lr, int64_t* rank) {
  if (!lr || !rank) return GSGPC_INVALID_ARGUMENT;
  *rank = lr->k;
  return GSGPC_OK;
}

gsgpc_status gsgpc_lowrank_cov_matrix(gsgpc_ctx* ctx, gsgpc_lowrank* lr, const gsgpc_points* pts, int64_t ns,
                                      double* cov) {
  return guard(ctx, [&] {
    if (!lr || !cov) invalid("NULL argument");
    check_points(pts, ns, false);
    if (ns == 0) return;
    const std::vector<double> c = lowrank_cov_raw(ctx, lr, pts, ns);
    for (int64_t i = 0; i < ns; ++i)
      for (int64_t j = 0; j < ns; ++j) cov[i * ns + j] = 0.5 * (c[i * ns + j] + c[j * ns + i]);
  });
}

gsgpc_status gsgpc_lowrank_query(gsgpc_ctx* ctx, gsgpc_lowrank* lr, const double* x, const double* x2, double* out) {
  return guard(ctx, [&] {
    if (!lr || !x || !x2 || !out) invalid("NULL argument");
    const int d = lr->g.d;
    std::vector<double> two(2 * d);
    for (int k = 0; k < d; ++k) {
      two[k] = x[k];
      two[d + k] = x2[k];
    }
    gsgpc_points p{};
    p.dtype = GSGPC_F64;
    p.x = two.data();
    p.x_row_stride = d;
    for (int k = 0; k < d; ++k) p.x_col_offset[k] = k;
    const std::vector<double> c = lowrank_cov_raw(ctx, lr, &p, 2);
    *out = c[1];  // prior(x, x2) − φ(x)ᵀ T⁻¹ φ(x2)
  });
}

}  // extern "C"
