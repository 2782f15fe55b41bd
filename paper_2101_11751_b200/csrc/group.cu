// group.cu — several GPUs driven from one process (gsgpc_ctx_create(device_ids[],
// ngpu); §8(e): the precompute shards by rows, one exchange step).
//
// A group holds one context per listed device.  gsgpc_group_sufficient_stats splits the rows
// into contiguous shards (device r: rows [r·n/G, (r+1)·n/G)), runs each shard's precompute on
// its device from its own host thread, finalizes, and sums the per-device statistics with ONE
// all-reduce — the reference's merge() (interp.cpp:202-210): W^T W, W^T y, yᵀy and n add up,
// and the W^T W structure (the touched pairs) is the union.  Every device ends with the full
// statistics, so the solve that follows runs replicated ("replicas only", §8(e)).
//
// Exchange: NCCL over NVLink/NVSwitch (ncclCommInitAll over the group's devices, one
// ncclAllReduce(sum) of the [stencil | W^T y | probe images | yᵀy | n] buffers and one
// ncclAllReduce(max) of the structure bytes, grouped).  libnccl is resolved at run time
// (dlopen of the already-loaded libnccl.so.2 when a framework brought one, else the
// system's), so the library keeps no link-time dependency that could clash with a host
// framework's NCCL.  A group that lists a device twice (or where NCCL is missing) sums on
// the first device in rank order through peer copies instead — same result, used by the
// single-GPU tests.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gsgpc.h"
#include "internal.cuh"

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  bool ok() const { return h && commInitAll && allReduce && groupStart && groupEnd && commDestroy; }
};

const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) return a;
    a.commInitAll = reinterpret_cast<decltype(a.commInitAll)>(dlsym(a.h, "ncclCommInitAll"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(a.h, "ncclAllReduce"));
    a.groupStart = reinterpret_cast<decltype(a.groupStart)>(dlsym(a.h, "ncclGroupStart"));
    a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(dlsym(a.h, "ncclGroupEnd"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.errStr = reinterpret_cast<decltype(a.errStr)>(dlsym(a.h, "ncclGetErrorString"));
    return a;
  }();
  return api;
}

__global__ void k_add_f64(int64_t n, double* __restrict__ dst, const double* __restrict__ src) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}

__global__ void k_max_u8(int64_t n, uint8_t* __restrict__ dst, const uint8_t* __restrict__ src) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = dst[i] > src[i] ? dst[i] : src[i];
}

void check(gsgpc_status st, gsgpc_ctx* ctx, const char* what) {
  if (st != GSGPC_OK) {
    std::string msg = std::string(what) + ": " + (ctx ? gsgpc_last_error(ctx) : "failed");
    throw gsgpc::Error(st, msg, ctx ? gsgpc_last_error_row(ctx) : 0);
  }
}

}  // namespace

struct gsgpc_group {
  std::vector<int> dev;
  std::vector<gsgpc_ctx*> ctx;
  std::vector<ncclComm_t> comm;  // empty: peer-copy exchange
  std::string err;
  int64_t err_row = 0;
  ~gsgpc_group() {
    if (!comm.empty() && nccl_api().ok())
      for (ncclComm_t c : comm) nccl_api().commDestroy(c);
    for (gsgpc_ctx* c : ctx)
      if (c) gsgpc_ctx_destroy(c);
  }
};

namespace {

template <class F>
gsgpc_status gguard(gsgpc_group* g, F&& f) {
  try {
    f();
    return GSGPC_OK;
  } catch (const gsgpc::Error& e) {
    if (g) {
      g->err = e.what();
      g->err_row = e.row;
    }
    return e.code;
  } catch (const std::exception& e) {
    if (g) g->err = e.what();
    return GSGPC_RUNTIME_ERROR;
  }
}

// Sum of the reduce buffers and OR of the structure bytes of one finalized stats object per
// device; afterwards every object holds the merged statistics (marked reduced).
void group_allreduce(gsgpc_group* g, gsgpc_stats** st) {
  const int G = static_cast<int>(g->ctx.size());
  std::vector<double*> buf(G);
  std::vector<uint8_t*> pat(G);
  int64_t count = -1, pcount = -1;
  for (int r = 0; r < G; ++r) {
    if (!st[r]) throw gsgpc::Error(GSGPC_INVALID_ARGUMENT, "gsgpc_group_allreduce_stats: NULL stats");
    int64_t c = 0, pc = 0;
    check(gsgpc_stats_pattern_buffer(g->ctx[r], st[r], &pat[r], &pc), g->ctx[r], "pattern buffer");
    check(gsgpc_stats_reduce_buffer(g->ctx[r], st[r], &buf[r], &c), g->ctx[r], "reduce buffer");
    if (r > 0 && (c != count || pc != pcount))
      throw gsgpc::Error(GSGPC_INVALID_ARGUMENT, "merge: grid or scheme mismatch");  // interp.cpp:203-205
    count = c;
    pcount = pc;
  }
  std::vector<cudaStream_t> s(G);
  for (int r = 0; r < G; ++r) s[r] = static_cast<cudaStream_t>(gsgpc_ctx_stream(g->ctx[r]));
  if (G > 1) {
    if (!g->comm.empty()) {
      const NcclApi& nc = nccl_api();
      auto nchk = [&](ncclResult_t e) {
        if (e != ncclSuccess)
          throw gsgpc::Error(GSGPC_CUDA_ERROR, std::string("NCCL: ") + (nc.errStr ? nc.errStr(e) : "error"));
      };
      nchk(nc.groupStart());
      for (int r = 0; r < G; ++r) {
        GSGPC_CUDA(cudaSetDevice(g->dev[r]));
        nchk(nc.allReduce(buf[r], buf[r], static_cast<size_t>(count), ncclFloat64, ncclSum, g->comm[r], s[r]));
        nchk(nc.allReduce(pat[r], pat[r], static_cast<size_t>(pcount), ncclUint8, ncclMax, g->comm[r], s[r]));
      }
      nchk(nc.groupEnd());
    } else {
      // rank order on device 0: buf0 += buf_r (r = 1..G-1), then copies back
      GSGPC_CUDA(cudaSetDevice(g->dev[0]));
      for (int r = 0; r < G; ++r) {
        GSGPC_CUDA(cudaSetDevice(g->dev[r]));
        GSGPC_CUDA(cudaStreamSynchronize(s[r]));
      }
      GSGPC_CUDA(cudaSetDevice(g->dev[0]));
      double* tmp = nullptr;
      uint8_t* tmpp = nullptr;
      GSGPC_CUDA(cudaMalloc(&tmp, sizeof(double) * count));
      GSGPC_CUDA(cudaMalloc(&tmpp, std::max<int64_t>(pcount, 1)));
      for (int r = 1; r < G; ++r) {
        GSGPC_CUDA(cudaMemcpyPeerAsync(tmp, g->dev[0], buf[r], g->dev[r], sizeof(double) * count, s[0]));
        k_add_f64<<<592, 256, 0, s[0]>>>(count, buf[0], tmp);
        GSGPC_CUDA(cudaMemcpyPeerAsync(tmpp, g->dev[0], pat[r], g->dev[r], pcount, s[0]));
        k_max_u8<<<592, 256, 0, s[0]>>>(pcount, pat[0], tmpp);
      }
      GSGPC_CUDA(cudaGetLastError());
      GSGPC_CUDA(cudaStreamSynchronize(s[0]));
      cudaFree(tmp);
      cudaFree(tmpp);
      for (int r = 1; r < G; ++r) {
        GSGPC_CUDA(cudaMemcpyPeerAsync(buf[r], g->dev[r], buf[0], g->dev[0], sizeof(double) * count, s[0]));
        GSGPC_CUDA(cudaMemcpyPeerAsync(pat[r], g->dev[r], pat[0], g->dev[0], pcount, s[0]));
      }
      GSGPC_CUDA(cudaStreamSynchronize(s[0]));
    }
  }
  for (int r = 0; r < G; ++r) check(gsgpc_stats_mark_reduced(g->ctx[r], st[r]), g->ctx[r], "mark reduced");
}

gsgpc_points shard_points(const gsgpc_points& p, int64_t lo) {
  gsgpc_points q = p;
  const size_t es = p.dtype == GSGPC_F32 ? 4 : 8;
  q.x = static_cast<const char*>(p.x) + static_cast<size_t>(lo * p.x_row_stride) * es;
  q.y = static_cast<const char*>(p.y) + static_cast<size_t>(lo * p.y_stride) * es;
  return q;
}

}  // namespace

extern "C" {

gsgpc_status gsgpc_group_create(const int* device_ids, int ngpu, gsgpc_group** out) {
  if (!out || !device_ids || ngpu < 1) return GSGPC_INVALID_ARGUMENT;
  *out = nullptr;
  auto g = std::make_unique<gsgpc_group>();
  const gsgpc_status st = gguard(g.get(), [&] {
    g->dev.assign(device_ids, device_ids + ngpu);
    for (int r = 0; r < ngpu; ++r) {
      gsgpc_ctx* c = nullptr;
      const gsgpc_status e = gsgpc_ctx_create(g->dev[r], &c);
      if (e != GSGPC_OK) throw gsgpc::Error(e, "gsgpc_group_create: device " + std::to_string(g->dev[r]));
      g->ctx.push_back(c);
    }
    std::vector<int> sorted = g->dev;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    if (ngpu > 1 && distinct && nccl_api().ok() && !getenv("GSGPC_GROUP_NO_NCCL")) {
      g->comm.resize(ngpu);
      if (nccl_api().commInitAll(g->comm.data(), ngpu, g->dev.data()) != ncclSuccess) g->comm.clear();
    }
  });
  if (st != GSGPC_OK) return st;
  *out = g.release();
  return GSGPC_OK;
}

gsgpc_status gsgpc_group_destroy(gsgpc_group* g) {
  delete g;
  return GSGPC_OK;
}

gsgpc_status gsgpc_group_info(const gsgpc_group* g, int* ngpu, int* uses_nccl) {
  if (!g) return GSGPC_INVALID_ARGUMENT;
  if (ngpu) *ngpu = static_cast<int>(g->ctx.size());
  if (uses_nccl) *uses_nccl = g->comm.empty() ? 0 : 1;
  return GSGPC_OK;
}

gsgpc_ctx* gsgpc_group_ctx(gsgpc_group* g, int rank) {
  if (!g || rank < 0 || rank >= static_cast<int>(g->ctx.size())) return nullptr;
  return g->ctx[rank];
}

const char* gsgpc_group_last_error(const gsgpc_group* g) { return g ? g->err.c_str() : "NULL group"; }
int64_t gsgpc_group_last_error_row(const gsgpc_group* g) { return g ? g->err_row : 0; }

gsgpc_status gsgpc_group_allreduce_stats(gsgpc_group* g, gsgpc_stats** stats) {
  if (!g || !stats) return GSGPC_INVALID_ARGUMENT;
  return gguard(g, [&] { group_allreduce(g, stats); });
}

gsgpc_status gsgpc_group_sufficient_stats(gsgpc_group* g, const gsgpc_grid* grid, int scheme, const gsgpc_points* pts,
                                          int64_t n, int probes, uint64_t seed, gsgpc_stats** out) {
  if (!g || !out || !pts || n < 0) return GSGPC_INVALID_ARGUMENT;
  const int G = static_cast<int>(g->ctx.size());
  for (int r = 0; r < G; ++r) out[r] = nullptr;
  std::vector<gsgpc_stats*> st(G, nullptr);
  const gsgpc_status status = gguard(g, [&] {
    for (int r = 0; r < G; ++r) {
      check(gsgpc_stats_create(g->ctx[r], grid, scheme, &st[r]), g->ctx[r], "stats_create");
      const int64_t lo = n * r / G;
      if (probes > 0)  // the shard's probe streams start at its first row (jump-ahead)
        check(gsgpc_stats_enable_probes_at(g->ctx[r], st[r], probes, seed, static_cast<uint64_t>(lo)), g->ctx[r],
              "enable_probes");
    }
    // one host thread per device; the first failing shard in row order decides the error
    std::vector<gsgpc_status> res(G, GSGPC_OK);
    std::vector<std::string> msg(G);
    std::vector<int64_t> row(G, 0);
    std::vector<std::thread> th;
    for (int r = 0; r < G; ++r) {
      th.emplace_back([&, r] {
        const int64_t lo = n * r / G, hi = n * (r + 1) / G;
        const gsgpc_points q = shard_points(*pts, lo);
        res[r] = gsgpc_stats_add(g->ctx[r], st[r], &q, hi - lo, nullptr, 0);
        if (res[r] == GSGPC_OK) res[r] = gsgpc_stats_finalize(g->ctx[r], st[r]);
        if (res[r] != GSGPC_OK) {
          msg[r] = gsgpc_last_error(g->ctx[r]);
          row[r] = gsgpc_last_error_row(g->ctx[r]) + (res[r] == GSGPC_OUT_OF_GRID ? lo : 0);
        }
      });
    }
    for (std::thread& t : th) t.join();
    for (int r = 0; r < G; ++r) {
      if (res[r] != GSGPC_OK) {
        if (res[r] == GSGPC_OUT_OF_GRID) {  // the shard's stream row → the batch's stream row
          const std::string tag = "stream row ";
          const size_t at = msg[r].find(tag);
          const size_t end = at == std::string::npos ? at : msg[r].find(':', at);
          if (at != std::string::npos && end != std::string::npos)
            msg[r] = msg[r].substr(0, at) + tag + std::to_string(row[r]) + msg[r].substr(end);
        }
        throw gsgpc::Error(res[r], msg[r], row[r]);
      }
    }
    group_allreduce(g, st.data());
  });
  if (status != GSGPC_OK) {
    for (int r = 0; r < G; ++r)
      if (st[r]) gsgpc_stats_destroy(st[r]);
    return status;
  }
  for (int r = 0; r < G; ++r) out[r] = st[r];
  return GSGPC_OK;
}

}  // extern "C"
