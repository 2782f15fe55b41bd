// probe_rng.cu — the reference's Rademacher probe streams on the device.
//
// rademacher_probe (gp.cpp:16-25): probe p draws one std::mt19937_64 output per row, in
// stream order, from a generator seeded with std::seed_seq{seed_lo, seed_hi, p_lo, p_hi}, and
// takes bit 0 (1 → +1, 0 → −1).  The streams are sequential, so each probe runs on one warp:
// the 312-word MT19937-64 twist is split into its three dependency phases (i < n−m from the
// old state; n−m ≤ i < n−1 from the new words i−(n−m); i = n−1 last), 32 words at a time, and
// the tempered outputs of a block are written one byte per row (coalesced).  The default is
// the block-per-probe variant below (k_probe_rng_blk: state in registers, one barrier per
// twist; config 5's 30 × 5e7 draws 112 → 44 ms), run over substreams of 1,048,320 draws each
// started by the GF(2) jump-ahead of mt_jump.cu (30 probes × 16 substreams per slab instead
// of 30 blocks on 148 SMs); GSGPC_PROBE_RNG_WARP=1 selects the warp kernel,
// GSGPC_PROBE_RNG_NOSPLIT=1 one block per probe.  A second kernel
// packs the bytes into one 64-bit word per row (bit p = probe p), the layout the binning
// carries with the rows.  The initial state is built on the host exactly as
// mersenne_twister_engine(seed_seq&) does ([rand.eng.mers]: generate 2n 32-bit words,
// x_i = a_{2i} + 2^32 a_{2i+1}, all-zero guard); each probe keeps (state, index) on the
// device across batches.
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <random>
#include <vector>

#include "internal.cuh"
#include "precompute.cuh"

namespace gsgpc {

constexpr int MT_N = 312, MT_M = 156;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ull;
constexpr uint64_t MT_UM = 0xFFFFFFFF80000000ull;  // upper w − r = 33 bits
constexpr uint64_t MT_LM = 0x7FFFFFFFull;          // lower r = 31 bits

void mt_seed_state(uint64_t seed, uint64_t p, uint64_t* st) {
  std::seed_seq seq{static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32),
                    static_cast<std::uint32_t>(p), static_cast<std::uint32_t>(p >> 32)};
  std::uint32_t a[2 * MT_N];
  seq.generate(a, a + 2 * MT_N);
  bool zero = true;
  for (int i = 0; i < MT_N; ++i) {
    st[i] = static_cast<uint64_t>(a[2 * i]) | (static_cast<uint64_t>(a[2 * i + 1]) << 32);
    if (i == 0 ? (st[0] & MT_UM) != 0 : st[i] != 0) zero = false;
  }
  if (zero) st[0] = 1ull << 63;
  st[MT_N] = MT_N;  // index: the first draw twists
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t hi_word, uint64_t lo_word, uint64_t far) {
  const uint64_t x = (hi_word & MT_UM) | (lo_word & MT_LM);
  return far ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
}

// Bit 0 of the tempered output (the only bit rademacher_probe reads).  Expanding the four
// tempering steps (y ^= (y>>29)&0x55…; y ^= (y<<17)&0x71D6…; y ^= (y<<37)&0xFFF7…; y ^= y>>43):
// bit 0 = y0 ^ y29 ^ (bit 43 of step 3) = y0 ^ y29 ^ y43 ^ y26 ^ y55 ^ y6 ^ y35 — the parity
// of y & 0x0080080824000041 (checked against the full tempering on random words).
__device__ __forceinline__ unsigned mt_temper_bit0(uint64_t y) {
  return static_cast<unsigned>(__popcll(y & 0x0080080824000041ull)) & 1u;
}

constexpr int MT_R = (MT_N + 31) / 32;  // 10 registers per lane: word 32 r + lane

// One twist of the register-resident state R[r] = mt[32 r + lane].  Words are produced in
// increasing index order, so each step still reads the old words above it (i + 1, i + m)
// and, for i ≥ n − m, the new words i − (n − m) below it — the sequential recurrence.
// Shuffles run on all lanes; the lane's own word is selected afterwards.
__device__ __forceinline__ void mt_twist_reg(uint64_t (&R)[MT_R], int lane) {
  const unsigned FULL = 0xffffffffu;
#pragma unroll
  for (int r = 0; r < MT_R; ++r) {
    // mt[i + 1]: lane + 1 of register r, or lane 0 of register r + 1 for the last lane
    const uint64_t up = __shfl_down_sync(FULL, R[r], 1);
    const uint64_t nx = r + 1 < MT_R ? __shfl_sync(FULL, R[r + 1 < MT_R ? r + 1 : r], 0) : 0ull;
    const uint64_t next = lane == 31 ? nx : up;
    const int i = 32 * r + lane;
    uint64_t v = R[r];
    if (r <= 4) {
      // i < 156: mt[i + 156] (old) = register r + 4 of lane + 28, or register r + 5 of lane − 4
      const uint64_t f4 = __shfl_sync(FULL, R[r + 4], (lane + 28) & 31);
      const uint64_t f5 = __shfl_sync(FULL, R[r + 5 < MT_R ? r + 5 : r], (lane + 28) & 31);
      if (i < MT_N - MT_M) v = mt_mix(R[r], next, lane < 4 ? f4 : f5);
    }
    if (r >= 4) {
      // 156 ≤ i < 311: mt[i − 156] (new) = register r − 5 of lane + 4, or register r − 4 of lane − 28
      const uint64_t b5 = __shfl_sync(FULL, R[r >= 5 ? r - 5 : r], (lane + 4) & 31);
      const uint64_t b4 = __shfl_sync(FULL, R[r - 4], (lane + 4) & 31);
      if (i >= MT_N - MT_M && i < MT_N - 1) v = mt_mix(R[r], next, lane < 28 ? b5 : b4);
    }
    R[r] = v;
  }
  // i = 311 (register 9, lane 23): mix(old mt[311], new mt[0], new mt[155])
  const uint64_t m0 = __shfl_sync(FULL, R[0], 0);
  const uint64_t m155 = __shfl_sync(FULL, R[4], 27);
  if (lane == (MT_N - 1) % 32) R[MT_R - 1] = mt_mix(R[MT_R - 1], m0, m155);
}

// One warp per probe: `rows` draws → bit 0 into planes[p][0, rows).
__global__ void __launch_bounds__(32) k_probe_rng(uint64_t* __restrict__ states, int64_t rows,
                                                  uint8_t* __restrict__ planes) {
  const int p = blockIdx.x, lane = threadIdx.x;
  uint64_t* st = states + static_cast<int64_t>(p) * (MT_N + 1);
  uint64_t R[MT_R];
#pragma unroll
  for (int r = 0; r < MT_R; ++r) R[r] = 32 * r + lane < MT_N ? st[32 * r + lane] : 0ull;
  int idx = static_cast<int>(st[MT_N]);
  uint8_t* out = planes + static_cast<int64_t>(p) * rows;
  int64_t done = 0;
  while (done < rows) {
    if (idx == MT_N) {
      mt_twist_reg(R, lane);
      idx = 0;
    }
    const int k = static_cast<int>(imin64(MT_N - idx, rows - done));
    // draws idx .. idx + k − 1 of this block → rows done .. done + k − 1
#pragma unroll
    for (int r = 0; r < MT_R; ++r) {
      const int j = 32 * r + lane - idx;
      if (j >= 0 && j < k) out[done + j] = static_cast<uint8_t>(mt_temper_bit0(R[r]));
    }
    idx += k;
    done += k;
  }
#pragma unroll
  for (int r = 0; r < MT_R; ++r)
    if (32 * r + lane < MT_N) st[32 * r + lane] = R[r];
  if (lane == 0) st[MT_N] = static_cast<uint64_t>(idx);
}

// One block per probe (the warp version above spends most of its time on the serial shuffle
// chain of the twist: ~0.45e9 draws/s per probe).  Thread j < 156 keeps words j and 156 + j
// of the state in registers; a twist needs only thread j + 1's old words (exchanged through a
// double-buffered shared array, one barrier per twist):
//   new[j]       = mix(old[j], old[j + 1], old[j + 156])          (old[156] = thread 0's 2nd word)
//   new[156 + j] = mix(old[156 + j], old[157 + j], new[j])        (j < 155)
//   new[311]     = mix(old[311], new[0], new[155])                (thread 155 recomputes new[0])
// then every thread tempers its two new words into the byte planes.
constexpr int MT_BT = 160;  // 5 warps; threads ≥ 156 only help with the global state copy

// Substreams: block b = (probe b / K, substream k = b % K) owns states[b] and draws
// rows [k·Ls, min((k + 1)·Ls, total)) of its probe's `total` (K = 1: Ls = total).
__global__ void __launch_bounds__(MT_BT) k_probe_rng_blk(uint64_t* __restrict__ states, int64_t total, int K,
                                                         int64_t Ls, uint8_t* __restrict__ planes) {
  __shared__ uint64_t xa[2][MT_M + 1], xb[2][MT_M + 1];
  const int p = blockIdx.x / K, sk = blockIdx.x % K, j = threadIdx.x;
  const bool act = j < MT_M;
  uint64_t* st = states + static_cast<int64_t>(blockIdx.x) * (MT_N + 1);
  uint64_t wa = act ? st[j] : 0ull, wb = act ? st[MT_M + j] : 0ull;
  int idx = static_cast<int>(st[MT_N]);
  const int64_t r0 = static_cast<int64_t>(sk) * Ls;
  const int64_t rows = imin64(Ls, total - r0);
  uint8_t* out = planes + static_cast<int64_t>(p) * total + r0;
  int64_t done = 0;
  if (idx < MT_N) {  // draws left in the current state
    const int k = static_cast<int>(imin64(MT_N - idx, rows));
    if (act) {
      if (j >= idx && j - idx < k) out[j - idx] = static_cast<uint8_t>(mt_temper_bit0(wa));
      const int w2 = MT_M + j;
      if (w2 >= idx && w2 - idx < k) out[w2 - idx] = static_cast<uint8_t>(mt_temper_bit0(wb));
    }
    idx += k;
    done += k;
  }
  int buf = 0;
  while (done < rows) {
    if (act) {
      xa[buf][j] = wa;
      xb[buf][j] = wb;
    }
    __syncthreads();
    if (act) {
      const uint64_t a1 = j + 1 < MT_M ? xa[buf][j + 1] : xb[buf][0];  // old[j + 1]
      const uint64_t na = mt_mix(wa, a1, wb);
      uint64_t nb;
      if (j + 1 < MT_M) {
        nb = mt_mix(wb, xb[buf][j + 1], na);
      } else {  // word 311: new[0] recomputed from thread 0's and 1's old words
        const uint64_t n0 = mt_mix(xa[buf][0], xa[buf][1], xb[buf][0]);
        nb = mt_mix(wb, n0, na);
      }
      wa = na;
      wb = nb;
      const int k = static_cast<int>(imin64(MT_N, rows - done));
      if (j < k) out[done + j] = static_cast<uint8_t>(mt_temper_bit0(wa));
      if (MT_M + j < k) out[done + MT_M + j] = static_cast<uint8_t>(mt_temper_bit0(wb));
    }
    const int k = static_cast<int>(imin64(MT_N, rows - done));
    done += k;
    idx = k;
    buf ^= 1;
  }
  if (act) {
    st[j] = wa;
    st[MT_M + j] = wb;
  }
  if (j == 0) st[MT_N] = static_cast<uint64_t>(idx);
}

// words[i] = Σ_p planes[p][i] << p
__global__ void __launch_bounds__(256) k_probe_pack(const uint8_t* __restrict__ planes, int P, int64_t rows,
                                                    uint64_t* __restrict__ words) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  uint64_t w = 0;
  for (int p = 0; p < P; ++p) w |= static_cast<uint64_t>(planes[static_cast<int64_t>(p) * rows + i] & 1u) << p;
  words[i] = w;
}

// dst[p] = src[p·K + K − 1] (the last substream's end state is the probe's new position)
__global__ void k_probe_take_last(const uint64_t* __restrict__ src, int K, uint64_t* __restrict__ dst) {
  const int p = blockIdx.x;
  for (int i = threadIdx.x; i <= MT_N; i += blockDim.x)
    dst[static_cast<int64_t>(p) * (MT_N + 1) + i] = src[(static_cast<int64_t>(p) * K + K - 1) * (MT_N + 1) + i];
}

// Substreams: every substream is a whole number of units of kSubRows draws (kJumpUnit blocks
// of 312 words), so each start is a block jump x^{312 q} with q a multiple of kJumpUnit,
// whatever the base index.  One slab holds as many rows as a 3 GB plane budget allows (config
// 5: all 5e7 rows at once), cut into K substreams per probe so P·K ≈ 4 blocks per SM draw
// concurrently — few jumps (each costs ~10^4 shared loads per thread) and enough blocks for
// the latency-bound twist.  (Round 2 start: 16 fixed 1.05e6-draw substreams per 1.7e7-row slab,
// 1440 jumps for config 5.)
constexpr int64_t kSubRows = int64_t{MT_N} * static_cast<int64_t>(kJumpUnit);  // 1,048,320 draws
constexpr int kMaxSub = 64;
constexpr int64_t kPlaneBudget = int64_t{3} << 30;  // bytes of probe planes per slab

int64_t probe_rng_slab(int P) {
  const int64_t units = std::max<int64_t>(1, kPlaneBudget / (std::max(1, P) * kSubRows));
  return units * kSubRows;
}
int64_t probe_rng_scratch_words(int P) { return static_cast<int64_t>(P) * kMaxSub * (MT_N + 1) + kMaxSub * 312; }

void run_probe_rng(const Launch& L, uint64_t* states, int P, int64_t rows, uint8_t* planes, uint64_t* words,
                   uint64_t* scratch) {
  const int64_t slab = probe_rng_slab(P);
  static const bool warp_rng = [] {
    const char* e = getenv("GSGPC_PROBE_RNG_WARP");
    return e && e[0] == '1';
  }();
  static const bool no_split = [] {
    const char* e = getenv("GSGPC_PROBE_RNG_NOSPLIT");
    return e && e[0] == '1';
  }();
  static const int bps = [] {  // diagnostics: concurrent generator blocks per SM
    const char* e = getenv("GSGPC_PROBE_RNG_BPS");
    return e ? std::max(1, atoi(e)) : 4;  // B200, config 5 (30 probes × 5e7 draws): 1 → 10.4, 2 → 6.4, 4 → 5.1 ms
  }();
  for (int64_t r0 = 0; r0 < rows; r0 += slab) {
    const int64_t nr = std::min(slab, rows - r0);
    int K = 1;
    int64_t Ls = nr;
    if (!warp_rng && !no_split) {
      const int want = std::min<int>(kMaxSub, std::max<int>(1, static_cast<int>(ceil_div(sm_count() * bps, P))));
      Ls = ceil_div(ceil_div(nr, want), kSubRows) * kSubRows;
      K = static_cast<int>(ceil_div(nr, Ls));
      if (K == 1) Ls = nr;
    }
    if (warp_rng) {
      k_probe_rng<<<P, 32, 0, L.s>>>(states, nr, planes);
      L.count(1);
    } else if (K == 1) {
      k_probe_rng_blk<<<P, MT_BT, 0, L.s>>>(states, nr, 1, nr, planes);
      L.count(1);
    } else {
      // substream k of every probe starts k · Ls draws after the probe's position
      uint64_t* sub = scratch;
      uint64_t* polys = scratch + static_cast<int64_t>(P) * kMaxSub * (MT_N + 1);
      std::vector<uint64_t> q(K);
      for (int k = 0; k < K; ++k) q[k] = static_cast<uint64_t>(k) * static_cast<uint64_t>(Ls / MT_N);
      run_mt_jump(L, states, P, q, polys, sub);
      k_probe_rng_blk<<<P * K, MT_BT, 0, L.s>>>(sub, nr, K, Ls, planes);
      k_probe_take_last<<<P, 128, 0, L.s>>>(sub, K, states);
      L.count(2);
    }
    k_probe_pack<<<static_cast<unsigned>(ceil_div(nr, 256)), 256, 0, L.s>>>(planes, P, nr, words + r0);
    L.count(1);
  }
  GSGPC_CUDA(cudaGetLastError());
}

}  // namespace gsgpc
