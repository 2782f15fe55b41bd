// probe_rng.cu — the reference's Rademacher probe streams on the device.
//
// rademacher_probe (gp.cpp:16-25): probe p draws one std::mt19937_64 output per row, in
// stream order, from a generator seeded with std::seed_seq{seed_lo, seed_hi, p_lo, p_hi}, and
// takes bit 0 (1 → +1, 0 → −1).  The streams are sequential, so each probe runs on one warp:
// the 312-word MT19937-64 twist is split into its three dependency phases (i < n−m from the
// old state; n−m ≤ i < n−1 from the new words i−(n−m); i = n−1 last), 32 words at a time, and
// the tempered outputs of a block are written one byte per row (coalesced).  A second kernel
// packs the bytes into one 64-bit word per row (bit p = probe p), the layout the binning
// carries with the rows.  The initial state is built on the host exactly as
// mersenne_twister_engine(seed_seq&) does ([rand.eng.mers]: generate 2n 32-bit words,
// x_i = a_{2i} + 2^32 a_{2i+1}, all-zero guard); each probe keeps (state, index) on the
// device across batches.
#include <cuda_runtime.h>

#include <cstdint>
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

// One twist of the warp-resident state (shared memory), lanes 0..31.
__device__ __forceinline__ void mt_twist(uint64_t* mt, int lane) {
  for (int base = 0; base < MT_N - MT_M; base += 32) {  // i < 156: old words only
    const int i = base + lane;
    uint64_t v = 0;
    if (i < MT_N - MT_M) v = mt_mix(mt[i], mt[i + 1], mt[i + MT_M]);
    __syncwarp();
    if (i < MT_N - MT_M) mt[i] = v;
    __syncwarp();
  }
  for (int base = MT_N - MT_M; base < MT_N - 1; base += 32) {  // 156 ≤ i < 311: new word i − 156
    const int i = base + lane;
    uint64_t v = 0;
    if (i < MT_N - 1) v = mt_mix(mt[i], mt[i + 1], mt[i - (MT_N - MT_M)]);
    __syncwarp();
    if (i < MT_N - 1) mt[i] = v;
    __syncwarp();
  }
  if (lane == 0) mt[MT_N - 1] = mt_mix(mt[MT_N - 1], mt[0], mt[MT_M - 1]);
  __syncwarp();
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// One warp per probe: `rows` draws → bit 0 into planes[p][0, rows).
__global__ void __launch_bounds__(32) k_probe_rng(uint64_t* __restrict__ states, int64_t rows,
                                                  uint8_t* __restrict__ planes) {
  __shared__ uint64_t mt[MT_N];
  const int p = blockIdx.x, lane = threadIdx.x;
  uint64_t* st = states + static_cast<int64_t>(p) * (MT_N + 1);
  for (int i = lane; i < MT_N; i += 32) mt[i] = st[i];
  int idx = static_cast<int>(st[MT_N]);
  __syncwarp();
  uint8_t* out = planes + static_cast<int64_t>(p) * rows;
  int64_t done = 0;
  while (done < rows) {
    if (idx == MT_N) {
      mt_twist(mt, lane);
      idx = 0;
    }
    const int k = static_cast<int>(imin64(MT_N - idx, rows - done));
    for (int j = lane; j < k; j += 32) out[done + j] = static_cast<uint8_t>(mt_temper(mt[idx + j]) & 1ull);
    idx += k;
    done += k;
  }
  __syncwarp();
  for (int i = lane; i < MT_N; i += 32) st[i] = mt[i];
  if (lane == 0) st[MT_N] = static_cast<uint64_t>(idx);
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

int64_t probe_rng_slab() { return int64_t{1} << 24; }

void run_probe_rng(const Launch& L, uint64_t* states, int P, int64_t rows, uint8_t* planes, uint64_t* words) {
  const int64_t slab = probe_rng_slab();
  for (int64_t r0 = 0; r0 < rows; r0 += slab) {
    const int64_t nr = std::min(slab, rows - r0);
    k_probe_rng<<<P, 32, 0, L.s>>>(states, nr, planes);
    k_probe_pack<<<static_cast<unsigned>(ceil_div(nr, 256)), 256, 0, L.s>>>(planes, P, nr, words + r0);
    L.count(2);
  }
  GSGPC_CUDA(cudaGetLastError());
}

}  // namespace gsgpc
