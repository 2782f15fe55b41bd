// mt_jump.cu — jump-ahead for the reference's MT19937-64 probe streams.
//
// rademacher_probe (gp.cpp:16-25) reads one std::mt19937_64 draw per row in stream order, so
// a probe stream is inherently sequential.  Two things need a stream started far from its
// seed without drawing every value in between:
//   * a rank (or an accumulator) whose rows start at global row o must draw outputs o, o+1, …
//     of each probe — the streams of one global pass, not a fresh stream per shard;
//   * one probe's draws for a 1.6e7-row slab are split into substreams of L rows, each on
//     its own block (30 probes × 16 substreams fill the 148 SMs instead of 30 blocks).
//
// The MT19937-64 state transition F is linear over GF(2).  Write the word sequence as
// x_{k+312} = mix(x_k, x_{k+1}, x_{k+156}) and a state as the window W_k = (x_k … x_{k+311}).
// With φ the characteristic polynomial of F (degree 19937; only the 31 low bits of x_k lie
// outside its span, and those bits are never read again), F^J W = g(F) W for
// g = x^J mod φ, and g(F) W = ⊕_{i : g_i = 1} W_{k+i}: word j of the jumped window is the XOR of
// x_{k+i+j} over the set coefficients — a correlation of g with the next 20248 words.
//   * φ: Berlekamp–Massey over bit 0 of 2·19937 tempered outputs (linear in the state, and
//     φ is irreducible, so the minimal polynomial of that bit sequence is φ itself).
//   * x^J mod φ: square-and-multiply over GF(2)[x] on 313-word bit vectors (carry-less
//     squaring by bit spreading, reduction by word-aligned XORs of 64 pre-shifted copies of φ).
//   * the correlation: one block per (stream, jump); the 20248 words live in shared memory
//     (162 KB), thread j accumulates word j while every thread walks the set bits of g.
// Jumps are taken in whole blocks of 312 words: a generator (window mt[0..311], index r)
// advanced by o draws is (F^{312 q} mt, r') with q = ⌊(r + o)/312⌋, r' = (r + o) mod 312.
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <random>
#include <vector>

#include "internal.cuh"
#include "precompute.cuh"

namespace gsgpc {

namespace {

constexpr int kN = 312, kM = 156;
constexpr int kDeg = 19937;                   // deg φ
constexpr int kPW = (kDeg + 64) / 64;         // 312 words: polynomials of degree ≤ 19967
constexpr int kSeq = kDeg + kN - 1;           // 20248 words of the sequence for one jump
constexpr uint64_t kA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUM = 0xFFFFFFFF80000000ull;
constexpr uint64_t kLM = 0x7FFFFFFFull;

using Poly = std::vector<uint64_t>;  // bit i = coefficient of x^i

inline int bit(const Poly& p, int64_t i) {
  return static_cast<int>((p[static_cast<size_t>(i >> 6)] >> (i & 63)) & 1u);
}

// p ^= q << s (q's length words, p long enough)
void xor_shifted(Poly& p, const Poly& q, int64_t s) {
  const int64_t w = s >> 6, b = s & 63;
  for (size_t i = 0; i < q.size(); ++i) {
    if (!q[i]) continue;
    p[w + i] ^= q[i] << b;
    if (b) p[w + i + 1] ^= q[i] >> (64 - b);
  }
}

struct Gf2Field {
  Poly phi;               // φ, degree kDeg
  std::vector<Poly> phs;  // phs[s] = φ << s, s < 64 (kPW + 1 words)

  Gf2Field() {
    // 2·deg bits of the linear sequence: bit 0 of consecutive std::mt19937_64 outputs
    const int n2 = 2 * kDeg;
    std::mt19937_64 gen(5489u);
    std::vector<uint8_t> s(n2);
    for (int i = 0; i < n2; ++i) s[i] = static_cast<uint8_t>(gen() & 1u);
    // reversed packed copy: R bit t = s[n2 − 1 − t], so s[n − i] for i = 0.. is R from n2 − 1 − n
    const int rw = (n2 + 63) / 64 + 2;
    Poly R(rw, 0);
    for (int t = 0; t < n2; ++t) R[t >> 6] |= static_cast<uint64_t>(s[n2 - 1 - t]) << (t & 63);
    // Berlekamp–Massey (connection polynomial C: Σ_{i=0..L} c_i s_{n−i} = 0, c_0 = 1)
    const int cw = kPW + 2;
    Poly C(cw, 0), B(cw, 0), T;
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int n = 0; n < n2; ++n) {
      const int off = n2 - 1 - n;
      const int w0 = off >> 6, sh = off & 63;
      const int nw = (L >> 6) + 1;
      uint64_t acc = 0;
      for (int q = 0; q < nw; ++q) {
        uint64_t win = R[w0 + q] >> sh;
        if (sh) win |= R[w0 + q + 1] << (64 - sh);
        acc ^= win & C[q];
      }
      // bits above L in the last word of C are zero, so only the L + 1 window bits count
      if (__builtin_popcountll(acc) & 1) {
        if (2 * L <= n) {
          T = C;
          xor_shifted(C, Poly(B.begin(), B.end() - 2), m);
          L = n + 1 - L;
          B = T;
          m = 1;
        } else {
          xor_shifted(C, Poly(B.begin(), B.end() - 2), m);
          ++m;
        }
      } else {
        ++m;
      }
    }
    if (L != kDeg) throw Error(GSGPC_RUNTIME_ERROR, "mt19937_64 jump: characteristic polynomial has degree " +
                                                        std::to_string(L));
    // φ(x) = x^L C(1/x)
    phi.assign(kPW, 0);
    for (int i = 0; i <= L; ++i)
      if (bit(C, L - i)) phi[i >> 6] |= 1ull << (i & 63);
    phs.assign(64, Poly(kPW + 1, 0));
    for (int s2 = 0; s2 < 64; ++s2) xor_shifted(phs[s2], phi, s2);
  }

  // r (any length ≥ kPW) mod φ → kPW words
  Poly reduce(Poly r) const {
    int64_t top = static_cast<int64_t>(r.size()) * 64 - 1;
    for (int64_t b = top; b >= kDeg; --b) {
      if (!bit(r, b)) continue;
      const int64_t s = b - kDeg;
      const Poly& q = phs[s & 63];
      const int64_t w = s >> 6;
      for (size_t i = 0; i < q.size() && w + static_cast<int64_t>(i) < static_cast<int64_t>(r.size()); ++i)
        r[w + i] ^= q[i];
    }
    r.resize(kPW);
    return r;
  }

  Poly sqr(const Poly& a) const {
    Poly r(2 * kPW, 0);
    for (int i = 0; i < kPW; ++i) {
      uint64_t lo = 0, hi = 0;
      const uint64_t v = a[i];
      for (int b = 0; b < 32; ++b) {
        lo |= ((v >> b) & 1ull) << (2 * b);
        hi |= ((v >> (b + 32)) & 1ull) << (2 * b);
      }
      r[2 * i] = lo;
      r[2 * i + 1] = hi;
    }
    return reduce(std::move(r));
  }

  Poly mul(const Poly& a, const Poly& b) const {
    std::vector<Poly> bs(64, Poly(kPW + 1, 0));
    for (int s = 0; s < 64; ++s) xor_shifted(bs[s], b, s);
    Poly r(2 * kPW + 2, 0);
    for (int64_t i = 0; i < static_cast<int64_t>(kPW) * 64; ++i) {
      if (!bit(a, i)) continue;
      const Poly& q = bs[i & 63];
      const int64_t w = i >> 6;
      for (size_t k = 0; k < q.size(); ++k) r[w + k] ^= q[k];
    }
    return reduce(std::move(r));
  }

  Poly xpow(uint64_t e) const {  // x^e mod φ
    Poly r(kPW, 0);
    r[0] = 1;
    int hb = 63;
    while (hb >= 0 && !((e >> hb) & 1ull)) --hb;
    for (int b = hb; b >= 0; --b) {
      r = sqr(r);
      if ((e >> b) & 1ull) {  // r *= x
        Poly t(kPW + 1, 0);
        xor_shifted(t, r, 1);
        r = reduce(std::move(t));
      }
    }
    return r;
  }
};

const Gf2Field& field() {
  static std::once_flag once;
  static Gf2Field* f = nullptr;
  std::call_once(once, [] { f = new Gf2Field(); });
  return *f;
}

std::mutex g_poly_mu;
std::map<uint64_t, Poly>& poly_cache() {
  static std::map<uint64_t, Poly> c;
  return c;
}

__device__ __forceinline__ uint64_t jmix(uint64_t hi_word, uint64_t lo_word, uint64_t far) {
  const uint64_t x = (hi_word & kUM) | (lo_word & kLM);
  return far ^ (x >> 1) ^ ((x & 1ull) ? kA : 0ull);
}

constexpr int kJT = 320;  // threads per jump block (312 window words)

// Block b = (stream s = b / K, jump k = b % K): out[s·K + k] = F^{312 q_k} in[s] (window
// mt[0..311]; the index word is copied).  polys[k] = x^{312 q_k} mod φ (kPW words); a
// polynomial equal to 1 copies the window.  The set coefficients of g are first compacted
// into a list of positions (~10^4 for a random jump), so the correlation runs 8 independent
// shared loads per step instead of a bit scan with one dependent load per set bit (the jump
// kernel was the largest part of config 5's probe generation).
__global__ void __launch_bounds__(kJT) k_mt_jump(const uint64_t* __restrict__ in, int K,
                                                 const uint64_t* __restrict__ polys, uint64_t* __restrict__ out) {
  extern __shared__ uint64_t smem[];
  uint64_t* y = smem;                                        // kSeq words
  uint64_t* g = smem + kSeq;                                 // kPW words
  uint16_t* pos = reinterpret_cast<uint16_t*>(g + kPW);      // ≤ kDeg positions
  __shared__ int wtot[kJT / 32 + 1];
  const int s = blockIdx.x / K, k = blockIdx.x % K, t = threadIdx.x;
  const int lane = t & 31, wid = t >> 5;
  const uint64_t* st = in + static_cast<int64_t>(s) * (kN + 1);
  for (int i = t; i < kN; i += kJT) y[i] = st[i];
  for (int i = t; i < kPW; i += kJT) g[i] = polys[static_cast<int64_t>(k) * kPW + i];
  __syncthreads();
  // positions of the set bits, in increasing order (thread t < kPW owns word t)
  const uint64_t gw = t < kPW ? g[t] : 0ull;
  const int c = __popcll(gw);
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wtot[wid] = incl;
  // the sequence: words [base + 312, base + 468) depend only on words below base + 312
  for (int base = 0; base + kN < kSeq; base += kM) {
    const int i = base + t;
    if (t < kM && i + kN < kSeq) y[i + kN] = jmix(y[i], y[i + 1], y[i + kM]);
    __syncthreads();
  }
  if (t == 0) {
    int run = 0;
    for (int w = 0; w < kJT / 32; ++w) {
      const int v = wtot[w];
      wtot[w] = run;
      run += v;
    }
    wtot[kJT / 32] = run;
  }
  __syncthreads();
  {
    int o = wtot[wid] + incl - c;
    uint64_t bits = gw;
    while (bits) {
      const int b = __ffsll(static_cast<long long>(bits)) - 1;
      bits &= bits - 1;
      pos[o++] = static_cast<uint16_t>(64 * t + b);
    }
  }
  __syncthreads();
  const int np = wtot[kJT / 32];
  const int j = t < kN ? t : 0;
  uint64_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int i = 0;
  for (; i + 8 <= np; i += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] ^= y[pos[i + u] + j];
  }
  for (; i < np; ++i) acc[0] ^= y[pos[i] + j];
  const uint64_t r = ((acc[0] ^ acc[1]) ^ (acc[2] ^ acc[3])) ^ ((acc[4] ^ acc[5]) ^ (acc[6] ^ acc[7]));
  uint64_t* o = out + (static_cast<int64_t>(s) * K + k) * (kN + 1);
  if (t < kN) o[t] = r;
  if (t == 0) o[kN] = st[kN];
}

}  // namespace

// x^{312 q} mod φ (cached; caller holds g_poly_mu).  Substream starts are multiples N·q0 of
// one unit (kJumpUnit blocks of 312 draws): x^{312 N q0} is the square of x^{312 (N/2) q0}
// (N even) or x^{312 (N−1) q0} · x^{312 q0} (N odd) — a few squarings and multiplications per
// new multiple instead of a full square-and-multiply chain.
static const Poly& jump_poly_locked(uint64_t q) {
  auto& c = poly_cache();
  auto it = c.find(q);
  if (it != c.end()) return it->second;
  const uint64_t q0 = kJumpUnit;
  Poly p;
  if (q > q0 && q % q0 == 0) {
    const uint64_t N = q / q0;
    if (N % 2 == 0) p = field().sqr(jump_poly_locked(q / 2));
    else p = field().mul(jump_poly_locked(q - q0), jump_poly_locked(q0));
  } else {
    p = field().xpow(312ull * q);
  }
  return c.emplace(q, std::move(p)).first->second;
}

static const Poly& jump_poly(uint64_t q) {
  std::lock_guard<std::mutex> lk(g_poly_mu);
  return jump_poly_locked(q);
}

int64_t mt_jump_smem_bytes() {
  return static_cast<int64_t>(sizeof(uint64_t)) * (kSeq + kPW) + static_cast<int64_t>(sizeof(uint16_t)) * (kDeg + 1);
}

// Device: for S streams (states in: S × 313) and K block-jumps q[0..K) (q = 0: copy),
// out[s·K + k] = stream s advanced by 312·q[k] draws (index word kept).  polys_dev: scratch
// ≥ K × 312 words on the device.
void run_mt_jump(const Launch& L, const uint64_t* in, int S, const std::vector<uint64_t>& q, uint64_t* polys_dev,
                 uint64_t* out) {
  const int K = static_cast<int>(q.size());
  std::vector<uint64_t> h(static_cast<size_t>(K) * kPW, 0);
  for (int k = 0; k < K; ++k) {
    if (q[k] == 0) {
      h[static_cast<size_t>(k) * kPW] = 1;
    } else {
      const Poly& p = jump_poly(q[k]);
      std::copy(p.begin(), p.end(), h.begin() + static_cast<size_t>(k) * kPW);
    }
  }
  GSGPC_CUDA(cudaMemcpyAsync(polys_dev, h.data(), sizeof(uint64_t) * h.size(), cudaMemcpyHostToDevice, L.s));
  set_max_dynamic_smem(reinterpret_cast<const void*>(k_mt_jump), static_cast<int>(mt_jump_smem_bytes()));
  k_mt_jump<<<S * K, kJT, mt_jump_smem_bytes(), L.s>>>(in, K, polys_dev, out);
  L.count(1);
  GSGPC_CUDA(cudaGetLastError());
  // the host staging vector must outlive the async copy
  GSGPC_CUDA(cudaStreamSynchronize(L.s));
}

// Host restatement of the same jump (test hook and the CPU-side check of the device kernel):
// state (313 words: window + index) advanced by `draws` draws.
void mt_jump_host(uint64_t* st, uint64_t draws) {
  const uint64_t r = st[kN];
  const uint64_t a = r + draws;
  const uint64_t q = a / kN, r2 = a % kN;
  if (q > 0) {
    const Poly& g = jump_poly(q);
    std::vector<uint64_t> y(kSeq);
    for (int i = 0; i < kN; ++i) y[i] = st[i];
    for (int i = 0; i + kN < kSeq; ++i) {
      const uint64_t x = (y[i] & kUM) | (y[i + 1] & kLM);
      y[i + kN] = y[i + kM] ^ (x >> 1) ^ ((x & 1ull) ? kA : 0ull);
    }
    for (int j = 0; j < kN; ++j) {
      uint64_t acc = 0;
      for (int i = 0; i < kDeg; ++i)
        if (bit(g, i)) acc ^= y[i + j];
      st[j] = acc;
    }
  }
  st[kN] = r2;
}

}  // namespace gsgpc
