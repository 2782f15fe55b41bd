// fftw_stand_in.cpp — TEST INFRASTRUCTURE.  The FFTW3 subset declared in fftw3.h on a
// self-written recursive mixed-radix FFT (radices 2, 3, 5; any other prime factor by a direct
// DFT).  r2c: the full complex N-d transform of the real input, of which the non-redundant
// half (last dimension 0..n/2) is written; c2r: the Hermitian half is expanded, transformed
// back, and the real parts written.  Unnormalised, like FFTW.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstddef>
#include <vector>

namespace {

using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846264338327950288;

int smallest_factor(int n) {
  for (int p : {2, 3, 5})
    if (n % p == 0) return p;
  for (int p = 7; p * p <= n; p += 2)
    if (n % p == 0) return p;
  return n;
}

// out[k] = Σ_j in[j·stride] w^{jk}, w = exp(sign·2πi/n); decimation in time by the smallest factor
void fft_rec(const cd* in, cd* out, int n, int stride, int sign, const std::vector<cd>& tw, int tw_step) {
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  const int p = smallest_factor(n), q = n / p;
  // sub-transforms of the p interleaved subsequences
  for (int r = 0; r < p; ++r) fft_rec(in + static_cast<std::ptrdiff_t>(r) * stride, out + r * q, q, stride * p, sign, tw, tw_step * p);
  // butterflies: X[k + q·s] = Σ_r w_n^{r(k + q s)} Y_r[k]
  std::vector<cd> t(static_cast<std::size_t>(p));
  const std::ptrdiff_t N = static_cast<std::ptrdiff_t>(tw.size());
  for (int k = 0; k < q; ++k) {
    for (int r = 0; r < p; ++r) t[r] = out[r * q + k];
    for (int s = 0; s < p; ++s) {
      const int kk = k + q * s;
      cd acc = t[0];
      for (int r = 1; r < p; ++r) {
        const std::ptrdiff_t idx = (static_cast<std::ptrdiff_t>(r) * kk % n) * tw_step % N;
        acc += t[r] * tw[static_cast<std::size_t>(idx)];
      }
      out[kk] = acc;
    }
  }
  (void)sign;
}

void fft_1d(cd* data, int n, std::ptrdiff_t stride, int sign, std::vector<cd>& scratch_in, std::vector<cd>& scratch_out,
            const std::vector<cd>& tw) {
  for (int j = 0; j < n; ++j) scratch_in[j] = data[j * stride];
  fft_rec(scratch_in.data(), scratch_out.data(), n, 1, sign, tw, 1);
  for (int j = 0; j < n; ++j) data[j * stride] = scratch_out[j];
}

void fft_nd(std::vector<cd>& a, const std::vector<int>& dims, int sign) {
  const int d = static_cast<int>(dims.size());
  std::ptrdiff_t total = 1;
  for (int n : dims) total *= n;
  std::ptrdiff_t inner = 1;
  for (int k = d - 1; k >= 0; --k) {
    const int n = dims[k];
    std::vector<cd> tw(static_cast<std::size_t>(n)), si(static_cast<std::size_t>(n)), so(static_cast<std::size_t>(n));
    for (int j = 0; j < n; ++j) {
      const double ang = sign * 2.0 * kPi * j / n;
      tw[j] = cd(std::cos(ang), std::sin(ang));
    }
    const std::ptrdiff_t outer = total / (inner * n);
    for (std::ptrdiff_t o = 0; o < outer; ++o)
      for (std::ptrdiff_t i = 0; i < inner; ++i) fft_1d(a.data() + o * n * inner + i, n, inner, sign, si, so, tw);
    inner *= n;
  }
}

}  // namespace

struct fftw_stand_in_plan {
  std::vector<int> dims;
  bool forward;
  double* r;
  fftw_complex* c;
  std::ptrdiff_t total, half_total;
  int nlast, nhalf;
};

static fftw_plan make_plan(int rank, const int* n, double* r, fftw_complex* c, bool forward) {
  auto* p = new fftw_stand_in_plan;
  p->dims.assign(n, n + rank);
  p->forward = forward;
  p->r = r;
  p->c = c;
  p->total = 1;
  for (int k = 0; k < rank; ++k) p->total *= n[k];
  p->nlast = n[rank - 1];
  p->nhalf = p->nlast / 2 + 1;
  p->half_total = p->total / p->nlast * p->nhalf;
  return p;
}

extern "C" {

fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double* in, fftw_complex* out, unsigned) {
  return make_plan(rank, n, in, out, true);
}
fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex* in, double* out, unsigned) {
  return make_plan(rank, n, out, in, false);
}

void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
  std::vector<cd> a(static_cast<std::size_t>(p->total));
  for (std::ptrdiff_t i = 0; i < p->total; ++i) a[i] = cd(in[i], 0.0);
  fft_nd(a, p->dims, -1);
  const std::ptrdiff_t lines = p->total / p->nlast;
  for (std::ptrdiff_t l = 0; l < lines; ++l)
    for (int k = 0; k < p->nhalf; ++k) {
      const cd v = a[l * p->nlast + k];
      out[l * p->nhalf + k][0] = v.real();
      out[l * p->nhalf + k][1] = v.imag();
    }
}

void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
  // X[k_1..k_d] for k_d > n_d/2 is the conjugate of X at the mirrored multi-index
  const int d = static_cast<int>(p->dims.size());
  std::vector<cd> a(static_cast<std::size_t>(p->total));
  std::vector<int> idx(d, 0);
  for (std::ptrdiff_t flat = 0; flat < p->total; ++flat) {
    if (idx[d - 1] < p->nhalf) {
      const std::ptrdiff_t l = flat / p->nlast;
      const fftw_complex& v = in[l * p->nhalf + idx[d - 1]];
      a[flat] = cd(v[0], v[1]);
    } else {
      std::ptrdiff_t l = 0;
      for (int k = 0; k + 1 < d; ++k) l = l * p->dims[k] + (idx[k] == 0 ? 0 : p->dims[k] - idx[k]);
      const fftw_complex& v = in[l * p->nhalf + (p->nlast - idx[d - 1])];
      a[flat] = cd(v[0], -v[1]);
    }
    for (int k = d - 1; k >= 0; --k) {
      if (++idx[k] < p->dims[k]) break;
      idx[k] = 0;
    }
  }
  fft_nd(a, p->dims, +1);
  for (std::ptrdiff_t i = 0; i < p->total; ++i) out[i] = a[i].real();
}

void fftw_execute(const fftw_plan p) {
  if (p->forward) fftw_execute_dft_r2c(p, p->r, p->c);
  else fftw_execute_dft_c2r(p, p->c, p->r);
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
