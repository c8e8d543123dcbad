// FFTW3-API shim (see fftw3.h).  Test infrastructure for the CPU oracle only.
//
// Each axis length n gets a 1-D plan: its factorisation (4s first, then 2,
// 3, 5, 7, remaining primes) and a table of the n roots of unity for the
// plan's sign.  A d-dimensional transform applies the 1-D transform to every
// line along every axis (lines copied to a contiguous scratch buffer).  The
// recursion is decimation in time; the combine step at each level is done in
// place over the p interleaved sub-results.

#include "fftw3.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

namespace {

using cplx = std::complex<double>;

int g_threads = 1;

struct Plan1D {
  int n = 1;
  std::vector<int> factors;
  std::vector<cplx> w;  // w[j] = exp(sign * 2 pi i j / n)

  Plan1D(int n_, int sign) : n(n_) {
    int m = n;
    while (m % 4 == 0) { factors.push_back(4); m /= 4; }
    for (int p : {2, 3, 5, 7})
      while (m % p == 0) { factors.push_back(p); m /= p; }
    for (int p = 11; m > 1; p += 2)
      while (m % p == 0) { factors.push_back(p); m /= p; }
    w.resize(n);
    for (int j = 0; j < n; ++j) {
      long double ang = 2.0L * 3.14159265358979323846264338327950288L * (long double)j / (long double)n;
      w[j] = cplx((double)cosl(ang), (double)(sign * sinl(ang)));
    }
  }

  // out[0..len) = DFT_len of in[0], in[is], ...; ws = n / len (twiddle stride)
  void rec(const cplx* in, long is, cplx* out, int len, int fi, int ws) const {
    if (len == 1) { out[0] = in[0]; return; }
    const int p = factors[fi];
    const int m = len / p;
    for (int r = 0; r < p; ++r) rec(in + r * is, is * p, out + r * m, m, fi + 1, ws * p);
    cplx t[64];
    std::vector<cplx> big;
    cplx* tp = t;
    if (p > 64) { big.resize(p); tp = big.data(); }
    const int nn = n;
    for (int k = 0; k < m; ++k) {
      tp[0] = out[k];
      for (int r = 1; r < p; ++r) tp[r] = out[r * m + k] * w[(long)r * k * ws];  // r k ws < n

      if (p == 2) {
        out[k] = tp[0] + tp[1];
        out[k + m] = tp[0] - tp[1];
      } else if (p == 4) {
        // w4 = w[n/4] = exp(sign*i*pi/2)
        const cplx j4 = w[nn / 4];
        cplx a0 = tp[0] + tp[2], a1 = tp[0] - tp[2];
        cplx b0 = tp[1] + tp[3], b1 = (tp[1] - tp[3]) * j4;
        out[k] = a0 + b0;
        out[k + m] = a1 + b1;
        out[k + 2 * m] = a0 - b0;
        out[k + 3 * m] = a1 - b1;
      } else {
        const int step = nn / p;
        for (int q = 0; q < p; ++q) {
          cplx s = 0.0;
          for (int r = 0; r < p; ++r) s += tp[r] * w[(long)((r * q) % p) * step];
          out[k + q * m] = s;
        }
      }
    }
  }

  void exec(const cplx* in, cplx* out) const { rec(in, 1, out, n, 0, 1); }
};

}  // namespace

struct fftw_plan_s {
  int rank = 0;
  std::vector<int> dims;
  int sign = FFTW_FORWARD;
  std::vector<std::unique_ptr<Plan1D>> axes;
};

extern "C" {

void fftw_shim_set_threads(int n) { g_threads = std::max(1, n); }
int fftw_shim_get_threads(void) { return g_threads; }

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex*, fftw_complex*, int sign, unsigned) {
  if (rank < 1) return nullptr;
  auto* p = new fftw_plan_s;
  p->rank = rank;
  p->sign = sign;
  for (int a = 0; a < rank; ++a) {
    if (n[a] < 1) { delete p; return nullptr; }
    p->dims.push_back(n[a]);
    p->axes.emplace_back(new Plan1D(n[a], sign));
  }
  return p;
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

void fftw_execute_dft(const fftw_plan p, fftw_complex* in_, fftw_complex* out_) {
  cplx* in = reinterpret_cast<cplx*>(in_);
  cplx* out = reinterpret_cast<cplx*>(out_);
  std::size_t total = 1;
  for (int d : p->dims) total *= (std::size_t)d;
  if (in != out) std::memcpy(out, in, total * sizeof(cplx));
  for (int a = 0; a < p->rank; ++a) {
    const int n = p->dims[a];
    if (n == 1) continue;
    std::size_t stride = 1;
    for (int b = a + 1; b < p->rank; ++b) stride *= (std::size_t)p->dims[b];
    const std::size_t outer = total / ((std::size_t)n * stride);
    const std::size_t lines = outer * stride;
    const Plan1D& pl = *p->axes[a];
    // Lines along a strided axis are processed in blocks of B neighbouring lines
    // (contiguous in memory): the block is copied with B-element row copies,
    // each column transformed, and copied back -- cache-friendly for the slow axes.
    constexpr std::size_t B = 16;
    const std::size_t nblk_per_outer = stride >= B ? (stride + B - 1) / B : stride;
    const bool blocked = stride >= B;
    const std::size_t units = blocked ? outer * nblk_per_outer : lines;
    auto work = [&](std::size_t u0, std::size_t u1) {
      std::vector<cplx> a_(n), b_(n);
      std::vector<cplx> blk(blocked ? (std::size_t)n * B : 0);
      for (std::size_t u = u0; u < u1; ++u) {
        if (!blocked) {
          const std::size_t o = u / stride, s = u % stride;
          cplx* base = out + o * (std::size_t)n * stride + s;
          for (int k = 0; k < n; ++k) a_[k] = base[(std::size_t)k * stride];
          pl.exec(a_.data(), b_.data());
          for (int k = 0; k < n; ++k) base[(std::size_t)k * stride] = b_[k];
          continue;
        }
        const std::size_t o = u / nblk_per_outer, s0 = (u % nblk_per_outer) * B;
        const std::size_t w = std::min(B, stride - s0);
        cplx* base = out + o * (std::size_t)n * stride + s0;
        for (int k = 0; k < n; ++k) std::memcpy(&blk[(std::size_t)k * B], base + (std::size_t)k * stride, w * sizeof(cplx));
        for (std::size_t j = 0; j < w; ++j) {
          for (int k = 0; k < n; ++k) a_[k] = blk[(std::size_t)k * B + j];
          pl.exec(a_.data(), b_.data());
          for (int k = 0; k < n; ++k) blk[(std::size_t)k * B + j] = b_[k];
        }
        for (int k = 0; k < n; ++k) std::memcpy(base + (std::size_t)k * stride, &blk[(std::size_t)k * B], w * sizeof(cplx));
      }
    };
    const int nth = (int)std::min<std::size_t>((std::size_t)g_threads, units);
    if (nth <= 1 || total < 32768) {
      work(0, units);
    } else {
      std::vector<std::thread> th;
      const std::size_t chunk = (units + nth - 1) / nth;
      for (int t = 0; t < nth; ++t) {
        std::size_t l0 = t * chunk, l1 = std::min(units, l0 + chunk);
        if (l0 < l1) th.emplace_back(work, l0, l1);
      }
      for (auto& x : th) x.join();
    }
  }
}

}  // extern "C"
