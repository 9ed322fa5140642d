/* TEST INFRASTRUCTURE ONLY (oracle). Not part of the product path.
 *
 * Minimal API-compatible stand-in for the FFTW3 subset used by the reference
 * (proj/core/src/spectral.cpp:47-62, 112-123): fftw_plan_dft_r2c / _c2r over a
 * rank-d row-major real array, unnormalised, half-complex last axis
 * (n_last/2 + 1 complex outputs).  FFTW3 is absent from this image.  The
 * transforms here are direct separable DFTs (O(m * sum(n_i))), which is exact
 * to round-off for the (2L-1)^3 <= 11^3 sizes the reference uses.  Written from
 * the DFT definition; nothing is copied from FFTW.
 */
#pragma once

#include <cmath>
#include <complex>
#include <vector>

typedef double fftw_complex[2];

#define FFTW_ESTIMATE (1U << 6)

struct ankh_shim_fftw_plan_s {
  int kind; /* 0 = r2c, 1 = c2r */
  std::vector<int> dims;
  double* real;
  fftw_complex* cplx;
};
typedef ankh_shim_fftw_plan_s* fftw_plan;

namespace ankh_shim_fftw {

/* In-place 1-D DFT along one axis of a row-major complex array.  sign = -1
 * forward, +1 backward; twiddles use the exact integer phase (j*k mod n). */
inline void dft_axis(std::vector<std::complex<double>>& a, const std::vector<int>& dims, int axis,
                     int sign) {
  const int n = dims[static_cast<std::size_t>(axis)];
  std::size_t stride = 1;
  for (std::size_t i = static_cast<std::size_t>(axis) + 1; i < dims.size(); ++i) stride *= static_cast<std::size_t>(dims[i]);
  std::size_t total = 1;
  for (int d : dims) total *= static_cast<std::size_t>(d);
  const std::size_t block = stride * static_cast<std::size_t>(n);
  std::vector<std::complex<double>> tw(static_cast<std::size_t>(n));
  const double two_pi = 6.283185307179586476925286766559;
  for (int k = 0; k < n; ++k) {
    const double ang = sign * two_pi * static_cast<double>(k) / static_cast<double>(n);
    tw[static_cast<std::size_t>(k)] = std::complex<double>(std::cos(ang), std::sin(ang));
  }
  std::vector<std::complex<double>> line(static_cast<std::size_t>(n)), out(static_cast<std::size_t>(n));
  for (std::size_t base = 0; base < total; base += block) {
    for (std::size_t s = 0; s < stride; ++s) {
      for (int j = 0; j < n; ++j) line[static_cast<std::size_t>(j)] = a[base + s + static_cast<std::size_t>(j) * stride];
      for (int k = 0; k < n; ++k) {
        std::complex<double> acc(0.0, 0.0);
        for (int j = 0; j < n; ++j) {
          const long long ph = (static_cast<long long>(j) * k) % n;
          acc += line[static_cast<std::size_t>(j)] * tw[static_cast<std::size_t>(ph)];
        }
        out[static_cast<std::size_t>(k)] = acc;
      }
      for (int k = 0; k < n; ++k) a[base + s + static_cast<std::size_t>(k) * stride] = out[static_cast<std::size_t>(k)];
    }
  }
}

}  // namespace ankh_shim_fftw

inline fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double* in, fftw_complex* out,
                                   unsigned /*flags*/) {
  if (rank < 1) return nullptr;
  fftw_plan p = new ankh_shim_fftw_plan_s;
  p->kind = 0;
  p->dims.assign(n, n + rank);
  p->real = in;
  p->cplx = out;
  return p;
}

inline fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex* in, double* out,
                                   unsigned /*flags*/) {
  if (rank < 1) return nullptr;
  fftw_plan p = new ankh_shim_fftw_plan_s;
  p->kind = 1;
  p->dims.assign(n, n + rank);
  p->real = out;
  p->cplx = in;
  return p;
}

inline void fftw_execute(const fftw_plan p) {
  std::size_t total = 1;
  for (int d : p->dims) total *= static_cast<std::size_t>(d);
  const int last = p->dims.back();
  const int half = last / 2 + 1;
  const std::size_t outer = total / static_cast<std::size_t>(last);
  const int rank = static_cast<int>(p->dims.size());
  std::vector<std::complex<double>> a(total);
  if (p->kind == 0) {
    for (std::size_t i = 0; i < total; ++i) a[i] = std::complex<double>(p->real[i], 0.0);
    for (int ax = 0; ax < rank; ++ax) ankh_shim_fftw::dft_axis(a, p->dims, ax, -1);
    for (std::size_t o = 0; o < outer; ++o)
      for (int k = 0; k < half; ++k) {
        const std::complex<double> v = a[o * static_cast<std::size_t>(last) + static_cast<std::size_t>(k)];
        p->cplx[o * static_cast<std::size_t>(half) + static_cast<std::size_t>(k)][0] = v.real();
        p->cplx[o * static_cast<std::size_t>(half) + static_cast<std::size_t>(k)][1] = v.imag();
      }
  } else {
    /* rebuild the full Hermitian spectrum: X[-k] = conj(X[k]) over all axes */
    std::vector<int> idx(static_cast<std::size_t>(rank));
    for (std::size_t flat = 0; flat < total; ++flat) {
      std::size_t rem = flat;
      for (int ax = rank - 1; ax >= 0; --ax) {
        idx[static_cast<std::size_t>(ax)] = static_cast<int>(rem % static_cast<std::size_t>(p->dims[static_cast<std::size_t>(ax)]));
        rem /= static_cast<std::size_t>(p->dims[static_cast<std::size_t>(ax)]);
      }
      const int kl = idx[static_cast<std::size_t>(rank - 1)];
      bool conj = kl >= half;
      std::size_t src = 0;
      for (int ax = 0; ax < rank; ++ax) {
        const int d = p->dims[static_cast<std::size_t>(ax)];
        int k = idx[static_cast<std::size_t>(ax)];
        if (conj) k = (d - k) % d;
        src = src * static_cast<std::size_t>(ax == rank - 1 ? half : d) + static_cast<std::size_t>(k);
      }
      std::complex<double> v(p->cplx[src][0], p->cplx[src][1]);
      a[flat] = conj ? std::conj(v) : v;
    }
    for (int ax = 0; ax < rank; ++ax) ankh_shim_fftw::dft_axis(a, p->dims, ax, +1);
    for (std::size_t i = 0; i < total; ++i) p->real[i] = a[i].real();
  }
}

inline void fftw_destroy_plan(fftw_plan p) { delete p; }
