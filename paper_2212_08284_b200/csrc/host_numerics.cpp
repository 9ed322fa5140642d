// Geometry-only precompute for the B200 plan (see host_numerics.hpp).
#include "host_numerics.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <random>
#include <stdexcept>
#include <thread>

namespace ankh_b200 {

namespace {
constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoOverSqrtPi = 1.1283791670955125739;

void cheb_values(int order, double x, double* t) {
  t[0] = 1.0;
  if (order > 1) t[1] = x;
  for (int m = 2; m < order; ++m) t[m] = 2.0 * x * t[m - 1] - t[m - 2];
}
}  // namespace

namespace {
using LD = long double;
const LD kTwoOverSqrtPiL = 1.12837916709551257389615890312154517L;

LD p_exact(LD s) {  // erf(sqrt s)/sqrt s = (2/sqrt(pi)) sum (-s)^n / (n! (2n+1)), s <= 0.25
  LD term = kTwoOverSqrtPiL, sum = 0.0L;
  for (int n = 0; n < 40; ++n) {
    sum += term / (2 * n + 1);
    term *= -s / (n + 1);
  }
  return sum;
}
LD g_exact(LD s) { return kTwoOverSqrtPiL * std::exp(-s); }

// Interpolate f at n Chebyshev nodes of [0, a]; monomial coefficients in s.
bool cheb_fit(LD (*f)(LD), LD a, int n, double* out) {
  std::vector<LD> u(n), y(n), m(static_cast<std::size_t>(n) * n);
  const LD pi = 3.14159265358979323846264338327950288L;
  for (int i = 0; i < n; ++i) {
    u[i] = (std::cos((2 * i + 1) * pi / (2 * n)) + 1.0L) / 2.0L;  // nodes of [0, 1]
    y[i] = f(u[i] * a);
    LD p = 1.0L;
    for (int k = 0; k < n; ++k) {
      m[static_cast<std::size_t>(i) * n + k] = p;
      p *= u[i];
    }
  }
  // Gaussian elimination with partial pivoting (n <= 12)
  std::vector<LD> c = y;
  std::vector<LD> a2 = m;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::fabs(a2[static_cast<std::size_t>(r) * n + col]) >
          std::fabs(a2[static_cast<std::size_t>(piv) * n + col]))
        piv = r;
    if (a2[static_cast<std::size_t>(piv) * n + col] == 0.0L) return false;
    if (piv != col) {
      for (int k = 0; k < n; ++k)
        std::swap(a2[static_cast<std::size_t>(piv) * n + k], a2[static_cast<std::size_t>(col) * n + k]);
      std::swap(c[piv], c[col]);
    }
    for (int r = col + 1; r < n; ++r) {
      const LD f2 = a2[static_cast<std::size_t>(r) * n + col] / a2[static_cast<std::size_t>(col) * n + col];
      for (int k = col; k < n; ++k)
        a2[static_cast<std::size_t>(r) * n + k] -= f2 * a2[static_cast<std::size_t>(col) * n + k];
      c[r] -= f2 * c[col];
    }
  }
  for (int r = n - 1; r >= 0; --r) {
    for (int k = r + 1; k < n; ++k) c[r] -= a2[static_cast<std::size_t>(r) * n + k] * c[k];
    c[r] /= a2[static_cast<std::size_t>(r) * n + r];
  }
  LD scale = 1.0L;
  for (int k = 0; k < n; ++k) {
    out[k] = static_cast<double>(c[k] / scale);  // u = s / a
    scale *= a;
  }
  return true;
}

// max relative error of the double-coefficient polynomial on [0, a]
LD fit_error(LD (*f)(LD), const double* c, int n, LD a) {
  LD worst = 0.0L;
  for (int i = 0; i <= 2000; ++i) {
    const LD s = a * i / 2000;
    LD h = c[n - 1];
    for (int k = n - 2; k >= 0; --k) h = h * s + c[k];
    worst = std::max(worst, std::fabs((h - f(s)) / f(s)));
  }
  return worst;
}
}  // namespace

RadialFit fit_radial(double s_max) {
  RadialFit r{};
  if (s_max <= 0.25) {
    const LD a = std::max(static_cast<LD>(s_max), 1e-12L);
    for (int n : {6, 7, 8, 9, 10, 12}) {
      double p[14] = {}, g[14] = {};
      if (!cheb_fit(p_exact, a, n, p) || !cheb_fit(g_exact, a, n, g)) continue;
      const LD e = std::max(fit_error(p_exact, p, n, a), fit_error(g_exact, g, n, a));
      // 2.5e-14 relative on P and G: the radial factors' absolute error is
      // then < 1e-15 of b0 and g at every near distance (xi P and g are
      // ~1 % of 1/r there), 1e4 below the 1e-11 component parity gate --
      // one Horner term less per polynomial than fitting to 2e-16 (config 3:
      // 6 instead of 7 terms, 2 of ~100 FP64 instructions per pair)
      if (e <= 2.5e-14L) {
        r.nterms = n;
        r.s_lim = s_max;
        r.max_err = static_cast<double>(e);
        std::copy(p, p + 14, r.p);
        std::copy(g, g + 14, r.g);
        return r;
      }
    }
  }
  // Maclaurin, 14 terms (truncation < 1e-18 for s <= 0.25), libm beyond
  r.nterms = 14;
  r.s_lim = 0.25;
  LD tp = kTwoOverSqrtPiL, tg = kTwoOverSqrtPiL;
  for (int k = 0; k < 14; ++k) {
    r.p[k] = static_cast<double>(tp / (2 * k + 1));
    r.g[k] = static_cast<double>(tg);
    tp *= -1.0L / (k + 1);
    tg *= -1.0L / (k + 1);
  }
  r.max_err = static_cast<double>(
      std::max(fit_error(p_exact, r.p, 14, 0.25L), fit_error(g_exact, r.g, 14, 0.25L)));
  return r;
}

double erfc_screen(double z) {
  if (z >= 0.0 && z <= 0.5) {
    const double z2 = z * z;
    double term = z, sum = 0.0;
    for (int n = 0; n < 13; ++n) {
      sum += term / (2 * n + 1);
      term *= -z2 / (n + 1);
    }
    return 1.0 - kTwoOverSqrtPi * sum;
  }
  return std::erfc(z);
}

std::vector<double> cheb_nodes(int order) {
  std::vector<double> n(order);
  for (int k = 0; k < order; ++k) n[k] = std::cos((2.0 * k + 1.0) * kPi / (2.0 * order));
  return n;
}

std::vector<double> equi_nodes(int order) {
  std::vector<double> n(order);
  for (int k = 0; k < order; ++k) n[k] = -1.0 + 2.0 * k / (order - 1.0);
  return n;
}

double lagrange_cheb(int order, int k, double x) {
  std::vector<double> t(order), tr(order);
  cheb_values(order, x, t.data());
  cheb_values(order, cheb_nodes(order)[k], tr.data());
  double s = 1.0;
  for (int m = 1; m < order; ++m) s += 2.0 * tr[m] * t[m];
  return s / order;
}

double lagrange_equi(int order, int k, double x) {
  std::vector<double> w(order);
  double b = 1.0;
  for (int j = 0; j < order; ++j) {
    w[j] = (j % 2 == 0) ? b : -b;
    b = b * (order - 1 - j) / (j + 1);
  }
  const std::vector<double> nodes = equi_nodes(order);
  double denom = 0.0;
  for (int m = 0; m < order; ++m) {
    const double dx = x - nodes[m];
    if (dx == 0.0) return m == k ? 1.0 : 0.0;
    denom += w[m] / dx;
  }
  return (w[k] / (x - nodes[k])) / denom;
}

std::array<std::vector<double>, 3> diff_operator(int order) {
  const int L = order;
  const std::vector<double> nodes = cheb_nodes(L);
  std::vector<double> h(L * L), d(L * L, 0.0), t(L);
  for (int k = 0; k < L; ++k) {
    cheb_values(L, nodes[k], t.data());
    h[k * L] = 1.0 / L;
    for (int m = 1; m < L; ++m) h[k * L + m] = 2.0 * t[m] / L;
  }
  for (int m = 1; m < L; ++m)
    for (int j = m - 1; j >= 0; j -= 2) d[m * L + j] = (j == 0) ? m : 2.0 * m;
  auto mul = [L](const std::vector<double>& a, const std::vector<double>& b) {
    std::vector<double> c(L * L, 0.0);
    for (int i = 0; i < L; ++i)
      for (int k = 0; k < L; ++k)
        for (int j = 0; j < L; ++j) c[i * L + j] += a[i * L + k] * b[k * L + j];
    return c;
  };
  std::array<std::vector<double>, 3> hd;
  hd[0] = h;
  hd[1] = mul(h, d);
  hd[2] = mul(hd[1], d);
  return hd;
}

std::vector<double> diff_operator_hd3(int order) {
  const int L = order;
  const auto hd = diff_operator(L);
  std::vector<double> d(L * L, 0.0), out(L * L, 0.0);
  for (int m = 1; m < L; ++m)
    for (int j = m - 1; j >= 0; j -= 2) d[m * L + j] = (j == 0) ? m : 2.0 * m;
  for (int i = 0; i < L; ++i)
    for (int k = 0; k < L; ++k)
      for (int j = 0; j < L; ++j) out[i * L + j] += hd[2][i * L + k] * d[k * L + j];
  return out;
}

std::vector<double> transfer_cheb(int order, const std::vector<double>& src) {
  const int n = static_cast<int>(src.size());
  std::vector<double> t(order * n);
  for (int l = 0; l < n; ++l)
    for (int k = 0; k < order; ++k) t[k * n + l] = lagrange_cheb(order, k, src[l]);
  return t;
}

std::vector<double> transfer_equi(int order, const std::vector<double>& src) {
  const int n = static_cast<int>(src.size());
  std::vector<double> t(order * n);
  for (int l = 0; l < n; ++l)
    for (int k = 0; k < order; ++k) t[k * n + l] = lagrange_equi(order, k, src[l]);
  return t;
}

std::vector<double> m2l_dense(int order, double cell_radius, const std::array<int, 3>& offset,
                              double xi) {
  const int L = order;
  const int K = L * L * L;
  const std::vector<double> nodes = cheb_nodes(L);
  std::vector<double> d2[3];
  for (int ax = 0; ax < 3; ++ax) {
    d2[ax].resize(L * L);
    const double shift = 2.0 * cell_radius * offset[ax];
    for (int a = 0; a < L; ++a)
      for (int b = 0; b < L; ++b) {
        const double d = cell_radius * (nodes[a] - nodes[b]) - shift;
        d2[ax][a * L + b] = d * d;
      }
  }
  std::vector<double> c(static_cast<std::size_t>(K) * K);
  for (int i0 = 0; i0 < L; ++i0)
    for (int i1 = 0; i1 < L; ++i1)
      for (int i2 = 0; i2 < L; ++i2) {
        const int row = (i0 * L + i1) * L + i2;
        for (int j0 = 0; j0 < L; ++j0) {
          const double a = d2[0][i0 * L + j0];
          for (int j1 = 0; j1 < L; ++j1) {
            const double ab = a + d2[1][i1 * L + j1];
            const int col_base = (j0 * L + j1) * L;
            for (int j2 = 0; j2 < L; ++j2) {
              const double r = std::sqrt(ab + d2[2][i2 * L + j2]);
              c[static_cast<std::size_t>(row) * K + col_base + j2] = erfc_screen(xi * r) / r;
            }
          }
        }
      }
  return c;
}

// --------------------------------------------------------------------- SVD
namespace {

// One-sided Jacobi on a column-major m x n matrix w (m >= n).  On return the
// columns of w are U*sigma and v (n x n, column-major) holds V.
// skip_rel > 0: pairs of columns whose norms are both below skip_rel times
// the largest column norm are not rotated -- they only mix directions far
// below a truncation cutoff (their span, the kept columns and the rank
// decision are unaffected).
void jacobi_colmajor(std::vector<double>& w, int m, int n, std::vector<double>& v,
                     double skip_rel) {
  v.assign(static_cast<std::size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) v[static_cast<std::size_t>(i) * n + i] = 1.0;
  const double eps = 2.220446049250313e-16;
  std::vector<double> norms(n);
  for (int j = 0; j < n; ++j) {
    const double* wj = w.data() + static_cast<std::size_t>(j) * m;
    double acc = 0.0;
    for (int i = 0; i < m; ++i) acc += wj[i] * wj[i];
    norms[j] = acc;
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    bool rotated = false;
    double skip2 = 0.0;  // squared norms
    if (skip_rel > 0.0) {
      double mx = 0.0;
      for (int j = 0; j < n; ++j) mx = std::max(mx, norms[j]);
      skip2 = mx * skip_rel * skip_rel;
    }
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        if (norms[p] < skip2 && norms[q] < skip2) continue;
        double* wp = w.data() + static_cast<std::size_t>(p) * m;
        double* wq = w.data() + static_cast<std::size_t>(q) * m;
        double gamma = 0.0;
        for (int i = 0; i < m; ++i) gamma += wp[i] * wq[i];
        const double alpha = norms[p], beta = norms[q];
        if (gamma == 0.0 || std::abs(gamma) <= eps * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        double np = 0.0, nq = 0.0;
        for (int i = 0; i < m; ++i) {
          const double x = wp[i], y = wq[i];
          const double a = cs * x - sn * y, b = sn * x + cs * y;
          wp[i] = a;
          wq[i] = b;
          np += a * a;
          nq += b * b;
        }
        norms[p] = np;
        norms[q] = nq;
        double* vp = v.data() + static_cast<std::size_t>(p) * n;
        double* vq = v.data() + static_cast<std::size_t>(q) * n;
        for (int i = 0; i < n; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
      }
    }
    if (!rotated) break;
  }
}

}  // namespace

void svd_thin(const std::vector<double>& a, int m, int n, std::vector<double>& u,
              std::vector<double>& sigma, std::vector<double>& v, double skip_rel) {
  const bool tall = m >= n;
  const int mm = tall ? m : n, nn = tall ? n : m;
  // column-major working copy of (tall ? a : a^T)
  std::vector<double> w(static_cast<std::size_t>(mm) * nn);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      const double x = a[static_cast<std::size_t>(i) * n + j];
      if (tall)
        w[static_cast<std::size_t>(j) * mm + i] = x;
      else
        w[static_cast<std::size_t>(i) * mm + j] = x;
    }
  std::vector<double> vv;
  jacobi_colmajor(w, mm, nn, vv, skip_rel);
  std::vector<double> sig(nn);
  for (int j = 0; j < nn; ++j) {
    const double* wj = w.data() + static_cast<std::size_t>(j) * mm;
    double acc = 0.0;
    for (int i = 0; i < mm; ++i) acc += wj[i] * wj[i];
    sig[j] = std::sqrt(acc);
  }
  std::vector<int> order(nn);
  for (int j = 0; j < nn; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sig[x] > sig[y]; });
  // left vectors of the working matrix: mm x nn ; right: nn x nn (row-major out)
  std::vector<double> uw(static_cast<std::size_t>(mm) * nn), vw(static_cast<std::size_t>(nn) * nn);
  sigma.assign(nn, 0.0);
  for (int jj = 0; jj < nn; ++jj) {
    const int j = order[jj];
    const double s = sig[j];
    sigma[jj] = s;
    for (int i = 0; i < mm; ++i)
      uw[static_cast<std::size_t>(i) * nn + jj] = s > 0.0 ? w[static_cast<std::size_t>(j) * mm + i] / s : 0.0;
    for (int i = 0; i < nn; ++i) vw[static_cast<std::size_t>(i) * nn + jj] = vv[static_cast<std::size_t>(j) * nn + i];
  }
  if (tall) {
    u.swap(uw);
    v.swap(vw);
  } else {
    u.swap(vw);
    v.swap(uw);
  }
}

namespace {

// Thin Q (m x q, row-major) of a full-column-rank m x q matrix y (row-major),
// by Householder reflections.
std::vector<double> householder_thin_q(const std::vector<double>& y, int m, int q) {
  std::vector<double> a(static_cast<std::size_t>(m) * q);  // column-major copy
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < q; ++j) a[static_cast<std::size_t>(j) * m + i] = y[static_cast<std::size_t>(i) * q + j];
  std::vector<double> tau(q, 0.0);
  for (int k = 0; k < q && k < m; ++k) {
    double* col = a.data() + static_cast<std::size_t>(k) * m;
    double norm2 = 0.0;
    for (int i = k; i < m; ++i) norm2 += col[i] * col[i];
    const double norm = std::sqrt(norm2);
    if (norm == 0.0) continue;
    const double alpha = col[k] >= 0.0 ? -norm : norm;
    col[k] -= alpha;
    double vn2 = 0.0;
    for (int i = k; i < m; ++i) vn2 += col[i] * col[i];
    if (vn2 == 0.0) continue;
    tau[k] = 2.0 / vn2;
    for (int j = k + 1; j < q; ++j) {
      double* cj = a.data() + static_cast<std::size_t>(j) * m;
      double s = 0.0;
      for (int i = k; i < m; ++i) s += col[i] * cj[i];
      s *= tau[k];
      for (int i = k; i < m; ++i) cj[i] -= s * col[i];
    }
  }
  // Q = H_0 ... H_{q-1} [I_q; 0]  (column-major m x q)
  std::vector<double> qm(static_cast<std::size_t>(m) * q, 0.0);
  for (int j = 0; j < q; ++j) qm[static_cast<std::size_t>(j) * m + j] = 1.0;
  for (int k = std::min(q, m) - 1; k >= 0; --k) {
    if (tau[k] == 0.0) continue;
    const double* v = a.data() + static_cast<std::size_t>(k) * m;
    for (int j = 0; j < q; ++j) {
      double* xj = qm.data() + static_cast<std::size_t>(j) * m;
      double s = 0.0;
      for (int i = k; i < m; ++i) s += v[i] * xj[i];
      s *= tau[k];
      for (int i = k; i < m; ++i) xj[i] -= s * v[i];
    }
  }
  std::vector<double> out(static_cast<std::size_t>(m) * q);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < q; ++j) out[static_cast<std::size_t>(i) * q + j] = qm[static_cast<std::size_t>(j) * m + i];
  return out;
}

// gaussian_matrix (fmm.cpp:25-36): column-major fill, Box-Muller with the
// log-argument draw first (the order GCC emits for the unsequenced pair).
std::vector<double> gaussian_rowmajor(int rows, int cols, std::uint64_t seed) {
  std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ULL);
  auto unit = [&rng]() { return ((rng() >> 11) + 0.5) * (1.0 / 9007199254740992.0); };
  constexpr double two_pi = 6.283185307179586477;
  std::vector<double> m(static_cast<std::size_t>(rows) * cols);
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < rows; ++i) {
      const double u1 = unit();
      const double u2 = unit();
      m[static_cast<std::size_t>(i) * cols + j] = std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
    }
  return m;
}

// c (m x k) = a (m x n) * b (n x k), row-major.  Every c_ij accumulates its
// n products in increasing l, one multiply-add at a time (the arithmetic of
// the plain triple loop, bit for bit); the loops are blocked so a (l, j)
// block of b stays cache-resident across all rows of a, and four rows of c
// share each load of b.
std::vector<double> matmul(const std::vector<double>& a, const std::vector<double>& b, int m, int n,
                           int k) {
  std::vector<double> c(static_cast<std::size_t>(m) * k, 0.0);
  constexpr int JB = 256, LB = 128;
  for (int j0 = 0; j0 < k; j0 += JB) {
    const int jn = std::min(JB, k - j0);
    for (int l0 = 0; l0 < n; l0 += LB) {
      const int l1 = std::min(n, l0 + LB);
      int i = 0;
      for (; i + 4 <= m; i += 4) {
        double* __restrict__ c0 = c.data() + static_cast<std::size_t>(i) * k + j0;
        double* __restrict__ c1 = c0 + k;
        double* __restrict__ c2 = c1 + k;
        double* __restrict__ c3 = c2 + k;
        const double* a0 = a.data() + static_cast<std::size_t>(i) * n;
        for (int l = l0; l < l1; ++l) {
          const double x0 = a0[l], x1 = a0[n + l], x2 = a0[2 * static_cast<std::size_t>(n) + l],
                       x3 = a0[3 * static_cast<std::size_t>(n) + l];
          const double* __restrict__ bl = b.data() + static_cast<std::size_t>(l) * k + j0;
          for (int j = 0; j < jn; ++j) {
            const double bv = bl[j];
            c0[j] += x0 * bv;
            c1[j] += x1 * bv;
            c2[j] += x2 * bv;
            c3[j] += x3 * bv;
          }
        }
      }
      for (; i < m; ++i) {
        double* __restrict__ ci = c.data() + static_cast<std::size_t>(i) * k + j0;
        for (int l = l0; l < l1; ++l) {
          const double x = a[static_cast<std::size_t>(i) * n + l];
          const double* __restrict__ bl = b.data() + static_cast<std::size_t>(l) * k + j0;
          for (int j = 0; j < jn; ++j) ci[j] += x * bl[j];
        }
      }
    }
  }
  return c;
}

void finish(Factors& f, const std::vector<double>& u, int ucols, const std::vector<double>& sv,
            const std::vector<double>& v, int vcols, int k_full, double svd_tol) {
  int rank = 1;
  while (rank < static_cast<int>(sv.size()) && sv[rank] > sv[0] * svd_tol) ++rank;
  f.rank = rank;
  f.k_full = k_full;
  f.lmat.assign(static_cast<std::size_t>(rank) * k_full, 0.0);
  f.rmat.assign(static_cast<std::size_t>(rank) * k_full, 0.0);
  for (int r = 0; r < rank; ++r)
    for (int j = 0; j < k_full; ++j) {
      f.lmat[static_cast<std::size_t>(r) * k_full + j] = u[static_cast<std::size_t>(j) * ucols + r] * sv[r];
      f.rmat[static_cast<std::size_t>(r) * k_full + j] = v[static_cast<std::size_t>(j) * vcols + r];
    }
}

}  // namespace

Factors compress_m2l(const std::vector<double>& c, int k_full, double svd_tol, std::uint64_t seed) {
  Factors f;
  if (k_full <= 150) {
    std::vector<double> u, s, v;
    // rank = 1 + #{sigma_i > sigma_0 tol}: directions 1e-3 below the cutoff
    // need not be resolved among themselves
    svd_thin(c, k_full, k_full, u, s, v, svd_tol * 1e-3);
    finish(f, u, k_full, s, v, k_full, k_full, svd_tol);
    return f;
  }
  int q = 48;
  while (true) {
    q = std::min(q, k_full);
    const std::vector<double> omega = gaussian_rowmajor(k_full, q, seed);
    const std::vector<double> y = matmul(c, omega, k_full, k_full, q);
    const std::vector<double> qmat = householder_thin_q(y, k_full, q);  // K x q
    // b = Q^T C (q x K)
    std::vector<double> qt(static_cast<std::size_t>(q) * k_full);
    for (int i = 0; i < k_full; ++i)
      for (int j = 0; j < q; ++j) qt[static_cast<std::size_t>(j) * k_full + i] = qmat[static_cast<std::size_t>(i) * q + j];
    const std::vector<double> b = matmul(qt, c, q, k_full, k_full);
    std::vector<double> ub, s, vb;
    svd_thin(b, q, k_full, ub, s, vb);  // ub q x q, vb K x q
    if (q == k_full || s[q - 1] <= s[0] * svd_tol * 1e-2) {
      const std::vector<double> u = matmul(qmat, ub, k_full, q, q);  // K x q
      finish(f, u, q, s, vb, q, k_full, svd_tol);
      return f;
    }
    q *= 2;
  }
}

Symmetry symmetry_of(const std::array<int, 3>& o) {
  Symmetry s;
  std::array<int, 3> axes{0, 1, 2};
  std::stable_sort(axes.begin(), axes.end(),
                   [&](int a, int b) { return std::abs(o[a]) > std::abs(o[b]); });
  for (int j = 0; j < 3; ++j) {
    s.rep[j] = std::abs(o[axes[j]]);
    s.perm[axes[j]] = j;
  }
  for (int a = 0; a < 3; ++a) s.sign[a] = o[a] < 0 ? -1 : 1;
  return s;
}

std::vector<int> node_permutation(const Symmetry& s, int L) {
  std::vector<int> p(static_cast<std::size_t>(L) * L * L);
  for (int k0 = 0; k0 < L; ++k0)
    for (int k1 = 0; k1 < L; ++k1)
      for (int k2 = 0; k2 < L; ++k2) {
        const int k[3] = {k0, k1, k2};
        int pk[3];
        for (int a = 0; a < 3; ++a) {
          const int src = k[s.perm[a]];
          pk[a] = s.sign[a] > 0 ? src : L - 1 - src;
        }
        p[(k0 * L + k1) * L + k2] = (pk[0] * L + pk[1]) * L + pk[2];
      }
  return p;
}

std::vector<double> r2c_3d(const std::vector<double>& a, int d0, int d1, int d2) {
  const int h2 = d2 / 2 + 1;
  const double two_pi = 6.283185307179586476925286766559;
  auto twiddles = [&](int n) {
    std::vector<double> c(n), s(n);
    for (int k = 0; k < n; ++k) {
      const double ang = -two_pi * k / n;
      c[k] = std::cos(ang);
      s[k] = std::sin(ang);
    }
    return std::make_pair(c, s);
  };
  // axis 2 (real -> half complex)
  std::vector<double> re(static_cast<std::size_t>(d0) * d1 * h2), im(re.size());
  {
    auto [c, s] = twiddles(d2);
    for (int i = 0; i < d0 * d1; ++i)
      for (int k = 0; k < h2; ++k) {
        double sr = 0.0, si = 0.0;
        for (int j = 0; j < d2; ++j) {
          const int ph = static_cast<int>((static_cast<long long>(j) * k) % d2);
          const double x = a[static_cast<std::size_t>(i) * d2 + j];
          sr += x * c[ph];
          si += x * s[ph];
        }
        re[static_cast<std::size_t>(i) * h2 + k] = sr;
        im[static_cast<std::size_t>(i) * h2 + k] = si;
      }
  }
  auto axis = [&](int n, std::size_t stride, std::size_t outer_stride, int outer, int inner) {
    auto [c, s] = twiddles(n);
    std::vector<double> lr(n), li(n);
    for (int o = 0; o < outer; ++o)
      for (int in = 0; in < inner; ++in) {
        const std::size_t base = static_cast<std::size_t>(o) * outer_stride + in;
        for (int j = 0; j < n; ++j) {
          lr[j] = re[base + j * stride];
          li[j] = im[base + j * stride];
        }
        for (int k = 0; k < n; ++k) {
          double sr = 0.0, si = 0.0;
          for (int j = 0; j < n; ++j) {
            const int ph = static_cast<int>((static_cast<long long>(j) * k) % n);
            sr += lr[j] * c[ph] - li[j] * s[ph];
            si += lr[j] * s[ph] + li[j] * c[ph];
          }
          re[base + k * stride] = sr;
          im[base + k * stride] = si;
        }
      }
  };
  axis(d1, h2, static_cast<std::size_t>(d1) * h2, d0, h2);                 // axis 1
  axis(d0, static_cast<std::size_t>(d1) * h2, 0, 1, d1 * h2);             // axis 0
  std::vector<double> out(2 * re.size());
  for (std::size_t i = 0; i < re.size(); ++i) {
    out[2 * i] = re[i];
    out[2 * i + 1] = im[i];
  }
  return out;
}

void parallel_for(int n, int threads, const std::function<void(int)>& fn) {
  if (n <= 0) return;
  if (threads <= 0) {
    const unsigned hw = std::thread::hardware_concurrency();
    threads = hw > 0 ? static_cast<int>(hw) : 1;
  }
  threads = std::min(threads, n);
  if (threads <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> pool;
  std::atomic<int> next{0};
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) fn(i);
    });
  for (auto& t : pool) t.join();
}

}  // namespace ankh_b200
