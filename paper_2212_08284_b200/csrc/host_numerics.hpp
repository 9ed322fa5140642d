// Host-side, geometry-only precompute of the B200 plan.  These run once per
// plan (they depend on box radius, order, depth, xi, p, svd_tol -- never on the
// particles) and their results are uploaded to HBM.  Each routine names the
// reference lines whose numerics it reproduces (paths relative to
// /root/reference/proj/core).
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <vector>

namespace ankh_b200 {

/// P2P radial polynomials in s = xi^2 r^2 on [0, s_max] (s_max from the
/// plan's largest near distance): P(s) = erf(sqrt s) / sqrt s and
/// G(s) = (2/sqrt(pi)) exp(-s), so that erfc(xi r) / r = 1/r - xi P(s) and
/// the Gaussian factor of radial (kernel.cpp:26-38) is xi G(s).  Fitted in
/// long double at Chebyshev nodes with the fewest terms (from 6..10, 12) whose
/// double coefficients stay within 2e-16 relative error of both functions on
/// a dense grid -- the accuracy of the reference's own series, with fewer
/// terms than a Maclaurin polynomial.  Beyond s_max = 0.25 (huge leaves):
/// 14-term Maclaurin up to s = 0.25 and libm erfc / exp past it (nterms 14).
struct RadialFit {
  int nterms;
  double s_lim;     // polynomial valid for s <= s_lim
  double max_err;   // measured max relative error of the fit on [0, s_lim]
  double p[14], g[14];
};
RadialFit fit_radial(double s_max);

/// kernel.cpp:14-23, 48-51: 13-term Maclaurin erf for 0 <= z <= 0.5, else erfc.
double erfc_screen(double z);

/// Grid1D::chebyshev (chebyshev.cpp:48-58) and ::equispaced (60-70).
std::vector<double> cheb_nodes(int order);
std::vector<double> equi_nodes(int order);

/// Cardinal Lagrange basis S_k(x) of the Chebyshev grid (chebyshev.cpp:72-83)
/// and of the equispaced grid (barycentric, chebyshev.cpp:19-44).
double lagrange_cheb(int order, int k, double x);
double lagrange_equi(int order, int k, double x);

/// DiffOperator (chebyshev.cpp:85-108): hd[n] = H D^n, n = 0..2, row-major L x L.
std::array<std::vector<double>, 3> diff_operator(int order);
/// H D^3 (L x L, row-major): the next basis derivative, for the forces' L2P.
std::vector<double> diff_operator_hd3(int order);

/// transfer_1d (chebyshev.cpp:236-244): T(k, l) = S_k^{dst}(src[l]), row-major.
std::vector<double> transfer_cheb(int order, const std::vector<double>& src_local);
std::vector<double> transfer_equi(int order, const std::vector<double>& src_local);

/// m2l_dense (fmm.cpp:60-96), row-major K x K, same operation order.
std::vector<double> m2l_dense(int order, double cell_radius, const std::array<int, 3>& offset,
                              double xi);

/// Truncated factors C ~= L^T R (fmm.cpp:98-133): L = (U_k S_k)^T, R = V_k^T,
/// k x K row-major; exact SVD for K <= 150, else the reference's seeded
/// randomized range finder (same Gaussian sketch, same stopping rule).
struct Factors {
  int rank = 0;
  int k_full = 0;
  std::vector<double> lmat, rmat;
};
Factors compress_m2l(const std::vector<double>& c, int k_full, double svd_tol, std::uint64_t seed);

/// fmm.hpp:42-44 and fmm.cpp:167-169.
inline std::int64_t offset_key(const std::array<int, 3>& o) {
  return (static_cast<std::int64_t>(o[0]) * 4096 + o[1]) * 4096 + o[2];
}
inline std::uint64_t m2l_seed(int level, std::int64_t key) {
  return static_cast<std::uint64_t>(level) * 0x100000001b3ULL + static_cast<std::uint64_t>(key);
}

/// Signed-permutation symmetry of the M2L block: offset o = g(rep) with
/// o_a = s_a * rep_{perm[a]}; then C_o(P k, P l) = C_rep(k, l) where
/// P(k)_a = k_{perm[a]} (s_a > 0) or L-1-k_{perm[a]} (s_a < 0).
struct Symmetry {
  std::array<int, 3> rep{};   // |o| sorted descending
  std::array<int, 3> perm{};
  std::array<int, 3> sign{};
};
Symmetry symmetry_of(const std::array<int, 3>& offset);
/// node index map P for the given symmetry: out[k] = P(k), k lex (i L + j) L + l.
std::vector<int> node_permutation(const Symmetry& s, int order);

/// One-sided Jacobi thin SVD of a (m x n, row-major).  U m x p, V n x p
/// (row-major), sigma descending, p = min(m, n).  skip_rel > 0: directions
/// with singular values below skip_rel * sigma_0 are not resolved among
/// themselves (for truncations at a much larger cutoff).
void svd_thin(const std::vector<double>& a, int m, int n, std::vector<double>& u,
              std::vector<double>& sigma, std::vector<double>& v, double skip_rel = 0.0);

/// Real-to-complex DFT of a row-major real array of dims d0 x d1 x d2 in the
/// FFTW half-complex layout (d2/2+1 on the last axis), unnormalised.  Returns
/// interleaved (re, im).
std::vector<double> r2c_3d(const std::vector<double>& a, int d0, int d1, int d2);

/// Run fn(i) for i in [0, n) on up to `threads` host threads (static chunks).
void parallel_for(int n, int threads, const std::function<void(int)>& fn);

}  // namespace ankh_b200
