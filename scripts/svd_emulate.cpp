// CPU emulation of k_jacobi_svd (16 lane-partial fma dots, butterfly sums,
// round-robin order): Jacobi sweeps per symmetry class at config 3 under the
// host skip rule (both columns small) and the GPU rule (either column small).
//   g++ -O2 -std=c++17 -Ipaper_2212_08284_b200/csrc scripts/svd_emulate.cpp \
//       paper_2212_08284_b200/csrc/host_numerics.cpp -o /tmp/svd_emulate -lpthread
#include <cmath>
#include <cstdio>
#include <vector>
#include <array>
#include <map>
#include "host_numerics.hpp"
using namespace ankh_b200;
static double wsum(double* v) {  // butterfly over a half-warp (xor), as half_sum
  for (int o = 8; o > 0; o >>= 1) { double t[16]; for (int l = 0; l < 16; ++l) t[l] = v[l] + v[l ^ o]; for (int l = 0; l < 16; ++l) v[l] = t[l]; }
  return v[0];
}
int run(const std::vector<double>& c, int K, double skip_rel, double tolmul, bool either) {
  std::vector<double> w(K * K), nrm(K);
  for (int i = 0; i < K; ++i) for (int j = 0; j < K; ++j) w[j * K + i] = c[i * K + j];
  for (int j = 0; j < K; ++j) { double p[32] = {}; for (int i = 0; i < K; ++i) p[i & 15] = std::fma(w[j*K+i], w[j*K+i], p[i & 15]); nrm[j] = wsum(p); }
  const double eps = 2.220446049250313e-16 * tolmul;
  const int np = K + (K & 1);
  int sweep = 0;
  for (; sweep < 100; ++sweep) {
    double mx = 0; for (double x : nrm) mx = std::fmax(mx, x);
    double sk2 = mx * skip_rel * skip_rel;
    int rot = 0;
    for (int step = 0; step < np - 1; ++step)
      for (int pi = 0; pi < np / 2; ++pi) {
        int p, q;
        if (pi == 0) { p = step; q = np - 1; } else { p = (step + pi) % (np - 1); q = (step - pi + np - 1) % (np - 1); }
        if (p > q) std::swap(p, q);
        if (q >= K) continue;
        double a = nrm[p], b = nrm[q];
        if (either ? (std::fmin(a, b) < sk2) : (a < sk2 && b < sk2)) continue;
        double* wp = &w[p * K]; double* wq = &w[q * K];
        double g[32] = {}; for (int i = 0; i < K; ++i) g[i & 15] = std::fma(wp[i], wq[i], g[i & 15]);
        double gg = wsum(g);
        if (gg == 0.0 || std::fabs(gg) <= eps * std::sqrt(a * b)) continue;
        double z = (b - a) / (2 * gg), t = (z >= 0 ? 1.0 : -1.0) / (std::fabs(z) + std::sqrt(1 + z * z));
        double cs = 1 / std::sqrt(1 + t * t), sn = cs * t;
        double pa[32] = {}, pb[32] = {};
        for (int i = 0; i < K; ++i) { double x = wp[i], y = wq[i]; double u = cs * x - sn * y, v = sn * x + cs * y; wp[i] = u; wq[i] = v; pa[i & 15] = std::fma(u, u, pa[i & 15]); pb[i & 15] = std::fma(v, v, pb[i & 15]); }
        nrm[p] = wsum(pa); nrm[q] = wsum(pb); ++rot;
      }
    if (!rot) break;
  }
  return sweep;
}
int main() {
  const int L = 5, K = 125; const double rb = 108.8;
  int worst = 0;
  std::map<int,int> hist;
  for (int level = 1; level <= 5; ++level)
    for (int a = 2; a <= 3; ++a) for (int b = 0; b <= a; ++b) for (int cc = 0; cc <= b; ++cc) {
      auto c = m2l_dense(L, rb / (1 << level), {a, b, cc}, 0.01);
      int s1 = run(c, K, 1e-10, 1.0, false), s2 = run(c, K, 1e-10, std::sqrt(125.0), true), s3 = run(c, K, 1e-13, std::sqrt(125.0), true);
      std::printf("level %d rep (%d,%d,%d): sweeps host-rule %d  either@1e-10 %d  either@1e-13 %d\n", level, a, b, cc, s1, s2, s3);
    }
}
