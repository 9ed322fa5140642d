// Runtime-order P2M and M2M for interpolation orders past the compiled
// kernels (L = 11 .. 64; the reference accepts order_cheb <= 64,
// chebyshev.cpp:86).  Same arithmetic as k_p2m_m2m.cu, with L a kernel
// argument and the per-leaf / per-parent working sets in shared memory while
// they fit (else in a global scratch slice per CTA):
//
// P2M (modified_charges, chebyshev.cpp:138-203; leaf_expansions,
// fmm.cpp:181-201): one CTA per leaf; per batch of PB particles the 1-D
// Chebyshev values, the bases S^(n) = radius^-n (H D^n) T and the
// moment-folded z factors are staged, then every thread owns output nodes
// (i, j, k) and accumulates
//   Q[i,j,k] += sum_p x0[i] w0[jk] + x1[i] w1[jk] + x2[i] w2[jk]
//   w0 = y0 A0 + y1 A1 + y2 A2,  w1 = y0 B0 + y1 B1,  w2 = y0 C0
// (the 10 terms regrouped by derivative order, as k_p2m_w).
//
// M2M (upward_pass, fmm.cpp:203-236; tensor3_apply, chebyshev.cpp:246-272):
// one CTA per parent (grid-stride), the 8 children applied axis by axis
// (z, y, x) into a parent accumulator.
#include "kernels.cuh"

namespace ankh_b200 {

namespace {

constexpr int kGenThreads = 256;

__device__ __forceinline__ double self_term_g(const double* r, double c_mu, double c_th) {
  // kernel.cpp:208-209 (record layout: x y z q mx my mz txx txy txz tyy tyz tzz tr)
  const double mu2 = fma(r[4], r[4], fma(r[5], r[5], r[6] * r[6]));
  const double th2 = fma(r[7], r[7], fma(r[10], r[10], r[12] * r[12])) +
                     2.0 * fma(r[8], r[8], fma(r[9], r[9], r[11] * r[11]));
  return fma(c_th, th2, fma(c_mu, mu2, r[3] * r[3]));
}

// smem per batch particle: record (14) + T (3L) + X (3L) + Y (3L) + raw z (3L) + Z (6L)
__host__ __device__ inline int p2m_gen_per(int L) { return 14 + 18 * L; }

__global__ void __launch_bounds__(kGenThreads) k_p2m_gen(const double* __restrict__ part,
                                                         const unsigned* __restrict__ leaf_off, int depth,
                                                         double rb, const double* __restrict__ hd,
                                                         double* __restrict__ exp_leaf, unsigned m_begin,
                                                         double* __restrict__ self_leaf, double c_mu,
                                                         double c_th, int L, int PB) {
  extern __shared__ __align__(16) double sm[];
  const int L2 = L * L, K = L2 * L, KS = exp_stride(K);
  double* rec = sm;               // PB x 14
  double* T = rec + PB * kRec;    // PB x 3 axes x L
  double* X = T + PB * 3 * L;     // PB x 3 orders x L
  double* Y = X + PB * 3 * L;     // PB x 3 orders x L
  double* Zr = Y + PB * 3 * L;    // PB x 3 orders x L (before the moment fold)
  double* Z = Zr + PB * 3 * L;    // PB x 6 x L: A0 A1 A2 B0 B1 C0
  __shared__ double s_self[kGenThreads];
  const int tid = threadIdx.x;
  const int n = 1 << depth;
  const unsigned m = m_begin + blockIdx.x;  // Morton leaf
  const int ci[3] = {static_cast<int>(morton_compact3(m >> 2)), static_cast<int>(morton_compact3(m >> 1)),
                     static_cast<int>(morton_compact3(m))};
  const unsigned leaf = (static_cast<unsigned>(ci[0]) * n + ci[1]) * n + ci[2];
  const unsigned begin = leaf_off[leaf];
  const int cnt = static_cast<int>(leaf_off[leaf + 1] - begin);
  ANKH_DASSERT(leaf_off[leaf + 1] >= begin && PB >= 1 && PB <= kGenThreads);
  double* out = exp_leaf + static_cast<std::size_t>(m) * KS;
  if (cnt == 0) {  // fmm.cpp:190-193
    for (int o = tid; o < K; o += kGenThreads) out[o] = 0.0;
    if (tid == 0) self_leaf[m] = 0.0;
    return;
  }
  // cell_geometry (octree.cpp:18-25)
  const double rad = rb / n, inv_rad = 1.0 / rad;
  double self_acc = 0.0;
  for (int p0 = 0; p0 < cnt; p0 += PB) {
    const int pb = min(PB, cnt - p0);
    __syncthreads();
    for (int w = tid; w < pb * 7; w += kGenThreads) {
      const int p = w / 7, c = w - 7 * (w / 7);
      const double2 v = __ldg(reinterpret_cast<const double2*>(part + static_cast<std::size_t>(begin + p0 + p) * kRec) + c);
      rec[p * kRec + 2 * c] = v.x;
      rec[p * kRec + 2 * c + 1] = v.y;
    }
    __syncthreads();
    if (tid < pb) self_acc += self_term_g(rec + tid * kRec, c_mu, c_th);
    // Chebyshev values T_m(local) per (particle, axis)
    for (int w = tid; w < pb * 3; w += kGenThreads) {
      const int p = w / 3, ax = w - 3 * (w / 3);
      const double center = -rb + rad * (2 * ci[ax] + 1);
      const double local = (rec[p * kRec + ax] - center) * inv_rad;
      double* t = T + (p * 3 + ax) * L;
      double a = 1.0, b = local;
      t[0] = a;
      if (L > 1) t[1] = b;
      for (int q = 2; q < L; ++q) {
        const double c = 2.0 * local * b - a;
        t[q] = c;
        a = b;
        b = c;
      }
    }
    __syncthreads();
    // bases S^(nd)[i] = radius^-nd sum_q (H D^nd)[i][q] T_q per (particle, axis, nd, i)
    for (int w = tid; w < pb * 9 * L; w += kGenThreads) {
      const int i = w % L, r = w / L, nd = r % 3, r2 = r / 3, ax = r2 % 3, p = r2 / 3;
      const double* h = hd + nd * L2 + i * L;
      const double* t = T + (p * 3 + ax) * L;
      double v = 0.0;
      for (int q = 0; q < L; ++q) v += h[q] * t[q];
      const double scale = nd == 0 ? 1.0 : (nd == 1 ? inv_rad : inv_rad * inv_rad);
      double* dst = ax == 0 ? X : (ax == 1 ? Y : Zr);
      dst[(p * 3 + nd) * L + i] = scale * v;
    }
    __syncthreads();
    // moments folded into the z factors
    for (int w = tid; w < pb * L; w += kGenThreads) {
      const int p = w / L, k = w - L * (w / L);
      const double* r = rec + p * kRec;
      const double z0 = Zr[(p * 3) * L + k], z1 = Zr[(p * 3 + 1) * L + k], z2 = Zr[(p * 3 + 2) * L + k];
      double* zf = Z + p * 6 * L + k;
      zf[0] = r[3] * z0 + r[6] * z1 + r[12] * z2;  // A0 = q z0 + mu_z z1 + Th_zz z2
      zf[L] = r[5] * z0 + (2.0 * r[11]) * z1;      // A1 = mu_y z0 + 2 Th_yz z1
      zf[2 * L] = r[10] * z0;                      // A2 = Th_yy z0
      zf[3 * L] = r[4] * z0 + (2.0 * r[9]) * z1;   // B0 = mu_x z0 + 2 Th_xz z1
      zf[4 * L] = (2.0 * r[8]) * z0;               // B1 = 2 Th_xy z0
      zf[5 * L] = r[7] * z0;                       // C0 = Th_xx z0
    }
    __syncthreads();
    for (int o = tid; o < K; o += kGenThreads) {
      const int i = o / L2, jk = o - L2 * (o / L2), j = jk / L, k = jk - L * (jk / L);
      double a = p0 == 0 ? 0.0 : out[o];
      for (int p = 0; p < pb; ++p) {
        const double* x = X + p * 3 * L + i;
        const double* y = Y + p * 3 * L + j;
        const double* z = Z + p * 6 * L + k;
        const double y0 = y[0], y1 = y[L], y2 = y[2 * L];
        const double w0 = fma(y0, z[0], fma(y1, z[L], y2 * z[2 * L]));
        const double w1 = fma(y0, z[3 * L], y1 * z[4 * L]);
        const double w2 = y0 * z[5 * L];
        a = fma(x[0], w0, fma(x[L], w1, fma(x[2 * L], w2, a)));
      }
      out[o] = a;
    }
  }
  // the leaf's self-energy sum, fixed order
  s_self[tid] = self_acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int k = 0; k < min(PB, kGenThreads); ++k) t += s_self[k];
    self_leaf[m] = t;
  }
}

// Parents [p_begin, p_begin + p_count) of one level, grid-stride; M[c][i][a]
// = T_c(i, a) the two 1-D transfer matrices (global, L1-resident).  buf: 3K
// doubles per CTA (shared memory, or gbuf + 3K blockIdx.x).
__global__ void __launch_bounds__(kGenThreads) k_m2m_gen(const double* __restrict__ child,
                                                         double* __restrict__ parent,
                                                         const double* __restrict__ M, int L,
                                                         unsigned p_begin, unsigned p_count,
                                                         double* __restrict__ gbuf) {
  extern __shared__ __align__(16) double sm[];
  const int L2 = L * L, K = L2 * L, KS = exp_stride(K);
  double* S1 = gbuf ? gbuf + static_cast<std::size_t>(blockIdx.x) * 3 * K : sm;
  double* S2 = S1 + K;
  double* A = S2 + K;
  for (unsigned pi = blockIdx.x; pi < p_count; pi += gridDim.x) {
    const unsigned p = p_begin + pi;
    ANKH_DASSERT(gbuf || 3 * K * sizeof(double) <= 200 * 1024);
    for (int c = 0; c < 8; ++c) {  // Morton children 8p + (cx<<2 | cy<<1 | cz)
      const int cx = c >> 2, cy = (c >> 1) & 1, cz = c & 1;
      const double* v = child + (8ull * p + c) * KS;
      __syncthreads();
      for (int e = threadIdx.x; e < K; e += kGenThreads) {  // z
        const int ab = e / L, k = e - L * (e / L);
        const double* m = M + cz * L2 + k * L;
        const double* x = v + ab * L;
        double acc = 0.0;
        for (int q = 0; q < L; ++q) acc += m[q] * x[q];
        S1[e] = acc;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < K; e += kGenThreads) {  // y
        const int a = e / L2, jk = e - L2 * (e / L2), j = jk / L, k = jk - L * (jk / L);
        const double* m = M + cy * L2 + j * L;
        const double* s = S1 + a * L2 + k;
        double acc = 0.0;
        for (int b = 0; b < L; ++b) acc += m[b] * s[b * L];
        S2[e] = acc;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < K; e += kGenThreads) {  // x, summed over the children
        const int i = e / L2, jk = e - L2 * (e / L2);
        const double* m = M + cx * L2 + i * L;
        const double* s = S2 + jk;
        double acc = 0.0;
        for (int a = 0; a < L; ++a) acc += m[a] * s[a * L2];
        A[e] = c == 0 ? acc : A[e] + acc;
      }
    }
    __syncthreads();
    double* out = parent + static_cast<std::size_t>(p) * KS;
    for (int e = threadIdx.x; e < K; e += kGenThreads) out[e] = A[e];
  }
}

constexpr std::size_t kGenSmemMax = 200 * 1024;

}  // namespace

void launch_p2m_generic(const double* part, const unsigned* leaf_off, int depth, int order, double box_radius,
                        const double* hd, double* exp_leaf, double* self_leaf, double xi, unsigned m_begin,
                        unsigned m_end, cudaStream_t st) {
  if (m_end <= m_begin) return;
  const double c_mu = 2.0 * xi * xi / 3.0, c_th = 8.0 * xi * xi * xi * xi / 5.0;  // kernel.cpp:209
  const int per = p2m_gen_per(order);
  const int pb = static_cast<int>(std::min<std::size_t>(32, kGenSmemMax / (sizeof(double) * per)));
  const std::size_t smem = sizeof(double) * per * pb;
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_p2m_gen, kGenSmemMax);
  k_p2m_gen<<<m_end - m_begin, kGenThreads, smem, st>>>(part, leaf_off, depth, box_radius, hd, exp_leaf,
                                                       m_begin, self_leaf, c_mu, c_th, order, pb);
}

std::size_t m2m_generic_scratch_doubles(int order) {
  const std::size_t K = static_cast<std::size_t>(order) * order * order;
  return 3 * K * sizeof(double) <= kGenSmemMax ? 0 : 3 * K * kM2MGenGlobalCtas;
}

void launch_m2m_generic(double* exp, const long long* level_off, int first, int top, int order, const double* m2m,
                        double* scratch, cudaStream_t st, unsigned p_begin, unsigned p_count) {
  if (first < top || first < 0) return;
  if (p_count == 0) p_count = 1u << (3 * first);
  const std::size_t K = static_cast<std::size_t>(order) * order * order;
  const bool in_smem = 3 * K * sizeof(double) <= kGenSmemMax;
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_m2m_gen, kGenSmemMax);
  for (int l = first; l >= top; --l) {
    const unsigned grid = in_smem ? p_count : std::min<unsigned>(p_count, kM2MGenGlobalCtas);
    k_m2m_gen<<<grid, kGenThreads, in_smem ? 3 * K * sizeof(double) : 0, st>>>(
        exp + level_off[l + 1], exp + level_off[l], m2m, order, p_begin, p_count, in_smem ? nullptr : scratch);
    // whole subtrees: the next level's parents are these cells' parents
    p_begin >>= 3;
    p_count = std::max(1u, p_count >> 3);
  }
}

}  // namespace ankh_b200
