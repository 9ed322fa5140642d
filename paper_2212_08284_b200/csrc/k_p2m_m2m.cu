// P2M (modified charges) and M2M (upward pass) on sm_100a.
//
// P2M restates modified_charges (chebyshev.cpp:138-203) / leaf_expansions
// (fmm.cpp:181-201):  Q[i,j,k] = sum_p sum_terms coef * Sx^(nx)[i] Sy^(ny)[j]
// Sz^(nz)[k] with S^(n) = radius^-n (H D^n) T(local).  The 10 terms are
// regrouped by the x-derivative order m = nx in {0,1,2}:
//   Q[i, jk] = sum_p sum_m Sx_m[p][i] * W_m[p][jk]
// i.e. one small GEMM (L x 3P) * (3P x L^2) per leaf, with W built in shared
// memory.  One CTA per leaf; empty leaves write zeros (fmm.cpp:190-193).
//
// M2M restates upward_pass (fmm.cpp:203-236) with tensor3_apply
// (chebyshev.cpp:246-272): parent += (Mx (x) My (x) Mz) child for the 8
// children, contracted axis by axis with the child sums folded in
// (z: 8 -> 4 partial sums, y: 4 -> 2, x: 2 -> 1).  One CTA per parent.
#include "kernels.cuh"

namespace ankh_b200 {

namespace {

constexpr int kP2MThreads = 128;
constexpr int kMaxOrder = 10;  // K <= 1000 (plan rejects larger orders)

__global__ void __launch_bounds__(kP2MThreads) k_p2m(const double* __restrict__ part,
                                                     const unsigned* __restrict__ leaf_off,
                                                     int depth, int L, double rb,
                                                     const double* __restrict__ hd_g,
                                                     double* __restrict__ exp_leaf, int pb_max,
                                                     const DevResult* __restrict__ res) {
  const bool charges_only = res->any_multipole == 0;
  extern __shared__ double sm[];
  const int L2 = L * L, K = L2 * L;
  double* hd = sm;                       // 3 L^2
  double* S = hd + 3 * L2;               // pb_max x 3 axes x 3 orders x L
  double* W = S + pb_max * 9 * L;        // pb_max x 3 x L^2
  const unsigned leaf = blockIdx.x;
  const int n = 1 << depth;
  const unsigned begin = leaf_off[leaf];
  const int cnt = static_cast<int>(leaf_off[leaf + 1] - begin);
  double* out = exp_leaf + static_cast<std::size_t>(leaf) * K;
  if (cnt == 0) {
    for (int o = threadIdx.x; o < K; o += kP2MThreads) out[o] = 0.0;
    return;
  }
  // cell_geometry (octree.cpp:18-25)
  const double rad = rb / n;
  const int ci[3] = {static_cast<int>(leaf) / (n * n), (static_cast<int>(leaf) / n) % n,
                     static_cast<int>(leaf) % n};
  double center[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) center[a] = -rb + rad * (2 * ci[a] + 1);
  const double inv_rad = 1.0 / rad;
  for (int w = threadIdx.x; w < 3 * L2; w += kP2MThreads) hd[w] = hd_g[w];

  constexpr int kOutMax = (kMaxOrder * kMaxOrder * kMaxOrder + kP2MThreads - 1) / kP2MThreads;
  double acc[kOutMax];
#pragma unroll
  for (int q = 0; q < kOutMax; ++q) acc[q] = 0.0;

  for (int p0 = 0; p0 < cnt; p0 += pb_max) {
    const int pb = min(pb_max, cnt - p0);
    __syncthreads();
    // phase A: 1-D basis derivatives per (particle, axis)
    for (int w = threadIdx.x; w < pb * 3; w += kP2MThreads) {
      const int p = w / 3, ax = w - 3 * (w / 3);
      const double* rec = part + static_cast<std::size_t>(begin + p0 + p) * kRec;
      const double local = (rec[ax] - center[ax]) * inv_rad;
      double t[kMaxOrder];
      t[0] = 1.0;
      if (L > 1) t[1] = local;
      for (int m = 2; m < L; ++m) t[m] = 2.0 * local * t[m - 1] - t[m - 2];
      double scale = 1.0;
      for (int nd = 0; nd < 3; ++nd) {
        double* s_out = S + ((p * 3 + ax) * 3 + nd) * L;
        const double* h = hd + nd * L2;
        for (int i = 0; i < L; ++i) {
          double v = 0.0;
          for (int m = 0; m < L; ++m) v += h[i * L + m] * t[m];
          s_out[i] = scale * v;
        }
        scale *= inv_rad;
      }
    }
    __syncthreads();
    // phase B: W_m[p][jk]
    for (int w = threadIdx.x; w < pb * L2; w += kP2MThreads) {
      const int p = w / L2, jk = w - L2 * (w / L2);
      const int j = jk / L, k = jk - L * (jk / L);
      const double* rec = part + static_cast<std::size_t>(begin + p0 + p) * kRec;
      const double* sy = S + (p * 3 + 1) * 3 * L;
      const double* sz = S + (p * 3 + 2) * 3 * L;
      const double y0 = sy[j], y1 = sy[L + j], y2 = sy[2 * L + j];
      const double z0 = sz[k], z1 = sz[L + k], z2 = sz[2 * L + k];
      double* wp = W + p * 3 * L2 + jk;
      if (charges_only) {
        wp[0] = rec[3] * (y0 * z0);
        wp[L2] = 0.0;
        wp[2 * L2] = 0.0;
      } else {
        const double q = rec[3], mx = rec[4], my = rec[5], mz = rec[6];
        const double txx = rec[7], txy = rec[8], txz = rec[9], tyy = rec[10], tyz = rec[11],
                     tzz = rec[12];
        wp[0] = q * (y0 * z0) + my * (y1 * z0) + mz * (y0 * z1) + tyy * (y2 * z0) +
                tzz * (y0 * z2) + (2.0 * tyz) * (y1 * z1);
        wp[L2] = mx * (y0 * z0) + (2.0 * txy) * (y1 * z0) + (2.0 * txz) * (y0 * z1);
        wp[2 * L2] = txx * (y0 * z0);
      }
    }
    __syncthreads();
    // phase C: Q[i, jk] += sum_p sum_m Sx_m[p][i] W_m[p][jk]
#pragma unroll
    for (int q = 0; q < kOutMax; ++q) {
      const int o = threadIdx.x + q * kP2MThreads;
      if (o < K) {
        const int i = o / L2, jk = o - L2 * (o / L2);
        double a = acc[q];
        for (int p = 0; p < pb; ++p) {
          const double* sx = S + (p * 3 + 0) * 3 * L;
          const double* wp = W + p * 3 * L2 + jk;
          a += sx[i] * wp[0];
          a += sx[L + i] * wp[L2];
          a += sx[2 * L + i] * wp[2 * L2];
        }
        acc[q] = a;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kOutMax; ++q) {
    const int o = threadIdx.x + q * kP2MThreads;
    if (o < K) out[o] = acc[q];
  }
}

constexpr int kM2MThreads = 128;

__global__ void __launch_bounds__(kM2MThreads) k_m2m(const double* __restrict__ child,
                                                     double* __restrict__ parent, int level,
                                                     int L, const double* __restrict__ m2m_g) {
  extern __shared__ double sm[];
  const int L2 = L * L, K = L2 * L;
  double* M = sm;               // 2 x L x L: M[c][i][a] = T_c(i, a)
  double* V = M + 2 * L2;       // 8 x K children
  double* S1 = V + 8 * K;       // 4 x K  (cx, cy) after z
  double* S2 = S1 + 4 * K;      // 2 x K  (cx) after y
  const int n = 1 << level, nc = 2 * n;
  const unsigned pcell = blockIdx.x;
  const int pi = static_cast<int>(pcell) / (n * n), pj = (static_cast<int>(pcell) / n) % n,
            pk = static_cast<int>(pcell) % n;
  for (int w = threadIdx.x; w < 2 * L2; w += kM2MThreads) M[w] = m2m_g[w];
  for (int w = threadIdx.x; w < 8 * K; w += kM2MThreads) {
    const int c = w / K, e = w - K * (w / K);
    const int cx = c >> 2, cy = (c >> 1) & 1, cz = c & 1;
    const std::size_t ch =
        (static_cast<std::size_t>(2 * pi + cx) * nc + (2 * pj + cy)) * nc + (2 * pk + cz);
    V[w] = child[ch * K + e];
  }
  __syncthreads();
  // z: S1[(cx,cy)][a,b,k] = sum_cz sum_c' Mz[cz](k,c') V[(cx,cy,cz)][a,b,c']
  for (int w = threadIdx.x; w < 4 * K; w += kM2MThreads) {
    const int q = w / K, e = w - K * (w / K);
    const int ab = e / L, k = e - L * (e / L);
    double acc = 0.0;
    for (int cz = 0; cz < 2; ++cz) {
      const double* v = V + (2 * q + cz) * K + ab * L;
      const double* m = M + cz * L2 + k * L;
      for (int c = 0; c < L; ++c) acc += m[c] * v[c];
    }
    S1[w] = acc;
  }
  __syncthreads();
  // y: S2[cx][a,j,k] = sum_cy sum_b My[cy](j,b) S1[(cx,cy)][a,b,k]
  for (int w = threadIdx.x; w < 2 * K; w += kM2MThreads) {
    const int cx = w / K, e = w - K * (w / K);
    const int a = e / L2, jk = e - L2 * (e / L2);
    const int j = jk / L, k = jk - L * (jk / L);
    double acc = 0.0;
    for (int cy = 0; cy < 2; ++cy) {
      const double* s = S1 + (2 * cx + cy) * K + a * L2 + k;
      const double* m = M + cy * L2 + j * L;
      for (int b = 0; b < L; ++b) acc += m[b] * s[b * L];
    }
    S2[w] = acc;
  }
  __syncthreads();
  // x: out[i,j,k] = sum_cx sum_a Mx[cx](i,a) S2[cx][a,j,k]
  double* out = parent + static_cast<std::size_t>(pcell) * K;
  for (int e = threadIdx.x; e < K; e += kM2MThreads) {
    const int i = e / L2, jk = e - L2 * (e / L2);
    double acc = 0.0;
    for (int cx = 0; cx < 2; ++cx) {
      const double* s = S2 + cx * K + jk;
      const double* m = M + cx * L2 + i * L;
      for (int a = 0; a < L; ++a) acc += m[a] * s[a * L2];
    }
    out[e] = acc;
  }
}

}  // namespace

void launch_p2m(const double* part, const unsigned* leaf_off, int depth, int order,
                double box_radius, const double* hd, double* exp_leaf, const DevResult* res,
                cudaStream_t st) {
  const int L = order, L2 = L * L;
  const int pb = L <= 6 ? 32 : 16;
  const std::size_t smem = sizeof(double) * (3 * L2 + pb * 9 * L + pb * 3 * L2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_p2m, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const unsigned leaves = 1u << (3 * depth);
  k_p2m<<<leaves, kP2MThreads, smem, st>>>(part, leaf_off, depth, L, box_radius, hd, exp_leaf, pb,
                                           res);
}

void launch_m2m(const double* child, double* parent, int parent_level, int order,
                const double* m2m, cudaStream_t st) {
  const int L = order, K = L * L * L;
  const std::size_t smem = sizeof(double) * (2 * L * L + 14 * K);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_m2m, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const unsigned cells = 1u << (3 * parent_level);
  k_m2m<<<cells, kM2MThreads, smem, st>>>(child, parent, parent_level, L, m2m);
}

}  // namespace ankh_b200
