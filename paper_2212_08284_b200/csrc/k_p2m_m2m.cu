// P2M (modified charges) and M2M (upward pass) on sm_100a, compile-time order L.
//
// P2M restates modified_charges (chebyshev.cpp:138-203) / leaf_expansions
// (fmm.cpp:181-201):  Q[i,j,k] = sum_p sum_terms coef * Sx^(nx)[i] Sy^(ny)[j]
// Sz^(nz)[k] with S^(n) = radius^-n (H D^n) T(local).  The 10 terms are
// regrouped by the x-derivative order m = nx in {0,1,2}:
//   Q[i, jk] = sum_p sum_m Sx_m[p][i] * W_m[p][jk]
// i.e. one small GEMM (L x 3P) * (3P x L^2) per leaf, with the particle
// records, the 1-D bases S and W staged in shared memory.  One CTA per leaf;
// empty leaves write zeros (fmm.cpp:190-193).
//
// M2M restates upward_pass (fmm.cpp:203-236) with tensor3_apply
// (chebyshev.cpp:246-272): parent += (Mx (x) My (x) Mz) child for the 8
// children, contracted axis by axis with the child sums folded in
// (z: 8 -> 4 partial sums, y: 4 -> 2, x: 2 -> 1).  One CTA per parent.
#include "kernels.cuh"

namespace ankh_b200 {

namespace {

constexpr int kP2MThreads = 128;
#ifndef ANKH_P2M_VEC
#define ANKH_P2M_VEC 1
#endif

// self_energy summand of one particle record (kernel.cpp:208-209): q^2 +
// c_mu |mu|^2 + c_th Theta:Theta (off-diagonals twice, SymMat3::contract)
__device__ __forceinline__ double self_term(double q, double mx, double my, double mz, double txx,
                                            double txy, double txz, double tyy, double tyz, double tzz,
                                            double c_mu, double c_th) {
  const double mu2 = fma(mx, mx, fma(my, my, mz * mz));
  const double th2 = fma(txx, txx, fma(tyy, tyy, tzz * tzz)) + 2.0 * fma(txy, txy, fma(txz, txz, tyz * tyz));
  return fma(c_th, th2, fma(c_mu, mu2, q * q));
}

// hd[n] = H D^n (chebyshev.cpp:85-115) for n = 0..2 depends only on the
// order L, so it lives in the constant bank (one slot per L = 2..10) and the
// basis DFMAs read it as an immediate operand instead of loading it per
// particle.  Written by upload_p2m_basis at plan build (identical bytes for
// every plan of the same L).
__host__ __device__ constexpr int hd_slot(int L) { return L <= 2 ? 0 : hd_slot(L - 1) + 3 * (L - 1) * (L - 1); }
__constant__ double c_hd[hd_slot(11)];
constexpr int kP2MWarps = kP2MThreads / 32;

// Warp-per-leaf P2M.  Each lane first evaluates the 1-D bases of one particle
// (S^(n) = radius^-n (H D^n) T(local) for the 3 axes) and folds the moments
// into the z factors:
//   W0[jk] = y0[j] A0[k] + y1[j] A1[k] + y2[j] A2[k],
//     A0 = q z0 + mu_z z1 + Th_zz z2,  A1 = mu_y z0 + 2 Th_yz z1,  A2 = Th_yy z0
//   W1[jk] = y0[j] B0[k] + y1[j] B1[k],  B0 = mu_x z0 + 2 Th_xz z1,  B1 = 2 Th_xy z0
//   W2[jk] = y0[j] C0[k],                C0 = Th_xx z0
// (the 10 terms of chebyshev.cpp:173-200 regrouped by derivative order);
// then lanes own (j, k) columns and accumulate Q[i, jk] += sum_m Sx_m[i] W_m[jk]
// over the leaf's particles in registers.  No CTA barriers.
template <int L>
struct P2MWShape {
  static constexpr int L2 = L * L, K = L2 * L;
  static constexpr int QJ = (L2 + 31) / 32;       // (j,k) columns per lane
  // kVec: per particle, 16-B aligned groups so the accumulation reads them
  // with 128-bit shared loads (shared-memory issue rivals FP64 there):
  //   X [m][i] (3L, padded even) | Y [j][4] = y0 y1 y2 - | Z [k][6] = A0 A1 A2 B0 B1 C0
  // (config 3: P2M + M2M 0.220 -> 0.213 ms).  L = 6 keeps the scalar layout
  // (the vector one spills there).  Else: X [m][i] | Y [m][j] | Z [f][k].
  static constexpr bool kVec = ANKH_P2M_VEC && L <= 5;
  static constexpr int XP = (3 * L + 1) / 2 * 2;
  static constexpr int YOFF = kVec ? XP : 3 * L, ZOFF = kVec ? XP + 4 * L : 6 * L;
  static constexpr int PER = kVec ? XP + 10 * L : 12 * L;  // staged doubles per particle
  static constexpr std::size_t smem_doubles = kP2MWarps * 32 * PER;
};

template <int L>
#ifndef ANKH_P2M_MINB
#define ANKH_P2M_MINB 4
#endif
__global__ void __launch_bounds__(kP2MThreads, ANKH_P2M_MINB) k_p2m_w(const double* __restrict__ part,
                                                       const unsigned* __restrict__ leaf_off,
                                                       int depth, double rb,
                                                       const double* __restrict__ hd_g,
                                                       double* __restrict__ exp_leaf,
                                                       unsigned m_begin, unsigned m_end,
                                                       const unsigned* __restrict__ list,
                                                       const unsigned* __restrict__ bounds,
                                                       double* __restrict__ self_leaf, double c_mu,
                                                       double c_th) {
  using Sh = P2MWShape<L>;
  constexpr int L2 = Sh::L2, K = Sh::K, PER = Sh::PER, KS = exp_stride(K);
  extern __shared__ __align__(16) double sm[];
  const double* hd = c_hd + hd_slot(L);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // per particle: sx[3][L] | sy[3][L] | A0 A1 A2 B0 B1 C0 [L]
  double* st = sm + warp * 32 * PER;
  (void)hd_g;
  const int n = 1 << depth;
  // leaves are visited (and their expansions stored) in Morton order
  // list mode (streamed host path): the leaves list[bounds[0] .. bounds[1]),
  // warps striding over them (the grid is sized without knowing the count)
  const unsigned stride = list ? gridDim.x * kP2MWarps : 0u;
  for (unsigned item = blockIdx.x * kP2MWarps + warp;; item += stride) {
  unsigned m;
  if (list) {
    if (item >= bounds[1] - bounds[0]) return;
    m = list[bounds[0] + item];
  } else {
    m = m_begin + item;
    if (m >= m_end) return;
  }
  const int ci0 = static_cast<int>(morton_compact3(m >> 2)),
            ci1 = static_cast<int>(morton_compact3(m >> 1)), ci2 = static_cast<int>(morton_compact3(m));
  const unsigned leaf = (static_cast<unsigned>(ci0) * n + ci1) * n + ci2;
  const unsigned begin = leaf_off[leaf];
  const int cnt = static_cast<int>(leaf_off[leaf + 1] - begin);
  double* out = exp_leaf + static_cast<std::size_t>(m) * KS;
  // cell_geometry (octree.cpp:18-25)
  const double rad = rb / n;
  const double c0 = -rb + rad * (2 * ci0 + 1), c1 = -rb + rad * (2 * ci1 + 1),
               c2 = -rb + rad * (2 * ci2 + 1);
  const double inv_rad = 1.0 / rad;

  double acc[Sh::QJ][L];
  int jj[Sh::QJ], kk[Sh::QJ];
#pragma unroll
  for (int q = 0; q < Sh::QJ; ++q) {
    const int jk = min(lane + 32 * q, L2 - 1);
    jj[q] = jk / L;
    kk[q] = jk - L * (jk / L);
#pragma unroll
    for (int i = 0; i < L; ++i) acc[q][i] = 0.0;
  }

  double self_acc = 0.0;
  for (int p0 = 0; p0 < cnt; p0 += 32) {
    const int pc = min(32, cnt - p0);
    __syncwarp();
    if (lane < pc) {
      const double2* r = reinterpret_cast<const double2*>(part + static_cast<std::size_t>(begin + p0 + lane) * kRec);
      const double2 v0 = __ldg(r), v1 = __ldg(r + 1), v2 = __ldg(r + 2), v3 = __ldg(r + 3),
                    v4 = __ldg(r + 4), v5 = __ldg(r + 5), v6 = __ldg(r + 6);
      const double q = v1.y, mx = v2.x, my = v2.y, mz = v3.x, txx = v3.y, txy = v4.x,
                   txz = v4.y, tyy = v5.x, tyz = v5.y, tzz = v6.x;
      self_acc += self_term(q, mx, my, mz, txx, txy, txz, tyy, tyz, tzz, c_mu, c_th);
      const double lx = (v0.x - c0) * inv_rad, ly = (v0.y - c1) * inv_rad,
                   lz = (v1.x - c2) * inv_rad;
      double* dst = st + lane * PER;
      double tx[L], ty[L], tz[L];
      tx[0] = ty[0] = tz[0] = 1.0;
      if (L > 1) {
        tx[1] = lx;
        ty[1] = ly;
        tz[1] = lz;
      }
#pragma unroll
      for (int m = 2; m < L; ++m) {
        tx[m] = 2.0 * lx * tx[m - 1] - tx[m - 2];
        ty[m] = 2.0 * ly * ty[m - 1] - ty[m - 2];
        tz[m] = 2.0 * lz * tz[m - 1] - tz[m - 2];
      }
      double scale = 1.0;
#pragma unroll
      for (int nd = 0; nd < 3; ++nd) {
        double zb[L];
#pragma unroll
        for (int i = 0; i < L; ++i) {
          double vx = 0.0, vy = 0.0, vz = 0.0;
#pragma unroll
          for (int m = 0; m < L; ++m) {
            const double h = hd[nd * L2 + i * L + m];
            vx += h * tx[m];
            vy += h * ty[m];
            vz += h * tz[m];
          }
          dst[nd * L + i] = scale * vx;                                     // x basis S^(nd)
          dst[Sh::YOFF + (Sh::kVec ? 4 * i + nd : nd * L + i)] = scale * vy;  // y basis
          zb[i] = scale * vz;
        }
        scale *= inv_rad;
        // fold the moments into the z factors (A0 A1 A2 B0 B1 C0)
#define ZF(f, i) dst[Sh::ZOFF + (Sh::kVec ? 6 * (i) + (f) : (f) * L + (i))]
#pragma unroll
        for (int i = 0; i < L; ++i) {
          const double z = zb[i];
          if (nd == 0) {
            ZF(0, i) = q * z;
            ZF(1, i) = my * z;
            ZF(2, i) = tyy * z;
            ZF(3, i) = mx * z;
            ZF(4, i) = (2.0 * txy) * z;
            ZF(5, i) = txx * z;
          } else if (nd == 1) {
            ZF(0, i) += mz * z;
            ZF(1, i) += (2.0 * tyz) * z;
            ZF(3, i) += (2.0 * txz) * z;
          } else {
            ZF(0, i) += tzz * z;
          }
        }
#undef ZF
      }
    }
    __syncwarp();
    for (int p = 0; p < pc; ++p) {
      const double* s = st + p * PER;
      if constexpr (Sh::kVec) {
      double xv[Sh::XP];
#pragma unroll
      for (int u = 0; u < Sh::XP / 2; ++u) {
        const double2 t = reinterpret_cast<const double2*>(s)[u];
        xv[2 * u] = t.x;
        xv[2 * u + 1] = t.y;
      }
#pragma unroll
      for (int q = 0; q < Sh::QJ; ++q) {
        const double2* y2p = reinterpret_cast<const double2*>(s + Sh::YOFF + 4 * jj[q]);
        const double2* z2p = reinterpret_cast<const double2*>(s + Sh::ZOFF + 6 * kk[q]);
        const double2 ya = y2p[0], yb = y2p[1], za = z2p[0], zb2 = z2p[1], zc = z2p[2];
        const double w0 = fma(ya.x, za.x, fma(ya.y, za.y, yb.x * zb2.x));
        const double w1 = fma(ya.x, zb2.y, ya.y * zc.x);
        const double w2 = ya.x * zc.y;
#pragma unroll
        for (int i = 0; i < L; ++i)
          acc[q][i] = fma(xv[i], w0, fma(xv[L + i], w1, fma(xv[2 * L + i], w2, acc[q][i])));
      }
      } else {
#pragma unroll
      for (int q = 0; q < Sh::QJ; ++q) {
        const int j = jj[q], k = kk[q];
        const double y0 = s[3 * L + j], y1 = s[4 * L + j], y2 = s[5 * L + j];
        const double w0 = fma(y0, s[6 * L + k], fma(y1, s[7 * L + k], y2 * s[8 * L + k]));
        const double w1 = fma(y0, s[9 * L + k], y1 * s[10 * L + k]);
        const double w2 = y0 * s[11 * L + k];
#pragma unroll
        for (int i = 0; i < L; ++i)
          acc[q][i] = fma(s[i], w0, fma(s[L + i], w1, fma(s[2 * L + i], w2, acc[q][i])));
      }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < Sh::QJ; ++q) {
    const int jk = lane + 32 * q;
    if (jk < L2) {
#pragma unroll
      for (int i = 0; i < L; ++i) out[i * L2 + jk] = acc[q][i];
    }
  }
  // the leaf's self-energy sum, fixed lane order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) self_acc += __shfl_down_sync(0xffffffffu, self_acc, o);
  if (lane == 0) self_leaf[m] = self_acc;
  if (!list) return;
  }  // list mode: next leaf
}

template <int L>
struct P2MShape {
  static constexpr int L2 = L * L, K = L2 * L;
  static constexpr int PB = L <= 6 ? 32 : 16;                     // particles per batch
  static constexpr int QN = (K + kP2MThreads - 1) / kP2MThreads;  // outputs per thread
  static constexpr int RS = 14;                                   // staged record stride
  static constexpr std::size_t smem_doubles = 3 * L2 + PB * RS + PB * 9 * L + PB * 3 * L2;
};

template <int L>
__global__ void __launch_bounds__(kP2MThreads) k_p2m(const double* __restrict__ part,
                                                     const unsigned* __restrict__ leaf_off,
                                                     int depth, double rb,
                                                     const double* __restrict__ hd_g,
                                                     double* __restrict__ exp_leaf,
                                                     const DevResult* __restrict__ res,
                                                     unsigned m_begin, double* __restrict__ self_leaf,
                                                     double c_mu, double c_th) {
  using Sh = P2MShape<L>;
  constexpr int L2 = Sh::L2, K = Sh::K, PB = Sh::PB, RS = Sh::RS, KS = exp_stride(K);
  extern __shared__ __align__(16) double sm[];
  double* hd = sm;              // 3 L^2
  double* rec = hd + 3 * L2;    // PB x RS
  double* S = rec + PB * RS;    // PB x 3 axes x 3 orders x L
  double* W = S + PB * 9 * L;   // PB x 3 x L^2
  const int tid = threadIdx.x;
  const int n = 1 << depth;
  const unsigned m = m_begin + blockIdx.x;  // Morton leaf
  const unsigned leaf = morton_to_lex(m, n);
  const unsigned begin = leaf_off[leaf];
  const int cnt = static_cast<int>(leaf_off[leaf + 1] - begin);
  double* out = exp_leaf + static_cast<std::size_t>(m) * KS;
  if (cnt == 0) {
    for (int o = tid; o < K; o += kP2MThreads) out[o] = 0.0;
    if (tid == 0) self_leaf[m] = 0.0;
    return;
  }
  double self_acc = 0.0;  // particle tid of each batch (PB <= kP2MThreads)
  const bool charges_only = res->any_multipole == 0;
  // cell_geometry (octree.cpp:18-25)
  const double rad = rb / n;
  const int ci0 = static_cast<int>(leaf) / (n * n), ci1 = (static_cast<int>(leaf) / n) % n,
            ci2 = static_cast<int>(leaf) % n;
  const double inv_rad = 1.0 / rad;
  for (int w = tid; w < 3 * L2; w += kP2MThreads) hd[w] = hd_g[w];

  double acc[Sh::QN];
  int oi[Sh::QN], ojk[Sh::QN];
#pragma unroll
  for (int q = 0; q < Sh::QN; ++q) {
    acc[q] = 0.0;
    const int o = tid + q * kP2MThreads;
    oi[q] = o / L2;
    ojk[q] = o - L2 * (o / L2);
  }

  for (int p0 = 0; p0 < cnt; p0 += PB) {
    const int pb = min(PB, cnt - p0);
    __syncthreads();
    for (int w = tid; w < pb * 7; w += kP2MThreads) {
      const int p = w / 7, c = w - 7 * (w / 7);
      const double2 v = __ldg(
          reinterpret_cast<const double2*>(part + static_cast<std::size_t>(begin + p0 + p) * kRec) + c);
      rec[p * RS + 2 * c] = v.x;
      rec[p * RS + 2 * c + 1] = v.y;
    }
    __syncthreads();
    if (tid < pb) {
      const double* r = rec + tid * RS;
      self_acc += self_term(r[3], r[4], r[5], r[6], r[7], r[8], r[9], r[10], r[11], r[12], c_mu, c_th);
    }
    // phase A: 1-D basis derivatives per (particle, axis)
    for (int w = tid; w < pb * 3; w += kP2MThreads) {
      const int p = w / 3, ax = w - 3 * (w / 3);
      const int cax = ax == 0 ? ci0 : (ax == 1 ? ci1 : ci2);
      const double center = -rb + rad * (2 * cax + 1);
      const double local = (rec[p * RS + ax] - center) * inv_rad;
      double t[L];
      t[0] = 1.0;
      if (L > 1) t[1] = local;
#pragma unroll
      for (int m = 2; m < L; ++m) t[m] = 2.0 * local * t[m - 1] - t[m - 2];
      double scale = 1.0;
#pragma unroll
      for (int nd = 0; nd < 3; ++nd) {
        double* s_out = S + ((p * 3 + ax) * 3 + nd) * L;
        const double* h = hd + nd * L2;
#pragma unroll
        for (int i = 0; i < L; ++i) {
          double v = 0.0;
#pragma unroll
          for (int m = 0; m < L; ++m) v += h[i * L + m] * t[m];
          s_out[i] = scale * v;
        }
        scale *= inv_rad;
      }
    }
    __syncthreads();
    // phase B: W_m[p][jk]
    for (int w = tid; w < pb * L2; w += kP2MThreads) {
      const int p = w / L2, jk = w - L2 * (w / L2);
      const int j = jk / L, k = jk - L * (jk / L);
      const double* r = rec + p * RS;
      const double* sy = S + (p * 3 + 1) * 3 * L;
      const double* sz = S + (p * 3 + 2) * 3 * L;
      const double y0 = sy[j], y1 = sy[L + j], y2 = sy[2 * L + j];
      const double z0 = sz[k], z1 = sz[L + k], z2 = sz[2 * L + k];
      double* wp = W + p * 3 * L2 + jk;
      if (charges_only) {
        wp[0] = r[3] * (y0 * z0);
        wp[L2] = 0.0;
        wp[2 * L2] = 0.0;
      } else {
        wp[0] = r[3] * (y0 * z0) + r[5] * (y1 * z0) + r[6] * (y0 * z1) + r[10] * (y2 * z0) +
                r[12] * (y0 * z2) + (2.0 * r[11]) * (y1 * z1);
        wp[L2] = r[4] * (y0 * z0) + (2.0 * r[8]) * (y1 * z0) + (2.0 * r[9]) * (y0 * z1);
        wp[2 * L2] = r[7] * (y0 * z0);
      }
    }
    __syncthreads();
    // phase C: Q[i, jk] += sum_p sum_m Sx_m[p][i] W_m[p][jk]
#pragma unroll
    for (int q = 0; q < Sh::QN; ++q) {
      if (tid + q * kP2MThreads < K) {
        double a = acc[q];
        const double* sx = S + oi[q];
        const double* wp = W + ojk[q];
        for (int p = 0; p < pb; ++p) {
          a += sx[0] * wp[0];
          a += sx[L] * wp[L2];
          a += sx[2 * L] * wp[2 * L2];
          sx += 9 * L;
          wp += 3 * L2;
        }
        acc[q] = a;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < Sh::QN; ++q)
    if (tid + q * kP2MThreads < K) out[tid + q * kP2MThreads] = acc[q];
  // the leaf's self-energy sum: PB threads, fixed order
  __shared__ double s_self[PB];
  if (tid < PB) s_self[tid] = self_acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int k = 0; k < PB; ++k) t += s_self[k];
    self_leaf[m] = t;
  }
}

constexpr int kM2MThreads = 128;

// One parent's M2M (upward_pass, fmm.cpp:203-236; tensor3_apply,
// chebyshev.cpp:246-272) by the whole CTA: parent[i,j,k] = sum over the 8
// children of T_cx(i,a) T_cy(j,b) T_cz(k,c) child[a,b,c], the child sums
// folded into each axis stage.  M (the two 1-D transfer matrices) is already
// in shared memory.  kCoherent: children written by other CTAs of the same
// launch (the chained kernel) are read past L1 (ld.global.cg).
template <int L, bool kCoherent>
__device__ __forceinline__ void m2m_parent(const double* __restrict__ child, double* __restrict__ parent,
                                           unsigned pcell, const double* M, double* V, double* S1, double* S2) {
  constexpr int L2 = L * L, K = L2 * L, KS = exp_stride(K);
  // Morton order: the children of parent p are rows 8p + (cx<<2 | cy<<1 | cz),
  // one contiguous 8 KS-double block: loaded as 16-B pieces, a batch of
  // loads in flight per thread before any shared-memory store
  const double2* ch0 = reinterpret_cast<const double2*>(child + static_cast<std::size_t>(pcell) * 8 * KS);
  double2* V2 = reinterpret_cast<double2*>(V);
  constexpr int NV = 8 * KS / 2, kBatch = 8;
  for (int w0 = 0; w0 < NV; w0 += kBatch * kM2MThreads) {
    double2 t[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int w = w0 + u * kM2MThreads + threadIdx.x;
      if (w < NV) t[u] = kCoherent ? __ldcg(ch0 + w) : __ldg(ch0 + w);
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int w = w0 + u * kM2MThreads + threadIdx.x;
      if (w < NV) V2[w] = t[u];
    }
  }
  __syncthreads();
  // z: S1[(cx,cy)][a,b,k] = sum_cz sum_c' Mz[cz](k,c') V[(cx,cy,cz)][a,b,c']
  for (int w = threadIdx.x; w < 4 * K; w += kM2MThreads) {
    const int q = w / K, e = w - K * (w / K);
    const int ab = e / L, k = e - L * (e / L);
    double acc = 0.0;
#pragma unroll
    for (int cz = 0; cz < 2; ++cz) {
      const double* v = V + (2 * q + cz) * KS + ab * L;
      const double* m = M + cz * L2 + k * L;
#pragma unroll
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
#pragma unroll
    for (int cy = 0; cy < 2; ++cy) {
      const double* s = S1 + (2 * cx + cy) * K + a * L2 + k;
      const double* m = M + cy * L2 + j * L;
#pragma unroll
      for (int b = 0; b < L; ++b) acc += m[b] * s[b * L];
    }
    S2[w] = acc;
  }
  __syncthreads();
  // x: out[i,j,k] = sum_cx sum_a Mx[cx](i,a) S2[cx][a,j,k]
  double* out = parent + static_cast<std::size_t>(pcell) * KS;
  for (int e = threadIdx.x; e < K; e += kM2MThreads) {
    const int i = e / L2, jk = e - L2 * (e / L2);
    double acc = 0.0;
#pragma unroll
    for (int cx = 0; cx < 2; ++cx) {
      const double* s = S2 + cx * K + jk;
      const double* m = M + cx * L2 + i * L;
#pragma unroll
      for (int a = 0; a < L; ++a) acc += m[a] * s[a * L2];
    }
    out[e] = acc;
  }
}

// The upward pass in ONE launch: CTA b computes parent p_begin + b at level
// `first`; the last of eight siblings to finish (per-cell arrival counter,
// threadfence pattern) goes on to their parent, and so on up to level `top`.
// Every sibling set lies inside the launch's cells (whole subtrees), so each
// cell is computed exactly once, by the CTA that completed its children.
// The counters reset themselves (the eighth arrival zeroes its slot).
template <int L>
__global__ void __launch_bounds__(kM2MThreads) k_m2m_chain(double* __restrict__ exp,
                                                           const long long* __restrict__ level_off, int first,
                                                           int top, unsigned p_begin,
                                                           unsigned* __restrict__ counters,
                                                           const double* __restrict__ m2m_g) {
  constexpr int L2 = L * L, K = L2 * L, KS = exp_stride(K);
  extern __shared__ __align__(16) double sm[];
  double* M = sm;           // 2 x L x L: M[c][i][a] = T_c(i, a)
  double* V = M + 2 * L2;   // 8 x KS children (rows as stored, zero tails)
  double* S1 = V + 8 * KS;  // 4 x K  (cx, cy) after z
  double* S2 = S1 + 4 * K;  // 2 x K  (cx) after y
  __shared__ int s_last;
  for (int w = threadIdx.x; w < 2 * L2; w += kM2MThreads) M[w] = m2m_g[w];
  unsigned p = p_begin + blockIdx.x;
  int l = first;
  for (;;) {
    if (l == first)
      m2m_parent<L, false>(exp + level_off[l + 1], exp + level_off[l], p, M, V, S1, S2);
    else
      m2m_parent<L, true>(exp + level_off[l + 1], exp + level_off[l], p, M, V, S1, S2);
    if (l == top) break;
    __threadfence();  // this parent row is visible before the arrival is counted
    __syncthreads();
    if (threadIdx.x == 0) {
      // counters of the parent level l - 1: cells [8^(l-1) - 1) / 7 ...
      unsigned* c = counters + ((1u << (3 * (l - 1))) - 1u) / 7u + (p >> 3);
      const unsigned old = atomicAdd(c, 1u);
      s_last = old == 7u;
      if (old == 7u) *c = 0u;
    }
    __syncthreads();
    if (!s_last) break;
    __threadfence();  // the siblings' rows, published before their arrivals
    p >>= 3;
    --l;
  }
}

template <int L>
void p2m_order(const double* part, const unsigned* leaf_off, int depth, double rb,
               const double* hd, double* exp_leaf, const DevResult* res, double* self_leaf, double xi,
               unsigned m_begin, unsigned m_end, const unsigned* list, const unsigned* bounds,
               unsigned list_count, cudaStream_t st) {
  const double c_mu = 2.0 * xi * xi / 3.0, c_th = 8.0 * xi * xi * xi * xi / 5.0;  // kernel.cpp:209
  const unsigned leaves = list ? list_count : (m_end > m_begin ? m_end - m_begin : 0u);
  if (leaves == 0) return;
  if (L > 6) {  // register budget of the warp-per-leaf variant: block-per-leaf instead
    if (list) return;  // (no list mode: the plan streams only for L <= 6)
    const std::size_t smem = sizeof(double) * P2MShape<L>::smem_doubles;
    static std::atomic<unsigned long long> attr_b{0};
    smem_opt_in(attr_b, k_p2m<L>, smem);
    k_p2m<L><<<leaves, kP2MThreads, smem, st>>>(part, leaf_off, depth, rb, hd, exp_leaf, res,
                                                m_begin, self_leaf, c_mu, c_th);
    return;
  }
  constexpr int LW = L > 6 ? 6 : L;  // (never launched with L > 6)
  const std::size_t smem = sizeof(double) * P2MWShape<LW>::smem_doubles;
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_p2m_w<LW>, smem);
  // list mode: list_count is an upper bound of the leaves (the warps stride)
  k_p2m_w<LW><<<(leaves + kP2MWarps - 1) / kP2MWarps, kP2MThreads, smem, st>>>(
      part, leaf_off, depth, rb, hd, exp_leaf, m_begin, m_end, list, bounds, self_leaf, c_mu, c_th);
}

}  // namespace

void upload_p2m_basis(int order, const double* hd, cudaStream_t st) {
  if (order < 2 || order > 10) return;
  const int L = order;
  cudaMemcpyToSymbolAsync(c_hd, hd, sizeof(double) * 3 * L * L, sizeof(double) * hd_slot(L),
                          cudaMemcpyHostToDevice, st);
}

namespace {

template <int L>
void m2m_chain_order(double* exp, const long long* level_off, int first, int top, unsigned p_begin,
                     unsigned p_count, unsigned* counters, const double* m2m, cudaStream_t st) {
  constexpr int K = L * L * L;
  const std::size_t smem = sizeof(double) * (2 * L * L + 8 * exp_stride(K) + 6 * K);
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_m2m_chain<L>, smem);
  k_m2m_chain<L><<<p_count, kM2MThreads, smem, st>>>(exp, level_off, first, top, p_begin, counters, m2m);
}

}  // namespace

#define ANKH_ORDER_SWITCH(L, CALL) \
  switch (L) {                     \
    case 2: CALL(2); break;        \
    case 3: CALL(3); break;        \
    case 4: CALL(4); break;        \
    case 5: CALL(5); break;        \
    case 6: CALL(6); break;        \
    case 7: CALL(7); break;        \
    case 8: CALL(8); break;        \
    case 9: CALL(9); break;        \
    case 10: CALL(10); break;      \
    default: break;                \
  }

void launch_p2m(const double* part, const unsigned* leaf_off, int depth, int order,
                double box_radius, const double* hd, double* exp_leaf, const DevResult* res,
                double* self_leaf, double xi, unsigned m_begin, unsigned m_end, cudaStream_t st,
                const unsigned* list, const unsigned* bounds, unsigned list_count) {
#define ANKH_P2M(N) \
  p2m_order<N>(part, leaf_off, depth, box_radius, hd, exp_leaf, res, self_leaf, xi, m_begin, m_end, list, \
               bounds, list_count, st)
  if (order > 10) {  // runtime-order kernel (k_generic.cu); no list mode (streamed path is L <= 6)
    if (!list) launch_p2m_generic(part, leaf_off, depth, order, box_radius, hd, exp_leaf, self_leaf, xi, m_begin,
                                  m_end, st);
    return;
  }
  ANKH_ORDER_SWITCH(order, ANKH_P2M)
#undef ANKH_P2M
}

std::size_t m2m_counter_count(int depth) {
  std::size_t c = 0;
  for (int l = 0; l < depth; ++l) c += std::size_t(1) << (3 * l);
  return c;
}

void launch_m2m_chain(double* exp, const long long* level_off, int first, int top, int order,
                      const double* m2m, unsigned* counters, cudaStream_t st, unsigned p_begin,
                      unsigned p_count) {
  if (first < top || first < 0) return;
  if (p_count == 0) p_count = 1u << (3 * first);
#define ANKH_M2M(N) m2m_chain_order<N>(exp, level_off, first, top, p_begin, p_count, counters, m2m, st)
  ANKH_ORDER_SWITCH(order, ANKH_M2M)
#undef ANKH_M2M
}

}  // namespace ankh_b200
