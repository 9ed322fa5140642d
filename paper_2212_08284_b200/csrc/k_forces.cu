// Forces F_a = -dE/dx_a of the ANKH-FMM energy (moments held fixed in the
// lab frame) -- SURVEY.md §8f-3, the paper's stated perspective
// (PAPER.md:541, 990).  The reference computes energies only; these kernels
// differentiate exactly the energy the reference defines (fmm.cpp:383-436):
//
//   near field  E_near = sum_pairs e(x_a - x_b - shift)   (fmm.cpp:278-327)
//     -> k_p2p_force_half (forces alone): the gradient of pair_interaction
//        (pair.cuh pair_grad_mp) over the energy's half shell, every
//        neighbour pair once (Newton's third law; source-side sums in 13
//        direction slots, deterministic, no atomics);
//     -> k_p2p_force (with the moment derivatives): per target particle over
//        its own leaf and all 26 neighbours (every thread owns its target's sum).
//   far field   E_far = sum_canonical (L_o M_t).(R_o M_s)  (fmm.cpp:238-276)
//     -> Lambda_c = dE/dM_c for every cell (k_m2l_local, DMMA): for every
//        partner p of c, L_o^T R_o M_p when (c, p) is the canonical instance,
//        R_o'^T L_o' M_p when (p, c) is (o' = -o) -- the factors the energy
//        uses, so the gradient is exact for every order;
//     -> the periodic term E_per = 1/2 v^T C v, v = (T x T x T) M_root
//        (fmm.cpp:421-427): Lambda_root += (T x T x T)^T C v (k_periodic_local;
//        C is the symmetric block-Toeplitz operator of the generator);
//     -> L2L, the transpose of M2M (fmm.cpp:203-236): Lambda_child +=
//        (T_cx x T_cy x T_cz)^T Lambda_parent (k_l2l);
//     -> L2P, the transpose of P2M differentiated once more (chebyshev.cpp:
//        138-203): dM_leaf/dx_a uses S^(n+1) = rad^-(n+1) H D^(n+1) T(local)
//        for every term S^(n) of modified_charges (k_l2p).
// The self energy does not depend on positions.
#include <algorithm>

#include "kernels.cuh"
#include "pair.cuh"

namespace ankh_b200 {

namespace {

__device__ __forceinline__ unsigned compact3f(unsigned v) {
  v &= 0x09249249u;
  v = (v ^ (v >> 2)) & 0x030c30c3u;
  v = (v ^ (v >> 4)) & 0x0300f00fu;
  v = (v ^ (v >> 8)) & 0x030000ffu;
  v = (v ^ (v >> 16)) & 0x000003ffu;
  return v;
}
__device__ __forceinline__ unsigned spread3f(unsigned v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
// split_extended (octree.cpp:11-14)
__device__ __forceinline__ void split_extf(int ext, int n, int& in_box, int& image) {
  image = ext >= 0 ? ext / n : -((-ext + n - 1) / n);
  in_box = ext - n * image;
}

// ---------------------------------------------------------------- near field
constexpr int kForceTPB = 256;

// kDsrc: also the derivative of the pair energies with respect to the
// target's 10 moments (pair_dsrc) into d_near[10 j] (sorted order);
// kGrad = false: the moment derivatives alone (a field evaluation of the
// induced-dipole solve: no pair gradient, f_near untouched)
template <int NT, bool kDsrc, bool kGrad = true>
__global__ void __launch_bounds__(kForceTPB, 2) k_p2p_force(const double* __restrict__ part,
                                                             const unsigned* __restrict__ leaf_off,
                                                             const unsigned* __restrict__ leaf_mp, int depth,
                                                             int periodic, double period,
                                                             const __grid_constant__ P2PParams pp, int cap,
                                                             double* __restrict__ f_near,
                                                             double* __restrict__ d_near) {
  extern __shared__ __align__(16) double sm[];  // cap x kRec staged sources
  __shared__ int seg_begin[27], seg_prefix[28], seg_n, any_mp;
  __shared__ double seg_shift[27][3];
  __shared__ double red[kForceTPB * 3];
  const int tid = threadIdx.x;
  const int n = 1 << depth;
  const unsigned morton = blockIdx.x;
  const int ax = static_cast<int>(compact3f(morton >> 2)), ay = static_cast<int>(compact3f(morton >> 1)),
            az = static_cast<int>(compact3f(morton));
  const unsigned leaf = static_cast<unsigned>((ax * n + ay) * n + az);
  const int a_begin = static_cast<int>(leaf_off[leaf]);
  const int na = static_cast<int>(leaf_off[leaf + 1]) - a_begin;
  if (na == 0) return;
  // segment table: lane 0 = own leaf, lanes 1..26 = the 26 neighbours
  if (tid < 32) {
    const int lane = tid;
    int bb = 0, nb = 0;
    bool lmp = false;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    if (lane == 0) {
      bb = a_begin;
      nb = na;
      lmp = leaf_mp[leaf] != 0u;
    } else if (lane <= 26) {
      const int d = lane < 14 ? lane - 1 : lane;  // skip the centre (13)
      const int ext[3] = {ax + d / 9 - 1, ay + (d / 3) % 3 - 1, az + d % 3 - 1};
      int in[3], img[3];
      bool ok = true;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (!periodic && (ext[k] < 0 || ext[k] >= n)) ok = false;
        split_extf(ext[k], n, in[k], img[k]);
      }
      if (ok) {
        const unsigned b = static_cast<unsigned>((in[0] * n + in[1]) * n + in[2]);
        bb = static_cast<int>(leaf_off[b]);
        nb = static_cast<int>(leaf_off[b + 1]) - bb;
        lmp = nb > 0 && leaf_mp[b] != 0u;
        sx = period * img[0];
        sy = period * img[1];
        sz = period * img[2];
      }
    }
    const unsigned keep = __ballot_sync(0xffffffffu, lane == 0 || nb > 0);
    const unsigned mps = __ballot_sync(0xffffffffu, lmp);
    int incl = nb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if ((keep >> lane) & 1u) {
      const int slot = __popc(keep & ((1u << lane) - 1u));
      seg_begin[slot] = bb;
      seg_shift[slot][0] = sx;
      seg_shift[slot][1] = sy;
      seg_shift[slot][2] = sz;
      seg_prefix[slot + 1] = incl;
    }
    if (lane == 0) {
      seg_prefix[0] = 0;
      seg_n = __popc(keep);
      any_mp = mps != 0u;
    }
  }
  __syncthreads();
  const int total = seg_prefix[seg_n];
  const bool mp = any_mp != 0;
  for (int t0 = 0; t0 < na; t0 += kForceTPB) {
    const int nt = min(kForceTPB, na - t0);
    const int S = kForceTPB / nt;
    const bool active = tid < S * nt;
    const int il = t0 + (active ? tid % nt : 0), sl = active ? tid / nt : 0;
    const Target tg = load_target(part + static_cast<std::size_t>(a_begin + il) * kRec);
    double grad[3] = {0.0, 0.0, 0.0};
    double ds[10] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int c0 = 0; c0 < total; c0 += cap) {
      const int cn = min(cap, total - c0);
      ANKH_DASSERT(cn > 0 && cn <= cap);
      __syncthreads();
      for (int q = tid; q < cn; q += kForceTPB) {
        const int g = c0 + q;
        int sgi = 0;
        while (g >= seg_prefix[sgi + 1]) ++sgi;
        const double2* r = reinterpret_cast<const double2*>(
            part + static_cast<std::size_t>(seg_begin[sgi] + (g - seg_prefix[sgi])) * kRec);
        double2* d = reinterpret_cast<double2*>(sm + static_cast<std::size_t>(q) * kRec);
        double2 v0 = __ldg(r), v1 = __ldg(r + 1);
        v0.x = v0.x + seg_shift[sgi][0];  // positions[iy] + shift (fmm.cpp:319)
        v0.y = v0.y + seg_shift[sgi][1];
        v1.x = v1.x + seg_shift[sgi][2];
        d[0] = v0;
        d[1] = v1;
#pragma unroll
        for (int k = 2; k < 7; ++k) d[k] = __ldg(r + k);
      }
      __syncthreads();
      if (!active) continue;
      const int skip = il - c0;  // the target itself (own leaf = virtual [0, na))
      if (mp) {
        for (int j = sl; j < cn; j += S)
          if (j != skip) {
            if (kGrad) pair_grad_mp<NT>(tg, sm + static_cast<std::size_t>(j) * kRec, pp, grad);
            if (kDsrc) pair_dsrc<NT>(tg, sm + static_cast<std::size_t>(j) * kRec, pp, ds);
          }
      } else {
        for (int j = sl; j < cn; j += S)
          if (j != skip) {
            if (kGrad) pair_grad_q<NT>(tg, sm + static_cast<std::size_t>(j) * kRec, pp, grad);
            if (kDsrc) pair_dsrc<NT>(tg, sm + static_cast<std::size_t>(j) * kRec, pp, ds);
          }
      }
    }
    // fixed-order sum over the target's slices; F = -grad
    __syncthreads();
    if (kGrad) {
#pragma unroll
      for (int d = 0; d < 3; ++d) red[3 * tid + d] = grad[d];
      __syncthreads();
      if (tid < nt) {
        double f[3] = {0.0, 0.0, 0.0};
        for (int s = 0; s < S; ++s)
#pragma unroll
          for (int d = 0; d < 3; ++d) f[d] += red[3 * (s * nt + tid) + d];
        double* out = f_near + 3 * static_cast<std::size_t>(a_begin + t0 + tid);
#pragma unroll
        for (int d = 0; d < 3; ++d) out[d] = -f[d];
      }
    }
    if (kDsrc) {  // the same fixed-order slice sum, staged in the (finished) source buffer
      ANKH_DASSERT(cap * kRec >= 10 * kForceTPB);
      __syncthreads();
#pragma unroll
      for (int d = 0; d < 10; ++d) sm[10 * tid + d] = ds[d];
      __syncthreads();
      if (tid < nt) {
        double v[10] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int s_ = 0; s_ < S; ++s_)
#pragma unroll
          for (int d = 0; d < 10; ++d) v[d] += sm[10 * (s_ * nt + tid) + d];
        double* out = d_near + 10 * static_cast<std::size_t>(a_begin + t0 + tid);
#pragma unroll
        for (int d = 0; d < 10; ++d) out[d] = v[d];
      }
    }
  }
}

// Forces only (no moment derivatives): the 13 lex-positive neighbours of the
// energy's half shell (fmm.cpp:284-292) with Newton's third law -- the pair
// energy depends on x_a - x_b - shift alone, so grad_b e = -grad_a e and every
// neighbour pair is evaluated once (half k_p2p_force's pair count; own-leaf
// pairs stay one-sided).  Deterministic, no atomics:
//  * a tile of <= 32 targets sits on P = 2^ceil(log2 nt) adjacent lanes, the
//    256 / P lane groups own disjoint contiguous blocks of the staged sources,
//    and lane il walks its group's block rotated by il: at every step the
//    lanes of a group touch distinct sources, a group never leaves its warp,
//    and __syncwarp() orders the steps, so the source-side sums fb[] (shared)
//    see one writer at a time in a fixed order;
//  * the target-side sums are reduced over the groups in a fixed order (as
//    in k_p2p_force) and belong to this CTA alone;
//  * the source-side sums go to f_slot[direction][particle]: leaf B's slot d
//    is written by the one CTA of leaf B - d, and k_force_out adds the 13
//    slots in a fixed order (slots of absent or empty neighbours stay at the
//    zero the launcher sets).
template <int NT>
__global__ void __launch_bounds__(kForceTPB, 2) k_p2p_force_half(const double* __restrict__ part,
                                                                  const unsigned* __restrict__ leaf_off,
                                                                  const unsigned* __restrict__ leaf_mp, int depth,
                                                                  int periodic, double period,
                                                                  const __grid_constant__ P2PParams pp, int cap,
                                                                  double* __restrict__ f_near,
                                                                  double* __restrict__ f_slot,
                                                                  std::size_t slot_stride) {
  extern __shared__ __align__(16) double sm[];  // cap x kRec staged sources + 3 x cap source-side sums
  __shared__ int seg_begin[14], seg_prefix[15], seg_dir[14], seg_n, any_mp;
  __shared__ double seg_shift[14][3];
  __shared__ double red[kForceTPB * 3];
  double* const fb = sm + static_cast<std::size_t>(cap) * kRec;  // fb[d * cap + j]
  const int tid = threadIdx.x;
  const int n = 1 << depth;
  const unsigned morton = blockIdx.x;
  const int ax = static_cast<int>(compact3f(morton >> 2)), ay = static_cast<int>(compact3f(morton >> 1)),
            az = static_cast<int>(compact3f(morton));
  const unsigned leaf = static_cast<unsigned>((ax * n + ay) * n + az);
  const int a_begin = static_cast<int>(leaf_off[leaf]);
  const int na = static_cast<int>(leaf_off[leaf + 1]) - a_begin;
  if (na == 0) return;
  // segment table: lane 0 = own leaf, lanes 1..13 = the lex-positive
  // directions (0,0,1), (0,1,-1..1), (1,-1..1,-1..1), as k_p2p orders them
  if (tid < 32) {
    const int lane = tid;
    int bb = 0, nb = 0;
    bool lmp = false;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    if (lane == 0) {
      bb = a_begin;
      nb = na;
      lmp = leaf_mp[leaf] != 0u;
    } else if (lane <= 13) {
      const int d = lane - 1;
      const int ox = d < 4 ? 0 : 1;
      const int oy = d == 0 ? 0 : (d < 4 ? 1 : (d - 4) / 3 - 1);
      const int oz = d == 0 ? 1 : (d < 4 ? d - 2 : (d - 4) % 3 - 1);
      const int ext[3] = {ax + ox, ay + oy, az + oz};
      int in[3], img[3];
      bool ok = true;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (!periodic && (ext[k] < 0 || ext[k] >= n)) ok = false;
        split_extf(ext[k], n, in[k], img[k]);
      }
      if (ok) {
        const unsigned b = static_cast<unsigned>((in[0] * n + in[1]) * n + in[2]);
        bb = static_cast<int>(leaf_off[b]);
        nb = static_cast<int>(leaf_off[b + 1]) - bb;
        lmp = nb > 0 && leaf_mp[b] != 0u;
        sx = period * img[0];
        sy = period * img[1];
        sz = period * img[2];
      }
    }
    const unsigned keep = __ballot_sync(0xffffffffu, lane == 0 || nb > 0);
    const unsigned mps = __ballot_sync(0xffffffffu, lmp);
    int incl = nb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if ((keep >> lane) & 1u) {
      const int slot = __popc(keep & ((1u << lane) - 1u));
      seg_begin[slot] = bb;
      seg_dir[slot] = lane;
      seg_shift[slot][0] = sx;
      seg_shift[slot][1] = sy;
      seg_shift[slot][2] = sz;
      seg_prefix[slot + 1] = incl;
    }
    if (lane == 0) {
      seg_prefix[0] = 0;
      seg_n = __popc(keep);
      any_mp = mps != 0u;
    }
  }
  __syncthreads();
  const int total = seg_prefix[seg_n];
  const bool mp = any_mp != 0;
  for (int c0 = 0; c0 < total; c0 += cap) {
    const int cn = min(cap, total - c0);
    ANKH_DASSERT(cn > 0 && cn <= cap);
    __syncthreads();  // the previous chunk's sums are flushed
    for (int q = tid; q < cn; q += kForceTPB) {
      const int g = c0 + q;
      int sgi = 0;
      while (g >= seg_prefix[sgi + 1]) ++sgi;
      const double2* r = reinterpret_cast<const double2*>(
          part + static_cast<std::size_t>(seg_begin[sgi] + (g - seg_prefix[sgi])) * kRec);
      double2* d = reinterpret_cast<double2*>(sm + static_cast<std::size_t>(q) * kRec);
      double2 v0 = __ldg(r), v1 = __ldg(r + 1);
      v0.x = v0.x + seg_shift[sgi][0];  // positions[iy] + shift (fmm.cpp:319)
      v0.y = v0.y + seg_shift[sgi][1];
      v1.x = v1.x + seg_shift[sgi][2];
      d[0] = v0;
      d[1] = v1;
#pragma unroll
      for (int k = 2; k < 7; ++k) d[k] = __ldg(r + k);
      fb[q] = 0.0;
      fb[cap + q] = 0.0;
      fb[2 * cap + q] = 0.0;
    }
    __syncthreads();
    const int own_end = na - c0;  // chunk entries below it are the own leaf's
    for (int t0 = 0; t0 < na; t0 += 32) {
      const int nt = min(32, na - t0);
      int P = 1;
      while (P < nt) P <<= 1;
      const int S = kForceTPB / P;  // lane groups = source blocks
      const int il = tid & (P - 1), grp = tid / P;
      const bool active = il < nt;
      const int m = (cn + S - 1) / S;  // sources per block
      const int R = max(m, P);         // rotation length: distinct lanes, distinct sources
      const int jb = grp * m;
      const int jn = min(m, cn - jb);  // <= 0: an empty block
      const Target tg = load_target(part + static_cast<std::size_t>(a_begin + t0 + (active ? il : 0)) * kRec);
      const int self = t0 + il - c0;  // the target itself (own leaf = entries [0, na) of the list)
      double grad[3] = {0.0, 0.0, 0.0};
      int p = il;
      for (int i = 0; i < R; ++i) {
        const int j = jb + p;
        if (active && p < jn && j != self) {
          double gp[3] = {0.0, 0.0, 0.0};
          const double* sb = sm + static_cast<std::size_t>(j) * kRec;
          if (mp)
            pair_grad_mp<NT>(tg, sb, pp, gp);
          else
            pair_grad_q<NT>(tg, sb, pp, gp);
          grad[0] += gp[0];
          grad[1] += gp[1];
          grad[2] += gp[2];
          if (j >= own_end) {  // F_b = -grad_b e = +grad_a e
            fb[j] += gp[0];
            fb[cap + j] += gp[1];
            fb[2 * cap + j] += gp[2];
          }
        }
        __syncwarp();
        if (++p == R) p = 0;
      }
      // fixed-order sum over the target's groups; F = -grad
#pragma unroll
      for (int d = 0; d < 3; ++d) red[3 * tid + d] = grad[d];
      __syncthreads();
      if (tid < nt) {
        double f[3] = {0.0, 0.0, 0.0};
        for (int s = 0; s < S; ++s)
#pragma unroll
          for (int d = 0; d < 3; ++d) f[d] += red[3 * (s * P + tid) + d];
        double* out = f_near + 3 * static_cast<std::size_t>(a_begin + t0 + tid);
#pragma unroll
        for (int d = 0; d < 3; ++d) out[d] = c0 == 0 ? -f[d] : out[d] - f[d];
      }
      __syncthreads();
    }
    // the neighbours' sums of this chunk, each (direction, particle) slot once
    for (int q = tid; q < cn; q += kForceTPB) {
      const int g = c0 + q;
      if (g < na) continue;
      int sgi = 0;
      while (g >= seg_prefix[sgi + 1]) ++sgi;
      const std::size_t b = static_cast<std::size_t>(seg_begin[sgi] + (g - seg_prefix[sgi]));
      double* out = f_slot + static_cast<std::size_t>(seg_dir[sgi] - 1) * slot_stride + 3 * b;
      out[0] = fb[q];
      out[1] = fb[cap + q];
      out[2] = fb[2 * cap + q];
    }
  }
}

// ------------------------------------------------- far field: dE/dM per cell
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}

// bulk (TMA 1-D) row copies completing on an mbarrier (ANKH_LOC_BULK variant)
__device__ __forceinline__ unsigned loc_saddr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void loc_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(loc_saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void loc_mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(loc_saddr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void loc_mbar_wait(unsigned long long* b, unsigned parity) {
  const unsigned a = loc_saddr(b);
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void loc_bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          loc_saddr(dst)),
      "l"(src), "r"(bytes), "r"(loc_saddr(bar))
      : "memory");
}

constexpr int kLocWarps = 4;              // 8 targets per warp, 32 per CTA
// A/B knobs (make variants VAR_SRC=k_forces), k_m2l_local at config 3: rows 32
// with 3 CTAs per SM asked for (160 registers) 7.32 ms; no minimum (162
// registers) 7.65; rows 16 / 4 CTAs 7.44; rows 24 / 4 CTAs 11.0 (ranks of 32
// take two passes); rows 16 / 5 CTAs (96 registers, spills) 13.8; two or four
// GEMM 1 accumulator sets 9.0 / 10.7; 48 rows (2 CTAs) 16.1; bulk row copies
// on mbarriers (ANKH_LOC_BULK) 7.30 against 7.40 in the same run; GEMM 1's
// partner rows as batches of eight 16-B loads per lane (with 16-B A fragments)
// 7.59 against 7.41.  Tiles of one
// boundary signature (one factor pass per offset instead of 1.12 on average)
// add 14 % more tiles and gain nothing: the kernel is bound by the per-pass
// latency chain (stage -> barrier -> GEMM 1 -> GEMM 2) at three CTAs per SM,
// the DMMA pipe ~60 % active.
#ifndef ANKH_LOC_ROWS
#define ANKH_LOC_ROWS 32
#endif
#ifndef ANKH_LOC_MINB
#define ANKH_LOC_MINB 3
#endif
#define ANKH_LOC_BOUNDS __launch_bounds__(kLocWarps * 32, ANKH_LOC_MINB)
constexpr int kLocRows = ANKH_LOC_ROWS;   // factor rows staged per pass (multiple of 8)
constexpr int kLocRowTiles = 16;          // Lambda rows per row group: 128

// One CTA = up to 32 target cells of one parity class at one level (Morton
// m = 8 (j0 + i) + cls); every warp owns 8 of them.  For each of the 189
// partner offsets of the class (octree.cpp:79-87) and each factor pass (the
// offset's own factors for canonical pairs, the mirror's for the others):
//   V = X [M_p ...]      (X = R_o, or L_o' swapped; rank rows x 8 partners)
//   Lambda += Y^T V      (Y = L_o, or R_o'; 128 node rows x 8 targets)
// GEMM 1 takes the partners' expansion rows straight from global (L2) as B
// fragments; V moves from the accumulator layout to GEMM 2's B layout by warp
// shuffles; Lambda stays in registers for all offsets (no atomics).
__global__ void ANKH_LOC_BOUNDS k_m2l_local(
    const double* __restrict__ exp, double* __restrict__ loc, const long long* __restrict__ level_off,
    const double* __restrict__ factors, const M2LOp* __restrict__ ops, const int2* __restrict__ op_of,
    const int4* __restrict__ tiles, int Kp, int periodic, int rows) {
  extern __shared__ __align__(16) double sm[];
  const int KS = Kp + 4;
  // rows (<= kLocRows, a multiple of 8): factor rows staged per pass, fewer
  // than kLocRows when the order's row length would not fit shared memory
  double* sX = sm;               // rows x KS
  double* sY = sX + rows * KS;   // rows x KS
#ifdef ANKH_LOC_BULK
  __shared__ unsigned long long bar_x, bar_y;
  if (threadIdx.x == 0) {
    loc_mbar_init(&bar_x, 1);
    loc_mbar_init(&bar_y, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned bar_phase = 0;
#endif
  const int4 tile = tiles[blockIdx.x];  // (level, cls, j0, count)
  const int level = tile.x, cls = tile.y, count = tile.w;
  const int n = 1 << level;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* E = exp + level_off[level];
  // this lane's B-fragment target (column lane/4) and its two accumulator
  // targets (columns 2 (lane%4) + {0, 1})
  const int ib = warp * 8 + (lane >> 2);
  const bool vb = ib < count;
  const unsigned mt = 8u * static_cast<unsigned>(tile.z + (vb ? ib : 0)) + static_cast<unsigned>(cls);
  const int tx = static_cast<int>(compact3f(mt >> 2)), ty = static_cast<int>(compact3f(mt >> 1)),
            tz = static_cast<int>(compact3f(mt));
  const unsigned t_lex = static_cast<unsigned>((tx * n + ty) * n + tz);
  const int cx = (cls >> 2) & 1, cy = (cls >> 1) & 1, cz = cls & 1;
  const int row_groups = (Kp + 8 * kLocRowTiles - 1) / (8 * kLocRowTiles);
  for (int rg = 0; rg < row_groups; ++rg) {
    const int rows0 = rg * 8 * kLocRowTiles;
    const int row_tiles = min(kLocRowTiles, (Kp - rows0) / 8);
    double lam[kLocRowTiles][2];
#pragma unroll
    for (int M = 0; M < kLocRowTiles; ++M) lam[M][0] = lam[M][1] = 0.0;
    for (int ox = -2 - cx; ox <= 3 - cx; ++ox)
      for (int oy = -2 - cy; oy <= 3 - cy; ++oy)
        for (int oz = -2 - cz; oz <= 3 - cz; ++oz) {
          if (max(max(abs(ox), abs(oy)), abs(oz)) < 2) continue;
          // partner of this lane's B target, and whether (t, p) is canonical
          // (fmm.cpp:246-250: t < s, or t == s with the image lex-positive)
          const int ext[3] = {tx + ox, ty + oy, tz + oz};
          int in[3], img[3];
          bool valid = vb;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            if (!periodic && (ext[k] < 0 || ext[k] >= n)) valid = false;
            split_extf(ext[k], n, in[k], img[k]);
          }
          const unsigned p_lex = static_cast<unsigned>((in[0] * n + in[1]) * n + in[2]);
          const bool lexpos = img[0] != 0 ? img[0] > 0 : (img[1] != 0 ? img[1] > 0 : img[2] > 0);
          const bool canon = t_lex < p_lex || (t_lex == p_lex && lexpos);
          const unsigned pm = (spread3f(static_cast<unsigned>(in[0])) << 2) |
                              (spread3f(static_cast<unsigned>(in[1])) << 1) | spread3f(static_cast<unsigned>(in[2]));
          const double* Mp = E + static_cast<std::size_t>(valid ? pm : 0u) * Kp;
          const int need0 = __syncthreads_or(valid && canon);
          const int need1 = __syncthreads_or(valid && !canon);
          for (int pass = 0; pass < 2; ++pass) {
            if (!(pass == 0 ? need0 : need1)) continue;
            // pass 0: this offset's factors (X = R_o, Y = L_o) for canonical
            // pairs; pass 1: the mirror offset's (X = L_-o, Y = R_-o)
            const int sx = pass == 0 ? ox : -ox, sy = pass == 0 ? oy : -oy, sz = pass == 0 ? oz : -oz;
            const int2 opr = op_of[level * 343 + ((sx + 3) * 7 + (sy + 3)) * 7 + (sz + 3)];
            const bool mine = valid && (pass == 0 ? canon : !canon);
            // every pair the energy counts has its operator (a missing one would drop terms)
            ANKH_DASSERT(!mine || (opr.x >= 0 && opr.y > 0));
            for (int blk = 0; blk < opr.y; ++blk) {
              const M2LOp op = ops[opr.x + blk];
              const double* Lg = factors + op.factor_off;
              const double* Rg = Lg + static_cast<std::size_t>(op.kp) * Kp;
              const double* Xg = pass == 0 ? Rg : Lg;
              const double* Yg = pass == 0 ? Lg : Rg;
              for (int r0 = 0; r0 < op.kp; r0 += rows) {
                const int rb = min(rows, op.kp - r0);  // multiple of 8
                __syncthreads();  // previous readers of sX / sY are done
#ifdef ANKH_LOC_BULK
                // one bulk copy per factor row (warp 0), X and Y on their own
                // barriers: GEMM 1 starts when X is in, Y lands meanwhile
                if (warp == 0) {
                  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                  if (lane == 0) {
                    loc_mbar_expect(&bar_x, static_cast<unsigned>(rb * Kp) * 8u);
                    loc_mbar_expect(&bar_y, static_cast<unsigned>(rb * Kp) * 8u);
                  }
                  __syncwarp();
                  for (int r = lane; r < rb; r += 32) {
                    loc_bulk_g2s(sX + r * KS, Xg + static_cast<std::size_t>(r0 + r) * Kp,
                                 static_cast<unsigned>(Kp) * 8u, &bar_x);
                    loc_bulk_g2s(sY + r * KS, Yg + static_cast<std::size_t>(r0 + r) * Kp,
                                 static_cast<unsigned>(Kp) * 8u, &bar_y);
                  }
                }
                loc_mbar_wait(&bar_x, bar_phase);
#else
                for (int w = threadIdx.x; w < rb * (Kp / 2); w += kLocWarps * 32) {
                  const int r = w / (Kp / 2), c2 = 2 * (w - (Kp / 2) * (w / (Kp / 2)));
                  cp_async16(sX + r * KS + c2, Xg + static_cast<std::size_t>(r0 + r) * Kp + c2);
                  cp_async16(sY + r * KS + c2, Yg + static_cast<std::size_t>(r0 + r) * Kp + c2);
                }
                asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
                __syncthreads();
#endif
                // GEMM 1: V (rb x 8) = X (rb x Kp) . [M_p] (Kp x 8)
                double v[kLocRows / 8][2];
#pragma unroll
                for (int m = 0; m < kLocRows / 8; ++m) v[m][0] = v[m][1] = 0.0;
                const int rb8 = rb / 8;
                for (int ks = 0; ks < Kp / 4; ++ks) {
                  const double b = mine ? __ldg(Mp + 4 * ks + (lane & 3)) : 0.0;
#pragma unroll
                  for (int m = 0; m < kLocRows / 8; ++m)
                    if (m < rb8) dmma(v[m], sX[(8 * m + (lane >> 2)) * KS + 4 * ks + (lane & 3)], b);
                }
#ifdef ANKH_LOC_BULK
                loc_mbar_wait(&bar_y, bar_phase);
                bar_phase ^= 1u;
#endif
                // GEMM 2: Lambda (rows x 8) += Y^T (rows x rb) . V (rb x 8)
#pragma unroll
                for (int s = 0; s < kLocRows / 4; ++s) {
                  if (s < rb / 4) {
                    const int src = 4 * ((lane & 3) + 4 * (s & 1)) + (lane >> 3);
                    double v0 = 0.0, v1 = 0.0;
#pragma unroll
                    for (int m = 0; m < kLocRows / 8; ++m)
                      if (m == (s >> 1)) {
                        v0 = __shfl_sync(0xffffffffu, v[m][0], src);
                        v1 = __shfl_sync(0xffffffffu, v[m][1], src);
                      }
                    const double bb = ((lane >> 2) & 1) ? v1 : v0;
                    const double* yrow = sY + (4 * s + (lane & 3)) * KS + rows0 + (lane >> 2);
#pragma unroll
                    for (int M = 0; M < kLocRowTiles; ++M)
                      if (M < row_tiles) dmma(lam[M], yrow[8 * M], bb);
                  }
                }
              }
            }
          }
        }
    // Lambda rows [rows0, rows0 + 8 row_tiles) of the targets of columns
    // 2 (lane%4) + {0, 1}
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ic = warp * 8 + 2 * (lane & 3) + h;
      if (ic >= count) continue;
      const unsigned mc = 8u * static_cast<unsigned>(tile.z + ic) + static_cast<unsigned>(cls);
      double* out = loc + level_off[level] + static_cast<std::size_t>(mc) * Kp + rows0 + (lane >> 2);
#pragma unroll
      for (int M = 0; M < kLocRowTiles; ++M)
        if (M < row_tiles) out[8 * M] = lam[M][h];
    }
  }
}

// ------------------------------------------------------- periodic far images
// Lambda_root += (T x T x T)^T C (T x T x T) M_root, C[x, y] = gen[(x - y) mod
// (2L-1)] per axis (the circulant embedding of spectral.cpp; gen[d] = gen[-d],
// so C is symmetric and dE_per/dv = C v for E_per = 1/2 v^T C v).
constexpr int kPerLocThreads = 256;
__global__ void __launch_bounds__(kPerLocThreads) k_periodic_local(const double* __restrict__ root,
                                                                   const double* __restrict__ T,
                                                                   const double* __restrict__ gen, int L,
                                                                   double* __restrict__ loc_root) {
  extern __shared__ double sm[];
  const int L2 = L * L, K = L2 * L, eb = 2 * L - 1;
  double* a = sm;      // K
  double* b = a + K;   // K
  double* c = b + K;   // K
  const int tid = threadIdx.x;
  for (int e = tid; e < K; e += kPerLocThreads) a[e] = root[e];
  __syncthreads();
  // v = (T x T x T) M: z, then y, then x (T(k, l) = T[k L + l])
  for (int e = tid; e < K; e += kPerLocThreads) {
    const int ij = e / L, k = e % L;
    double s = 0.0;
    for (int l = 0; l < L; ++l) s += T[k * L + l] * a[ij * L + l];
    b[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < K; e += kPerLocThreads) {
    const int i = e / L2, j = (e / L) % L, k = e % L;
    double s = 0.0;
    for (int l = 0; l < L; ++l) s += T[j * L + l] * b[(i * L + l) * L + k];
    c[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < K; e += kPerLocThreads) {
    const int i = e / L2, jk = e % L2;
    double s = 0.0;
    for (int l = 0; l < L; ++l) s += T[i * L + l] * c[l * L2 + jk];
    a[e] = s;  // v
  }
  __syncthreads();
  // w = C v on the L^3 block
  for (int e = tid; e < K; e += kPerLocThreads) {
    const int xi = e / L2, xj = (e / L) % L, xk = e % L;
    double s = 0.0;
    for (int f = 0; f < K; ++f) {
      const int yi = f / L2, yj = (f / L) % L, yk = f % L;
      const int di = xi - yi, dj = xj - yj, dk = xk - yk;
      const int gi = di >= 0 ? di : di + eb, gj = dj >= 0 ? dj : dj + eb, gk = dk >= 0 ? dk : dk + eb;
      s += gen[(gi * eb + gj) * eb + gk] * a[f];
    }
    b[e] = s;
  }
  __syncthreads();
  // Lambda += (T^T x T^T x T^T) w
  for (int e = tid; e < K; e += kPerLocThreads) {
    const int ij = e / L, c0 = e % L;
    double s = 0.0;
    for (int k = 0; k < L; ++k) s += T[k * L + c0] * b[ij * L + k];
    c[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < K; e += kPerLocThreads) {
    const int i = e / L2, b0 = (e / L) % L, c0 = e % L;
    double s = 0.0;
    for (int j = 0; j < L; ++j) s += T[j * L + b0] * c[(i * L + j) * L + c0];
    a[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < K; e += kPerLocThreads) {
    const int a0 = e / L2, bc = e % L2;
    double s = 0.0;
    for (int i = 0; i < L; ++i) s += T[i * L + a0] * a[i * L2 + bc];
    loc_root[e] += s;
  }
}

// ----------------------------------------------------------------- L2L
// Lambda_child(cx,cy,cz)[a,b,c] += sum_ijk T_cx(i,a) T_cy(j,b) T_cz(k,c) Lambda_parent[i,j,k]
// (the transpose of M2M: parent[i,j,k] += sum T_cx(i,a) T_cy(j,b) T_cz(k,c) child[a,b,c]).
constexpr int kL2LThreads = 128;
template <int L>
__global__ void __launch_bounds__(kL2LThreads) k_l2l(const double* __restrict__ loc_parent,
                                                     double* __restrict__ loc_child,
                                                     const double* __restrict__ m2m_g) {
  constexpr int L2 = L * L, K = L2 * L, KS = exp_stride(K);
  extern __shared__ __align__(16) double sm[];
  double* M = sm;        // 2 x L x L: M[c][i][a] = T_c(i, a)
  double* P = M + 2 * L2;  // K
  double* U1 = P + K;    // 2 K: [cz][i][j][c]
  double* U2 = U1 + 2 * K;  // 4 K: [cy][cz][i][b][c]
  const unsigned p = blockIdx.x;
  for (int w = threadIdx.x; w < 2 * L2; w += kL2LThreads) M[w] = m2m_g[w];
  for (int w = threadIdx.x; w < K; w += kL2LThreads) P[w] = loc_parent[static_cast<std::size_t>(p) * KS + w];
  __syncthreads();
  for (int w = threadIdx.x; w < 2 * K; w += kL2LThreads) {
    const int cz = w / K, e = w % K, ij = e / L, c = e % L;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < L; ++k) s += M[cz * L2 + k * L + c] * P[ij * L + k];
    U1[w] = s;
  }
  __syncthreads();
  for (int w = threadIdx.x; w < 4 * K; w += kL2LThreads) {
    const int q = w / K, cy = q >> 1, cz = q & 1, e = w % K;
    const int i = e / L2, b = (e / L) % L, c = e % L;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < L; ++j) s += M[cy * L2 + j * L + b] * U1[cz * K + (i * L + j) * L + c];
    U2[w] = s;
  }
  __syncthreads();
  for (int w = threadIdx.x; w < 8 * K; w += kL2LThreads) {
    const int ch = w / K, cx = ch >> 2, q = ch & 3, e = w % K;
    const int a = e / L2, bc = e % L2;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) s += M[cx * L2 + i * L + a] * U2[q * K + i * L2 + bc];
    loc_child[(8 * static_cast<std::size_t>(p) + ch) * KS + e] += s;
  }
}

// ----------------------------------------------------------------- L2P
// dE_far/dx_a = sum_terms coef * (d/dx)[S_x^(nx) S_y^(ny) S_z^(nz)] . Lambda_leaf
// with d/dx S^(n) = S^(n+1) (chebyshev.cpp:85-115: S^(n) = rad^-n H D^n T(local)).
constexpr int kL2PThreads = 64;
template <int L>
__global__ void __launch_bounds__(kL2PThreads) k_l2p(const double* __restrict__ part,
                                                     const unsigned* __restrict__ leaf_off, int depth,
                                                     double rb, const double* __restrict__ hd4,
                                                     const double* __restrict__ loc_leaf,
                                                     double* __restrict__ f_far, double* __restrict__ d_far) {
  constexpr int L2 = L * L, K = L2 * L, KS = exp_stride(K);
  __shared__ double lam[K];
  __shared__ double hd[4 * L2];  // H D^n, n = 0..3
  const unsigned m = blockIdx.x;
  const int n = 1 << depth;
  const int ci0 = static_cast<int>(compact3f(m >> 2)), ci1 = static_cast<int>(compact3f(m >> 1)),
            ci2 = static_cast<int>(compact3f(m));
  const unsigned leaf = (static_cast<unsigned>(ci0) * n + ci1) * n + ci2;
  const unsigned begin = leaf_off[leaf];
  const int cnt = static_cast<int>(leaf_off[leaf + 1] - begin);
  if (cnt == 0) return;
  for (int w = threadIdx.x; w < K; w += kL2PThreads) lam[w] = loc_leaf[static_cast<std::size_t>(m) * KS + w];
  for (int w = threadIdx.x; w < 4 * L2; w += kL2PThreads) hd[w] = hd4[w];
  __syncthreads();
  // cell_geometry (octree.cpp:18-25)
  const double rad = rb / n;
  const double cc[3] = {-rb + rad * (2 * ci0 + 1), -rb + rad * (2 * ci1 + 1), -rb + rad * (2 * ci2 + 1)};
  const double inv_rad = 1.0 / rad;
  for (int pi = threadIdx.x; pi < cnt; pi += kL2PThreads) {
    const double* r = part + static_cast<std::size_t>(begin + pi) * kRec;
    double s[3][4][L];  // axis, derivative order 0..3, node
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const double l = (r[ax] - cc[ax]) * inv_rad;
      double t[L];
      t[0] = 1.0;
      if (L > 1) t[1] = l;
#pragma unroll
      for (int q = 2; q < L; ++q) t[q] = 2.0 * l * t[q - 1] - t[q - 2];
      double scale = 1.0;
#pragma unroll
      for (int d = 0; d < 4; ++d) {
#pragma unroll
        for (int i = 0; i < L; ++i) {
          double v = 0.0;
#pragma unroll
          for (int q = 0; q < L; ++q) v += hd[d * L2 + i * L + q] * t[q];
          s[ax][d][i] = scale * v;
        }
        scale *= inv_rad;
      }
    }
    // W[dx][dy][dz] = sum_ijk lam[i,j,k] Sx^(dx)_i Sy^(dy)_j Sz^(dz)_k for dx + dy + dz <= 3
    double W[4][4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) W[a][b][c] = 0.0;
    for (int i = 0; i < L; ++i) {
      double Y[4][4];  // [dy][dz]
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) Y[b][c] = 0.0;
      for (int j = 0; j < L; ++j) {
        double Z[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < L; ++k) {
          const double lv = lam[(i * L + j) * L + k];
#pragma unroll
          for (int c = 0; c < 4; ++c) Z[c] += lv * s[2][c][k];
        }
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int c = 0; c + b < 4; ++c) Y[b][c] += s[1][b][j] * Z[c];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; a + b < 4; ++b)
#pragma unroll
          for (int c = 0; a + b + c < 4; ++c) W[a][b][c] += s[0][a][i] * Y[b][c];
    }
    // the 10 terms of modified_charges (chebyshev.cpp:173-184)
    const double q = r[3], mx = r[4], my = r[5], mz = r[6], txx = r[7], txy = r[8], txz = r[9],
                 tyy = r[10], tyz = r[11], tzz = r[12];
    struct Term {
      double c;
      int x, y, z;
    };
    const Term terms[10] = {{q, 0, 0, 0},          {mx, 1, 0, 0},        {my, 0, 1, 0},
                            {mz, 0, 0, 1},         {txx, 2, 0, 0},       {tyy, 0, 2, 0},
                            {tzz, 0, 0, 2},        {2.0 * txy, 1, 1, 0}, {2.0 * txz, 1, 0, 1},
                            {2.0 * tyz, 0, 1, 1}};
    double g[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int t = 0; t < 10; ++t) {
      g[0] += terms[t].c * W[terms[t].x + 1][terms[t].y][terms[t].z];
      g[1] += terms[t].c * W[terms[t].x][terms[t].y + 1][terms[t].z];
      g[2] += terms[t].c * W[terms[t].x][terms[t].y][terms[t].z + 1];
    }
    double* out = f_far + 3 * static_cast<std::size_t>(begin + pi);
    out[0] = -g[0];
    out[1] = -g[1];
    out[2] = -g[2];
    if (d_far) {  // dE_far/ds_a: the terms' own basis products (no extra derivative)
      double* o = d_far + 10 * static_cast<std::size_t>(begin + pi);
      o[0] = W[0][0][0];
      o[1] = W[1][0][0];
      o[2] = W[0][1][0];
      o[3] = W[0][0][1];
      o[4] = W[2][0][0];
      o[5] = 2.0 * W[1][1][0];
      o[6] = 2.0 * W[1][0][1];
      o[7] = W[0][2][0];
      o[8] = 2.0 * W[0][1][1];
      o[9] = W[0][0][2];
    }
  }
}

// dE/ds[idx[j]] = near[j] + far[j] + the self energy's derivative
// (kernel.cpp:206-213: -xi/sqrt(pi) (q^2 + c_mu |mu|^2 + c_th Theta:Theta),
// Theta:Theta with the off-diagonals twice)
__global__ void k_dsrc_out(const double* __restrict__ d_near, const double* __restrict__ d_far,
                           const double* __restrict__ part, const unsigned* __restrict__ sorted, std::size_t n,
                           double self_scale, double c_mu, double c_th, double* __restrict__ out) {
  const std::size_t j = static_cast<std::size_t>(blockIdx.x) * 256 + threadIdx.x;
  if (j >= n) return;
  const double* r = part + j * kRec;  // x y z q mx my mz txx txy txz tyy tyz tzz tr
  const double self[10] = {2.0 * r[3],        2.0 * c_mu * r[4], 2.0 * c_mu * r[5], 2.0 * c_mu * r[6],
                           2.0 * c_th * r[7], 4.0 * c_th * r[8], 4.0 * c_th * r[9], 2.0 * c_th * r[10],
                           4.0 * c_th * r[11], 2.0 * c_th * r[12]};
  double* o = out + 10 * static_cast<std::size_t>(sorted[j]);
#pragma unroll
  for (int d = 0; d < 10; ++d) o[d] = (d_near[10 * j + d] + d_far[10 * j + d]) + self_scale * self[d];
}

// forces[idx[j]] = near[j] + far[j]: back to the caller's particle order
// (+ the 13 source-side slots of k_p2p_force_half, added in direction order)
__global__ void k_force_out(const double* __restrict__ f_near, const double* __restrict__ f_far,
                            const double* __restrict__ f_slot, std::size_t slot_stride,
                            const unsigned* __restrict__ sorted, std::size_t n, double* __restrict__ out) {
  const std::size_t j = static_cast<std::size_t>(blockIdx.x) * 256 + threadIdx.x;
  if (j >= n) return;
  const std::size_t i = sorted[j];
  double f[3] = {f_near[3 * j], f_near[3 * j + 1], f_near[3 * j + 2]};
  if (f_slot) {
#pragma unroll
    for (int k = 0; k < 13; ++k) {
      const double* s = f_slot + k * slot_stride + 3 * j;
#pragma unroll
      for (int d = 0; d < 3; ++d) f[d] += s[d];
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) out[3 * i + d] = f[d] + f_far[3 * j + d];
}

P2PParams make_force_params(double xi, const P2PRadial& rad) {
  P2PParams pp{};
  pp.xi = xi;
  pp.xi2 = xi * xi;
  pp.tx = 2.0 * xi * xi;
  pp.s_lim = rad.s_lim;
  double w = xi;  // xi^(2k+1), as the P2P kernels fold it
  for (int k = 0; k < 14; ++k) {
    pp.p[k] = rad.p[k] * w;
    pp.g[k] = rad.g[k] * w;
    w *= pp.xi2;
  }
  return pp;
}

template <int NT>
void launch_force_near_t(const double* part, const unsigned* leaf_off, const unsigned* leaf_mp, int depth,
                         int periodic, double period, const P2PParams& pp, int cap, double* f_near,
                         double* d_near, double* f_slot, std::size_t slot_stride, cudaStream_t st) {
  const std::size_t smem = sizeof(double) * static_cast<std::size_t>(cap) * kRec;
  if (d_near && !f_near) {
    static std::atomic<unsigned long long> attr{0};
    smem_opt_in(attr, k_p2p_force<NT, true, false>, sizeof(double) * force_max_cap() * kRec);
    k_p2p_force<NT, true, false><<<1u << (3 * depth), kForceTPB, smem, st>>>(
        part, leaf_off, leaf_mp, depth, periodic, period, pp, cap, nullptr, d_near);
  } else if (d_near) {
    static std::atomic<unsigned long long> attr{0};
    smem_opt_in(attr, k_p2p_force<NT, true>, sizeof(double) * force_max_cap() * kRec);
    k_p2p_force<NT, true><<<1u << (3 * depth), kForceTPB, smem, st>>>(part, leaf_off, leaf_mp, depth, periodic,
                                                                      period, pp, cap, f_near, d_near);
  } else if (f_slot) {
    static std::atomic<unsigned long long> attr{0};
    smem_opt_in(attr, k_p2p_force_half<NT>, sizeof(double) * force_half_max_cap() * (kRec + 3));
    k_p2p_force_half<NT><<<1u << (3 * depth), kForceTPB, sizeof(double) * static_cast<std::size_t>(cap) * (kRec + 3),
                           st>>>(part, leaf_off, leaf_mp, depth, periodic, period, pp, cap, f_near, f_slot,
                                 slot_stride);
  } else {
    static std::atomic<unsigned long long> attr{0};
    smem_opt_in(attr, k_p2p_force<NT, false>, sizeof(double) * force_max_cap() * kRec);
    k_p2p_force<NT, false><<<1u << (3 * depth), kForceTPB, smem, st>>>(part, leaf_off, leaf_mp, depth, periodic,
                                                                       period, pp, cap, f_near, nullptr);
  }
}

}  // namespace

int force_max_cap() { return 960; }       // 960 x 112 B = 105 KB: two CTAs per SM
int force_half_max_cap() { return 768; }  // 768 x 136 B = 102 KB (+ 7 KB static): two CTAs per SM

void launch_force_near(const double* part, const unsigned* leaf_off, const unsigned* leaf_mp, int depth,
                       int periodic, double period, double xi, const P2PRadial& rad, int cap, double* f_near,
                       cudaStream_t st, double* d_near, double* f_slot, std::size_t slot_stride) {
  const int cap_max = (f_slot && !d_near) ? force_half_max_cap() : force_max_cap();
  cap = cap < 64 ? 64 : (cap > cap_max ? cap_max : cap);
  if (d_near && cap < kForceTPB) cap = kForceTPB;  // the moment sums are staged in the source buffer
  const P2PParams pp = make_force_params(xi, rad);
#define ANKH_F_NT(N)                                                                                         \
  launch_force_near_t<N>(part, leaf_off, leaf_mp, depth, periodic, period, pp, cap, f_near, d_near, f_slot, \
                         slot_stride, st)
  switch (rad.nterms) {
    case 6: ANKH_F_NT(6); break;
    case 7: ANKH_F_NT(7); break;
    case 8: ANKH_F_NT(8); break;
    case 9: ANKH_F_NT(9); break;
    case 10: ANKH_F_NT(10); break;
    case 12: ANKH_F_NT(12); break;
    default: ANKH_F_NT(14); break;
  }
#undef ANKH_F_NT
}

// factor rows staged per pass: kLocRows, or what the order's row length
// leaves room for (orders 8..10: 24, 16, 8 rows)
int m2l_local_rows(int Kp) {
  const std::size_t row = sizeof(double) * 2 * static_cast<std::size_t>(Kp + 4);
  const int fit = static_cast<int>((224 * 1024) / row) / 8 * 8;
  return std::max(8, std::min(kLocRows, fit));
}
std::size_t m2l_local_smem(int Kp) {
  return sizeof(double) * 2 * m2l_local_rows(Kp) * static_cast<std::size_t>(Kp + 4);
}

void launch_m2l_local(const double* exp, double* loc, const long long* level_off, const double* factors,
                      const M2LOp* ops, const int2* op_of, const int4* tiles, int n_tiles, int Kp, int periodic,
                      cudaStream_t st) {
  if (n_tiles <= 0) return;
  const std::size_t smem = m2l_local_smem(Kp);
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_m2l_local, 225 * 1024);  // the device maximum less the static part: plans of any order
  k_m2l_local<<<n_tiles, kLocWarps * 32, smem, st>>>(exp, loc, level_off, factors, ops, op_of, tiles, Kp,
                                                     periodic, m2l_local_rows(Kp));
}

void launch_periodic_local(const double* root, const double* to_equi, const double* gen, int order,
                           double* loc_root, cudaStream_t st) {
  const int K = order * order * order;
  const std::size_t smem = sizeof(double) * 3 * K;
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_periodic_local, sizeof(double) * 3 * 1000);  // L <= 10
  k_periodic_local<<<1, kPerLocThreads, smem, st>>>(root, to_equi, gen, order, loc_root);
}

#define ANKH_FORCE_ORDERS(CALL) \
  switch (order) {              \
    case 2: CALL(2); break;     \
    case 3: CALL(3); break;     \
    case 4: CALL(4); break;     \
    case 5: CALL(5); break;     \
    case 6: CALL(6); break;     \
    case 7: CALL(7); break;     \
    case 8: CALL(8); break;     \
    case 9: CALL(9); break;     \
    case 10: CALL(10); break;   \
    default: break;             \
  }

void launch_l2l(const double* loc_parent, double* loc_child, int parent_level, int order, const double* m2m,
                cudaStream_t st) {
  const unsigned parents = 1u << (3 * parent_level);
#define ANKH_L2L(N)                                                                       \
  {                                                                                       \
    const std::size_t smem = sizeof(double) * (2 * N * N + 7 * N * N * N);                \
    static std::atomic<unsigned long long> attr{0};                                       \
    smem_opt_in(attr, k_l2l<N>, smem);                                                    \
    k_l2l<N><<<parents, kL2LThreads, smem, st>>>(loc_parent, loc_child, m2m);             \
  }
  ANKH_FORCE_ORDERS(ANKH_L2L)
#undef ANKH_L2L
}

void launch_l2p(const double* part, const unsigned* leaf_off, int depth, int order, double rb, const double* hd4,
                const double* loc_leaf, double* f_far, cudaStream_t st, double* d_far) {
  const unsigned leaves = 1u << (3 * depth);
#define ANKH_L2P(N) k_l2p<N><<<leaves, kL2PThreads, 0, st>>>(part, leaf_off, depth, rb, hd4, loc_leaf, f_far, d_far)
  ANKH_FORCE_ORDERS(ANKH_L2P)
#undef ANKH_L2P
}

void launch_force_out(const double* f_near, const double* f_far, const unsigned* sorted, std::size_t n,
                      double* out, cudaStream_t st, const double* f_slot, std::size_t slot_stride) {
  if (n == 0) return;
  k_force_out<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(f_near, f_far, f_slot, slot_stride, sorted,
                                                                      n, out);
}

void launch_dsrc_out(const double* d_near, const double* d_far, const double* part, const unsigned* sorted,
                     std::size_t n, double xi, int include_self, double* out, cudaStream_t st) {
  if (n == 0) return;
  constexpr double kInvSqrtPiD = 0.56418958354775628695;
  const double self_scale = include_self ? -xi * kInvSqrtPiD : 0.0;
  const double c_mu = 2.0 * xi * xi / 3.0, c_th = 8.0 * xi * xi * xi * xi / 5.0;  // kernel.cpp:209-210
  k_dsrc_out<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(d_near, d_far, part, sorted, n, self_scale,
                                                                     c_mu, c_th, out);
}

}  // namespace ankh_b200
