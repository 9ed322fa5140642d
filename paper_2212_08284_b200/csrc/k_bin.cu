// Validation, leaf binning, stable sort and gather (sm_100a).
//
// Reference: validate_system (types.cpp:16-63), build_tree (octree.cpp:27-45),
// self_energy (kernel.cpp:206-213).  Binning is bit-exact with the reference:
// shifted = (x + r_B) * inv_side with inv_side = n / (2 r_B) computed on the
// host exactly as octree.cpp:35, IEEE round-to-nearest add and multiply (no
// FMA contraction), floor, clamp to [0, n-1].  Particles are bucketed by a
// counting sort (leaf histogram and arrival slots from k_bin, a scan, a
// scatter) and each leaf's indices are put back in ascending order, which is
// the reference's bucket order (bit-exact leaf CSR).  All of it is HBM-bound
// (104 B read, 8 B of keys/slots, 112-B records written per atom).
#include <algorithm>

#include <cub/cub.cuh>

#include "kernels.cuh"

namespace ankh_b200 {

namespace {

__device__ __forceinline__ int bin_axis(double x, double rb, double inv_side, int n) {
  const double shifted = __dmul_rn(__dadd_rn(x, rb), inv_side);
  double f = floor(shifted);
  f = fmin(fmax(f, 0.0), static_cast<double>(n - 1));
  return static_cast<int>(f);
}

// The moment half of validate_system (types.cpp:16-63) for particle i:
// first non-finite index, and whether moment_order (kernel.cpp:40-44) > 0.
// Returns the multipole flag (false for a non-finite particle).
__device__ __forceinline__ bool check_moments(const double* __restrict__ s, std::size_t i, DevResult* res) {
  bool finite = true, mp = false;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    finite = finite && isfinite(s[k]);
    mp = mp || (k > 0 && s[k] != 0.0);
  }
  if (!finite) atomicMin(&res->min_nonfinite, static_cast<unsigned long long>(i));
  return finite && mp;
}

// Lanes of a warp with the same key take consecutive slots of one counter
// with a single atomic (consecutive particles mostly share a leaf, so
// per-lane atomics would serialise on a handful of addresses); the leader
// also raises the leaf's largest index (the streamed path's readiness).
// key == ~0u: lane inactive.  Returns the lane's slot.
__device__ __forceinline__ unsigned warp_count(unsigned key, unsigned* counts, unsigned* leafmax, unsigned i) {
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
  unsigned base = 0;
  if (lane == leader && key != ~0u) {
    base = atomicAdd(&counts[key], static_cast<unsigned>(__popc(peers)));
    // indices ascend with the lane: the highest peer holds the largest
    if (leafmax) atomicMax(&leafmax[key], i + static_cast<unsigned>((31 - __clz(peers)) - lane));
  }
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + static_cast<unsigned>(__popc(peers & ((1u << lane) - 1u)));
}

// particles [256 block0, n): one range of the positions (the streamed path
// bins each arrived chunk) or all of them (block0 = 0)
__global__ void __launch_bounds__(256) k_bin(const double* __restrict__ pos,
                                             const double* __restrict__ src, std::size_t n,
                                             double rb, double inv_side, int nax,
                                             unsigned* __restrict__ keys,
                                             unsigned* __restrict__ idx,
                                             unsigned* __restrict__ counts,
                                             const unsigned char* __restrict__ need, DevResult* res,
                                             unsigned block0, unsigned* __restrict__ leafmax) {
  const std::size_t i = (static_cast<std::size_t>(block0) + blockIdx.x) * 256 + threadIdx.x;
  bool mp = false;
  unsigned key = 0;
  bool counted = false;
  if (i < n) {
    const double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
    bool finite = isfinite(x) && isfinite(y) && isfinite(z);
    if (src) {  // src == nullptr: positions only (the moments are checked elsewhere)
      double s[10];
#pragma unroll
      for (int k = 0; k < 10; ++k) s[k] = src[10 * i + k];
#pragma unroll
      for (int k = 0; k < 10; ++k) finite = finite && isfinite(s[k]);
      mp = finite && check_moments(s, i, res);
    }
    if (!finite) {
      atomicMin(&res->min_nonfinite, static_cast<unsigned long long>(i));
    } else {
      if (fabs(x) > rb || fabs(y) > rb || fabs(z) > rb)
        atomicMin(&res->min_outside, static_cast<unsigned long long>(i));
      const int ix = bin_axis(x, rb, inv_side, nax);
      const int iy = bin_axis(y, rb, inv_side, nax);
      const int iz = bin_axis(z, rb, inv_side, nax);
      key = static_cast<unsigned>((ix * nax + iy) * nax + iz);
    }
    keys[i] = key;
    // without counts (validation path) idx is the identity for the radix sort;
    // a shard (need != nullptr) sorts only the leaves it reads: the others
    // stay empty in its CSR (every particle is still validated above)
    if (!counts)
      idx[i] = static_cast<unsigned>(i);
    else if (need && !need[key])
      idx[i] = ~0u;
    else
      counted = true;
  }
  // counting sort: idx receives the particle's arrival slot in its leaf
  // (ascending order inside the leaf is restored by k_leaf_gather)
  if (counts) {  // uniform across the grid: every lane takes part
    const unsigned slot = warp_count(counted ? key : ~0u, counts, leafmax, static_cast<unsigned>(i));
    if (counted) idx[i] = slot;
  }
  if (__syncthreads_or(mp) && threadIdx.x == 0) atomicOr(&res->any_multipole, 1);
}

// Exclusive scan of n uints in one pass (the leaf histogram -> the CSR
// offsets): tiles of 4096 taken in ticket order, each publishes its
// aggregate and then its inclusive prefix (decoupled look-back over the
// predecessors' status words: flag in bits 62-63, value below).  The state
// (status[tiles], ticket, done) resets itself: the last tile to finish
// zeroes it for the next launch (zero-initialised once by the plan).
constexpr int kScanThreads = 256, kScanItems = 16, kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kScanAgg = 1ull << 62, kScanIncl = 2ull << 62, kScanVal = (1ull << 62) - 1;

__global__ void __launch_bounds__(kScanThreads) k_scan(const unsigned* __restrict__ in, unsigned* __restrict__ out,
                                                       unsigned n, unsigned long long* status, unsigned* ctr) {
  __shared__ unsigned s_tile, s_prefix, s_last, s_warp[kScanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(&ctr[0], 1u);
  __syncthreads();
  const unsigned tile = s_tile;
  ANKH_DASSERT(tile < gridDim.x);  // tickets: one per block (the state was reset by the last launch)
  const std::size_t base = static_cast<std::size_t>(tile) * kScanTile + static_cast<std::size_t>(tid) * kScanItems;
  unsigned v[kScanItems];
  if (base + kScanItems <= n) {
    const uint4* p = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      const uint4 w = p[q];
      v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = base + k < n ? in[base + k] : 0u;
  }
  unsigned tsum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) tsum += v[k];
  unsigned incl = tsum;  // warp-inclusive scan of the thread sums
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    // block aggregate and the warps' exclusive offsets
    const unsigned wv = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
    unsigned wi = wv;
#pragma unroll
    for (int o = 1; o < kScanThreads / 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    const unsigned agg = __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
    if (lane < kScanThreads / 32) s_warp[lane] = wi - wv;
    volatile unsigned long long* st = status;
    unsigned long long excl = 0;
    if (tile == 0) {
      if (lane == 0) st[0] = kScanIncl | agg;
    } else {
      if (lane == 0) st[tile] = kScanAgg | agg;
      // warp-wide look-back: 32 predecessors per round trip, nearest first;
      // stop at the nearest one that published its inclusive prefix
      for (long long j = static_cast<long long>(tile) - 1; j >= 0; j -= 32) {
        const long long idx = j - lane;
        unsigned long long w = kScanIncl + 0ull;  // before tile 0: inclusive 0
        if (idx >= 0) w = st[idx];
        while (__any_sync(0xffffffffu, (w & ~kScanVal) == 0))
          if ((w & ~kScanVal) == 0) w = st[idx];
        const unsigned incl_mask = __ballot_sync(0xffffffffu, (w & ~kScanVal) == kScanIncl);
        const int stop = incl_mask ? __ffs(incl_mask) - 1 : 31;  // lanes 0..stop contribute
        unsigned long long v = lane <= stop ? (w & kScanVal) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        excl += __shfl_sync(0xffffffffu, v, 0);
        if (incl_mask) break;
      }
      if (lane == 0) st[tile] = kScanIncl | (excl + agg);
    }
    if (lane == 0) s_prefix = static_cast<unsigned>(excl);
  }
  __syncthreads();
  unsigned run = s_prefix + s_warp[warp] + (incl - tsum);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
  // self-reset: the last tile to finish clears the state for the next launch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&ctr[1], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    for (unsigned j = tid; j < gridDim.x; j += kScanThreads) status[j] = 0ull;
    if (tid == 0) {
      ctr[0] = 0u;
      ctr[1] = 0u;
    }
  }
}

// Counting-sort scatter: particle i goes to offsets[key] + slot (leaf order is
// final, order inside a leaf is arrival order).
__global__ void __launch_bounds__(256) k_scatter(const unsigned* __restrict__ keys,
                                                 const unsigned* __restrict__ slots,
                                                 const unsigned* __restrict__ offsets,
                                                 std::size_t n, unsigned* __restrict__ unsorted) {
  const std::size_t i = static_cast<std::size_t>(blockIdx.x) * 256 + threadIdx.x;
  if (i >= n || slots[i] == ~0u) return;  // ~0u: a leaf this shard does not read
  ANKH_DASSERT(offsets[keys[i]] + slots[i] < offsets[keys[i] + 1]);
  unsorted[offsets[keys[i]] + slots[i]] = static_cast<unsigned>(i);
}

#ifndef ANKH_LEAF_THREADS
#define ANKH_LEAF_THREADS 64  // 32 / 64 / 128: binning phase 0.100 / 0.096 / 0.102 ms at config 3
#endif
constexpr int kLeafThreads = ANKH_LEAF_THREADS;
constexpr int kLeafSmem = 512;  // leaves up to this size are sorted in shared memory

__device__ __forceinline__ void write_record(const double* __restrict__ pos,
                                             const double* __restrict__ src, std::size_t i,
                                             double* __restrict__ rec) {
  double r[kRec];
  r[0] = pos[3 * i];
  r[1] = pos[3 * i + 1];
  r[2] = pos[3 * i + 2];
#pragma unroll
  for (int k = 0; k < 10; ++k) r[3 + k] = src[10 * i + k];
  r[13] = (r[7] + r[10]) + r[12];  // SymMat3::trace (types.hpp:57)
  double2* out = reinterpret_cast<double2*>(rec);
#pragma unroll
  for (int k = 0; k < kRec / 2; ++k) out[k] = make_double2(r[2 * k], r[2 * k + 1]);
}

// One CTA per leaf: put the leaf's particle indices in ascending order (the
// reference's bucket order, octree.cpp:42 -- indices are unique, so a rank is
// a position) and gather its records.  Small leaves: rank sort in shared
// memory; large ones: bottom-up merge passes in global memory (ping-pong
// between the leaf's slices of `unsorted` and `scratch`).
// With `check_src` the leaf's moments are also validated here (the moment
// half of validate_system) -- k_bin then reads positions only, and the
// moments are read once, by this gather, instead of twice.
__global__ void __launch_bounds__(kLeafThreads) k_leaf_gather(
    const double* __restrict__ pos, const double* __restrict__ src,
    const unsigned* __restrict__ offsets, unsigned* __restrict__ unsorted,
    unsigned* __restrict__ scratch, unsigned* __restrict__ sorted,
    const unsigned char* __restrict__ need, double* __restrict__ part, bool check_src,
    DevResult* res, unsigned* __restrict__ leaf_mp, unsigned* __restrict__ inv) {
  __shared__ unsigned a[kLeafSmem], b[kLeafSmem];
  const unsigned leaf = blockIdx.x;
  if (need && !need[leaf]) return;  // another shard's leaf
  const unsigned base = offsets[leaf];
  const int c = static_cast<int>(offsets[leaf + 1] - base);
  ANKH_DASSERT(offsets[leaf + 1] >= base);
  if (c == 0) {
    if (part && leaf_mp && threadIdx.x == 0) leaf_mp[leaf] = 0u;
    return;
  }
  const unsigned* order;
  if (c <= kLeafSmem) {
    for (int e = threadIdx.x; e < c; e += kLeafThreads) a[e] = unsorted[base + e];
    __syncthreads();
    for (int e = threadIdx.x; e < c; e += kLeafThreads) {
      const unsigned v = a[e];
      int rank = 0;
      for (int j = 0; j < c; ++j) rank += a[j] < v;
      b[rank] = v;
      sorted[base + rank] = v;
      if (inv) inv[v] = base + rank;  // the sorted slot of particle v
    }
    __syncthreads();
    order = b;
  } else {
    unsigned* x = unsorted + base;
    unsigned* y = scratch + base;
    for (int w = 1; w < c; w *= 2) {
      for (int p = threadIdx.x; p < c; p += kLeafThreads) {
        const int run = p / w, rs = run * w, ps = (run ^ 1) * w;
        const int plen = ps < c ? min(w, c - ps) : 0;
        const unsigned v = x[p];
        int lo = 0, hi = plen;  // elements of the partner run below v
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (x[ps + mid] < v) lo = mid + 1; else hi = mid;
        }
        y[min(rs, ps) + (p - rs) + lo] = v;
      }
      __syncthreads();
      unsigned* t = x;
      x = y;
      y = t;
    }
    for (int p = threadIdx.x; p < c; p += kLeafThreads) {
      sorted[base + p] = x[p];
      if (inv) inv[x[p]] = base + p;
    }
    __syncthreads();
    order = sorted + base;
  }
  if (!part) return;  // sort only (positions bound ahead of the moments)
  // four threads (a lane quad) per particle: the moments row (80 B, 16-B
  // aligned) is read as five 16-B pieces s0..s4 = (q,mx) (my,mz) (txx,txy)
  // (txz,tyy) (tyz,tzz) -- lane k takes s_k, lane 0 also s4 and (x, y), lane 1
  // z -- and the record's 16-B pieces {k, k+4} are assembled by quad shuffles:
  //   0 (x, y)  1 (z, q)  2 (mx, my)  3 (mz, txx)  4 (txy, txz)  5 (tyy, tyz)  6 (tzz, tr)
  // Each lane checks the moments it read (together every one of q, mu, Theta).
  bool mp = false;
  const int k = threadIdx.x & 3;
  for (int e0 = 0; e0 < 4 * c; e0 += kLeafThreads) {
    const int e = e0 + threadIdx.x;
    const bool ok = e < 4 * c;  // whole quads: 4c is a multiple of 4
    const int p = ok ? e >> 2 : 0;
    const std::size_t i = order[p];
    const double2* s2 = reinterpret_cast<const double2*>(src + 10 * i);
    double2 mine = ok ? __ldg(s2 + k) : make_double2(0.0, 0.0);
    double2 s4 = make_double2(0.0, 0.0), xy = make_double2(0.0, 0.0);
    double z = 0.0;
    if (ok && k == 0) {
      s4 = __ldg(s2 + 4);
      xy = make_double2(__ldg(pos + 3 * i), __ldg(pos + 3 * i + 1));
    }
    if (ok && k == 1) z = __ldg(pos + 3 * i + 2);
    // quad exchange (all lanes take part; lane q's pieces from __shfl ... width 4)
    const double p0x = __shfl_sync(0xffffffffu, mine.x, 0, 4), p0y = __shfl_sync(0xffffffffu, mine.y, 0, 4);
    const double p1x = __shfl_sync(0xffffffffu, mine.x, 1, 4), p1y = __shfl_sync(0xffffffffu, mine.y, 1, 4);
    const double p2x = __shfl_sync(0xffffffffu, mine.x, 2, 4), p2y = __shfl_sync(0xffffffffu, mine.y, 2, 4);
    const double p3x = __shfl_sync(0xffffffffu, mine.x, 3, 4), p3y = __shfl_sync(0xffffffffu, mine.y, 3, 4);
    const double p4x = __shfl_sync(0xffffffffu, s4.x, 0, 4), p4y = __shfl_sync(0xffffffffu, s4.y, 0, 4);
    if (!ok) continue;
    double2* out = reinterpret_cast<double2*>(part + static_cast<std::size_t>(base + p) * kRec);
    if (k == 0) {
      out[0] = xy;
      out[4] = make_double2(p2y, p3x);
    } else if (k == 1) {
      out[1] = make_double2(z, p0x);
      out[5] = make_double2(p3y, p4x);
    } else if (k == 2) {
      out[2] = make_double2(p0y, p1x);
      out[6] = make_double2(p4y, (p2x + p3y) + p4y);  // SymMat3::trace (types.hpp:57)
    } else {
      out[3] = make_double2(p1y, p2x);
    }
    bool fin = isfinite(mine.x) && isfinite(mine.y);
    if (k == 0) fin = fin && isfinite(s4.x) && isfinite(s4.y);
    if (check_src && !fin) atomicMin(&res->min_nonfinite, static_cast<unsigned long long>(i));
    // multipole: anything but q (lane 0's s0.x) nonzero
    mp = mp || (k != 0 && mine.x != 0.0) || mine.y != 0.0 || (k == 0 && (s4.x != 0.0 || s4.y != 0.0));
  }
  mp = __syncthreads_or(mp);
  if (threadIdx.x == 0) {
    if (leaf_mp) leaf_mp[leaf] = mp ? 1u : 0u;  // the P2P kernel's per-leaf pair code
    if (check_src && mp) atomicOr(&res->any_multipole, 1);
  }
}

// Records in leaf order from an existing sorted index (the moments of a
// plan whose positions were bound by ankh_plan_set_positions_v1).
// Per-leaf multipole flag of a scattered record: lanes with the same leaf
// combine first (consecutive particles mostly share a leaf), one atomic each.
__device__ __forceinline__ void flag_leaf(bool active, bool mp, unsigned key, unsigned* leaf_mp) {
  const bool want = active && mp;
  const unsigned k = want ? key : ~0u;
  const unsigned peers = __match_any_sync(0xffffffffu, k);
  if (want && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1)) atomicOr(&leaf_mp[key], 1u);
}

__device__ __forceinline__ bool src_has_multipole(const double* __restrict__ s) {
  bool m = false;
#pragma unroll
  for (int k = 1; k < 10; ++k) m = m || s[k] != 0.0;
  return m;
}

__global__ void __launch_bounds__(256) k_gather_sorted(const double* __restrict__ pos,
                                                       const double* __restrict__ src,
                                                       const unsigned* __restrict__ sorted,
                                                       std::size_t n, double* __restrict__ part,
                                                       const unsigned* __restrict__ keys,
                                                       unsigned* __restrict__ leaf_mp) {
  const std::size_t j = static_cast<std::size_t>(blockIdx.x) * 256 + threadIdx.x;
  const bool ok = j < n;
  const unsigned i = ok ? sorted[j] : 0u;
  if (ok) write_record(pos, src, i, part + j * kRec);
  if (leaf_mp) flag_leaf(ok, ok && src_has_multipole(src + 10 * static_cast<std::size_t>(i)), ok ? keys[i] : 0u, leaf_mp);
}

// The moment half of validate_system (types.cpp:16-63) for particles
// [block0 256, n): the bound-positions path (all particles), a shard's index
// slice, or -- streamed host path -- one arrived chunk, each particle's
// record then also scattered to its sorted slot inv[i].
__global__ void __launch_bounds__(256) k_src_check(const double* __restrict__ src, std::size_t n,
                                                   DevResult* res, unsigned block0,
                                                   const double* __restrict__ pos,
                                                   const unsigned* __restrict__ inv,
                                                   double* __restrict__ part,
                                                   const unsigned* __restrict__ keys,
                                                   unsigned* __restrict__ leaf_mp) {
  const std::size_t i = (static_cast<std::size_t>(block0) + blockIdx.x) * 256 + threadIdx.x;
  bool mp = false;
  if (i < n) {
    if (inv) write_record(pos, src, static_cast<unsigned>(i), part + static_cast<std::size_t>(inv[i]) * kRec);
    mp = check_moments(src + 10 * i, i, res);
  }
  if (leaf_mp) flag_leaf(i < n, src_has_multipole(src + 10 * (i < n ? i : 0)), i < n ? keys[i] : 0u, leaf_mp);
  if (__syncthreads_or(mp) && threadIdx.x == 0) atomicOr(&res->any_multipole, 1);
}

// Streamed host path, per Morton leaf m: the chunk after which its records
// are complete (the chunk of its largest particle index, leafmax from k_bin)
// and the chunk after which its 13 half-shell neighbours are too (P2P's
// source set, k_p2p); counts per chunk in cnt[0..C) (P2M) / cnt[C..2C) (P2P).
__device__ __forceinline__ int chunk_of(unsigned i, const StreamChunks& ch) {
  int lo = 0, hi = ch.n - 1;  // the last c with start[c] <= i
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ch.start[mid] <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void stream_ready_leaf(unsigned m, const unsigned* __restrict__ leafmax, int depth,
                                                  int periodic, const StreamChunks& ch,
                                                  unsigned char* __restrict__ ready, unsigned* key_p2m,
                                                  unsigned* key_p2p) {
  const int n = 1 << depth;
  const int ax = static_cast<int>(morton_compact3(m >> 2)), ay = static_cast<int>(morton_compact3(m >> 1)),
            az = static_cast<int>(morton_compact3(m));
  auto leaf_ready = [&](int x, int y, int z) -> int {
    return chunk_of(leafmax[static_cast<unsigned>((x * n + y) * n + z)], ch);  // empty: 0
  };
  const int r = leaf_ready(ax, ay, az);
  int p = r;
  for (int d = 0; d < 13; ++d) {  // the 13 lex-positive directions, as k_p2p
    const int dx = d < 4 ? 0 : 1;
    const int dy = d == 0 ? 0 : (d < 4 ? 1 : (d - 4) / 3 - 1);
    const int dz = d == 0 ? 1 : (d < 4 ? d - 2 : (d - 4) % 3 - 1);
    int e[3] = {ax + dx, ay + dy, az + dz};
    bool ok = true;
    for (int k = 0; k < 3; ++k) {
      if (e[k] < 0 || e[k] >= n) {
        if (!periodic) ok = false;
        e[k] = ((e[k] % n) + n) % n;
      }
    }
    if (ok) p = max(p, leaf_ready(e[0], e[1], e[2]));
  }
  ready[2 * m] = static_cast<unsigned char>(r);
  ready[2 * m + 1] = static_cast<unsigned char>(p);
  *key_p2m = static_cast<unsigned>(r);
  *key_p2p = static_cast<unsigned>(ch.n + p);
}

// Warp-aggregated slot in a shared-memory counter per key: the lanes with
// equal keys take consecutive slots with one shared atomic per distinct key
// (leaves of one warp mostly share a chunk, so per-lane atomics on a handful
// of counters serialise).  key == ~0u: lane inactive.
__device__ __forceinline__ unsigned warp_slot(unsigned key, unsigned* s_cnt) {
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
  unsigned base = 0;
  if (lane == leader && key != ~0u) base = atomicAdd(&s_cnt[key], static_cast<unsigned>(__popc(peers)));
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + static_cast<unsigned>(__popc(peers & ((1u << lane) - 1u)));
}

// cnt[0 .. 2C) and cursor[0 .. 2C) zeroed by the caller (one memset)
__global__ void __launch_bounds__(256) k_stream_ready(const unsigned* __restrict__ leafmax, int depth,
                                                      int periodic, StreamChunks ch,
                                                      unsigned char* __restrict__ ready,
                                                      unsigned* __restrict__ cnt) {
  __shared__ unsigned s_cnt[2 * kMaxStreamChunks];
  if (threadIdx.x < 2 * kMaxStreamChunks) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const unsigned m = blockIdx.x * 256 + threadIdx.x;
  unsigned k0 = ~0u, k1 = ~0u;
  if (m < (1u << (3 * depth))) stream_ready_leaf(m, leafmax, depth, periodic, ch, ready, &k0, &k1);
  warp_slot(k0, s_cnt);
  warp_slot(k1, s_cnt);
  __syncthreads();
  if (threadIdx.x < 2 * ch.n && s_cnt[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], s_cnt[threadIdx.x]);
}

// Per-chunk leaf lists: bucket starts = exclusive scans of the two count
// sets (every block computes them; block 0 also stores the bounds the chunk
// kernels read: bounds[0..C] P2M, bounds[C+1..2C+1] P2P); each block
// reserves one contiguous range per key inside the buckets, its leaves take
// warp-aggregated slots inside it.
__global__ void __launch_bounds__(256) k_stream_lists(const unsigned char* __restrict__ ready, unsigned n_leaves,
                                                      int n_chunks, const unsigned* __restrict__ cnt,
                                                      unsigned* __restrict__ cursor, unsigned* __restrict__ bounds,
                                                      unsigned* __restrict__ list_p2m,
                                                      unsigned* __restrict__ list_p2p) {
  __shared__ unsigned s_cnt[2 * kMaxStreamChunks], s_base[2 * kMaxStreamChunks];
  const int tid = threadIdx.x;
  if (tid < 2 * kMaxStreamChunks) s_cnt[tid] = 0;
  if (tid < 2 * n_chunks) {
    const int set = tid / n_chunks, c = tid - set * n_chunks;
    unsigned start = 0;
    for (int j = 0; j < c; ++j) start += cnt[set * n_chunks + j];
    s_base[tid] = start;
    if (blockIdx.x == 0) {
      bounds[set * (n_chunks + 1) + c] = start;
      if (c == n_chunks - 1) bounds[set * (n_chunks + 1) + n_chunks] = start + cnt[tid];
    }
  }
  __syncthreads();
  const unsigned m = blockIdx.x * 256 + tid;
  const bool ok = m < n_leaves;
  const unsigned k0 = ok ? ready[2 * m] : ~0u;
  const unsigned k1 = ok ? n_chunks + ready[2 * m + 1] : ~0u;
  const unsigned s0 = warp_slot(k0, s_cnt);
  const unsigned s1 = warp_slot(k1, s_cnt);
  __syncthreads();
  if (tid < 2 * n_chunks && s_cnt[tid]) s_base[tid] += atomicAdd(&cursor[tid], s_cnt[tid]);
  __syncthreads();
  if (!ok) return;
  list_p2m[s_base[k0] + s0] = m;
  list_p2p[s_base[k1] + s1] = m;
}

// Result flags / energies, and (counts != nullptr) the leaf histogram zeroed
// in the same launch (one graph node instead of a memset plus a kernel).
__global__ void k_init_result(DevResult* res, int any_multipole, unsigned* counts, unsigned n_counts) {
  const unsigned g = blockIdx.x * blockDim.x + threadIdx.x;
  if (counts)
    for (unsigned e = g; e < n_counts; e += gridDim.x * blockDim.x) counts[e] = 0u;
  if (g != 0) return;
  for (int k = 0; k < kRedCount; ++k) res->red[k] = 0.0;
  res->min_nonfinite = ~0ull;
  res->min_outside = ~0ull;
  res->any_multipole = any_multipole;
  res->spare = 0;
}

// Exact-duplicate scan over (key, index)-sorted particles: duplicates share a
// leaf, so only runs of equal keys are compared (validate_system's rule,
// types.cpp:45-61).  Used on the error path where no P2P pass runs.
__global__ void k_dup_check(const unsigned* __restrict__ keys, const unsigned* __restrict__ idx,
                            const double* __restrict__ pos, std::size_t n, DevResult* res) {
  const std::size_t i = static_cast<std::size_t>(blockIdx.x) * 256 + threadIdx.x;
  if (i >= n) return;
  const std::size_t a = idx[i];
  for (std::size_t j = i + 1; j < n && keys[j] == keys[i]; ++j) {
    const std::size_t b = idx[j];
    if (pos[3 * a] == pos[3 * b] && pos[3 * a + 1] == pos[3 * b + 1] &&
        pos[3 * a + 2] == pos[3 * b + 2]) {
      res->red[kDuplicate] = 1.0;  // benign race: every writer stores 1
      return;
    }
  }
}

}  // namespace

void launch_init_result(DevResult* res, cudaStream_t st, int any_multipole, unsigned* counts,
                        unsigned n_counts) {
  const unsigned blocks = counts ? std::min(1024u, (n_counts + 255) / 256) : 1u;
  k_init_result<<<blocks, counts ? 256 : 1, 0, st>>>(res, any_multipole, counts, n_counts);
}

void launch_dup_check(const unsigned* keys_sorted, const unsigned* idx_sorted, const double* pos,
                      std::size_t n, DevResult* res, cudaStream_t st) {
  if (n < 2) return;
  k_dup_check<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(keys_sorted, idx_sorted, pos,
                                                                     n, res);
}

void launch_bin(const double* pos, const double* src, std::size_t n, double box_radius,
                double inv_side, int n_axis, unsigned* keys, unsigned* idx, unsigned* counts,
                DevResult* res, cudaStream_t st, const unsigned char* need, std::size_t i0, std::size_t i1,
                unsigned* leafmax) {
  i1 = std::min(i1, n);
  if (i1 <= i0) return;  // i0: a multiple of 256
  const unsigned blocks = static_cast<unsigned>((i1 - i0 + 255) / 256);
  k_bin<<<blocks, 256, 0, st>>>(pos, src, i1, box_radius, inv_side, n_axis, keys, idx, counts, need, res,
                                static_cast<unsigned>(i0 / 256), leafmax);
}

std::size_t scan_tiles(std::size_t n) { return (n + kScanTile - 1) / kScanTile; }

void launch_scan(const unsigned* in, unsigned* out, std::size_t n, ScanWork w, cudaStream_t st) {
  if (n == 0) return;
  k_scan<<<static_cast<unsigned>(scan_tiles(n)), kScanThreads, 0, st>>>(in, out, static_cast<unsigned>(n),
                                                                         w.status, w.ctr);
}

void launch_bucket_gather(ScanWork scan, const double* pos, const double* src,
                          const unsigned* keys, const unsigned* slots, const unsigned* counts,
                          unsigned* offsets, unsigned* unsorted, unsigned* scratch,
                          unsigned* sorted, std::size_t n, int n_leaves,
                          const unsigned char* need, double* part, cudaStream_t st,
                          bool check_src, DevResult* res, unsigned* leaf_mp, unsigned* inv) {
  launch_scan(counts, offsets, static_cast<std::size_t>(n_leaves) + 1, scan, st);
  if (n == 0) return;
  k_scatter<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(keys, slots, offsets, n,
                                                                    unsorted);
  k_leaf_gather<<<static_cast<unsigned>(n_leaves), kLeafThreads, 0, st>>>(
      pos, src, offsets, unsorted, scratch, sorted, need, part, check_src && part != nullptr, res, leaf_mp, inv);
}

void launch_src_gather(const double* pos, const double* src, const unsigned* sorted,
                       std::size_t n, DevResult* res, double* part, cudaStream_t st,
                       const unsigned* keys, unsigned* leaf_mp) {
  if (n == 0) return;
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  k_src_check<<<blocks, 256, 0, st>>>(src, n, res, 0u, nullptr, nullptr, nullptr, nullptr, nullptr);
  k_gather_sorted<<<blocks, 256, 0, st>>>(pos, src, sorted, n, part, keys, leaf_mp);
}

void launch_src_chunk(const double* pos, const double* src, const unsigned* inv, std::size_t i0,
                      std::size_t i1, DevResult* res, double* part, cudaStream_t st,
                      const unsigned* keys, unsigned* leaf_mp) {
  if (i1 <= i0) return;  // i0 is a multiple of 256
  const unsigned blocks = static_cast<unsigned>((i1 - i0 + 255) / 256);
  k_src_check<<<blocks, 256, 0, st>>>(src, i1, res, static_cast<unsigned>(i0 / 256), pos, inv, part, keys,
                                      leaf_mp);
}

void launch_stream_lists(const unsigned* leafmax, int depth, int periodic, const StreamChunks& ch,
                         unsigned char* ready, unsigned* cnt_cursor, unsigned* bounds, unsigned* list_p2m,
                         unsigned* list_p2p, cudaStream_t st) {
  const unsigned n_leaves = 1u << (3 * depth);
  cudaMemsetAsync(cnt_cursor, 0, 4 * kMaxStreamChunks * sizeof(unsigned), st);
  k_stream_ready<<<(n_leaves + 255) / 256, 256, 0, st>>>(leafmax, depth, periodic, ch, ready, cnt_cursor);
  k_stream_lists<<<(n_leaves + 255) / 256, 256, 0, st>>>(ready, n_leaves, ch.n, cnt_cursor,
                                                        cnt_cursor + 2 * kMaxStreamChunks, bounds, list_p2m,
                                                        list_p2p);
}

std::size_t sort_temp_bytes(std::size_t n) {
  std::size_t a = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<const unsigned*>(nullptr),
                                  static_cast<unsigned*>(nullptr),
                                  static_cast<const unsigned*>(nullptr),
                                  static_cast<unsigned*>(nullptr), static_cast<int>(n), 0, 32);
  return a + 256;
}

// validation path only (validate_only: no tree, duplicates by a radix sort)
void launch_sort(void* temp, std::size_t temp_bytes, const unsigned* keys_in, unsigned* keys_out,
                 const unsigned* idx_in, unsigned* idx_out, std::size_t n, int end_bit, cudaStream_t st) {
  if (n == 0) return;
  std::size_t bytes = temp_bytes;
  cub::DeviceRadixSort::SortPairs(temp, bytes, keys_in, keys_out, idx_in, idx_out, static_cast<int>(n), 0,
                                  end_bit > 0 ? end_bit : 1, st);
}

}  // namespace ankh_b200
