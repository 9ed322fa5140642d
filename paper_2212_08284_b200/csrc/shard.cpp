#include "shard.hpp"

#include <algorithm>
#include <cstdlib>

#include "host_numerics.hpp"

namespace ankh_b200 {

namespace {
std::uint32_t spread3(std::uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
}  // namespace

std::uint32_t morton3(std::uint32_t x, std::uint32_t y, std::uint32_t z) {
  return (spread3(x) << 2) | (spread3(y) << 1) | spread3(z);
}

void shard_leaf_range(int depth, int rank, int world, std::int64_t* begin, std::int64_t* end) {
  const std::int64_t nl = std::int64_t(1) << (3 * depth);
  *begin = nl * rank / world;
  *end = nl * (rank + 1) / world;
}

void shard_src_slice(std::size_t n, int rank, int world, std::size_t* i0, std::size_t* i1) {
  const std::size_t blocks = (n + 255) / 256, r = static_cast<std::size_t>(rank), g = static_cast<std::size_t>(world);
  *i0 = std::min(n, blocks * r / g * 256);
  *i1 = std::min(n, blocks * (r + 1) / g * 256);
}

int shard_exchange_level(int depth, int world) {
  int l0 = depth;
  for (int l = depth; l >= 1 && (std::int64_t(1) << (3 * l)) % world == 0; --l) l0 = l;
  return l0;
}

namespace {
std::uint32_t compact3(std::uint32_t v) {
  v &= 0x09249249u;
  v = (v ^ (v >> 2)) & 0x030c30c3u;
  v = (v ^ (v >> 4)) & 0x0300f00fu;
  v = (v ^ (v >> 8)) & 0x030000ffu;
  v = (v ^ (v >> 16)) & 0x000003ffu;
  return v;
}
}  // namespace

int shard_halo_level(int depth, int world) {
  return world <= 1 ? depth + 1 : shard_exchange_level(depth, world) + 1;
}

std::vector<std::uint32_t> shard_halo_cells(int level, int depth, bool periodic, int src, int dst,
                                            int world) {
  std::vector<std::uint32_t> out;
  const std::int64_t cells = std::int64_t(1) << (3 * level);
  if (world <= 1 || src == dst || cells % world != 0) return out;
  (void)depth;
  const int n = 1 << level;
  // dst's region: the Morton-aligned block [dst cells/G, (dst+1) cells/G) is a
  // box; its first and last cells are its min and max corners
  const std::uint32_t m0 = static_cast<std::uint32_t>(cells * dst / world);
  const std::uint32_t m1 = static_cast<std::uint32_t>(cells * (dst + 1) / world) - 1;
  const int lo[3] = {static_cast<int>(compact3(m0 >> 2)), static_cast<int>(compact3(m0 >> 1)),
                     static_cast<int>(compact3(m0))};
  const int hi[3] = {static_cast<int>(compact3(m1 >> 2)), static_cast<int>(compact3(m1 >> 1)),
                     static_cast<int>(compact3(m1))};
  // Reach of the interaction lists past the region's faces: Lambda(t)
  // offsets are s - t in [-2-c, 3-c] with c = t & 1 (octree.cpp:79-87), so
  // past an even lower face (odd upper face) only 2 cells can pair with a
  // cell inside -- in either direction of the unordered instance -- and 3
  // past a face of the other parity (regions one cell wide).  n is even, so
  // parities survive the periodic wrap.
  auto near = [&](int x, int a) {
    if (x >= lo[a] && x <= hi[a]) return true;
    const int reach_lo = (lo[a] & 1) ? 3 : 2, reach_hi = (hi[a] & 1) ? 2 : 3;
    if (periodic) {
      const int below = ((lo[a] - x) % n + n) % n, above = ((x - hi[a]) % n + n) % n;
      return below <= reach_lo || above <= reach_hi;
    }
    return x < lo[a] ? lo[a] - x <= reach_lo : x - hi[a] <= reach_hi;
  };
  const std::uint32_t s0 = static_cast<std::uint32_t>(cells * src / world);
  const std::uint32_t s1 = static_cast<std::uint32_t>(cells * (src + 1) / world);
  for (std::uint32_t m = s0; m < s1; ++m)
    if (near(static_cast<int>(compact3(m >> 2)), 0) && near(static_cast<int>(compact3(m >> 1)), 1) &&
        near(static_cast<int>(compact3(m)), 2))
      out.push_back(m);
  return out;
}

void shard_exchange_bytes(int depth, bool periodic, int row_doubles, int rank, int world, bool halo,
                          std::size_t* recv, std::size_t* send) {
  *recv = *send = 0;
  if (world <= 1) return;
  const int l0 = shard_exchange_level(depth, world);
  const int lh = halo ? shard_halo_level(depth, world) : depth + 1;
  const std::size_t row = static_cast<std::size_t>(row_doubles) * sizeof(double);
  for (int l = l0; l <= std::min(lh - 1, depth); ++l) {
    const std::size_t cells = std::size_t(1) << (3 * l);
    *recv += (cells - cells / world) * row;
    *send += (cells / world) * row;
  }
  for (int l = lh; l <= depth; ++l)
    for (int q = 0; q < world; ++q) {
      if (q == rank) continue;
      *recv += shard_halo_cells(l, depth, periodic, q, rank, world).size() * row;
      *send += shard_halo_cells(l, depth, periodic, rank, q, world).size() * row;
    }
}

int shard_m2l_owner(int level, std::uint32_t t, std::uint32_t s, int depth, int world) {
  if (world <= 1) return 0;
  // the owner of t or of s, by a hash of the pair: every cell has the same
  // number of interaction partners, so each shard gets half of the instances
  // of its targets and half of those of its sources -- balanced, whereas the
  // target alone favours low cell indices under the t < s canonical rule
  // (12 % excess on 8 shards at config 3)
  const std::uint32_t h = t * 0x9E3779B1u ^ (s + 0x7F4A7C15u) * 0x85EBCA77u;
  return shard_cell_owner(level, ((h >> 15) & 1u) ? s : t, depth, world);
}

int shard_cell_owner(int level, std::uint32_t cell, int depth, int world) {
  if (world <= 1) return 0;
  const int n = 1 << level;
  const std::uint32_t i = cell / (n * n), j = (cell / n) % n, k = cell % n;
  const std::int64_t first_leaf = static_cast<std::int64_t>(morton3(i, j, k)) << (3 * (depth - level));
  const std::int64_t nl = std::int64_t(1) << (3 * depth);
  int r = static_cast<int>(first_leaf * world / nl);
  std::int64_t b, e;
  while (true) {
    shard_leaf_range(depth, r, world, &b, &e);
    if (first_leaf < b) --r;
    else if (first_leaf >= e) ++r;
    else return r;
  }
}

void enumerate_offset(OffsetInstances& w, bool periodic, int depth, int rank, int world) {
  const int nl = 1 << w.level;
  int lo[3], step[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = 0;
    step[a] = 1;
    if (w.offset[a] == 3) step[a] = 2;                  // only even t_a
    if (w.offset[a] == -3) { lo[a] = 1; step[a] = 2; }  // only odd t_a
  }
  for (int tx = lo[0]; tx < nl; tx += step[0])
    for (int ty = lo[1]; ty < nl; ty += step[1])
      for (int tz = lo[2]; tz < nl; tz += step[2]) {
        const int ext[3] = {tx + w.offset[0], ty + w.offset[1], tz + w.offset[2]};
        int in[3], img[3];
        bool ok = true;
        for (int a = 0; a < 3; ++a) {
          if (!periodic && (ext[a] < 0 || ext[a] >= nl)) ok = false;
          img[a] = ext[a] >= 0 ? ext[a] / nl : -((-ext[a] + nl - 1) / nl);
          in[a] = ext[a] - nl * img[a];
        }
        if (!ok) continue;
        const std::uint32_t t = static_cast<std::uint32_t>((tx * nl + ty) * nl + tz);
        const std::uint32_t s = static_cast<std::uint32_t>((in[0] * nl + in[1]) * nl + in[2]);
        const bool lexpos = img[0] != 0 ? img[0] > 0 : (img[1] != 0 ? img[1] > 0 : img[2] > 0);
        if (!(t < s || (t == s && lexpos))) continue;
        if (rank >= 0 && shard_m2l_owner(w.level, t, s, depth, world) != rank) continue;
        w.t.push_back(t);
        w.s.push_back(s);
      }
}

std::vector<OffsetInstances> enumerate_m2l(int depth, bool periodic, int rank, int world,
                                           int threads) {
  std::vector<OffsetInstances> work;
  for (int level = 1; level <= depth; ++level)
    for (int ox = -3; ox <= 3; ++ox)
      for (int oy = -3; oy <= 3; ++oy)
        for (int oz = -3; oz <= 3; ++oz)
          if (std::max({std::abs(ox), std::abs(oy), std::abs(oz)}) >= 2) {
            OffsetInstances w;
            w.level = level;
            w.offset = {ox, oy, oz};
            work.push_back(std::move(w));
          }
  parallel_for(static_cast<int>(work.size()), threads,
               [&](int i) { enumerate_offset(work[i], periodic, depth, rank, world); });
  work.erase(std::remove_if(work.begin(), work.end(),
                            [](const OffsetInstances& w) { return w.t.empty(); }),
             work.end());
  return work;
}

}  // namespace ankh_b200
