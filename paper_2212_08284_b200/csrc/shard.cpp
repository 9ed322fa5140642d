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
