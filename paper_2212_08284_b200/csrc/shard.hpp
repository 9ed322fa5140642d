// Spatial sharding and M2L instance enumeration (host only, no CUDA).
//
// Shards own contiguous Morton ranges of leaves.  A level-l
// cell belongs to the shard that owns its first descendant leaf, so for
// world | 8 every shard owns whole level-1 subtrees.  P2P work is owned by
// the target leaf; a canonical M2L instance (t, s, image) (fmm.cpp:246-250)
// by the owner of t or of s, picked by a hash of (t, s) for balance; every
// unordered pair / instance is therefore counted by exactly one shard.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <vector>

namespace ankh_b200 {

/// Interleave (x, y, z) bits: x in bit 3k+2, y in 3k+1, z in 3k.
std::uint32_t morton3(std::uint32_t x, std::uint32_t y, std::uint32_t z);

/// Morton leaf range [begin, end) owned by `rank` of `world` at `depth`.
void shard_leaf_range(int depth, int rank, int world, std::int64_t* begin, std::int64_t* end);
/// Particle-index slice [i0, i1) whose moments shard `rank` validates (whole
/// 256-particle blocks; the slices partition [0, n)).
void shard_src_slice(std::size_t n, int rank, int world, std::size_t* i0, std::size_t* i1);
/// Lowest level l >= 1 whose 8^l cells split evenly over `world` shards, up to
/// `depth` (the upward exchange all-gathers levels l .. depth).
int shard_exchange_level(int depth, int world);

/// M2L halo of the deep levels: Morton cells of `level`
/// (ascending) that shard `src` owns and shard `dst` reads -- every cell that
/// can form an M2L instance with a cell of dst's own region (an instance is
/// owned by the owner of t or of s, fmm.cpp:43-50): within 2 cells of the
/// region's faces (3 past a face of odd parity), periodic wrap when
/// `periodic`.  Requires world | 8^level (shard regions are then
/// Morton-aligned boxes); src == dst or world == 1 gives an empty list.
std::vector<std::uint32_t> shard_halo_cells(int level, int depth, bool periodic, int src, int dst,
                                            int world);
/// Lowest level whose cells are exchanged as a halo instead of an all-gather:
/// shard_exchange_level + 1 (the exchange level itself is all-gathered, the
/// redundant M2M above it needs every cell).  > depth: no halo levels.
int shard_halo_level(int depth, int world);

/// Bytes shard `rank` receives / sends in one upward exchange (rows of
/// `row_doubles` doubles): the all-gathered levels exch .. halo-1 plus the
/// deep-level halos.  `halo` false: the whole-level all-gather of every level
/// exch .. depth (the former schedule, for comparison).
void shard_exchange_bytes(int depth, bool periodic, int row_doubles, int rank, int world, bool halo,
                          std::size_t* recv, std::size_t* send);

/// Owner shard of lex cell `cell` at `level` in a depth-`depth` tree.
int shard_cell_owner(int level, std::uint32_t cell, int depth, int world);

/// Shard that evaluates the canonical M2L instance (t, s) at `level`.
int shard_m2l_owner(int level, std::uint32_t t, std::uint32_t s, int depth, int world);

/// Canonical M2L instances of one (level, offset): Lambda(t) offsets are
/// s - t in [-2-c, 3-c] per axis with c = t & 1 (octree.cpp:79-87), wrapped
/// with split_extended (octree.cpp:11-14) when periodic, kept iff
/// t < s or (t == s and image lex-positive) (fmm.cpp:246-250).  Only instances
/// owned by `rank` (shard_m2l_owner) are returned (rank < 0: all), as (t, s)
/// pairs in lex t order.
struct OffsetInstances {
  int level = 0;
  std::array<int, 3> offset{};
  std::vector<std::uint32_t> t, s;
};
void enumerate_offset(OffsetInstances& w, bool periodic, int depth, int rank, int world);

/// All (level, offset) groups with at least one instance owned by `rank`.
std::vector<OffsetInstances> enumerate_m2l(int depth, bool periodic, int rank, int world,
                                           int threads);

}  // namespace ankh_b200
