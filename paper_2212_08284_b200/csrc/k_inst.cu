// M2L instance lists on the GPU (plan precompute): the
// canonical (target, source) cell pairs of every (level, offset) operator --
// fmm.cpp:238-276 with the closed-form offset set of §8a a8 -- written straight
// into the plan's instance array in the layout the host enumeration produced
// (shard.cpp enumerate_offset, then a sort by target Morton index):
//
//   op order   level 1..depth, then offset (ox, oy, oz) lexicographic, max |o| >= 2
//   per op     targets in ascending Morton order, each at most once
//   filters    t_a even for o_a = 3, odd for o_a = -3 (children of the
//              parent's neighbours); source inside the box unless periodic;
//              canonical t < s or (t == s and the image is lex-positive)
//              (fmm.cpp:43-56); shard ownership shard_m2l_owner
//
// Candidates are the 8^level Morton indices of each op, padded to whole
// 256-thread blocks so a block belongs to one op.  k_inst_count writes per-block
// counts, an exclusive scan turns them into write offsets (and per-op counts at
// the op boundaries), k_inst_write compacts in order.
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace ankh_b200 {

namespace {

constexpr int kInstBlock = 256;

__device__ __forceinline__ unsigned spread3d(unsigned v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__device__ __forceinline__ unsigned compact3d(unsigned v) {
  v &= 0x09249249u;
  v = (v ^ (v >> 2)) & 0x030c30c3u;
  v = (v ^ (v >> 4)) & 0x0300f00fu;
  v = (v ^ (v >> 8)) & 0x030000ffu;
  v = (v ^ (v >> 16)) & 0x000003ffu;
  return v;
}
__device__ __forceinline__ unsigned morton3d(unsigned x, unsigned y, unsigned z) {
  return (spread3d(x) << 2) | (spread3d(y) << 1) | spread3d(z);
}

// shard.cpp shard_leaf_range / shard_cell_owner / shard_m2l_owner
__device__ int cell_owner(int level, unsigned cell, int depth, int world) {
  const unsigned n = 1u << level;
  const unsigned i = cell / (n * n), j = (cell / n) % n, k = cell % n;
  const long long first_leaf = static_cast<long long>(morton3d(i, j, k)) << (3 * (depth - level));
  const long long nl = 1ll << (3 * depth);
  int r = static_cast<int>(first_leaf * world / nl);
  while (true) {
    const long long b = nl * r / world, e = nl * (r + 1) / world;
    if (first_leaf < b)
      --r;
    else if (first_leaf >= e)
      ++r;
    else
      return r;
  }
}
__device__ __forceinline__ int m2l_owner(int level, unsigned t, unsigned s, int depth, int world) {
  if (world <= 1) return 0;
  const unsigned h = t * 0x9E3779B1u ^ (s + 0x7F4A7C15u) * 0x85EBCA77u;
  return cell_owner(level, ((h >> 15) & 1u) ? s : t, depth, world);
}

// candidate Morton index m of operator (level, o): source Morton index or -1
__device__ __forceinline__ long long instance_source(int level, int ox, int oy, int oz, unsigned m,
                                                     int periodic, int depth, int rank, int world) {
  const int nl = 1 << level;
  if (m >= (1u << (3 * level))) return -1;
  const int t[3] = {static_cast<int>(compact3d(m >> 2)), static_cast<int>(compact3d(m >> 1)),
                    static_cast<int>(compact3d(m))};
  const int o[3] = {ox, oy, oz};
  int in[3], img[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (o[a] == 3 && (t[a] & 1)) return -1;
    if (o[a] == -3 && !(t[a] & 1)) return -1;
    const int ext = t[a] + o[a];
    if (!periodic && (ext < 0 || ext >= nl)) return -1;
    img[a] = ext >= 0 ? ext / nl : -((-ext + nl - 1) / nl);
    in[a] = ext - nl * img[a];
  }
  const unsigned tl = static_cast<unsigned>((t[0] * nl + t[1]) * nl + t[2]);
  const unsigned sl = static_cast<unsigned>((in[0] * nl + in[1]) * nl + in[2]);
  const bool lexpos = img[0] != 0 ? img[0] > 0 : (img[1] != 0 ? img[1] > 0 : img[2] > 0);
  if (!(tl < sl || (tl == sl && lexpos))) return -1;
  if (rank >= 0 && m2l_owner(level, tl, sl, depth, world) != rank) return -1;
  return morton3d(in[0], in[1], in[2]);
}

struct InstLevel {
  int level, n_ops, blocks_per_op;
  long long first_block;  // block index of this level's first op
};

// grid (blocks_per_op, n_ops of the level)
__global__ void __launch_bounds__(kInstBlock) k_inst_count(const int4* __restrict__ offs,
                                                           InstLevel lv, int periodic, int depth,
                                                           int rank, int world,
                                                           unsigned* __restrict__ counts) {
  const int4 o = offs[blockIdx.y];
  const unsigned m = blockIdx.x * kInstBlock + threadIdx.x;
  const bool keep = instance_source(lv.level, o.x, o.y, o.z, m, periodic, depth, rank, world) >= 0;
  const int c = __syncthreads_count(keep);
  if (threadIdx.x == 0)
    counts[lv.first_block + static_cast<long long>(blockIdx.y) * lv.blocks_per_op + blockIdx.x] = c;
}

__global__ void __launch_bounds__(kInstBlock) k_inst_write(const int4* __restrict__ offs,
                                                           InstLevel lv, int periodic, int depth,
                                                           int rank, int world,
                                                           const unsigned* __restrict__ offsets,
                                                           uint2* __restrict__ inst) {
  __shared__ unsigned warp_base[kInstBlock / 32];
  const int4 o = offs[blockIdx.y];
  const unsigned m = blockIdx.x * kInstBlock + threadIdx.x;
  const long long s = instance_source(lv.level, o.x, o.y, o.z, m, periodic, depth, rank, world);
  const unsigned ballot = __ballot_sync(0xffffffffu, s >= 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) warp_base[warp] = __popc(ballot);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned acc = 0;
    for (int w = 0; w < kInstBlock / 32; ++w) {
      const unsigned c = warp_base[w];
      warp_base[w] = acc;
      acc += c;
    }
  }
  __syncthreads();
  if (s >= 0) {
    const unsigned pos = offsets[lv.first_block + static_cast<long long>(blockIdx.y) * lv.blocks_per_op +
                                 blockIdx.x] +
                         warp_base[warp] + __popc(ballot & ((1u << lane) - 1u));
    inst[pos] = make_uint2(m, static_cast<unsigned>(s));
  }
}

}  // namespace

// Per-op instance counts (op order as above) into op_counts; returns the
// total.  With inst == nullptr only counts (and the device offsets) are built;
// call again with inst sized to the total to write the instances.
std::size_t m2l_instances_device(int depth, int periodic, int rank, int world, const int4* d_offs,
                                 int n_offs, unsigned* d_counts, unsigned* d_offsets,
                                 std::size_t n_blocks_total, void* d_temp, std::size_t temp_bytes,
                                 uint2* inst, cudaStream_t st) {
  long long first = 0;
  for (int level = 1; level <= depth; ++level) {
    const unsigned cand = 1u << (3 * level);
    InstLevel lv{level, n_offs, static_cast<int>((cand + kInstBlock - 1) / kInstBlock), first};
    if (inst == nullptr)
      k_inst_count<<<dim3(lv.blocks_per_op, n_offs), kInstBlock, 0, st>>>(d_offs, lv, periodic, depth,
                                                                          rank, world, d_counts);
    else
      k_inst_write<<<dim3(lv.blocks_per_op, n_offs), kInstBlock, 0, st>>>(
          d_offs, lv, periodic, depth, rank, world, d_offsets, inst);
    first += static_cast<long long>(lv.blocks_per_op) * n_offs;
  }
  if (inst == nullptr) {
    // counts[n_blocks_total] is the scan's extra slot (zero) -> total at the end
    std::size_t bytes = temp_bytes;
    cub::DeviceScan::ExclusiveSum(d_temp, bytes, d_counts, d_offsets,
                                  static_cast<int>(n_blocks_total + 1), st);
  }
  return static_cast<std::size_t>(first);
}

std::size_t m2l_instances_temp_bytes(std::size_t n_blocks_total) {
  std::size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const unsigned*>(nullptr),
                                static_cast<unsigned*>(nullptr), static_cast<int>(n_blocks_total + 1));
  return bytes;
}

std::size_t m2l_instance_blocks(int depth, int n_offs) {
  std::size_t b = 0;
  for (int level = 1; level <= depth; ++level)
    b += static_cast<std::size_t>(((1u << (3 * level)) + kInstBlock - 1) / kInstBlock) * n_offs;
  return b;
}

int m2l_instance_block_size() { return kInstBlock; }

}  // namespace ankh_b200
