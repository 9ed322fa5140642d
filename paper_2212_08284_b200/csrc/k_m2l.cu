// M2L far-field energy on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
//
// Restates far_field_energy (fmm.cpp:238-276): for every canonical instance
// (t, s) of one (level, offset) operator with factors L, R (k x K, from
// compress_m2l fmm.cpp:98-133)
//     e += (L M_t) . (R M_s)
// As a grouped GEMM: a CTA takes 64 instances of one operator, streams the
// factor rows (padded to kp = 8*KP8) and the 2 x 64 gathered expansions
// through shared memory in kChunk-node chunks (kStages-deep cp.async
// pipeline, one CTA barrier per chunk), and
// each warp accumulates U = L [M_t...] and V = R [M_s...] for its 8*NTW
// instances in DMMA fragments (rank rows = M dim, instances = N dim, nodes =
// K dim; every factor fragment feeds NTW instance tiles).  The energy of the
// tile is sum(U o V), reduced in a fixed order into one partial per tile.
// FP64-pipe bound: 4kK + 2k flops per instance.
#include "kernels.cuh"

namespace ankh_b200 {

namespace {

#ifndef ANKH_M2L_CHUNK
#define ANKH_M2L_CHUNK 8
#endif
#ifndef ANKH_M2L_STAGES
#define ANKH_M2L_STAGES 2
#endif
constexpr int kChunk = ANKH_M2L_CHUNK;   // node columns per pipeline stage
constexpr int kStages = ANKH_M2L_STAGES; // cp.async pipeline depth
constexpr int kStride = kChunk + 4;      // smem row stride (doubles): fragment loads in the minimal 2 wavefronts

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}

// 16-byte copy, zero-filled when !valid (src is not read then)
__device__ __forceinline__ void cp_async16z(double* dst, const double* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src),
               "r"(valid ? 16 : 0));
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// KP8 = padded rank / 8 (DMMA M tiles), NTW = 8-instance N tiles per warp.
// A warp reuses each factor fragment for its NTW instance tiles; the CTA has
// 64 / (8 NTW) warps and covers one 64-instance tile of one operator.
template <int KP8, int NTW>
__global__ void __launch_bounds__(kM2LTile * 4 / NTW) k_m2l(const double* __restrict__ exp,
                                                          const long long* __restrict__ level_off,
                                                          const double* __restrict__ factors,
                                                          const M2LOp* __restrict__ ops,
                                                          const M2LTile* __restrict__ tiles,
                                                          const int* __restrict__ tile_ids,
                                                          const uint2* __restrict__ inst, int K,
                                                          int Kp, double* __restrict__ far_partial) {
  constexpr int kp = 8 * KP8;
  constexpr int kThr = kM2LTile * 4 / NTW;  // 32 lanes per 8 NTW instances
  constexpr int kWarps = kThr / 32;
  constexpr int kStage = (2 * kp + 2 * kM2LTile) * kStride;  // doubles per pipeline stage
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[kWarps];
  __shared__ const double* s_row[2 * kM2LTile];  // expansion row of each target / source

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile_index = tile_ids[blockIdx.x];
  const M2LTile tile = tiles[tile_index];
  const M2LOp op = ops[tile.op];
  const double* Lg = factors + op.factor_off;
  const double* Rg = Lg + static_cast<long long>(kp) * Kp;
  const double* E = exp + level_off[tile.level];  // rows of Kp doubles, zero tail
  for (int q = tid; q < kM2LTile; q += kThr) {
    const uint2 ts = q < tile.count ? inst[tile.begin + q] : make_uint2(0u, 0u);
    ANKH_DASSERT(tile.count <= kM2LTile && ts.x < (1u << (3 * tile.level)) && ts.y < (1u << (3 * tile.level)));
    ANKH_DASSERT(op.kp == kp);
    s_row[q] = E + static_cast<long long>(ts.x) * Kp;
    s_row[kM2LTile + q] = E + static_cast<long long>(ts.y) * Kp;
  }
  __syncthreads();

  // stage chunk [k0, k0 + kChunk) of L, R and the 64 target / source expansions
  auto issue = [&](int k0, double* st) {
    double* sL = st;
    double* sR = sL + kp * kStride;
    double* sT = sR + kp * kStride;  // followed by the 64 source rows (sS)
    for (int w = tid; w < kp * (kChunk / 2); w += kThr) {
      const int r = w / (kChunk / 2), c = 2 * (w - (kChunk / 2) * (w / (kChunk / 2)));
      cp_async16(sL + r * kStride + c, Lg + static_cast<long long>(r) * Kp + k0 + c);
      cp_async16(sR + r * kStride + c, Rg + static_cast<long long>(r) * Kp + k0 + c);
    }
    // 2 x 64 rows x (kChunk / 2) 16-B pieces; sT and sS are contiguous in smem
    for (int w = tid; w < 2 * kM2LTile * (kChunk / 2); w += kThr) {
      const int q = w / (kChunk / 2), c = 2 * (w - (kChunk / 2) * (w / (kChunk / 2)));
      const bool ok = (q & (kM2LTile - 1)) < tile.count;
      cp_async16z(sT + q * kStride + c, s_row[q] + k0 + c, ok);
    }
  };

  double u[NTW][KP8][2], v[NTW][KP8][2];
#pragma unroll
  for (int t = 0; t < NTW; ++t)
#pragma unroll
    for (int m = 0; m < KP8; ++m) u[t][m][0] = u[t][m][1] = v[t][m][0] = v[t][m][1] = 0.0;

  const int row = lane >> 2, col = lane & 3;
  const int nchunks = Kp / kChunk;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nchunks) issue(s * kChunk, sm + s * kStage);
    cp_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    // chunk c has landed once at most kStages - 2 younger groups are pending;
    // the barrier also retires every reader of the buffer refilled next
    cp_wait<kStages - 2>();
    __syncthreads();
    if (c + kStages - 1 < nchunks)
      issue((c + kStages - 1) * kChunk, sm + ((c + kStages - 1) % kStages) * kStage);
    cp_commit();
    const double* st = sm + (c % kStages) * kStage;
    const double* sL = st;
    const double* sR = sL + kp * kStride;
    const double* bT = sR + kp * kStride + (warp * 8 * NTW + row) * kStride + col;
    const double* bS = bT + kM2LTile * kStride;
#pragma unroll
    for (int ks = 0; ks < kChunk / 4; ++ks) {
      double bt[NTW], bs[NTW];
#pragma unroll
      for (int t = 0; t < NTW; ++t) {
        bt[t] = bT[t * 8 * kStride + 4 * ks];
        bs[t] = bS[t * 8 * kStride + 4 * ks];
      }
#pragma unroll
      for (int m = 0; m < KP8; ++m) {
        const double al = sL[(8 * m + row) * kStride + 4 * ks + col];
        const double ar = sR[(8 * m + row) * kStride + 4 * ks + col];
#pragma unroll
        for (int t = 0; t < NTW; ++t) {
          dmma(u[t][m], al, bt[t]);
          dmma(v[t][m], ar, bs[t]);
        }
      }
    }
  }
  double e = 0.0;
#pragma unroll
  for (int t = 0; t < NTW; ++t)
#pragma unroll
    for (int m = 0; m < KP8; ++m) e += u[t][m][0] * v[t][m][0] + u[t][m][1] * v[t][m][1];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_down_sync(0xffffffffu, e, o);
  if (lane == 0) red[warp] = e;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) t += red[w];
    far_partial[tile_index] = t;
  }
}

template <int KP8>
void launch_class(const double* exp, const long long* level_off, const double* factors,
                  const M2LOp* ops, const M2LTile* tiles, int n_tiles, const int* tile_ids,
                  const uint2* inst, int K, int Kp, double* far_partial, cudaStream_t st) {
  // two instance tiles per warp for the common small-rank classes (register budget)
#ifndef ANKH_M2L_NTW_SMALL
#define ANKH_M2L_NTW_SMALL 2  // instance tiles per warp for KP8 <= 3
#endif
  constexpr int NTW = KP8 <= 3 ? ANKH_M2L_NTW_SMALL : (KP8 <= 5 ? 2 : 1);
  constexpr int kThr = kM2LTile * 4 / NTW;
  const std::size_t smem = kStages * sizeof(double) * (2 * 8 * KP8 + 2 * kM2LTile) * kStride;
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_m2l<KP8, NTW>, smem);
  k_m2l<KP8, NTW><<<n_tiles, kThr, smem, st>>>(exp, level_off, factors, ops, tiles, tile_ids,
                                               inst, K, Kp, far_partial);
}

}  // namespace

void launch_m2l(const double* exp, const long long* level_off, const double* factors,
                const M2LOp* ops, const M2LTile* tiles, int n_tiles_class, int kp8,
                const int* tile_ids, const uint2* inst, int K, int Kp, double* far_partial,
                cudaStream_t st) {
  if (n_tiles_class <= 0) return;
#define ANKH_M2L_CASE(N)                                                                    \
  case N:                                                                                   \
    launch_class<N>(exp, level_off, factors, ops, tiles, n_tiles_class, tile_ids, inst, K, \
                    Kp, far_partial, st);                                                   \
    break;
  switch (kp8) {
    ANKH_M2L_CASE(1)
    ANKH_M2L_CASE(2)
    ANKH_M2L_CASE(3)
    ANKH_M2L_CASE(4)
    ANKH_M2L_CASE(5)
    ANKH_M2L_CASE(6)
    ANKH_M2L_CASE(7)
    ANKH_M2L_CASE(8)
    ANKH_M2L_CASE(9)
    ANKH_M2L_CASE(10)
    ANKH_M2L_CASE(11)
    ANKH_M2L_CASE(12)
    ANKH_M2L_CASE(13)
    ANKH_M2L_CASE(14)
    ANKH_M2L_CASE(15)
    ANKH_M2L_CASE(16)
    default:
      break;
  }
#undef ANKH_M2L_CASE
}

}  // namespace ankh_b200
