// Halo exchange of the deep expansion levels: pack the rows a
// shard sends (its own cells that a peer's M2L reads) into one contiguous
// buffer per peer, and unpack received rows into their Morton slots of the
// level-major expansion array.  Pure HBM copies (one 8*Kp-byte row per warp,
// 16-B accesses); the row lists are built once per plan (shard.cpp
// shard_halo_cells) as offsets in doubles into the expansion array.
#include "kernels.cuh"

namespace ankh_b200 {

namespace {

constexpr int kHaloThreads = 256;
constexpr int kRowsPerBlock = kHaloThreads / 32;

// dir 0: buf[j] = exp[row_off[j]] (pack); dir 1: exp[row_off[j]] = buf[j] (unpack)
__global__ void __launch_bounds__(kHaloThreads) k_halo_rows(double* __restrict__ exp,
                                                            const long long* __restrict__ row_off,
                                                            long long n_rows, int Kp,
                                                            double* __restrict__ buf, int dir) {
  const long long j = static_cast<long long>(blockIdx.x) * kRowsPerBlock + (threadIdx.x >> 5);
  if (j >= n_rows) return;
  const int lane = threadIdx.x & 31;
  double2* e = reinterpret_cast<double2*>(exp + row_off[j]);
  double2* b = reinterpret_cast<double2*>(buf + j * Kp);
  for (int k = lane; k < Kp / 2; k += 32) {
    if (dir == 0)
      b[k] = e[k];
    else
      e[k] = b[k];
  }
}

}  // namespace

void launch_halo_rows(double* exp, const long long* row_off, long long n_rows, int Kp, double* buf,
                      bool unpack, cudaStream_t st) {
  if (n_rows <= 0) return;
  const unsigned blocks = static_cast<unsigned>((n_rows + kRowsPerBlock - 1) / kRowsPerBlock);
  k_halo_rows<<<blocks, kHaloThreads, 0, st>>>(exp, row_off, n_rows, Kp, buf, unpack ? 1 : 0);
}

}  // namespace ankh_b200
