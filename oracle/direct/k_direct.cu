// TEST INFRASTRUCTURE ONLY (checker, not the product): built into
// oracle/direct/libankh_direct.so, loaded by tests/ through oracle/direct.py.
//
// Direct screened lattice sum on sm_100a -- the exact quantity the FMM
// approximates, for validating it (SPEC's `direct` method; the reference has no
// direct engine):
//
//   E_lattice = 1/2 sum_{|I|inf <= p} sum_{i, j; (i != j or I != 0)}
//               pair_interaction(x_i, x_j + 2 r_B I)
//
// with the same screened pair energy as the near field (pair.cuh, i.e.
// kernel.cpp:157-204 with erfc(xi r)/r); e_total = E_lattice + self_energy.
// SURVEY.md Appendix B uses this definition to check the reference (relative
// FMM errors 1.2e-4 / 6.7e-6 / 7.2e-7 at L = 4 / 6 / 8).  Cost n^2 (2p+1)^3
// pair evaluations: a validation tool for n up to a few thousand.
//
// Grid: (target tiles of 64) x (2p+1)^2 image columns (I_x, I_y); each CTA
// stages the sources in shared memory in tiles and walks I_z; a thread keeps
// its target in registers and shifts it by -2 r_B I (r = x_i - 2 r_B I - x_j).
// Per-CTA partials, summed in a fixed order on the host (deterministic).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "pair.cuh"

namespace ankh_b200 {

namespace {

constexpr int kDirThreads = 64;
constexpr int kDirTile = 128;  // staged sources per pass

__global__ void k_direct_records(const double* __restrict__ pos, const double* __restrict__ src,
                                 std::size_t n, double* __restrict__ rec) {
  const std::size_t i = static_cast<std::size_t>(blockIdx.x) * 256 + threadIdx.x;
  if (i >= n) return;
  double* r = rec + i * kRec;
  r[0] = pos[3 * i];
  r[1] = pos[3 * i + 1];
  r[2] = pos[3 * i + 2];
  for (int k = 0; k < 10; ++k) r[3 + k] = src[10 * i + k];
  r[13] = (r[7] + r[10]) + r[12];  // SymMat3::trace (types.hpp:57)
}

__global__ void __launch_bounds__(kDirThreads) k_direct(const double* __restrict__ rec, int n,
                                                        int p, double period,
                                                        const __grid_constant__ P2PParams pp,
                                                        double* __restrict__ partial) {
  __shared__ __align__(16) double sm[kDirTile * kRec];
  __shared__ double red[kDirThreads / 32];
  const int tid = threadIdx.x;
  const int i = blockIdx.x * kDirThreads + tid;
  const int side = 2 * p + 1;
  const int ix = static_cast<int>(blockIdx.y) / side - p, iy = static_cast<int>(blockIdx.y) % side - p;
  Target a{};
  if (i < n) a = load_target(rec + static_cast<std::size_t>(i) * kRec);
  const double ax = a.x - period * ix, ay = a.y - period * iy, az = a.z;
  double acc = 0.0;
  for (int j0 = 0; j0 < n; j0 += kDirTile) {
    const int cnt = min(kDirTile, n - j0);
    __syncthreads();
    for (int w = tid; w < cnt * kRec; w += kDirThreads) sm[w] = rec[static_cast<std::size_t>(j0) * kRec + w];
    __syncthreads();
    if (i < n) {
      for (int iz = -p; iz <= p; ++iz) {
        a.x = ax;
        a.y = ay;
        a.z = az - period * iz;
        const bool central = ix == 0 && iy == 0 && iz == 0;
        for (int j = 0; j < cnt; ++j) {
          if (central && j0 + j == i) continue;  // the x = y term of the central cell
          acc = pair_mp<14>(a, sm + j * kRec, pp, acc);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kDirThreads / 32; ++w) t += red[w];
    partial[blockIdx.y * gridDim.x + blockIdx.x] = 0.5 * t;
  }
}

}  // namespace

int direct_partials(int n, int p) {
  const int side = 2 * p + 1;
  return ((n + kDirThreads - 1) / kDirThreads) * side * side;
}

void launch_direct(const double* pos, const double* src, int n, double box_radius, double xi,
                   int p, const P2PRadial& rad, double* rec, double* partial, cudaStream_t st) {
  if (n <= 0) return;
  k_direct_records<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(pos, src, n, rec);
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
  const int side = 2 * p + 1;
  dim3 grid(static_cast<unsigned>((n + kDirThreads - 1) / kDirThreads),
            static_cast<unsigned>(side * side));
  k_direct<<<grid, kDirThreads, 0, st>>>(rec, n, p, 2.0 * box_radius, pp, partial);
}

}  // namespace ankh_b200

// C-ABI of the checker.  The radial polynomials come from the product's
// ankh_radial_fit_v1(1e9) (valid to s = 0.25, libm beyond: any distance).
//   *e_lattice = 1/2 sum_{|I|inf <= p} sum_{i,j: i != j or I != 0}
//                pair_interaction(x_i, x_j + 2 r_B I)          (kernel.cpp:157-204)
// Returns 0, or 1 with a message in err.
extern "C" int ankh_direct_lattice_v1(size_t n, const double* positions, const double* sources,
                                      double box_radius, double xi, int p, int nterms, double s_lim,
                                      const double* pcoef, const double* gcoef, double* e_lattice,
                                      char* err, size_t errlen) {
  using namespace ankh_b200;
  auto fail = [&](const std::string& m) {
    if (err && errlen) {
      std::strncpy(err, m.c_str(), errlen - 1);
      err[errlen - 1] = '\0';
    }
    return 1;
  };
  *e_lattice = 0.0;
  if (n == 0) return 0;
  if (n >= (1u << 30)) return fail("direct: too many particles");
  const int ni = static_cast<int>(n);
  const int np = direct_partials(ni, p);
  P2PRadial rad{};
  rad.nterms = nterms;
  rad.s_lim = s_lim;
  std::memcpy(rad.p, pcoef, sizeof rad.p);
  std::memcpy(rad.g, gcoef, sizeof rad.g);
  double *d_pos = nullptr, *d_src = nullptr, *d_rec = nullptr, *d_part = nullptr;
  cudaError_t e = cudaSuccess;
  std::vector<double> part(np);
  if ((e = cudaMalloc(&d_pos, n * 3 * sizeof(double))) == cudaSuccess &&
      (e = cudaMalloc(&d_src, n * 10 * sizeof(double))) == cudaSuccess &&
      (e = cudaMalloc(&d_rec, n * kRec * sizeof(double))) == cudaSuccess &&
      (e = cudaMalloc(&d_part, np * sizeof(double))) == cudaSuccess &&
      (e = cudaMemcpy(d_pos, positions, n * 3 * sizeof(double), cudaMemcpyHostToDevice)) == cudaSuccess &&
      (e = cudaMemcpy(d_src, sources, n * 10 * sizeof(double), cudaMemcpyHostToDevice)) == cudaSuccess) {
    launch_direct(d_pos, d_src, ni, box_radius, xi, p, rad, d_rec, d_part, nullptr);
    if ((e = cudaGetLastError()) == cudaSuccess)
      e = cudaMemcpy(part.data(), d_part, np * sizeof(double), cudaMemcpyDeviceToHost);
  }
  cudaFree(d_pos);
  cudaFree(d_src);
  cudaFree(d_rec);
  cudaFree(d_part);
  if (e != cudaSuccess) return fail(std::string("direct: ") + cudaGetErrorString(e));
  double acc = 0.0;
  for (double v : part) acc += v;  // fixed order
  *e_lattice = acc;
  return 0;
}
