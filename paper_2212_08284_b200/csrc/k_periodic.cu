// Periodic far-image term and the final deterministic reduction (sm_100a).
//
// Precompute (plan): the circulant generator of build_periodic_operator
// (fmm.cpp:333-377): gen[a,b,c] = sum_{2 <= |I|_inf <= p} H(z - 2 r_B I),
// z = h (a if a < L else a - (2L-1)) per axis, h = 2 r_B / (L-1).  One CTA per
// generator entry, fixed-order block reduction (run-to-run deterministic).
//
// Evaluation: periodic_far_energy (fmm.cpp:421-427 with
// CirculantSpectrum::quadratic_form, spectral.cpp:73-104) in ONE CTA:
//   root_equi = (T (x) T (x) T) M_root   (T = Chebyshev -> equispaced)
//   w = r2c( pad(root_equi) ) over (2L-1)^3, separable DFT in shared memory
//   e = 0.5 * (1/m) sum_k mult_k Re(spec_k) |w_k|^2
#include "kernels.cuh"

namespace ankh_b200 {

namespace {

constexpr double kTwoOverSqrtPi = 1.1283791670955125739;

__device__ __forceinline__ double erfc_screen_dev(double z) {
  // kernel.cpp:14-23, 48-51
  if (z >= 0.0 && z <= 0.5) {
    const double z2 = z * z;
    double term = z, sum = 0.0;
#pragma unroll
    for (int n = 0; n < 13; ++n) {
      sum += term / (2 * n + 1);
      term *= -z2 / (n + 1);
    }
    return 1.0 - kTwoOverSqrtPi * sum;
  }
  return erfc(z);
}

__global__ void __launch_bounds__(256) k_periodic_gen(double* __restrict__ gen, int L, double rb,
                                                      double xi, int p) {
  __shared__ double red[8];
  const int eb = 2 * L - 1;
  const int idx = blockIdx.x;
  const int a = idx / (eb * eb), b = (idx / eb) % eb, c = idx % eb;
  const double h = 2.0 * rb / (L - 1);
  const double z0 = h * (a < L ? a : a - eb), z1 = h * (b < L ? b : b - eb),
               z2 = h * (c < L ? c : c - eb);
  const double period = 2.0 * rb;
  const int w = 2 * p + 1;
  const long long total = static_cast<long long>(w) * w * w;
  double acc = 0.0;
  for (long long s = threadIdx.x; s < total; s += 256) {
    const int ix = static_cast<int>(s / (w * w)) - p;
    const int iy = static_cast<int>((s / w) % w) - p;
    const int iz = static_cast<int>(s % w) - p;
    if (max(max(abs(ix), abs(iy)), abs(iz)) < 2) continue;
    const double dx = z0 - period * ix, dy = z1 - period * iy, dz = z2 - period * iz;
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    acc += erfc_screen_dev(xi * r) / r;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += red[k];
    gen[idx] = t;
  }
}

constexpr int kPerThreads = 256;

__global__ void __launch_bounds__(kPerThreads) k_periodic_eval(const double* __restrict__ root,
                                                               const double* __restrict__ T,
                                                               const double* __restrict__ spec_re,
                                                               int L, double* __restrict__ out,
                                                               double* __restrict__ gbuf) {
  extern __shared__ double sm[];
  const int eb = 2 * L - 1, L2 = L * L, K = L2 * L;
  // working set in shared memory, or (large orders) in a global scratch
  double* v = gbuf ? gbuf : sm;   // K   (root, then scratch)
  double* t1 = v + K;             // K
  double* t2 = t1 + K;            // K
  double* tw_c = t2 + K;          // eb twiddles
  double* tw_s = tw_c + eb;
  double* w2r = tw_s + eb;        // L x L x L  (a, b, kz)
  double* w2i = w2r + K;
  double* w1r = w2i + K;          // L x eb x L (a, ky, kz)
  double* w1i = w1r + L * eb * L;
  double* red = w1i + L * eb * L; // kPerThreads
  const int tid = threadIdx.x;
  for (int e = tid; e < K; e += kPerThreads) v[e] = root[e];
  for (int k = tid; k < eb; k += kPerThreads) {
    double s, c;
    sincospi(-2.0 * k / eb, &s, &c);
    tw_c[k] = c;
    tw_s[k] = s;
  }
  __syncthreads();
  // tensor3_apply(T, T, T, root): z, then y, then x  (chebyshev.cpp:246-272)
  for (int e = tid; e < K; e += kPerThreads) {
    const int ab = e / L, k = e - L * (e / L);
    double acc = 0.0;
    for (int c = 0; c < L; ++c) acc += T[k * L + c] * v[ab * L + c];
    t1[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < K; e += kPerThreads) {
    const int a = e / L2, jk = e - L2 * (e / L2), j = jk / L, k = jk - L * (jk / L);
    double acc = 0.0;
    for (int b = 0; b < L; ++b) acc += T[j * L + b] * t1[a * L2 + b * L + k];
    t2[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < K; e += kPerThreads) {
    const int i = e / L2, jk = e - L2 * (e / L2);
    double acc = 0.0;
    for (int a = 0; a < L; ++a) acc += T[i * L + a] * t2[a * L2 + jk];
    v[e] = acc;  // root_equi
  }
  __syncthreads();
  // r2c along z: kz in [0, L) (= eb/2 + 1), inputs c in [0, L)
  for (int e = tid; e < K; e += kPerThreads) {
    const int ab = e / L, kz = e - L * (e / L);
    double sr = 0.0, si = 0.0;
    for (int c = 0; c < L; ++c) {
      const int ph = (c * kz) % eb;
      sr += v[ab * L + c] * tw_c[ph];
      si += v[ab * L + c] * tw_s[ph];
    }
    w2r[e] = sr;
    w2i[e] = si;
  }
  __syncthreads();
  // y: ky in [0, eb), inputs b in [0, L)
  for (int e = tid; e < L * eb * L; e += kPerThreads) {
    const int a = e / (eb * L), rem = e - (eb * L) * (e / (eb * L)), ky = rem / L,
              kz = rem - L * (rem / L);
    double sr = 0.0, si = 0.0;
    for (int b = 0; b < L; ++b) {
      const int ph = (b * ky) % eb;
      const double xr = w2r[(a * L + b) * L + kz], xi = w2i[(a * L + b) * L + kz];
      sr += xr * tw_c[ph] - xi * tw_s[ph];
      si += xr * tw_s[ph] + xi * tw_c[ph];
    }
    w1r[e] = sr;
    w1i[e] = si;
  }
  __syncthreads();
  // x: kx in [0, eb); accumulate mult * Re(spec) * |w|^2
  double acc = 0.0;
  for (int e = tid; e < eb * eb * L; e += kPerThreads) {
    const int kx = e / (eb * L), rem = e - (eb * L) * (e / (eb * L)), ky = rem / L,
              kz = rem - L * (rem / L);
    double sr = 0.0, si = 0.0;
    for (int a = 0; a < L; ++a) {
      const int ph = (a * kx) % eb;
      const double xr = w1r[(a * eb + ky) * L + kz], xi = w1i[(a * eb + ky) * L + kz];
      sr += xr * tw_c[ph] - xi * tw_s[ph];
      si += xr * tw_s[ph] + xi * tw_c[ph];
    }
    const double mult = kz == 0 ? 1.0 : 2.0;
    acc += mult * spec_re[e] * (sr * sr + si * si);
  }
  red[tid] = acc;
  __syncthreads();
  for (int s = kPerThreads / 2; s > 0; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  if (tid == 0) out[0] = 0.5 * red[0] / static_cast<double>(eb * eb * eb);
}

constexpr int kFinThreads = 256;
constexpr int kFinBlocks = 64;  // first level: contiguous slices, fixed order
static_assert(3 * kFinBlocks <= kFinThreads, "k_finalize stages the slices in red[]");

__device__ double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = kFinThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

__device__ unsigned long long block_sum_u64(unsigned long long v, unsigned long long* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = kFinThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const unsigned long long r = red[0];
  __syncthreads();
  return r;
}

template <typename T>
__device__ T slice_sum(const T* __restrict__ a, int n) {
  const int lo = static_cast<int>(static_cast<long long>(n) * blockIdx.x / kFinBlocks);
  const int hi = static_cast<int>(static_cast<long long>(n) * (blockIdx.x + 1) / kFinBlocks);
  T acc = 0;
  if (a)
    for (int i = lo + threadIdx.x; i < hi; i += kFinThreads) acc += a[i];
  return acc;
}

// Level 1: block b sums slice b of every partial array (fixed order per
// slice).  Level 2 runs in the block that finishes last (completion counter
// after a release fence): one pass over the kFinBlocks slices in slice order,
// so the result is bitwise independent of which block that is.  The counter
// is left at zero for the next evaluation (and CUDA-graph replays).
__global__ void __launch_bounds__(kFinThreads) k_finalize(
    const double* __restrict__ near_partial, int n_near,
    const unsigned long long* __restrict__ pair_count, int n_count,
    const double* __restrict__ far_partial, int n_far, const double* __restrict__ self_partial,
    int n_self, double* slices, unsigned long long* slice_pairs, unsigned* done,
    double self_scale, const double* __restrict__ periodic, int use_periodic, int include_self,
    DevResult* res) {
  __shared__ double red[kFinThreads];
  __shared__ unsigned long long redu[kFinThreads];
  __shared__ bool last;
  const double a = block_sum(slice_sum(near_partial, n_near), red);
  const double b = block_sum(slice_sum(far_partial, n_far), red);
  const double c = block_sum(slice_sum(self_partial, n_self), red);
  const unsigned long long p = block_sum_u64(slice_sum(pair_count, n_count), redu);
  if (threadIdx.x == 0) {
    slices[3 * blockIdx.x + 0] = a;
    slices[3 * blockIdx.x + 1] = b;
    slices[3 * blockIdx.x + 2] = c;
    slice_pairs[blockIdx.x] = p;
    __threadfence();
    last = atomicAdd(done, 1u) == kFinBlocks - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the other blocks' slices: one L2 load per thread, then the fixed-order sum
  if (threadIdx.x < kFinBlocks) {
    red[threadIdx.x] = __ldcg(slices + 3 * threadIdx.x);
    red[kFinBlocks + threadIdx.x] = __ldcg(slices + 3 * threadIdx.x + 1);
    red[2 * kFinBlocks + threadIdx.x] = __ldcg(slices + 3 * threadIdx.x + 2);
    redu[threadIdx.x] = __ldcg(slice_pairs + threadIdx.x);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double e_near = 0.0, e_far = 0.0, self_acc = 0.0;
  unsigned long long pairs = 0;
  for (int k = 0; k < kFinBlocks; ++k) {
    e_near += red[k];
    e_far += red[kFinBlocks + k];
    self_acc += red[2 * kFinBlocks + k];
    pairs += redu[k];
  }
  res->red[kENear] = e_near;
  res->red[kEFar] = e_far;
  res->red[kESelf] = include_self ? self_scale * self_acc : 0.0;  // -xi/sqrt(pi) acc (kernel.cpp:212)
  res->red[kEPeriodic] = use_periodic ? periodic[0] : 0.0;
  res->red[kNearPairs] = static_cast<double>(pairs);
  *done = 0u;
}

}  // namespace

void launch_periodic_gen(double* gen, int order, double box_radius, double xi, int p,
                         cudaStream_t st) {
  const int eb = 2 * order - 1;
  k_periodic_gen<<<eb * eb * eb, 256, 0, st>>>(gen, order, box_radius, xi, p);
}

namespace {
constexpr std::size_t kPerSmemMax = 200 * 1024;
std::size_t periodic_eval_doubles(int L) {
  const std::size_t eb = 2 * L - 1, K = static_cast<std::size_t>(L) * L * L;
  return 3 * K + 2 * eb + 2 * K + 2 * L * eb * L + kPerThreads;
}
}  // namespace

std::size_t periodic_eval_scratch_doubles(int order) {
  const std::size_t d = periodic_eval_doubles(order);
  return d * sizeof(double) <= kPerSmemMax ? 0 : d;
}

void launch_periodic_eval(const double* root, const double* to_equi, const double* spec_re,
                          int order, double* out, cudaStream_t st, double* scratch) {
  const int L = order;
  const bool global = periodic_eval_scratch_doubles(L) != 0;
  const std::size_t smem = global ? 0 : sizeof(double) * periodic_eval_doubles(L);
  static std::atomic<unsigned long long> attr{0};
  smem_opt_in(attr, k_periodic_eval, kPerSmemMax);
  k_periodic_eval<<<1, kPerThreads, smem, st>>>(root, to_equi, spec_re, L, out, global ? scratch : nullptr);
}

void launch_finalize(const double* near_partial, int n_near, const unsigned long long* pair_count,
                     int n_count, const double* far_partial, int n_far, const double* self_partial,
                     int n_self, double self_scale, const double* periodic, int use_periodic,
                     int include_self, double* scratch, DevResult* res, cudaStream_t st) {
  // scratch: kFinBlocks x 3 doubles, kFinBlocks uint64, the completion
  // counter (finalize_scratch_bytes; zeroed once at allocation)
  unsigned long long* slice_pairs = reinterpret_cast<unsigned long long*>(scratch + 3 * kFinBlocks);
  unsigned* done = reinterpret_cast<unsigned*>(slice_pairs + kFinBlocks);
  k_finalize<<<kFinBlocks, kFinThreads, 0, st>>>(near_partial, n_near, pair_count, n_count, far_partial, n_far,
                                                 include_self ? self_partial : nullptr, n_self, scratch,
                                                 slice_pairs, done, self_scale, periodic, use_periodic,
                                                 include_self, res);
}

std::size_t finalize_scratch_bytes() {
  return kFinBlocks * (3 * sizeof(double) + sizeof(unsigned long long)) + 16;
}

}  // namespace ankh_b200
