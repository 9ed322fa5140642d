// FP64 pipe peak probe (roofline denominator).  MEASURED_PEAKS.json carries
// HBM and bf16 figures only, so bench.py measures the DFMA peak in-process,
// right before its timed region: the best of a few DFMA-chain shapes (8 / 16
// / 32 independent chains per thread, 2 / 4 / 8 CTAs of 256 threads per SM),
// timed with CUDA events.
#include <algorithm>

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ankh_b200 {

namespace {
template <int CH>
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double b, double c) {
  double a[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 128 / CH; ++r) {
#pragma unroll
      for (int k = 0; k < CH; ++k) a[k] = fma(a[k], b, c);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

// FP64 tensor-core (DMMA) peak: SHAPE 0 = m8n8k4 (256 FMA / instruction),
// 1 = m16n8k8 (1024), 2 = m16n8k16 (2048; sm_90+ shapes).  8 independent
// accumulators per warp, register operands only.
template <int SHAPE>
__global__ void __launch_bounds__(256) k_dmma(double* out, int iters) {
  double a[8], b[4], c[8][4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1e-3 * (threadIdx.x + k);
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = 1e-3 * (threadIdx.x - k);
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int k = 0; k < 4; ++k) c[t][k] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1])
                     : "d"(a[0]), "d"(b[0]));
      } else if (SHAPE == 1) {
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};\n"
            : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
            "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
            : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
              "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int k = 0; k < 4; ++k) s += c[t][k];
  if (s == 12345.678) out[0] = s;
}

// Do DFMA (FP64 pipe) and DMMA (FP64 tensor subpipe) share issue capacity?
// MODE 0: every warp runs DFMA chains; 1: every warp runs m8n8k4 DMMAs; 2: even
// warps DFMA, odd warps DMMA (half of each).  With the iteration counts
// balanced so that T0 ~ T1, T2 ~ T0 means one shared pipe, T2 ~ T0/2 two.
template <int MODE>
__global__ void __launch_bounds__(256) k_mix(double* out, int it_f, int it_m) {
  const bool f = MODE == 0 || (MODE == 2 && ((threadIdx.x >> 5) & 1) == 0);
  double s = 0.0;
  if (f) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < it_f; ++i) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 0.999999, 1e-7);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
  } else {
    double c[8][2];
    const double a = 1e-3 * threadIdx.x, b = 1e-3 * (threadIdx.x + 1);
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
    for (int i = 0; i < it_m; ++i) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1])
                     : "d"(a), "d"(b));
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  }
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
float time_mix(int it_f, int it_m, int blocks, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mix<MODE><<<blocks, 256>>>(d, it_f / 4 + 1, it_m / 4 + 1);
  cudaEventRecord(e0);
  k_mix<MODE><<<blocks, 256>>>(d, it_f, it_m);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms;
}

template <int SHAPE>
double time_dmma(int iters, int sms, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4;
  k_dmma<SHAPE><<<blocks, 256>>>(d, iters / 4 + 1);
  cudaEventRecord(e0);
  k_dmma<SHAPE><<<blocks, 256>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double fma_per = SHAPE == 0 ? 256.0 : (SHAPE == 1 ? 1024.0 : 2048.0);
  const double flops = 2.0 * fma_per * 8 * static_cast<double>(iters) * blocks * (256 / 32);
  return ms > 0 ? flops / (ms * 1e-3) / 1e12 : 0.0;
}
}  // namespace

double probe_dmma_tflops(int shape, int iters) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  cudaMalloc(&d, sizeof(double));
  double r = 0.0;
  if (shape == 0) r = time_dmma<0>(iters, sms, d);
  else if (shape == 1) r = time_dmma<1>(iters / 4, sms, d);
  else r = time_dmma<2>(iters / 8, sms, d);
  cudaFree(d);
  return r;
}

double probe_fp64_mix_ms(int mode, int it_f, int it_m) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  cudaMalloc(&d, sizeof(double));
  float ms = 0.f;
  if (mode == 0) ms = time_mix<0>(it_f, it_m, sms * 4, d);
  else if (mode == 1) ms = time_mix<1>(it_f, it_m, sms * 4, d);
  else ms = time_mix<2>(it_f, it_m, sms * 4, d);
  cudaFree(d);
  return ms;
}

double probe_fp64_tflops(int iters) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  cudaMalloc(&d, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // the best of a few shapes (independent chains per thread x resident CTAs
  // per SM): 128 FMA per thread per iteration in every case
  double best = 0.0;
  auto run = [&](auto kernel, int per_sm) {
    const int blocks = sms * per_sm;
    kernel<<<blocks, 256>>>(d, iters / 4 + 1, 0.999999, 1e-7);  // warm-up / clock ramp
    cudaEventRecord(e0);
    kernel<<<blocks, 256>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 128 * static_cast<double>(iters) * blocks * 256;
    if (ms > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  };
  run(k_dfma<8>, 4);
  run(k_dfma<8>, 8);
  run(k_dfma<16>, 4);
  run(k_dfma<16>, 2);
  run(k_dfma<32>, 2);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return best;
}

}  // namespace ankh_b200
