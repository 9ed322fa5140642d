// FP64 pipe peak probe (roofline denominator).  MEASURED_PEAKS.json carries
// HBM and bf16 figures only, so bench.py measures the DFMA peak in-process,
// right before its timed region, with this kernel: 8 independent FMA chains
// per thread, 4 CTAs x 256 threads per SM, timed with CUDA events.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ankh_b200 {

namespace {
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double b, double c) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}
}  // namespace

double probe_fp64_tflops(int iters) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  cudaMalloc(&d, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4;
  k_dfma<<<blocks, 256>>>(d, iters / 4 + 1, 0.999999, 1e-7);  // warm-up / clock ramp
  cudaEventRecord(e0);
  k_dfma<<<blocks, 256>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * 256;
  return ms > 0 ? flops / (ms * 1e-3) / 1e12 : 0.0;
}

}  // namespace ankh_b200
