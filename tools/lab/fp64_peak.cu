// Measured FP64 FMA throughput of this B200 (the binding roof of the element
// assembly K2): every thread runs 8 independent DFMA chains.
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 123.456) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 1 << 14, block = 256, grid = sms * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_dfma<<<grid, block>>>(out, iters, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_dfma<<<grid, block>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8.0 * iters * (double)grid * block;
  printf("{\"fp64_fma_tflops\": %.2f, \"sms\": %d, \"how\": \"%d CTAs x %d threads x 8 independent DFMA chains x %d "
         "iterations, best of 5, CUDA events\"}\n", flops / (best * 1e-3) / 1e12, sms, grid, block, iters);
  return 0;
}
