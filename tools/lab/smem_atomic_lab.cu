// Throughput of shared-memory fp64 atomicAdd (CAS loop on sm_100a) vs plain
// LDS/STS read-modify-write, random addresses in a 16 KB window (the access
// pattern of a symmetric SpMV's transposed half inside a 2048-row tile).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_atom(double* out, int iters, int mode) {
  __shared__ double y[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) y[i] = 0.0;
  __syncthreads();
  unsigned s = 1234567u * (threadIdx.x + 1) + blockIdx.x;
  double v = 1.0 + threadIdx.x * 1e-3;
  double acc2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int it = 0; it < iters; it += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // 8 independent operations per iteration
      s = s * 1664525u + 1013904223u;
      const int j = (threadIdx.x * 7 + (s >> 21)) & 2047;  // mostly distinct within a warp
      if (mode == 0) atomicAdd(&y[j], v);
      else if (mode == 1) y[j] += v;               // racy RMW (cost reference only)
      else acc2[u] += y[j];                        // plain load
    }
  }
  for (int u = 0; u < 8; ++u) v += acc2[u];
  __syncthreads();
  double acc = 0.0;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) acc += y[i];
  if (acc == 123.456) out[0] = acc + v;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, grid = 148 * 8, block = 256;
  for (int mode = 0; mode < 3; ++mode) {
    k_atom<<<grid, block>>>(d, iters, mode);
    cudaEventRecord(a);
    k_atom<<<grid, block>>>(d, iters, mode);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)grid * block * iters;
    printf("mode %d (%s): %.3f ms, %.1f Gop/s, %.2f lane-ops/clk/SM at 1.9 GHz\n", mode,
           mode == 0 ? "atomicAdd f64 smem" : mode == 1 ? "LDS+DADD+STS" : "LDS", ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
