// Bandwidth of 1-D bulk asynchronous copies (cp.async.bulk global->shared)
// streamed through a shared-memory ring, one CTA per SM (lab, not product).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool mtest(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
  return ok;
}

// NP producer threads (lanes of warp 0, one sub-ring each), consumer warps 1..NC
template <int NP>
__global__ void k_bulk(const char* src, int64_t bytes_per_cta, int chunk, int slots, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)slots * chunk);
  uint64_t* empty = full + slots;
  volatile int* seq = reinterpret_cast<volatile int*>(empty + slots);
  const char* base = src + (int64_t)blockIdx.x * bytes_per_cta;
  const int nchunks = (int)(bytes_per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int k = 0; k < slots; ++k) {
      seq[k] = -1;
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + k)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(empty + k)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nc = blockDim.x / 32 - 1;
  if (warp == 0) {
    if (lane < NP) {
      // producer p handles chunks q = p, p + NP, ... ; slot = q % slots
      for (int q = lane; q < nchunks; q += NP) {
        const int slot = q % slots;
        const uint32_t par = (uint32_t)((q / slots) & 1);
        if (q >= slots) while (!mtest(empty + slot, par ^ 1u)) {}
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + slot)), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(sm + (size_t)slot * chunk)), "l"(base + (int64_t)q * chunk), "r"(chunk), "r"(sa(full + slot)) : "memory");
        seq[slot] = q;
      }
    }
    return;
  }
  unsigned long long acc = 0;
  for (int q = warp - 1; q < nchunks; q += nc) {
    const int slot = q % slots;
    while (seq[slot] != q) {}
    while (!mtest(full + slot, (uint32_t)((q / slots) & 1))) {}
    acc += reinterpret_cast<const unsigned long long*>(sm + (size_t)slot * chunk)[lane];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + slot)) : "memory");
  }
  if (acc == 0x1234567ull) sink[0] = acc;
}

__global__ void k_ldg(const double* src, int64_t n, double* sink) {
  double acc = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) acc += __ldcs(src + k);
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  const int64_t total = 1ll << 30;  // 1 GiB
  char* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 64);
  char* flush;
  cudaMalloc(&flush, 512 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int ncta = 148;
  const int64_t per = (total / ncta) / 16384 * 16384;
  auto run = [&](auto kern, int np, int chunk, int slots, int nwarps) {
    const size_t smem = (size_t)slots * chunk + 24 * slots;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(flush, r, 512 << 20);
      cudaEventRecord(a);
      kern<<<ncta, nwarps * 32, smem>>>(src, per, chunk, slots, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("bulk np=%d chunk=%6d slots=%3d warps=%2d: %7.1f GB/s %s\n", np, chunk, slots, nwarps,
           (double)per * ncta / best / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  for (int chunk : {1024, 2048, 4096, 8192, 16384})
    for (int np : {1, 4})
      for (int slots : {8, 24}) {
        if ((size_t)slots * chunk > 200 * 1024) continue;
        if (np == 1) run(k_bulk<1>, 1, chunk, slots, 17);
        else run(k_bulk<4>, 4, chunk, slots, 17);
      }
  run(k_bulk<4>, 4, 4096, 40, 17);
  run(k_bulk<8>, 8, 4096, 40, 17);
  run(k_bulk<8>, 8, 2048, 80, 17);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaMemset(flush, r, 512 << 20);
    cudaEventRecord(a);
    k_ldg<<<148 * 4, 512>>>((const double*)src, total / 8, (double*)sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("ldg: %7.1f GB/s\n", (double)total / best / 1e6);
  return 0;
}
