// Shared device helpers for libalyab200 (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <string>

#include "../../include/alyab200.h"

namespace ab {

extern std::atomic<int64_t> g_launches;
void set_error(const std::string& msg);

// Launch-status check used by every API entry point.
inline int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return AB_ECUDA;
  }
  return AB_OK;
}

inline int fail(const char* msg) {
  set_error(msg);
  return AB_EINVAL;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// ---------------------------------------------------------------------------
// 256-bit global accesses (LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100a).
// Node vectors are [n][4] doubles, 32-byte aligned.
// ---------------------------------------------------------------------------
struct d4 { double x, y, z, w; };

__device__ __forceinline__ d4 ld4_nc(const double* p) {
  d4 r;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ d4 ld4(const double* p) {
  d4 r;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st4(double* p, d4 v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
               : "memory");
}

// fp64 reduction to global memory (REDG.E.ADD.F64.RN), no return value.
__device__ __forceinline__ void red_add(double* p, double v) { atomicAdd(p, v); }

// ---------------------------------------------------------------------------
// Deterministic grid-wide sums: per-block partials + "last block" finalize.
// The last block sums the partials in a fixed order, so results do not
// depend on block scheduling.
// ---------------------------------------------------------------------------
template <int NV, int BLOCK>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem /* NV * BLOCK/32 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) smem[k * (BLOCK / 32) + warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = lane < BLOCK / 32 ? smem[k * (BLOCK / 32) + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      v[k] = t;  // valid in warp 0
    }
  }
}

// Returns true in exactly one block (the last to finish); in that block
// `tot[k]` holds the grid total of value k.  Two-level and deterministic:
// blocks are grouped by kGroup; the last block of each group sums the
// group's partials in index order, and the last group sums the group totals
// in index order.  A single counter hit by every block serialises at one L2
// slice (~1 atomic per few ns, measured ~8 us for 2754 blocks); grouped
// counters keep each address to <= kGroup arrivals.
// part: >= NV * (nb + ceil(nb / kGroup)) doubles; cnt: >= 1 + ceil(nb / kGroup)
// zero-initialised uint32 (re-armed here).
constexpr int kGroup = 64;

template <int NV, int BLOCK>
__device__ __forceinline__ bool grid_sum(double (&v)[NV], double* part, uint32_t* cnt, double (&tot)[NV]) {
  __shared__ double sm[NV * (BLOCK / 32)];
  __shared__ int stage;  // 0: not last in group, 1: last in group, 2: last overall
  block_sum<NV, BLOCK>(v, sm);
  const int nb = gridDim.x;
  const int ng = (nb + kGroup - 1) / kGroup;
  const int g = blockIdx.x / kGroup;
  const int gsize = (g == ng - 1) ? nb - g * kGroup : kGroup;
  double* gpart = part + (size_t)NV * nb;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) part[(size_t)k * nb + blockIdx.x] = v[k];
    __threadfence();
    const unsigned prev = atomicAdd(&cnt[1 + g], 1u);
    stage = (prev == (unsigned)gsize - 1) ? 1 : 0;
  }
  __syncthreads();
  if (stage == 0) return false;
  __threadfence();
  // last block of group g: ordered sum of the group's partials
  if (threadIdx.x < 32) {
    double acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      acc[k] = 0.0;
      for (int b = threadIdx.x; b < gsize; b += 32) acc[k] += __ldcg(&part[(size_t)k * nb + g * kGroup + b]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    }
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) gpart[(size_t)k * ng + g] = acc[k];
      cnt[1 + g] = 0u;
      __threadfence();
      const unsigned prev = atomicAdd(&cnt[0], 1u);
      stage = (prev == (unsigned)ng - 1) ? 2 : 1;
    }
  }
  __syncthreads();
  if (stage != 2) return false;
  __threadfence();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double acc = 0.0;
      for (int b = threadIdx.x; b < ng; b += 32) acc += __ldcg(&gpart[(size_t)k * ng + b]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      tot[k] = acc;  // valid in warp 0
    }
    if (threadIdx.x == 0) cnt[0] = 0u;
  }
  return true;
}

}  // namespace ab
