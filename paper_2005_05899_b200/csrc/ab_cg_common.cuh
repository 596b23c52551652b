// Device helpers shared by the resident CG kernels (ab_solver.cu, ab_cg_dd.cu):
// one 1024-thread CTA per SM, grid barriers on a monotone arrival counter,
// ordered all-sums of per-CTA partials, SELL-32 rows with 16-bit CTA-local
// columns read against z in shared memory.
#pragma once
#include "ab_common.cuh"

namespace ab {

constexpr int kResBlock = 1024;
#ifndef LOC_CHUNK
#define LOC_CHUNK 8
#endif
constexpr int kLocChunk = LOC_CHUNK;

// Grid barrier on a monotone arrival counter (zeroed before launch): the
// k-th barrier completes when the counter reaches k * gridDim.x.  One
// release-reduction per CTA and one acquire-polling thread per CTA; the
// CTA barriers on both sides extend the ordering to all threads.  Data
// exchanged across it is read with L2-only loads (ld.cg), so no stale L1
// lines are possible.
__device__ __forceinline__ void grid_barrier(unsigned* cnt, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__device__ __forceinline__ void prefetch_slice16(const int64_t* tsp, const uint16_t* lcol, const double* sval,
                                                 int sl) {
  const int64_t b = tsp[sl];
  const uint32_t cnt = (uint32_t)(tsp[sl + 1] - b);
  if (cnt == 0) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lcol + b), "r"(cnt * 2u) : "memory");
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sval + b), "r"(cnt * 8u) : "memory");
}

// tsp: slice pointers of the CTA's slices (local index sl, shared or global)
template <int CH>
__device__ __forceinline__ double sell_row_dot_smem(const int64_t* tsp, const uint16_t* __restrict__ lcol,
                                                    const double* __restrict__ sval, const double* zs, int sl,
                                                    int lane) {
  const int64_t b0 = tsp[sl];
  const int64_t base = b0 + lane;
  const int width = (int)((tsp[sl + 1] - b0) >> 5);
  double acc = 0.0;
  for (int j0 = 0; j0 < width; j0 += CH) {
    unsigned c[CH];
    double a[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const bool ok = j0 + u < width;
      c[u] = ok ? (unsigned)__ldcs(lcol + base + (int64_t)(j0 + u) * 32) : 0u;
      a[u] = ok ? __ldcs(sval + base + (int64_t)(j0 + u) * 32) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) acc = fma(a[u], zs[c[u]], acc);
  }
  return acc;
}

constexpr int kChunk = 16;

// (A z)_i for one SELL row: all column/value loads of a 16-wide chunk first,
// then the gathers, then the FMAs.  CG = true gathers through L2 only (z is
// rewritten inside the resident kernel).
template <bool CG = false>
__device__ __forceinline__ double sell_row_dot(const int64_t* __restrict__ sp, const int32_t* __restrict__ scol,
                                               const double* __restrict__ sval, const double* zv, int64_t i) {
  const int64_t s = i >> 5;
  const int lane = (int)(i & 31);
  const int64_t base = sp[s] + lane;
  const int width = (int)((sp[s + 1] - sp[s]) >> 5);
  double acc = 0.0;
  for (int j0 = 0; j0 < width; j0 += kChunk) {
    int c[kChunk];
    double a[kChunk];
#pragma unroll
    for (int u = 0; u < kChunk; ++u) {
      const bool ok = j0 + u < width;
      c[u] = ok ? __ldcs(scol + base + (int64_t)(j0 + u) * 32) : 0;
      a[u] = ok ? __ldcs(sval + base + (int64_t)(j0 + u) * 32) : 0.0;
    }
    double g[kChunk];
#pragma unroll
    for (int u = 0; u < kChunk; ++u) g[u] = CG ? __ldcg(zv + c[u]) : zv[c[u]];
#pragma unroll
    for (int u = 0; u < kChunk; ++u) acc = fma(a[u], g[u], acc);
  }
  return acc;
}


// Replicated per-CTA partials (resident solvers): the NV values of CTA b are
// written to kRep copies of a [NV][nbp] table (nbp = nb rounded up to 4),
// and CTA b reads copy b % kRep with 16-byte loads, so each 32-byte sector is
// requested by nb / kRep CTAs once instead of by every CTA four times.  The
// sum is a fixed tree (per-thread 4, warp xor tree, two warps per value):
// identical in every CTA, deterministic.  Needs nb <= 256.
constexpr int kRep = 4;
__host__ __device__ inline int rep_nbp(int nb) { return (nb + 3) & ~3; }

template <int NV>
__device__ __forceinline__ void put_partial_rep(double* tab, int nb, const double (&v)[NV]) {
  const int nbp = rep_nbp(nb);
#pragma unroll
  for (int r = 0; r < kRep; ++r)
#pragma unroll
    for (int k = 0; k < NV; ++k) tab[((size_t)r * NV + k) * nbp + blockIdx.x] = v[k];
}

template <int NV>
__device__ __forceinline__ void all_sum_rep(const double* tab, int nb, double* srep /* >= 2 * NV */,
                                            double (&out)[NV]) {
  const int nbp = rep_nbp(nb);
  const double* rp = tab + (size_t)(blockIdx.x % kRep) * NV * nbp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2 * NV) {
    const int k = warp >> 1, c = ((warp & 1) << 5) + lane, i = 4 * c;
    double s = 0.0;
    if (i < nb) {
      const double2 a = __ldcg(reinterpret_cast<const double2*>(rp + (size_t)k * nbp + i));
      const double2 b = __ldcg(reinterpret_cast<const double2*>(rp + (size_t)k * nbp + i + 2));
      s = a.x;
      if (i + 1 < nb) s += a.y;
      if (i + 2 < nb) s += b.x;
      if (i + 3 < nb) s += b.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) srep[warp] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = srep[2 * k] + srep[2 * k + 1];
}

// Ordered sum of nb (<= blockDim) per-CTA partials, all loads in flight at
// once (one L2 round trip), fixed reduction tree: identical in every CTA.
template <int NV>
__device__ __forceinline__ void all_sum_par(const double* part, int nb, double* sred, double* bcast,
                                            double (&out)[NV]) {
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = (int)threadIdx.x < nb ? __ldcg(part + (size_t)k * nb + threadIdx.x) : 0.0;
  block_sum<NV, kResBlock>(v, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) bcast[k] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = bcast[k];
}


__device__ __forceinline__ uint32_t sa32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMEM: one double per thread = two 32-bit columns of the thread's lane.
__device__ __forceinline__ void tm_ld(uint32_t a, uint32_t& lo, uint32_t& hi) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(a) : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double tm_val(uint32_t lo, uint32_t hi) {
  asm volatile("" : "+r"(lo), "+r"(hi));  // keep uses after tcgen05.wait::ld
  return __hiloint2double((int)hi, (int)lo);
}
__device__ __forceinline__ void tm_st(uint32_t a, double v) {
  const uint32_t lo = (uint32_t)__double2loint(v), hi = (uint32_t)__double2hiint(v);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "r"(lo), "r"(hi) : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 8 doubles / 8 packed 16-bit values per thread (16 / 4 columns)
__device__ __forceinline__ void tm_st8d(uint32_t a, const double (&v)[8]) {
  uint32_t w[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    w[2 * k] = (uint32_t)__double2loint(v[k]);
    w[2 * k + 1] = (uint32_t)__double2hiint(v[k]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(a),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
      "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
      : "memory");
}
__device__ __forceinline__ void tm_ld8d(uint32_t a, uint32_t (&w)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]),
        "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
      : "r"(a)
      : "memory");
}
__device__ __forceinline__ void tm_st4u(uint32_t a, const uint32_t (&w)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[0]), "r"(w[1]),
               "r"(w[2]), "r"(w[3])
               : "memory");
}
__device__ __forceinline__ void tm_ld4u(uint32_t a, uint32_t (&w)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
               : "r"(a)
               : "memory");
}
template <int N>
__device__ __forceinline__ void tm_fence_regs(uint32_t (&w)[N]) {  // keep uses after tcgen05.wait::ld
#pragma unroll
  for (int k = 0; k < N; ++k) asm volatile("" : "+r"(w[k]));
}

// TMEM allocation of all 512 columns by warp 0 (one CTA per SM), address in *slot.
__device__ __forceinline__ uint32_t tmem_alloc_all(uint32_t* slot) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa32(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  return *slot;
}
__device__ __forceinline__ void tmem_free_all(uint32_t taddr) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
  }
}

}  // namespace ab
