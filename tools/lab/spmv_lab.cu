// Microbenchmark variants of the CG SpMV / update (not part of the product;
// built by tools/lab/run_lab.py into tools/lab/liblab.so).
#include <cuda_runtime.h>
#include <stdint.h>

// pure stream of the SELL arrays (upper bound for the matrix traffic)
__global__ void k_stream(int64_t n_entries, const int32_t* __restrict__ cols, const double* __restrict__ vals,
                         double* out) {
  double acc = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_entries; k += (int64_t)gridDim.x * blockDim.x)
    acc += __ldcs(vals + k) * (double)__ldcs(cols + k);
  if (acc == 123.456) out[0] = acc;
}

// SELL SpMV with UNROLL-way batched loads: all cols/vals of a chunk first,
// then the gathers, then the FMAs.
template <int UNROLL>
__global__ void k_spmv_batch(int64_t n, const int64_t* __restrict__ sp, const int32_t* __restrict__ scol,
                             const double* __restrict__ sval, const double2* __restrict__ zp, double beta,
                             double* __restrict__ q) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i >> 5;
    const int lane = (int)(i & 31);
    const int64_t base = sp[s] + lane;
    const int width = (int)((sp[s + 1] - sp[s]) >> 5);
    double acc = 0.0;
    for (int j0 = 0; j0 < width; j0 += UNROLL) {
      int c[UNROLL];
      double a[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const bool ok = j0 + u < width;
        c[u] = ok ? __ldcs(scol + base + (int64_t)(j0 + u) * 32) : 0;
        a[u] = ok ? __ldcs(sval + base + (int64_t)(j0 + u) * 32) : 0.0;
      }
      double2 g[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) g[u] = __ldg(zp + c[u]);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) acc = fma(a[u], fma(beta, g[u].y, g[u].x), acc);
    }
    q[i] = acc;
  }
}

// same with one 8-byte gather (plain SpMV of x)
template <int UNROLL>
__global__ void k_spmv_x(int64_t n, const int64_t* __restrict__ sp, const int32_t* __restrict__ scol,
                         const double* __restrict__ sval, const double* __restrict__ x, double* __restrict__ q) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i >> 5;
    const int lane = (int)(i & 31);
    const int64_t base = sp[s] + lane;
    const int width = (int)((sp[s + 1] - sp[s]) >> 5);
    double acc = 0.0;
    for (int j0 = 0; j0 < width; j0 += UNROLL) {
      int c[UNROLL];
      double a[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const bool ok = j0 + u < width;
        c[u] = ok ? __ldcs(scol + base + (int64_t)(j0 + u) * 32) : 0;
        a[u] = ok ? __ldcs(sval + base + (int64_t)(j0 + u) * 32) : 0.0;
      }
      double g[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) g[u] = __ldg(x + c[u]);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) acc = fma(a[u], g[u], acc);
    }
    q[i] = acc;
  }
}

extern "C" {
int lab_stream(int64_t ne, const int32_t* cols, const double* vals, double* out, int grid, int block, void* s) {
  k_stream<<<grid, block, 0, (cudaStream_t)s>>>(ne, cols, vals, out);
  return (int)cudaGetLastError();
}

int lab_spmv_batch(int unroll, int64_t n, const int64_t* sp, const int32_t* scol, const double* sval,
                   const double* zp, double beta, double* q, int grid, int block, void* s) {
  const double2* z2 = reinterpret_cast<const double2*>(zp);
  cudaStream_t st = (cudaStream_t)s;
  switch (unroll) {
    case 4: k_spmv_batch<4><<<grid, block, 0, st>>>(n, sp, scol, sval, z2, beta, q); break;
    case 8: k_spmv_batch<8><<<grid, block, 0, st>>>(n, sp, scol, sval, z2, beta, q); break;
    case 16: k_spmv_batch<16><<<grid, block, 0, st>>>(n, sp, scol, sval, z2, beta, q); break;
    default: return -1;
  }
  return (int)cudaGetLastError();
}

int lab_spmv_x(int unroll, int64_t n, const int64_t* sp, const int32_t* scol, const double* sval, const double* x,
               double* q, int grid, int block, void* s) {
  cudaStream_t st = (cudaStream_t)s;
  switch (unroll) {
    case 4: k_spmv_x<4><<<grid, block, 0, st>>>(n, sp, scol, sval, x, q); break;
    case 8: k_spmv_x<8><<<grid, block, 0, st>>>(n, sp, scol, sval, x, q); break;
    case 16: k_spmv_x<16><<<grid, block, 0, st>>>(n, sp, scol, sval, x, q); break;
    default: return -1;
  }
  return (int)cudaGetLastError();
}
}

// ---- reduction overhead experiments ---------------------------------------
#include "../../paper_2005_05899_b200/csrc/ab_common.cuh"
namespace ab {
std::atomic<int64_t> g_launches{0};
void set_error(const std::string&) {}
}  // namespace ab

template <int BLOCK, int MODE>
__global__ void __launch_bounds__(BLOCK) k_dot(int64_t n, const double* __restrict__ p, const double* __restrict__ q,
                                               double* red, double* part, uint32_t* cnt) {
  double v[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK)
    v[0] += p[i] * q[i];
  if (MODE == 0) {  // block partial only
    __shared__ double sm[BLOCK / 32];
    ab::block_sum<1, BLOCK>(v, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
  } else if (MODE == 1) {  // two-level grid sum
    double t[1];
    if (ab::grid_sum<1, BLOCK>(v, part, cnt, t) && threadIdx.x == 0) red[0] = t[0];
  } else {  // fence only, no atomics
    __shared__ double sm[BLOCK / 32];
    ab::block_sum<1, BLOCK>(v, sm);
    if (threadIdx.x == 0) {
      part[blockIdx.x] = v[0];
      __threadfence();
    }
  }
}

extern "C" int lab_dot(int mode, int block, int64_t n, const double* p, const double* q, double* red, double* part,
                       uint32_t* cnt, int grid, void* s) {
  cudaStream_t st = (cudaStream_t)s;
  if (block == 256) {
    if (mode == 0) k_dot<256, 0><<<grid, 256, 0, st>>>(n, p, q, red, part, cnt);
    if (mode == 1) k_dot<256, 1><<<grid, 256, 0, st>>>(n, p, q, red, part, cnt);
    if (mode == 2) k_dot<256, 2><<<grid, 256, 0, st>>>(n, p, q, red, part, cnt);
  } else {
    if (mode == 0) k_dot<1024, 0><<<grid, 1024, 0, st>>>(n, p, q, red, part, cnt);
    if (mode == 1) k_dot<1024, 1><<<grid, 1024, 0, st>>>(n, p, q, red, part, cnt);
    if (mode == 2) k_dot<1024, 2><<<grid, 1024, 0, st>>>(n, p, q, red, part, cnt);
  }
  return (int)cudaGetLastError();
}
