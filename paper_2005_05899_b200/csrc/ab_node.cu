// Node-wise kernels (single HBM pass each): K3 RK stage update, K7 velocity
// correction, boundary values, halo pack/unpack, and the SFC key kernels of
// the domain decomposition.
#include "ab_common.cuh"

namespace ab {

// K3: uout = a u0 + b (uprev + k minv (rhs - gp)); rhs <- 0.
// 32-byte node records move with one 256-bit load/store each.
__global__ void k_rk_stage(int64_t n, double a, double b, double k, const double* __restrict__ u0,
                           const double* uprev, double* __restrict__ rhs, const double* __restrict__ gp,
                           const double* __restrict__ minv, double* uout) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const d4 r = ld4(rhs + 4 * i);
  const d4 g = ld4_nc(gp + 4 * i);
  const d4 up = ld4(uprev + 4 * i);
  const double km = k * __ldg(minv + i);
  d4 o;
  if (a != 0.0) {
    const d4 z = ld4_nc(u0 + 4 * i);
    o.x = fma(a, z.x, b * fma(km, r.x - g.x, up.x));
    o.y = fma(a, z.y, b * fma(km, r.y - g.y, up.y));
    o.z = fma(a, z.z, b * fma(km, r.z - g.z, up.z));
  } else {
    o.x = b * fma(km, r.x - g.x, up.x);
    o.y = b * fma(km, r.y - g.y, up.y);
    o.z = b * fma(km, r.z - g.z, up.z);
  }
  o.w = 0.0;
  st4(uout + 4 * i, o);
  st4(rhs + 4 * i, d4{0.0, 0.0, 0.0, 0.0});
}

// K7: uout = uin - k minv gd; p += dp; gp += gd; gd <- 0.
__global__ void k_correct(int64_t n, double k, const double* uin, double* uout, double* __restrict__ gd,
                          const double* __restrict__ minv, double* __restrict__ p, const double* __restrict__ dp,
                          double* __restrict__ gp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const d4 d = ld4(gd + 4 * i);
  d4 v = ld4(uin + 4 * i);
  d4 g = ld4(gp + 4 * i);
  const double km = k * __ldg(minv + i);
  v.x = fma(-km, d.x, v.x);
  v.y = fma(-km, d.y, v.y);
  v.z = fma(-km, d.z, v.z);
  g.x += d.x;
  g.y += d.y;
  g.z += d.z;
  st4(uout + 4 * i, v);
  st4(gp + 4 * i, g);
  st4(gd + 4 * i, d4{0.0, 0.0, 0.0, 0.0});
  p[i] += dp[i];
}

__global__ void k_velocity_bc(int64_t nf, const int32_t* __restrict__ idx, const uint8_t* __restrict__ mask,
                              const double* __restrict__ vals, double* __restrict__ u4) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  const int64_t node = idx[i];
  const uint8_t m = mask[i];
#pragma unroll
  for (int c = 0; c < 3; ++c)
    if (m & (1u << c)) u4[4 * node + c] = vals[3 * i + c];
}

__global__ void k_reciprocal(int64_t n, const double* __restrict__ in, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = 1.0 / in[i];
}

__global__ void k_halo_pack(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ f, int stride,
                            int ncomp, double* __restrict__ buf) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * ncomp) return;
  const int64_t i = t / ncomp;
  const int c = (int)(t - i * ncomp);
  buf[t] = f[(int64_t)idx[i] * stride + c];
}

__global__ void k_halo_unpack_add(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ buf,
                                  int stride, int ncomp, double* __restrict__ f) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * ncomp) return;
  const int64_t i = t / ncomp;
  const int c = (int)(t - i * ncomp);
  // one node may be shared with several neighbours: accumulate atomically
  red_add(f + (int64_t)idx[i] * stride + c, buf[t]);
}

// 3D Hilbert index, transpose-form (Skilling) with MSB-first interleave,
// equal bit for bit to reference sfc.py:45-81 / :114-148.
__device__ __forceinline__ int64_t hilbert3(int64_t x0, int64_t x1, int64_t x2, int level) {
  int64_t x[3] = {x0, x1, x2};
  int64_t q = (int64_t)1 << (level - 1);
  while (q > 1) {
    const int64_t p = q - 1;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (x[i] & q) {
        x[0] ^= p;
      } else {
        const int64_t t = (x[0] ^ x[i]) & p;
        x[0] ^= t;
        x[i] ^= t;
      }
    }
    q >>= 1;
  }
  x[1] ^= x[0];
  x[2] ^= x[1];
  int64_t t = 0;
  for (q = (int64_t)1 << (level - 1); q > 1; q >>= 1)
    if (x[2] & q) t ^= q - 1;
  x[0] ^= t;
  x[1] ^= t;
  x[2] ^= t;
  int64_t key = 0;
  for (int j = level - 1; j >= 0; --j)
#pragma unroll
    for (int i = 0; i < 3; ++i) key = (key << 1) | ((x[i] >> j) & 1);
  return key;
}

// cell = clip(floor((c - lo) / span * 2^L), 0, 2^L - 1) without contraction
// (reference sfc.py:184-192), then the Hilbert key.
__global__ void k_hilbert_keys(int64_t n, const double* __restrict__ cent, const double* __restrict__ lo,
                               const double* __restrict__ span, int level, int64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t side = (int64_t)1 << level;
  int64_t c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double rel = __ddiv_rn(__dsub_rn(cent[3 * i + d], lo[d]), span[d]);
    double f = floor(__dmul_rn(rel, (double)side));
    int64_t v = (int64_t)f;
    c[d] = v < 0 ? 0 : (v > side - 1 ? side - 1 : v);
  }
  keys[i] = hilbert3(c[0], c[1], c[2], level);
}

__global__ void k_hilbert_cells(int64_t n, const int64_t* __restrict__ cells, int level, int64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = hilbert3(cells[3 * i], cells[3 * i + 1], cells[3 * i + 2], level);
}

// Ordered segmented sum: out[s] = sum of vals[ptr[s]..ptr[s+1]) left to right
// (scatter_global's ascending-element-id accumulation, assembly.py:320-326).
__global__ void k_segment_sum(int64_t nseg, const int64_t* __restrict__ sp, const double* __restrict__ v,
                              double* __restrict__ out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  double acc = 0.0;
  for (int64_t k = sp[s]; k < sp[s + 1]; ++k) acc = __dadd_rn(acc, v[k]);
  out[s] = acc;
}

}  // namespace ab

using namespace ab;

extern "C" {

int ab_rk_stage(int64_t n, double a, double b, double k, const double* u0, const double* uprev, double* rhs,
                const double* gp, const double* minv, double* uout, void* stream) {
  if (n <= 0) return AB_OK;
  if (!uprev || !rhs || !gp || !minv || !uout || (a != 0.0 && !u0)) return fail("ab_rk_stage: null argument");
  k_rk_stage<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, a, b, k, u0, uprev, rhs, gp, minv, uout);
  return check_launch("ab_rk_stage");
}

int ab_correct(int64_t n, double k, const double* uin, double* uout, double* gd, const double* minv, double* p,
               const double* dp, double* gp, void* stream) {
  if (n <= 0) return AB_OK;
  k_correct<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, k, uin, uout, gd, minv, p, dp, gp);
  return check_launch("ab_correct");
}

int ab_apply_velocity_bc(int64_t nf, const int32_t* idx, const uint8_t* mask, const double* vals, double* u4,
                         void* stream) {
  if (nf <= 0) return AB_OK;
  k_velocity_bc<<<grid_for(nf, 256), 256, 0, S(stream)>>>(nf, idx, mask, vals, u4);
  return check_launch("ab_apply_velocity_bc");
}

int ab_reciprocal(int64_t n, const double* in, double* out, void* stream) {
  if (n <= 0) return AB_OK;
  k_reciprocal<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, in, out);
  return check_launch("ab_reciprocal");
}

int ab_halo_pack(int64_t n, const int32_t* idx, const double* f, int32_t stride, int32_t ncomp, double* buf,
                 void* stream) {
  if (n <= 0) return AB_OK;
  if (ncomp < 1 || stride < ncomp) return fail("ab_halo_pack: bad stride/ncomp");
  k_halo_pack<<<grid_for(n * ncomp, 256), 256, 0, S(stream)>>>(n, idx, f, stride, ncomp, buf);
  return check_launch("ab_halo_pack");
}

int ab_halo_unpack_add(int64_t n, const int32_t* idx, const double* buf, int32_t stride, int32_t ncomp, double* f,
                       void* stream) {
  if (n <= 0) return AB_OK;
  if (ncomp < 1 || stride < ncomp) return fail("ab_halo_unpack_add: bad stride/ncomp");
  k_halo_unpack_add<<<grid_for(n * ncomp, 256), 256, 0, S(stream)>>>(n, idx, buf, stride, ncomp, f);
  return check_launch("ab_halo_unpack_add");
}

int ab_hilbert_keys(int64_t n, const double* cent, const double* lo, const double* span, int32_t level,
                    int64_t* keys, void* stream) {
  if (level < 1 || level > 20) return fail("ab_hilbert_keys: level must be in [1, 20]");
  if (n <= 0) return AB_OK;
  k_hilbert_keys<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, cent, lo, span, level, keys);
  return check_launch("ab_hilbert_keys");
}

int ab_segment_sum(int64_t nseg, const int64_t* seg_ptr, const double* vals, double* out, void* stream) {
  if (nseg <= 0) return AB_OK;
  k_segment_sum<<<grid_for(nseg, 256), 256, 0, S(stream)>>>(nseg, seg_ptr, vals, out);
  return check_launch("ab_segment_sum");
}

int ab_hilbert_cells(int64_t n, const int64_t* cells, int32_t level, int64_t* keys, void* stream) {
  if (level < 1 || level > 20) return fail("ab_hilbert_cells: level must be in [1, 20]");
  if (n <= 0) return AB_OK;
  k_hilbert_cells<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, cells, level, keys);
  return check_launch("ab_hilbert_cells");
}

}  // extern "C"
