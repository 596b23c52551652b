// K4 / K6 / K7 as sparse products with the assembled discrete gradient
// operator B_ab = int N_a grad N_b (ab_gradop_csr):
//   div:      out[a] += scale * sum_b B_ab . u_b                (K4)
//   grad:     out4[a] += scale * sum_b B_ab p_b                 (K6)
//   grad+cor: gd = sum_b B_ab dp_b; uout = uin - k minv gd;     (K6 + K7 in
//             p += dp; gp += gd                                  one HBM pass)
// The element loops they replace are bound by shared-memory traffic of the
// node windows (~7x their HBM floor); the products stream the operator
// (3 fp64 planes + int32 columns in SELL-32, lane-innermost) at HBM speed
// and gather the node vectors through L2.  One thread per row, rows in
// slices of 32, loads batched per 8 entries (columns and values first, then
// the gathers, then the FMAs).
#include "ab_common.cuh"

namespace ab {

constexpr int kGoBlock = 256;
constexpr int kGoChunk = 8;

struct GoRow {
  int64_t base;
  int width;
};
__device__ __forceinline__ GoRow go_row(const int64_t* __restrict__ sp, int64_t i) {
  const int64_t s = i >> 5;
  const int64_t b = sp[s];
  return {b + (i & 31), (int)((sp[s + 1] - b) >> 5)};
}

__global__ void __launch_bounds__(kGoBlock) k_go_div(int64_t n, const int64_t* __restrict__ sp,
                                                     const int32_t* __restrict__ cols, const double* __restrict__ vx,
                                                     const double* __restrict__ vy, const double* __restrict__ vz,
                                                     const double* __restrict__ u4, double scale,
                                                     double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * kGoBlock + threadIdx.x;
  if (i >= n) return;
  const GoRow r = go_row(sp, i);
  double acc = 0.0;
  for (int j0 = 0; j0 < r.width; j0 += kGoChunk) {
    int c[kGoChunk];
    double a[kGoChunk][3];
#pragma unroll
    for (int u = 0; u < kGoChunk; ++u) {
      const bool ok = j0 + u < r.width;
      const int64_t k = r.base + (int64_t)(j0 + u) * 32;
      c[u] = ok ? __ldcs(cols + k) : 0;
      a[u][0] = ok ? __ldcs(vx + k) : 0.0;
      a[u][1] = ok ? __ldcs(vy + k) : 0.0;
      a[u][2] = ok ? __ldcs(vz + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kGoChunk; ++u) {
      const d4 v = ld4_nc(u4 + 4 * (int64_t)c[u]);
      acc = fma(a[u][0], v.x, acc);
      acc = fma(a[u][1], v.y, acc);
      acc = fma(a[u][2], v.z, acc);
    }
  }
  out[i] += scale * acc;
}

template <bool CORRECT>
__global__ void __launch_bounds__(kGoBlock) k_go_grad(int64_t n, const int64_t* __restrict__ sp,
                                                      const int32_t* __restrict__ cols, const double* __restrict__ vx,
                                                      const double* __restrict__ vy, const double* __restrict__ vz,
                                                      const double* __restrict__ p, double scale,
                                                      double* __restrict__ out4, double k, const double* uin,
                                                      double* uout, const double* __restrict__ minv,
                                                      double* __restrict__ pacc, double* __restrict__ gp) {
  const int64_t i = (int64_t)blockIdx.x * kGoBlock + threadIdx.x;
  if (i >= n) return;
  const GoRow r = go_row(sp, i);
  double g0 = 0.0, g1 = 0.0, g2 = 0.0;
  for (int j0 = 0; j0 < r.width; j0 += kGoChunk) {
    int c[kGoChunk];
    double a[kGoChunk][3];
#pragma unroll
    for (int u = 0; u < kGoChunk; ++u) {
      const bool ok = j0 + u < r.width;
      const int64_t kk = r.base + (int64_t)(j0 + u) * 32;
      c[u] = ok ? __ldcs(cols + kk) : 0;
      a[u][0] = ok ? __ldcs(vx + kk) : 0.0;
      a[u][1] = ok ? __ldcs(vy + kk) : 0.0;
      a[u][2] = ok ? __ldcs(vz + kk) : 0.0;
    }
    double pv[kGoChunk];
#pragma unroll
    for (int u = 0; u < kGoChunk; ++u) pv[u] = __ldg(p + c[u]);
#pragma unroll
    for (int u = 0; u < kGoChunk; ++u) {
      g0 = fma(a[u][0], pv[u], g0);
      g1 = fma(a[u][1], pv[u], g1);
      g2 = fma(a[u][2], pv[u], g2);
    }
  }
  g0 *= scale;
  g1 *= scale;
  g2 *= scale;
  if (!CORRECT) {
    d4 o = ld4(out4 + 4 * i);
    o.x += g0;
    o.y += g1;
    o.z += g2;
    st4(out4 + 4 * i, o);
  } else {
    // K7: uout = uin - k minv gd; p += dp; gp += gd
    const double km = k * minv[i];
    d4 u = ld4(uin + 4 * i);
    u.x = fma(-km, g0, u.x);
    u.y = fma(-km, g1, u.y);
    u.z = fma(-km, g2, u.z);
    st4(uout + 4 * i, u);
    pacc[i] += p[i];
    d4 q = ld4(gp + 4 * i);
    q.x += g0;
    q.y += g1;
    q.z += g2;
    st4(gp + 4 * i, q);
  }
}

}  // namespace ab

using namespace ab;

extern "C" {

static int go_check(const ab_sell3* b) {
  if (!b || !b->slice_ptr || !b->cols || !b->vx || !b->vy || !b->vz) return fail("gradient operator: null matrix");
  return AB_OK;
}

int ab_gradop_div(const ab_sell3* b, const double* u4, double scale, double* out, void* stream) {
  if (int rc = go_check(b)) return rc;
  if (!u4 || !out) return fail("ab_gradop_div: null argument");
  if (b->n_rows <= 0) return AB_OK;
  k_go_div<<<grid_for(b->n_rows, kGoBlock), kGoBlock, 0, S(stream)>>>(b->n_rows, b->slice_ptr, b->cols, b->vx,
                                                                      b->vy, b->vz, u4, scale, out);
  return check_launch("ab_gradop_div");
}

int ab_gradop_grad(const ab_sell3* b, const double* p, double scale, double* out4, void* stream) {
  if (int rc = go_check(b)) return rc;
  if (!p || !out4) return fail("ab_gradop_grad: null argument");
  if (b->n_rows <= 0) return AB_OK;
  k_go_grad<false><<<grid_for(b->n_rows, kGoBlock), kGoBlock, 0, S(stream)>>>(
      b->n_rows, b->slice_ptr, b->cols, b->vx, b->vy, b->vz, p, scale, out4, 0.0, nullptr, nullptr, nullptr, nullptr,
      nullptr);
  return check_launch("ab_gradop_grad");
}

int ab_gradop_correct(const ab_sell3* b, const double* dp, double k, const double* uin, double* uout,
                      const double* minv, double* p, double* gp, void* stream) {
  if (int rc = go_check(b)) return rc;
  if (!dp || !uin || !uout || !minv || !p || !gp) return fail("ab_gradop_correct: null argument");
  if (dp == p) return fail("ab_gradop_correct: dp must not alias p");
  if (b->n_rows <= 0) return AB_OK;
  k_go_grad<true><<<grid_for(b->n_rows, kGoBlock), kGoBlock, 0, S(stream)>>>(
      b->n_rows, b->slice_ptr, b->cols, b->vx, b->vy, b->vz, dp, 1.0, nullptr, k, uin, uout, minv, p, gp);
  return check_launch("ab_gradop_correct");
}

}  // extern "C"
