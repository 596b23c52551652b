// Pressure-Poisson Jacobi-PCG on a
// sliced-ELL (SELL-32) matrix: one thread per row, slice = warp, column
// index and value arrays lane-innermost so every warp load is one 128/256 B
// transaction.  Per iteration two fused kernels:
//   spmv:   p_new = z + beta p_old (evaluated at gather time), q = A p_new,
//           p.q partial sums;
//   update: x += alpha p, r -= alpha q, z = D^-1 r, r.z and r.r partials.
// Scalars (alpha, beta) are formed on the device from the reduction slots,
// so the loop never synchronises with the host.
#include "ab_common.cuh"

namespace ab {

constexpr int kCgBlock = 256;

// ---------------------------------------------------------------------------
// Setup: Dirichlet rows -> identity, CSR -> SELL-32 (+ diagonal extraction)
// ---------------------------------------------------------------------------
__global__ void k_csr_dirichlet(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                double* __restrict__ vals, const uint8_t* __restrict__ fixed) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool fi = fixed[i] != 0;
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
    const int c = cols[k];
    if (fi || fixed[c]) vals[k] = (c == i) ? 1.0 : 0.0;
  }
}

__global__ void k_csr_to_sell(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                              const double* __restrict__ vals, const int64_t* __restrict__ sp,
                              int32_t* __restrict__ scol, double* __restrict__ sval, double* __restrict__ diag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = i >> 5;
  const int lane = (int)(i & 31);
  const int64_t base = sp[s];
  const int64_t width = (sp[s + 1] - base) >> 5;
  const int64_t r0 = rp[i], nnz = rp[i + 1] - r0;
  double d = 0.0;
  for (int64_t j = 0; j < width; ++j) {
    int32_t c = (int32_t)i;
    double v = 0.0;
    if (j < nnz) {
      c = cols[r0 + j];
      v = vals[r0 + j];
      if (c == i) d += v;
    }
    scol[base + j * 32 + lane] = c;
    sval[base + j * 32 + lane] = v;
  }
  if (diag) diag[i] = d;
}

__global__ void k_sell_spmv(int64_t n, const int64_t* __restrict__ sp, const int32_t* __restrict__ scol,
                            const double* __restrict__ sval, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = i >> 5;
  const int lane = (int)(i & 31);
  const int64_t base = sp[s], end = sp[s + 1];
  double acc = 0.0;
  for (int64_t k = base + lane; k < end; k += 32) acc = fma(__ldcs(sval + k), __ldg(x + __ldcs(scol + k)), acc);
  y[i] = acc;
}

// ---------------------------------------------------------------------------
// CG kernels
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kCgBlock) k_cg_init(int64_t n, const double* __restrict__ b_in, double* b_zero,
                                                      const uint8_t* __restrict__ fixed,
                                                      const double* __restrict__ dinv, double* __restrict__ x,
                                                      double* __restrict__ r, double* __restrict__ z,
                                                      double* __restrict__ pold, const double* __restrict__ own,
                                                      double* red, double* sc, double* part, uint32_t* cnt) {
  const int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x;
  double v[2] = {0.0, 0.0};
  if (i < n) {
    double ri = b_in[i];
    if (fixed && fixed[i]) ri = 0.0;
    if (b_zero) b_zero[i] = 0.0;
    const double zi = dinv[i] * ri;
    r[i] = ri;
    z[i] = zi;
    x[i] = 0.0;
    pold[i] = 0.0;
    const double w = own ? own[i] : 1.0;
    v[0] = w * ri * zi;
    v[1] = w * ri * ri;
  }
  double t[2];
  if (grid_sum<2, kCgBlock>(v, part, cnt, t) && threadIdx.x == 0) {
    red[AB_RED_RZN] = t[0];
    red[AB_RED_RR] = t[1];
    sc[AB_SC_RZ] = 0.0;
  }
}

// Copy red[RR] -> sc[BB] after the (optionally all-reduced) init sums.
__global__ void k_cg_set_bb(const double* red, double* sc) { sc[AB_SC_BB] = red[AB_RED_RR]; }

template <bool DOT>
__global__ void __launch_bounds__(kCgBlock) k_cg_spmv(int64_t n, const int64_t* __restrict__ sp,
                                                      const int32_t* __restrict__ scol,
                                                      const double* __restrict__ sval, const double* __restrict__ z,
                                                      const double* __restrict__ pold, double* __restrict__ pnew,
                                                      double* __restrict__ q, const double* __restrict__ own,
                                                      double* red, double* sc, double* part, uint32_t* cnt) {
  const double rz_old = sc[AB_SC_RZ];
  const double rz_new = red[AB_RED_RZN];
  const double beta = rz_old != 0.0 ? rz_new / rz_old : 0.0;
  const int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x;
  double v[1] = {0.0};
  if (i < n) {
    const int64_t s = i >> 5;
    const int lane = (int)(i & 31);
    const int64_t base = sp[s], end = sp[s + 1];
    double acc = 0.0;
    for (int64_t k = base + lane; k < end; k += 32) {
      const int c = __ldcs(scol + k);
      const double pc = fma(beta, __ldg(pold + c), __ldg(z + c));
      acc = fma(__ldcs(sval + k), pc, acc);
    }
    const double pi = fma(beta, pold[i], z[i]);
    pnew[i] = pi;
    q[i] = acc;
    if (DOT) v[0] = (own ? own[i] : 1.0) * pi * acc;
  }
  if (DOT) {
    double t[1];
    if (grid_sum<1, kCgBlock>(v, part, cnt, t) && threadIdx.x == 0) {
      red[AB_RED_PQ] = t[0];
      sc[AB_SC_RZ] = rz_new;
    }
  }
  // decomposed path (DOT=false): the rz shift is done by k_cg_dot's last block
}

// p.q after the interface sum of q (decomposed path); the last block also
// performs the rz shift that k_cg_spmv<true> does in the single-domain path.
__global__ void __launch_bounds__(kCgBlock) k_cg_dot(int64_t n, const double* __restrict__ p,
                                                     const double* __restrict__ q, const double* __restrict__ own,
                                                     double* red, double* sc, double* part, uint32_t* cnt) {
  const int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x;
  double v[1] = {0.0};
  if (i < n) v[0] = (own ? own[i] : 1.0) * p[i] * q[i];
  double t[1];
  if (grid_sum<1, kCgBlock>(v, part, cnt, t) && threadIdx.x == 0) {
    red[AB_RED_PQ] = t[0];
    sc[AB_SC_RZ] = red[AB_RED_RZN];
  }
}

__global__ void __launch_bounds__(kCgBlock) k_cg_update(int64_t n, const double* __restrict__ p,
                                                        const double* __restrict__ q,
                                                        const double* __restrict__ dinv, double* __restrict__ x,
                                                        double* __restrict__ r, double* __restrict__ z,
                                                        const double* __restrict__ own, double* red,
                                                        const double* sc, double* part, uint32_t* cnt) {
  const double pq = red[AB_RED_PQ];
  const double alpha = pq != 0.0 ? sc[AB_SC_RZ] / pq : 0.0;
  const int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x;
  double v[2] = {0.0, 0.0};
  if (i < n) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    const double zi = dinv[i] * ri;
    r[i] = ri;
    z[i] = zi;
    const double w = own ? own[i] : 1.0;
    v[0] = w * ri * zi;
    v[1] = w * ri * ri;
  }
  double t[2];
  if (grid_sum<2, kCgBlock>(v, part, cnt, t) && threadIdx.x == 0) {
    red[AB_RED_RZN] = t[0];
    red[AB_RED_RR] = t[1];
  }
}

}  // namespace ab

using namespace ab;

extern "C" {

int ab_csr_dirichlet(int64_t n, const int64_t* rp, const int32_t* cols, double* vals, const uint8_t* fixed,
                     void* stream) {
  if (n <= 0) return AB_OK;
  if (!rp || !cols || !vals || !fixed) return fail("ab_csr_dirichlet: null argument");
  k_csr_dirichlet<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, rp, cols, vals, fixed);
  return check_launch("ab_csr_dirichlet");
}

int ab_csr_to_sell(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals, const int64_t* sp,
                   int32_t* scol, double* sval, double* diag, void* stream) {
  if (n <= 0) return AB_OK;
  k_csr_to_sell<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, rp, cols, vals, sp, scol, sval, diag);
  return check_launch("ab_csr_to_sell");
}

int ab_sell_spmv(const ab_sell* a, const double* x, double* y, void* stream) {
  if (!a || !x || !y) return fail("ab_sell_spmv: null argument");
  if (a->n_rows <= 0) return AB_OK;
  k_sell_spmv<<<grid_for(a->n_rows, 256), 256, 0, S(stream)>>>(a->n_rows, a->slice_ptr, a->cols, a->vals, x, y);
  return check_launch("ab_sell_spmv");
}

int ab_cg_init(int64_t n, const double* b_in, double* b_zero, const uint8_t* fixed, const double* dinv, double* x,
               double* r, double* z, double* p_old, const double* own, double* red, double* sc, double* part,
               uint32_t* cnt, void* stream) {
  if (n <= 0) return fail("ab_cg_init: empty system");
  k_cg_init<<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(n, b_in, b_zero, fixed, dinv, x, r, z, p_old, own,
                                                               red, sc, part, cnt);
  return check_launch("ab_cg_init");
}

int ab_cg_set_bb(double* red, double* sc, void* stream) {
  k_cg_set_bb<<<1, 1, 0, S(stream)>>>(red, sc);
  return check_launch("ab_cg_set_bb");
}

int ab_cg_spmv(const ab_sell* a, const double* z, const double* p_old, double* p_new, double* q, int32_t with_dot,
               const double* own, double* red, double* sc, double* part, uint32_t* cnt, void* stream) {
  if (!a) return fail("ab_cg_spmv: null matrix");
  const int64_t n = a->n_rows;
  if (with_dot)
    k_cg_spmv<true><<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(n, a->slice_ptr, a->cols, a->vals, z, p_old,
                                                                       p_new, q, own, red, sc, part, cnt);
  else
    k_cg_spmv<false><<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(n, a->slice_ptr, a->cols, a->vals, z, p_old,
                                                                        p_new, q, own, red, sc, part, cnt);
  return check_launch("ab_cg_spmv");
}

int ab_cg_dot(int64_t n, const double* p, const double* q, const double* own, double* red, double* sc, double* part,
              uint32_t* cnt, void* stream) {
  k_cg_dot<<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(n, p, q, own, red, sc, part, cnt);
  return check_launch("ab_cg_dot");
}

int ab_cg_update(int64_t n, const double* p, const double* q, const double* dinv, double* x, double* r, double* z,
                 const double* own, double* red, const double* sc, double* part, uint32_t* cnt, void* stream) {
  k_cg_update<<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(n, p, q, dinv, x, r, z, own, red, sc, part, cnt);
  return check_launch("ab_cg_update");
}

}  // extern "C"
