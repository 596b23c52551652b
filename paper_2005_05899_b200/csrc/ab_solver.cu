// Pressure-Poisson Jacobi-PCG on a
// sliced-ELL (SELL-32) matrix: one thread per row, slice = warp, column
// index and value arrays lane-innermost so every warp load is one 128/256 B
// transaction.  Forms:
//   resident: the whole solve in one cooperative kernel (k_cg_resident_local,
//     systems that fit on chip);
//   tiled single pass (default for larger systems): one kernel per iteration
//     on 2048-row tiles staged in shared memory (k_cg_tile_iter);
//   two kernels per iteration (options and the decomposed NCCL path):
//     spmv:   p_new = z + beta p_old, q = A p_new, p.q partial sums;
//     update: x += alpha p, r -= alpha q, z = D^-1 r, r.z and r.r partials.
// Scalars (alpha, beta) are formed on the device from the reduction slots,
// so the loop never synchronises with the host.
#include "ab_cg_common.cuh"

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
// CG kernels.  The SpMV is applied to the preconditioned
// residual z and the product A p is formed recursively,
//     p = z + beta p_old,   q = A p = A z + beta q_old,
// so each non-zero costs one 8-byte gather.  All kernels are row-per-thread
// with deterministic two-level grid reductions; alpha and beta are formed on
// the device from the reduction slots, so the loop never synchronises with
// the host.
// ---------------------------------------------------------------------------
constexpr int kCgGrid = 148 * 8;

__global__ void __launch_bounds__(kCgBlock) k_cg_init(int64_t n, const double* __restrict__ b_in, double* b_zero,
                                                      const uint8_t* __restrict__ fixed,
                                                      const double* __restrict__ dinv, double* __restrict__ x,
                                                      double* __restrict__ r, double* __restrict__ z,
                                                      double* __restrict__ p, double* __restrict__ q,
                                                      const double* __restrict__ own, double* red, double* sc,
                                                      double* part, uint32_t* cnt) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCgBlock) {
    double ri = b_in[i];
    if (fixed && fixed[i]) ri = 0.0;
    if (b_zero) b_zero[i] = 0.0;
    const double zi = dinv[i] * ri;
    r[i] = ri;
    z[i] = zi;
    x[i] = 0.0;
    p[i] = 0.0;
    q[i] = 0.0;
    const double w = own ? own[i] : 1.0;
    v[0] += w * ri * zi;
    v[1] += w * ri * ri;
  }
  double t[2];
  if (grid_sum<2, kCgBlock>(v, part, cnt, t) && threadIdx.x == 0) {
    red[AB_RED_RZN] = t[0];
    red[AB_RED_RR] = t[1];
    sc[AB_SC_RZ] = 0.0;
  }
}

// Single-domain init on P A P^T straight from the node-order right-hand
// side: r_i = b[perm[i]] (b zeroed behind it), and sc[BB] = r.r (no
// separate set_bb: nothing is all-reduced in between).
__global__ void __launch_bounds__(kCgBlock) k_cg_init_perm(int64_t n, const int64_t* __restrict__ perm, double* b,
                                                           int zero_b, const uint8_t* __restrict__ fixed,
                                                           const double* __restrict__ dinv, double* __restrict__ x,
                                                           double* __restrict__ r, double* __restrict__ z,
                                                           double* __restrict__ p, double* __restrict__ q, double* red,
                                                           double* sc, double* part, uint32_t* cnt) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCgBlock) {
    const int64_t ni = perm[i];
    double ri = b[ni];
    if (fixed && fixed[i]) ri = 0.0;
    const double zi = dinv[i] * ri;
    r[i] = ri;
    z[i] = zi;
    x[i] = 0.0;
    p[i] = 0.0;
    q[i] = 0.0;
    v[0] += ri * zi;
    v[1] += ri * ri;
  }
  double t[2];
  if (grid_sum<2, kCgBlock>(v, part, cnt, t) && threadIdx.x == 0) {
    red[AB_RED_RZN] = t[0];
    red[AB_RED_RR] = t[1];
    sc[AB_SC_RZ] = 0.0;
    sc[AB_SC_BB] = t[1];
  }
}

__global__ void k_perm_scatter(int64_t n, const int64_t* __restrict__ perm, const double* __restrict__ in,
                               double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[perm[i]] = in[i];
}

// ---------------------------------------------------------------------------
// Symmetrically scaled form (single domain, two kernels).  Jacobi-PCG on A
// is plain CG on A' = D^-1/2 A D^-1/2 with r' = D^-1/2 r, x = D^-1/2 x'
// (the same iterates in exact arithmetic): z = D^-1 r becomes r' itself, so
// per iteration the z write and the D^-1 read disappear (16 bytes per row)
// and r.z = r'.r'.  ||r||^2 = sum d r'^2 is formed only when a tolerance is
// tested (d non-NULL).
// ---------------------------------------------------------------------------
__global__ void k_sell_symscale(int64_t n, const int64_t* __restrict__ sp, const int32_t* __restrict__ scol,
                                double* __restrict__ sval, const double* __restrict__ s) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t sl = i >> 5;
  const int lane = (int)(i & 31);
  const double si = s[i];
  for (int64_t k = sp[sl] + lane; k < sp[sl + 1]; k += 32) sval[k] *= si * s[scol[k]];
}

__global__ void __launch_bounds__(kCgBlock) k_cg_init_scaled(int64_t n, const int64_t* __restrict__ perm, double* b,
                                                             int zero_b, const uint8_t* __restrict__ fixed,
                                                             const double* __restrict__ s,
                                                             const double* __restrict__ d, double* __restrict__ x,
                                                             double* __restrict__ r, double* __restrict__ p,
                                                             double* __restrict__ q, double* red, double* sc,
                                                             double* part, uint32_t* cnt) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCgBlock) {
    const int64_t ni = perm[i];
    double bi = b[ni];
    if (fixed && fixed[i]) bi = 0.0;
    const double ri = s[i] * bi;
    r[i] = ri;
    x[i] = 0.0;
    p[i] = 0.0;
    q[i] = 0.0;
    v[0] += ri * ri;
    v[1] += d ? d[i] * ri * ri : ri * ri;
  }
  double t[2];
  if (grid_sum<2, kCgBlock>(v, part, cnt, t) && threadIdx.x == 0) {
    red[AB_RED_RZN] = t[0];
    red[AB_RED_RR] = t[1];
    sc[AB_SC_RZ] = 0.0;
    sc[AB_SC_BB] = t[1];
  }
}

__global__ void __launch_bounds__(kCgBlock) k_cg_update_scaled(int64_t n, const double* __restrict__ p,
                                                               const double* __restrict__ q, double* __restrict__ x,
                                                               double* __restrict__ r, const double* __restrict__ d,
                                                               double* red, const double* sc, double* part,
                                                               uint32_t* cnt) {
  double v[2] = {0.0, 0.0};
  const int64_t i = 2 * ((int64_t)blockIdx.x * kCgBlock + threadIdx.x);
  const double pq = red[AB_RED_PQ];
  const double rz = sc[AB_SC_RZ];
  const double alpha = pq != 0.0 ? rz / pq : 0.0;
  if (i + 1 < n) {
    const double2 pv = *reinterpret_cast<const double2*>(p + i);
    const double2 xv = *reinterpret_cast<const double2*>(x + i);
    const double2 qv = *reinterpret_cast<const double2*>(q + i);
    const double2 rv = *reinterpret_cast<const double2*>(r + i);
    const double r0 = fma(-alpha, qv.x, rv.x), r1 = fma(-alpha, qv.y, rv.y);
    *reinterpret_cast<double2*>(x + i) = make_double2(fma(alpha, pv.x, xv.x), fma(alpha, pv.y, xv.y));
    *reinterpret_cast<double2*>(r + i) = make_double2(r0, r1);
    v[0] = r0 * r0 + r1 * r1;
    if (d) {
      const double2 dv = __ldg(reinterpret_cast<const double2*>(d + i));
      v[1] = dv.x * r0 * r0 + dv.y * r1 * r1;
    } else {
      v[1] = v[0];
    }
  } else if (i < n) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    v[0] = ri * ri;
    v[1] = d ? d[i] * ri * ri : ri * ri;
  }
  double tot[2];
  if (grid_sum<2, kCgBlock>(v, part, cnt, tot) && threadIdx.x == 0) {
    red[AB_RED_RZN] = tot[0];
    red[AB_RED_RR] = tot[1];
  }
}

// out[j] = s_i x'_i with i = iperm[j] (node j's solver row): coalesced
// writes, gathered reads (a scatter through perm writes partial sectors)
__global__ void k_cg_finish_scaled(int64_t n, const int64_t* __restrict__ iperm, const double* __restrict__ s,
                                   const double* __restrict__ x, double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    const int64_t i = iperm[j];
    out[j] = s[i] * x[i];
  }
}

// Copy red[RR] -> sc[BB] after the (optionally all-reduced) init sums.
__global__ void k_cg_set_bb(const double* red, double* sc) { sc[AB_SC_BB] = red[AB_RED_RR]; }

// Single domain (DOT): p = z + beta p, q = A z + beta q, p.q partials, then
// sc[RZ] := red[RZN].  Decomposed (!DOT): t = (A z)_local only; the
// interface sum of t and k_cg_dot follow.
template <bool DOT>
__global__ void __launch_bounds__(kCgBlock) k_cg_spmv(int64_t n, const int64_t* __restrict__ sp,
                                                      const int32_t* __restrict__ scol,
                                                      const double* __restrict__ sval, const double* __restrict__ z,
                                                      double* __restrict__ p, double* __restrict__ q,
                                                      double* __restrict__ t, const double* __restrict__ own,
                                                      double* red, double* sc, double* part, uint32_t* cnt) {
  const int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x;
  const double rz_old = sc[AB_SC_RZ];
  const double rz_new = red[AB_RED_RZN];
  const double beta = rz_old != 0.0 ? rz_new / rz_old : 0.0;
  double v[1] = {0.0};
  if (i < n) {
    const double az = sell_row_dot(sp, scol, sval, z, i);
    if (DOT) {
      const double pi = fma(beta, p[i], z[i]);
      const double qi = fma(beta, q[i], az);
      p[i] = pi;
      q[i] = qi;
      v[0] = (own ? own[i] : 1.0) * pi * qi;
    } else {
      t[i] = az;
    }
  }
  if (DOT) {
    double tot[1];
    if (grid_sum<1, kCgBlock>(v, part, cnt, tot) && threadIdx.x == 0) {
      red[AB_RED_PQ] = tot[0];
      sc[AB_SC_RZ] = rz_new;
    }
  }
}

// Single domain, symmetrically scaled matrix with its unit diagonal NOT
// stored (ab_cg_spmv_unit): (A' z)_i = z_i + sum_{j != i} a'_ij z_j, the z_i
// the recurrence reads anyway; 12 bytes per row less than storing the 1.
__global__ void __launch_bounds__(kCgBlock) k_cg_spmv_unit(int64_t n, const int64_t* __restrict__ sp,
                                                           const int32_t* __restrict__ scol,
                                                           const double* __restrict__ sval,
                                                           const double* __restrict__ z, double* __restrict__ p,
                                                           double* __restrict__ q, double* red, double* sc,
                                                           double* part, uint32_t* cnt) {
  const int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x;
  const double rz_old = sc[AB_SC_RZ];
  const double rz_new = red[AB_RED_RZN];
  const double beta = rz_old != 0.0 ? rz_new / rz_old : 0.0;
  double v[1] = {0.0};
  if (i < n) {
    const double zi = z[i];
    const double az = sell_row_dot(sp, scol, sval, z, i) + zi;
    const double pi = fma(beta, p[i], zi);
    const double qi = fma(beta, q[i], az);
    p[i] = pi;
    q[i] = qi;
    v[0] = pi * qi;
  }
  double tot[1];
  if (grid_sum<1, kCgBlock>(v, part, cnt, tot) && threadIdx.x == 0) {
    red[AB_RED_PQ] = tot[0];
    sc[AB_SC_RZ] = rz_new;
  }
}

// Tiled form of k_cg_spmv_unit: CTA b owns rows [b R, (b+1) R) of the
// (SFC-ordered) system; it stages its own z and its ghost rows' z (the
// remote columns, ab_cg_local ghost lists) in shared memory, then streams
// its slices with 16-bit tile-local columns (10 instead of 12 bytes per
// stored entry) and reads every z from shared memory: no per-entry global
// gather, whose latency bounds the int32 form once the stream is near the
// HBM roof.  Each row product has k_cg_spmv_unit's FMA order
// (bitwise equal); the p.q partials are grouped per tile.
#ifndef TILE_CHUNK
#define TILE_CHUNK 8
#endif
#ifndef TILE_MINB
#define TILE_MINB 1
#endif
constexpr int kTileBlock = 256;
__global__ void __launch_bounds__(kTileBlock, TILE_MINB) k_cg_spmv_tile(
    int64_t n, int rows_per_tile, const int64_t* __restrict__ sp, const uint16_t* __restrict__ lcol,
    const double* __restrict__ sval, const int32_t* __restrict__ ghost_ptr, const int32_t* __restrict__ ghost,
    const double* __restrict__ z, double* __restrict__ p, double* __restrict__ q, double* red, double* sc,
    double* part, uint32_t* cnt) {
  extern __shared__ __align__(16) double zs[];
  const int R = rows_per_tile;
  const int64_t row0 = (int64_t)blockIdx.x * R;
  const int rows = (int)(n - row0 < R ? n - row0 : R);
  const double rz_old = sc[AB_SC_RZ];
  const double rz_new = red[AB_RED_RZN];
  const double beta = rz_old != 0.0 ? rz_new / rz_old : 0.0;
  // own rows (16-byte loads; R and row0 are even)
  {
    const double2* z2 = reinterpret_cast<const double2*>(z + row0);
    double2* s2 = reinterpret_cast<double2*>(zs);
    const int h = rows >> 1;
    for (int k = threadIdx.x; k < h; k += kTileBlock) s2[k] = __ldcg(z2 + k);
    if ((rows & 1) && threadIdx.x == 0) zs[rows - 1] = __ldcg(z + row0 + rows - 1);
  }
  const int g0 = ghost_ptr[blockIdx.x], ng = ghost_ptr[blockIdx.x + 1] - g0;
  for (int k = threadIdx.x; k < ng; k += kTileBlock) zs[R + k] = __ldcg(z + __ldg(ghost + g0 + k));
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s0 = row0 >> 5;
  const int nsl = (rows + 31) >> 5;
  double v[1] = {0.0};
  for (int sl = warp; sl < nsl; sl += kTileBlock / 32) {
    const double acc = sell_row_dot_smem<TILE_CHUNK>(sp + s0, lcol, sval, zs, sl, lane);
    const int li = sl * 32 + lane;
    if (li < rows) {
      const int64_t i = row0 + li;
      const double zi = zs[li];
      const double az = acc + zi;
      const double pi = fma(beta, p[i], zi);
      const double qi = fma(beta, q[i], az);
      p[i] = pi;
      q[i] = qi;
      v[0] += pi * qi;
    }
  }
  double tot[1];
  if (grid_sum<1, kTileBlock>(v, part, cnt, tot) && threadIdx.x == 0) {
    red[AB_RED_PQ] = tot[0];
    sc[AB_SC_RZ] = rz_new;
  }
}

// ---------------------------------------------------------------------------
// Tiled single-pass scaled CG: ONE kernel per iteration (ab_cg_tile_iter).
// The two-kernel loop moves 88 vector bytes per row and iteration (SpMV: z,
// p, q; update: x, r, p, q).  Kernel j instead forms, per tile, r'_j =
// r'_{j-1} - alpha q_{j-1} while staging the tile's rows and ghost rows in
// shared memory (from 16-byte (r', q) pairs: own rows coalesced, one gather
// per ghost), then x_j = x_{j-1} + alpha p_{j-1}, p_j = r'_j + beta p_{j-1},
// q_j = A' r'_j + beta q_{j-1}: 64 bytes per row ((r', q) read from one
// buffer and written to the other, (x, p) in place) plus the ghosts.
// alpha_{j-1} = r'r'_{j-1} / p.q_{j-1} comes from the previous kernel's
// sums; beta_{j-1} needs r'r'_j before any tile has formed r'_j, so it uses
// the recurrence r'r'_j = r'r'_{j-1} - 2 alpha r'.q_{j-1} + alpha^2 q.q_{j-1}
// of the previous kernel's three dots (the true r'r'_j summed here feeds
// alpha_j, so the error does not accumulate).  Iterates equal the two-kernel
// form's up to that rounding-level difference in beta (tests: 1e-15 of the
// oracle after 50 iterations on the 705k-row C2 system).
// red slots: RZN = r'.r' of the r' formed, RR = sum d r'^2 (d given) or
// r'.r', PQ = p.q, RQ = r'.q, QQ = q.q.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kCgBlock) k_cg_tile_init(int64_t n, const int64_t* __restrict__ perm,
                                                           const double* __restrict__ b,
                                                           const uint8_t* __restrict__ fixed,
                                                           const double* __restrict__ s,
                                                           const double* __restrict__ d, double2* __restrict__ xp,
                                                           double2* __restrict__ rq, double* red, double* sc,
                                                           double* part, uint32_t* cnt) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCgBlock) {
    double bi = b[perm[i]];
    if (fixed && fixed[i]) bi = 0.0;
    const double ri = s[i] * bi;
    rq[i] = make_double2(ri, 0.0);
    xp[i] = make_double2(0.0, 0.0);
    v[0] += ri * ri;
    v[1] += d ? d[i] * ri * ri : ri * ri;
  }
  double t[2];
  if (grid_sum<2, kCgBlock>(v, part, cnt, t) && threadIdx.x == 0) {
    red[AB_RED_RZN] = t[0];
    red[AB_RED_RR] = t[1];
    red[AB_RED_PQ] = 0.0;  // alpha_{-1} = 0: the first iteration keeps r'_0 = b' and x = 0
    red[AB_RED_RQ] = 0.0;
    red[AB_RED_QQ] = 0.0;
    sc[AB_SC_RZ] = 0.0;
    sc[AB_SC_BB] = t[1];
  }
}

#ifndef TSP_PERSIST
#define TSP_PERSIST 1  // persistent CTAs over the tiles: 8.1M rows 294.7 -> 286.9 us per iteration
#endif
#ifndef TSP_MINB
#define TSP_MINB 4  // 63 registers: 4 CTAs of 2048-row tiles per SM (8.1M rows: 291 us vs 402 us uncapped, 86 registers)
#endif
// RPT rows per thread: R = 256 RPT rows per tile; warp w multiplies the
// tile's slices w, w + 8, ...
template <int RPT>
__global__ void __launch_bounds__(kTileBlock, TSP_MINB) k_cg_tile_iter(
    int64_t n, const int64_t* __restrict__ sp, const uint16_t* __restrict__ lcol, const double* __restrict__ sval,
    const int32_t* __restrict__ ghost_ptr, const int32_t* __restrict__ ghost, const double2* __restrict__ rq_in,
    double2* __restrict__ rq_out, double2* __restrict__ xp, const double* __restrict__ d, double* red, double* part,
    uint32_t* cnt) {
  constexpr int R = kTileBlock * RPT;
  extern __shared__ __align__(16) double qs[];  // [R] q_{j-1} of the own rows, then zs
  double* zs = qs + R;                          // [R + ghosts] r'_j of the own and ghost rows
  const double RR = red[AB_RED_RZN], PQ = red[AB_RED_PQ], RQ = red[AB_RED_RQ], QQ = red[AB_RED_QQ];
  const double alpha = PQ != 0.0 ? RR / PQ : 0.0;
  double rr_next = fma(alpha, fma(alpha, QQ, -2.0 * RQ), RR);
  if (rr_next < 0.0) rr_next = 0.0;
  const double beta = RR != 0.0 ? rr_next / RR : 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int64_t n_tiles = (n + R - 1) / R;
  // persistent CTAs walk the tiles (grid = resident CTAs when TSP_PERSIST)
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
  const int64_t row0 = tile * R;
  const int rows = (int)(n - row0 < R ? n - row0 : R);
  __syncthreads();  // the previous tile's shared-memory reads are done
  // own rows: r' = r' - alpha q and q_{j-1} into shared memory
  for (int li = threadIdx.x; li < rows; li += kTileBlock) {
    const double2 w = rq_in[row0 + li];
    qs[li] = w.y;
    zs[li] = fma(-alpha, w.y, w.x);
  }
  const int g0 = ghost_ptr[tile], ng = ghost_ptr[tile + 1] - g0;
  for (int k = threadIdx.x; k < ng; k += kTileBlock) {
    const double2 w = rq_in[__ldg(ghost + g0 + k)];
    zs[R + k] = fma(-alpha, w.y, w.x);
  }
  __syncthreads();
  const int64_t s0 = row0 >> 5;
#pragma unroll 1
  for (int k = 0; k < RPT; ++k) {
    const int sl = warp + 8 * k;
    if (sl * 32 >= rows) break;
    const double acc = sell_row_dot_smem<TILE_CHUNK>(sp + s0, lcol, sval, zs, sl, lane);
    const int li = sl * 32 + lane;
    if (li < rows) {
      const int64_t i = row0 + li;
      const double ri = zs[li];
      const double ar = acc + ri;
      const double2 w = xp[i];
      const double pi = fma(beta, w.y, ri);
      const double qi = fma(beta, qs[li], ar);
      rq_out[i] = make_double2(ri, qi);
      xp[i] = make_double2(fma(alpha, w.y, w.x), pi);
      v[0] += ri * ri;
      v[1] += d ? __ldg(d + i) * ri * ri : ri * ri;
      v[2] += pi * qi;
      v[3] += ri * qi;
      v[4] += qi * qi;
    }
  }
  }
  double tot[5];
  if (grid_sum<5, kTileBlock>(v, part, cnt, tot) && threadIdx.x == 0) {
    red[AB_RED_RZN] = tot[0];
    red[AB_RED_RR] = tot[1];
    red[AB_RED_PQ] = tot[2];
    red[AB_RED_RQ] = tot[3];
    red[AB_RED_QQ] = tot[4];
  }
}

// out[j] = s_i x'_i (i = iperm[j]); `apply`: x' += alpha p first (the x
// update of the last iteration, alpha = red[RZN] / red[PQ]).
__global__ void k_cg_tile_finish(int64_t n, const int64_t* __restrict__ iperm, const double* __restrict__ s,
                                 const double2* __restrict__ xp, const double* __restrict__ red, int apply,
                                 double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    const int64_t i = iperm[j];
    const double2 w = xp[i];
    double xi = w.x;
    if (apply) {
      const double PQ = red[AB_RED_PQ];
      const double alpha = PQ != 0.0 ? red[AB_RED_RZN] / PQ : 0.0;
      xi = fma(alpha, w.y, xi);
    }
    out[j] = s[i] * xi;
  }
}


// Decomposed path, after the interface sum of t = A z: p = z + beta p,
// q = t + beta q, p.q partials; the last block shifts sc[RZ] := red[RZN].
__global__ void __launch_bounds__(kCgBlock) k_cg_dot(int64_t n, const double* __restrict__ z,
                                                     const double* __restrict__ t, double* __restrict__ p,
                                                     double* __restrict__ q, const double* __restrict__ own,
                                                     double* red, double* sc, double* part, uint32_t* cnt) {
  const double rz_old = sc[AB_SC_RZ];
  const double rz_new = red[AB_RED_RZN];
  const double beta = rz_old != 0.0 ? rz_new / rz_old : 0.0;
  double v[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCgBlock) {
    const double pi = fma(beta, p[i], z[i]);
    const double qi = fma(beta, q[i], t[i]);
    p[i] = pi;
    q[i] = qi;
    v[0] += (own ? own[i] : 1.0) * pi * qi;
  }
  double tot[1];
  if (grid_sum<1, kCgBlock>(v, part, cnt, tot) && threadIdx.x == 0) {
    red[AB_RED_PQ] = tot[0];
    sc[AB_SC_RZ] = rz_new;
  }
}

// x += alpha p; r -= alpha q; z = dinv r; r.z and r.r partials.  Two
// consecutive rows per thread with 128-bit accesses.
__global__ void __launch_bounds__(kCgBlock) k_cg_update(int64_t n, const double* __restrict__ p,
                                                        const double* __restrict__ q,
                                                        const double* __restrict__ dinv, double* __restrict__ x,
                                                        double* __restrict__ r, double* __restrict__ z,
                                                        const double* __restrict__ own, double* red,
                                                        const double* sc, double* part, uint32_t* cnt) {
  double v[2] = {0.0, 0.0};
  const int64_t i = 2 * ((int64_t)blockIdx.x * kCgBlock + threadIdx.x);
  const double pq = red[AB_RED_PQ];
  const double rz = sc[AB_SC_RZ];
  if (i + 1 < n) {
    const double2 pv = *reinterpret_cast<const double2*>(p + i);
    const double2 xv = *reinterpret_cast<const double2*>(x + i);
    const double2 qv = *reinterpret_cast<const double2*>(q + i);
    const double2 rv = *reinterpret_cast<const double2*>(r + i);
    const double2 dv = __ldg(reinterpret_cast<const double2*>(dinv + i));
    const double alpha = pq != 0.0 ? rz / pq : 0.0;
    const double r0 = fma(-alpha, qv.x, rv.x), r1 = fma(-alpha, qv.y, rv.y);
    const double z0 = dv.x * r0, z1 = dv.y * r1;
    *reinterpret_cast<double2*>(x + i) = make_double2(fma(alpha, pv.x, xv.x), fma(alpha, pv.y, xv.y));
    *reinterpret_cast<double2*>(r + i) = make_double2(r0, r1);
    *reinterpret_cast<double2*>(z + i) = make_double2(z0, z1);
    double w0 = 1.0, w1 = 1.0;
    if (own) { w0 = own[i]; w1 = own[i + 1]; }
    v[0] = w0 * r0 * z0 + w1 * r1 * z1;
    v[1] = w0 * r0 * r0 + w1 * r1 * r1;
  } else if (i < n) {
    const double alpha = pq != 0.0 ? rz / pq : 0.0;
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    const double zi = dinv[i] * ri;
    r[i] = ri;
    z[i] = zi;
    const double w = own ? own[i] : 1.0;
    v[0] = w * ri * zi;
    v[1] = w * ri * ri;
  }
  double tot[2];
  if (grid_sum<2, kCgBlock>(v, part, cnt, tot) && threadIdx.x == 0) {
    red[AB_RED_RZN] = tot[0];
    red[AB_RED_RR] = tot[1];
  }
}


// ---------------------------------------------------------------------------
// Resident CG over a CTA-local column map (ab_cg_local).  Every CTA gathers
// the z values of its ghost rows (columns it references outside its own
// row range) ONCE per iteration into shared memory behind its own z, and
// the SpMV then reads z exclusively from shared memory through 16-bit local
// column indices: the per-non-zero L2 gathers of k_cg_resident (10.4M per
// iteration on C2) become ~0.3M per-ghost gathers, and the column stream
// shrinks from 4 to 2 bytes per non-zero.  Same iterates, same order of
// floating-point operations per row as k_cg_resident.
// Shared memory: r, p, q [RB] | x [RB] (XS only; else x lives in x_out) |
// z [RB] followed by the ghost values [max_ghost].
// ---------------------------------------------------------------------------

// Optional phase timeline of the resident solvers (ab_debug_timeline):
// globaltimer stamps of thread 0 of every CTA at the phase boundaries of
// iteration 10, tl[cta * 8 + k].
__device__ int64_t* g_timeline = nullptr;
// tl: g_timeline read once at kernel start (a global load per stamp sat on
// the critical path after every barrier)
__device__ __forceinline__ void stamp(int64_t* tl, int it, int k) {
  if (tl && it == 10 && threadIdx.x == 0) {
    int64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tl[blockIdx.x * 8 + k] = t;
  }
}

constexpr int kLocRowsPerThread = 8;  // rows_per_cta <= 8 * kResBlock

template <bool XS, bool TB>
__global__ void __launch_bounds__(kResBlock, 1) k_cg_resident_local(
    int64_t n, int64_t rows_per_cta, int max_ghost, const int64_t* __restrict__ sp,
    const uint16_t* __restrict__ lcol, const double* __restrict__ sval, const int32_t* __restrict__ gptr,
    const int32_t* __restrict__ gidx, const int32_t* __restrict__ perm, const double* __restrict__ b_in,
    double* b_zero,
    const uint8_t* __restrict__ fixed, const double* __restrict__ dinv, double* __restrict__ x_out, double* zg,
    int maxit, double tol, double* red, double* sc, double* part, unsigned* bar, int pf_depth) {
  int64_t* const tl = g_timeline;
  extern __shared__ double smem[];
  __shared__ double sred[2 * (kResBlock / 32)];
  __shared__ double srep[4];
  __shared__ uint32_t s_taddr;
  const int nb = gridDim.x;
  const int64_t RB = rows_per_cta;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int64_t r1 = r0 + RB < n ? r0 + RB : n;
  const int nloc = r1 > r0 ? (int)(r1 - r0) : 0;
  double* sr = smem;
  double* spp = sr + RB;
  double* sq = spp + RB;
  double* sd = sq + RB;               // XS: D^-1 of the rows (x is in tensor memory)
  double* sz = XS ? sd + RB : sd;     // [RB] own rows, then [max_ghost] ghosts
  // TB: the CTA's slice pointers and ghost ids copied to shared memory
  int64_t* tsp_s = reinterpret_cast<int64_t*>(sz + RB + max_ghost);
  int32_t* tg_s = reinterpret_cast<int32_t*>(tsp_s + RB / 32 + 1);
  // replicated partial tables (all_sum_rep): A 1 value, B and I 2 values;
  // behind the barrier counter at part + 5 nb (host: ab_cg_resident_local)
  double* partA = part + 8 * (size_t)nb;
  double* partB = partA + (size_t)kRep * rep_nbp(nb);
  double* partI = partA + (size_t)3 * kRep * rep_nbp(nb);
  unsigned nbar = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nsl = (nloc + 31) >> 5;
  const int64_t s_first = r0 >> 5;
  const int g0 = gptr[blockIdx.x];
  const int ng = gptr[blockIdx.x + 1] - g0;
  if (TB) {
    for (int k = threadIdx.x; k <= nsl; k += kResBlock) tsp_s[k] = sp[s_first + k];
    for (int k = threadIdx.x; k < ng; k += kResBlock) tg_s[k] = gidx[g0 + k];
    __syncthreads();
  }
  const int64_t* tsp = TB ? tsp_s : sp + s_first;
  const int32_t* tg = TB ? tg_s : gidx + g0;
  // XS: x of this thread's phase-B rows l = threadIdx.x + k * kResBlock in
  // tensor memory, columns 2k, 2k + 1 of the thread's lane
  uint32_t taddr = 0, tx = 0;
  if (XS) {
    taddr = tmem_alloc_all(&s_taddr);
    tx = taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
#pragma unroll
    for (int k = 0; k < kLocRowsPerThread; ++k) tm_st(tx + 2 * k, 0.0);
    tm_wait_st();
  }
  // XS: the warp's first slice (if at most 16 wide) stays in tensor memory
  // for the whole solve - values in columns 16-47, 16-bit columns packed two
  // per 32-bit column in 48-55 - so every iteration starts computing without
  // waiting for the matrix stream
  bool tm_slice = false;
  int w0 = 0;
  if (XS && warp < nsl) {
    w0 = (int)((tsp[warp + 1] - tsp[warp]) >> 5);
    tm_slice = w0 <= 16;
  }
  if (XS && tm_slice) {
    const int64_t base = tsp[warp] + lane;
#pragma unroll
    for (int j0 = 0; j0 < 16; j0 += 8) {
      double a[8];
      uint32_t cw[4];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = j0 + u < w0 ? __ldcs(sval + base + (int64_t)(j0 + u) * 32) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned c0 = j0 + 2 * u < w0 ? (unsigned)__ldcs(lcol + base + (int64_t)(j0 + 2 * u) * 32) : 0u;
        const unsigned c1 = j0 + 2 * u + 1 < w0 ? (unsigned)__ldcs(lcol + base + (int64_t)(j0 + 2 * u + 1) * 32)
                                                 : 0u;
        cw[u] = c0 | (c1 << 16);
      }
      tm_st8d(tx + 16 + 2 * j0, a);
      tm_st4u(tx + 48 + j0 / 2, cw);
    }
    tm_wait_st();
  }

  double a0 = 0.0, a1 = 0.0;
  for (int l = threadIdx.x; l < nloc; l += kResBlock) {
    const int64_t i = r0 + l;
    const int64_t ni = perm ? (int64_t)perm[i] : i;
    double ri = b_in[ni];
    if (fixed && fixed[i]) ri = 0.0;
    if (b_zero) b_zero[ni] = 0.0;
    const double zi = dinv[i] * ri;
    sr[l] = ri; sz[l] = zi; spp[l] = 0.0; sq[l] = 0.0;
    if (XS) sd[l] = dinv[i]; else x_out[ni] = 0.0;
    zg[i] = zi;
    a0 += ri * zi;
    a1 += ri * ri;
  }
  if (lane == 0)
    for (int d = (XS && tm_slice) ? 1 : 0; d < pf_depth + ((XS && tm_slice) ? 1 : 0); ++d)
      if (warp + d * (kResBlock / 32) < nsl) prefetch_slice16(tsp, lcol, sval, warp + d * (kResBlock / 32));
  {
    double v[2] = {a0, a1};
    block_sum<2, kResBlock>(v, sred);
    if (threadIdx.x == 0) put_partial_rep<2>(partI, nb, v);
  }
  grid_barrier(bar, ++nbar * nb);
  double t2[2];
  all_sum_rep<2>(partI, nb, srep, t2);
  double rz = t2[0], rr = t2[1];
  const double bb = rr;
  double rz_old = 0.0;
  int it = 0;
  for (; it < maxit; ++it) {
    if (tol > 0.0 && (bb == 0.0 || sqrt(rr / bb) <= tol)) break;
    const double beta = rz_old != 0.0 ? rz / rz_old : 0.0;
    stamp(tl, it, 0);
    // ---- ghost z values of this CTA's columns -> shared memory
    for (int k = threadIdx.x; k < ng; k += kResBlock) sz[RB + k] = __ldcg(zg + tg[k]);
    __syncthreads();
    stamp(tl, it, 1);
    // ---- phase A: p = z + beta p; q = A z + beta q (z from shared memory)
    double pq = 0.0;
#pragma unroll 1
    for (int sl = warp; sl < nsl; sl += kResBlock / 32) {
      if (lane == 0 && sl + pf_depth * (kResBlock / 32) < nsl)
        prefetch_slice16(tsp, lcol, sval, sl + pf_depth * (kResBlock / 32));
      double az;
      if (XS && sl == warp && tm_slice) {  // __syncwarp-uniform branch: whole warp
        az = 0.0;
#pragma unroll
        for (int j0 = 0; j0 < 16; j0 += 8) {
          uint32_t aw[16], cw[4];
          tm_ld8d(tx + 16 + 2 * j0, aw);
          tm_ld4u(tx + 48 + j0 / 2, cw);
          tm_wait_ld();
          tm_fence_regs(aw);
          tm_fence_regs(cw);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const unsigned c = (cw[u >> 1] >> (16 * (u & 1))) & 0xffffu;
            az = fma(__hiloint2double((int)aw[2 * u + 1], (int)aw[2 * u]), sz[c], az);
          }
        }
      } else {
        az = sell_row_dot_smem<kLocChunk>(tsp, lcol, sval, sz, sl, lane);
      }
      if (sl == warp) stamp(tl, it, 7);
      const int l = sl * 32 + lane;
      if (l < nloc) {
        const double p = fma(beta, spp[l], sz[l]);
        const double q = fma(beta, sq[l], az);
        spp[l] = p;
        sq[l] = q;
        pq += p * q;
      }
    }
    // D^-1 of this thread's phase-B rows (global form): in flight across the reduction
    double dv[kLocRowsPerThread];
    if (!XS) {
#pragma unroll
      for (int k = 0; k < kLocRowsPerThread; ++k) {
        const int l = threadIdx.x + k * kResBlock;
        dv[k] = l < nloc ? __ldg(dinv + r0 + l) : 0.0;
      }
    }
    {
      double v[1] = {pq};
      block_sum<1, kResBlock>(v, sred);
      if (threadIdx.x == 0) put_partial_rep<1>(partA, nb, v);
    }
    stamp(tl, it, 2);
    grid_barrier(bar, ++nbar * nb);
    double t1[1];
    all_sum_rep<1>(partA, nb, srep, t1);
    stamp(tl, it, 3);
    const double alpha = t1[0] != 0.0 ? rz / t1[0] : 0.0;
    // ---- phase B: x += alpha p, r -= alpha q, z = D^-1 r
    if (lane == 0 && it + 1 < maxit)
      for (int d = (XS && tm_slice) ? 1 : 0; d < pf_depth + ((XS && tm_slice) ? 1 : 0); ++d)
        if (warp + d * (kResBlock / 32) < nsl)
          prefetch_slice16(tsp, lcol, sval, warp + d * (kResBlock / 32));
    double b0 = 0.0, b1 = 0.0;
    uint32_t xw[kLocRowsPerThread][2];
    if (XS) {
#pragma unroll
      for (int k = 0; k < kLocRowsPerThread; ++k) tm_ld(tx + 2 * k, xw[k][0], xw[k][1]);
      tm_wait_ld();
    }
#pragma unroll
    for (int k = 0; k < kLocRowsPerThread; ++k) {
      const int l = threadIdx.x + k * kResBlock;
      if (XS) {
        const double xo = tm_val(xw[k][0], xw[k][1]);
        tm_st(tx + 2 * k, l < nloc ? fma(alpha, spp[l], xo) : xo);
      }
      if (l < nloc) {
        if (!XS) {
          const int64_t ni = perm ? (int64_t)perm[r0 + l] : r0 + l;
          x_out[ni] = fma(alpha, spp[l], x_out[ni]);
        }
        const double ri = fma(-alpha, sq[l], sr[l]);
        const double zi = (XS ? sd[l] : dv[k]) * ri;
        sr[l] = ri;
        sz[l] = zi;
        zg[r0 + l] = zi;
        b0 += ri * zi;
        b1 += ri * ri;
      }
    }
    stamp(tl, it, 6);
    {
      double v[2] = {b0, b1};
      block_sum<2, kResBlock>(v, sred);
      if (threadIdx.x == 0) put_partial_rep<2>(partB, nb, v);
    }
    stamp(tl, it, 4);
    grid_barrier(bar, ++nbar * nb);
    all_sum_rep<2>(partB, nb, srep, t2);
    stamp(tl, it, 5);
    rz_old = rz;
    rz = t2[0];
    rr = t2[1];
  }
  if (XS) {
    tm_wait_st();
#pragma unroll
    for (int k = 0; k < kLocRowsPerThread; ++k) {
      uint32_t lo, hi;
      tm_ld(tx + 2 * k, lo, hi);
      tm_wait_ld();
      const int l = threadIdx.x + k * kResBlock;
      if (l < nloc) x_out[perm ? (int64_t)perm[r0 + l] : r0 + l] = tm_val(lo, hi);
    }
    tmem_free_all(taddr);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    red[AB_RED_RZN] = rz;
    red[AB_RED_RR] = rr;
    red[AB_RED_ITERS] = (double)it;
    sc[AB_SC_BB] = bb;
  }
}


static unsigned cg_grid(int64_t n) {
  const int64_t g = (n + kCgBlock - 1) / kCgBlock;
  return (unsigned)(g < kCgGrid ? g : kCgGrid);
}

}  // namespace ab

using namespace ab;

template <int RPT>
static int tile_iter_launch(const ab_sell* a, const ab_cg_local* m, const double* rq_in, double* rq_out, double* xp,
                            const double* d, double* red, double* part, uint32_t* cnt, cudaStream_t st) {
  constexpr int R = kTileBlock * RPT;
  const int64_t n = a->n_rows;
  const size_t smem = (size_t)(2 * R + m->max_ghost) * sizeof(double);
  static size_t smem_set = 0;
  auto kern = k_cg_tile_iter<RPT>;
  if (smem > 48 * 1024 && smem > smem_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return fail("ab_cg_tile_iter: shared memory request rejected (too many ghost rows)");
    smem_set = smem;
  }
  int64_t grid = (n + R - 1) / R;
#if TSP_PERSIST
  static int resident = 0;
  if (!resident) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTileBlock, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident = (per_sm > 0 ? per_sm : 1) * sms;
  }
  if (grid > resident) grid = resident;
#endif
  kern<<<(unsigned)grid, kTileBlock, smem, st>>>(
      n, a->slice_ptr, m->cols, a->vals, m->ghost_ptr, m->ghost, reinterpret_cast<const double2*>(rq_in),
      reinterpret_cast<double2*>(rq_out), reinterpret_cast<double2*>(xp), d, red, part, cnt);
  return check_launch("ab_cg_tile_iter");
}

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
               double* r, double* z, double* p, double* q, const double* own, double* red, double* sc, double* part,
               uint32_t* cnt, void* stream) {
  if (n <= 0) return fail("ab_cg_init: empty system");
  k_cg_init<<<cg_grid(n), kCgBlock, 0, S(stream)>>>(n, b_in, b_zero, fixed, dinv, x, r, z, p, q, own, red, sc, part,
                                                    cnt);
  return check_launch("ab_cg_init");
}

int ab_sell_symscale(const ab_sell* a, const double* s, void* stream) {
  if (!a || !s) return fail("ab_sell_symscale: null argument");
  if (a->n_rows > 0)
    k_sell_symscale<<<grid_for(a->n_rows, 256), 256, 0, S(stream)>>>(a->n_rows, a->slice_ptr, a->cols,
                                                                     const_cast<double*>(a->vals), s);
  return check_launch("ab_sell_symscale");
}

int ab_cg_init_scaled(int64_t n, const int64_t* perm, double* b, int32_t zero_b, const uint8_t* fixed,
                      const double* s, const double* d, double* x, double* r, double* p, double* q, double* red,
                      double* sc, double* part, uint32_t* cnt, void* stream) {
  if (n <= 0 || !perm || !b || !s) return fail("ab_cg_init_scaled: empty system or null argument");
  k_cg_init_scaled<<<cg_grid(n), kCgBlock, 0, S(stream)>>>(n, perm, b, zero_b, fixed, s, d, x, r, p, q, red, sc, part,
                                                           cnt);
  // b is zeroed by a coalesced pass once every row has read it (a scattered
  // b[perm[i]] = 0 in the kernel costs a partial-sector write per row)
  if (zero_b && cudaMemsetAsync(b, 0, (size_t)n * sizeof(double), S(stream)) != cudaSuccess)
    return fail("ab_cg_init_scaled: cannot zero b");
  return check_launch("ab_cg_init_scaled");
}

int ab_cg_update_scaled(int64_t n, const double* p, const double* q, double* x, double* r, const double* d,
                        double* red, const double* sc, double* part, uint32_t* cnt, void* stream) {
  k_cg_update_scaled<<<grid_for((n + 1) / 2, kCgBlock), kCgBlock, 0, S(stream)>>>(n, p, q, x, r, d, red, sc, part,
                                                                                cnt);
  return check_launch("ab_cg_update_scaled");
}

int ab_cg_finish_scaled(int64_t n, const int64_t* iperm, const double* s, const double* x, double* out,
                        void* stream) {
  if (n > 0) k_cg_finish_scaled<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, iperm, s, x, out);
  return check_launch("ab_cg_finish_scaled");
}

int ab_cg_spmv_tile(const ab_sell* a, const ab_cg_local* m, const double* z, double* p, double* q, double* red,
                    double* sc, double* part, uint32_t* cnt, void* stream) {
  if (!a || !m || !m->cols || !m->ghost_ptr || !m->ghost) return fail("ab_cg_spmv_tile: null argument");
  const int64_t n = a->n_rows;
  const int64_t R = m->rows_per_cta;
  if (R < 64 || R % 64 || (int64_t)m->n_cta * R < n || R + m->max_ghost > 65536)
    return fail("ab_cg_spmv_tile: tile map does not match the matrix (rows_per_cta % 64, n_cta * R >= n, "
                "R + max_ghost <= 65536)");
  if ((uintptr_t)z & 15) return fail("ab_cg_spmv_tile: z must be 16-byte aligned");
  const size_t smem = (size_t)(R + m->max_ghost) * sizeof(double);
  static size_t smem_set = 0;
  if (smem > 48 * 1024 && smem > smem_set) {
    if (cudaFuncSetAttribute(k_cg_spmv_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return fail("ab_cg_spmv_tile: shared memory request rejected (tile too large)");
    smem_set = smem;
  }
  const unsigned grid = (unsigned)((n + R - 1) / R);
  k_cg_spmv_tile<<<grid, kTileBlock, smem, S(stream)>>>(n, (int)R, a->slice_ptr, m->cols, a->vals, m->ghost_ptr,
                                                        m->ghost, z, p, q, red, sc, part, cnt);
  return check_launch("ab_cg_spmv_tile");
}

int ab_cg_tile_init(int64_t n, const int64_t* perm, double* b, int32_t zero_b, const uint8_t* fixed,
                    const double* s, const double* d, double* xp, double* rq, double* red, double* sc, double* part,
                    uint32_t* cnt, void* stream) {
  if (n <= 0 || !perm || !b || !s || !xp || !rq) return fail("ab_cg_tile_init: empty system or null argument");
  if (((uintptr_t)xp | (uintptr_t)rq) & 15) return fail("ab_cg_tile_init: xp, rq must be 16-byte aligned");
  k_cg_tile_init<<<cg_grid(n), kCgBlock, 0, S(stream)>>>(n, perm, b, fixed, s, d, reinterpret_cast<double2*>(xp),
                                                         reinterpret_cast<double2*>(rq), red, sc, part, cnt);
  if (zero_b && cudaMemsetAsync(b, 0, (size_t)n * sizeof(double), S(stream)) != cudaSuccess)
    return fail("ab_cg_tile_init: cannot zero b");
  return check_launch("ab_cg_tile_init");
}

int ab_cg_tile_iter(const ab_sell* a, const ab_cg_local* m, const double* rq_in, double* rq_out, double* xp,
                    const double* d, double* red, double* part, uint32_t* cnt, void* stream) {
  if (!a || !m || !m->cols || !m->ghost_ptr || !m->ghost || !rq_in || !rq_out || !xp)
    return fail("ab_cg_tile_iter: null argument");
  if (rq_in == rq_out) return fail("ab_cg_tile_iter: rq_in and rq_out must be different buffers (ping-pong)");
  if (((uintptr_t)xp | (uintptr_t)rq_in | (uintptr_t)rq_out) & 15)
    return fail("ab_cg_tile_iter: xp, rq must be 16-byte aligned");
  const int64_t R = m->rows_per_cta;
  if ((int64_t)m->n_cta * R < a->n_rows || R + m->max_ghost > 65536)
    return fail("ab_cg_tile_iter: tile map does not match the matrix");
  switch (R) {
    case 1024: return tile_iter_launch<4>(a, m, rq_in, rq_out, xp, d, red, part, cnt, S(stream));
    case 2048: return tile_iter_launch<8>(a, m, rq_in, rq_out, xp, d, red, part, cnt, S(stream));
    case 4096: return tile_iter_launch<16>(a, m, rq_in, rq_out, xp, d, red, part, cnt, S(stream));
    default: return fail("ab_cg_tile_iter: rows_per_cta must be 1024, 2048 or 4096");
  }
}

int ab_cg_tile_finish(int64_t n, const int64_t* iperm, const double* s, const double* xp, const double* red,
                      int32_t apply, double* out, void* stream) {
  if (n > 0)
    k_cg_tile_finish<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, iperm, s, reinterpret_cast<const double2*>(xp), red,
                                                              apply, out);
  return check_launch("ab_cg_tile_finish");
}

int ab_cg_init_perm(int64_t n, const int64_t* perm, double* b, int32_t zero_b, const uint8_t* fixed,
                    const double* dinv, double* x, double* r, double* z, double* p, double* q, double* red, double* sc,
                    double* part, uint32_t* cnt, void* stream) {
  if (n <= 0 || !perm || !b) return fail("ab_cg_init_perm: empty system or null permutation");
  k_cg_init_perm<<<cg_grid(n), kCgBlock, 0, S(stream)>>>(n, perm, b, zero_b, fixed, dinv, x, r, z, p, q, red, sc,
                                                         part, cnt);
  if (zero_b && cudaMemsetAsync(b, 0, (size_t)n * sizeof(double), S(stream)) != cudaSuccess)
    return fail("ab_cg_init_perm: cannot zero b");
  return check_launch("ab_cg_init_perm");
}

int ab_perm_scatter(int64_t n, const int64_t* perm, const double* in, double* out, void* stream) {
  if (n <= 0) return AB_OK;
  k_perm_scatter<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, perm, in, out);
  return check_launch("ab_perm_scatter");
}

int ab_cg_set_bb(double* red, double* sc, void* stream) {
  k_cg_set_bb<<<1, 1, 0, S(stream)>>>(red, sc);
  return check_launch("ab_cg_set_bb");
}

int ab_cg_spmv(const ab_sell* a, const double* z, double* p, double* q, double* t, int32_t with_dot,
               const double* own, double* red, double* sc, double* part, uint32_t* cnt, void* stream) {
  if (!a) return fail("ab_cg_spmv: null matrix");
  if (!with_dot && !t) return fail("ab_cg_spmv: the decomposed form needs t");
  const int64_t n = a->n_rows;
  if (with_dot)
    k_cg_spmv<true><<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(n, a->slice_ptr, a->cols, a->vals, z, p, q, t,
                                                                       own, red, sc, part, cnt);
  else
    k_cg_spmv<false><<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(n, a->slice_ptr, a->cols, a->vals, z, p, q,
                                                                        t, own, red, sc, part, cnt);
  return check_launch("ab_cg_spmv");
}

int ab_cg_spmv_unit(const ab_sell* a, const double* z, double* p, double* q, double* red, double* sc, double* part,
                    uint32_t* cnt, void* stream) {
  if (!a) return fail("ab_cg_spmv_unit: null matrix");
  const int64_t n = a->n_rows;
  k_cg_spmv_unit<<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(n, a->slice_ptr, a->cols, a->vals, z, p, q, red, sc,
                                                                    part, cnt);
  return check_launch("ab_cg_spmv_unit");
}


int ab_cg_dot(int64_t n, const double* z, const double* t, double* p, double* q, const double* own, double* red,
              double* sc, double* part, uint32_t* cnt, void* stream) {
  k_cg_dot<<<cg_grid(n), kCgBlock, 0, S(stream)>>>(n, z, t, p, q, own, red, sc, part, cnt);
  return check_launch("ab_cg_dot");
}

int ab_cg_update(int64_t n, const double* p, const double* q, const double* dinv, double* x, double* r, double* z,
                 const double* own, double* red, const double* sc, double* part, uint32_t* cnt, void* stream) {
  k_cg_update<<<grid_for((n + 1) / 2, kCgBlock), kCgBlock, 0, S(stream)>>>(n, p, q, dinv, x, r, z, own, red, sc, part,
                                                                        cnt);
  return check_launch("ab_cg_update");
}

int ab_cg_resident_fits(int64_t n, int64_t* rows_per_cta, int32_t* n_cta) {
  int dev = 0, sms = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  int64_t rb = ((n + sms - 1) / sms + 31) / 32 * 32;
  const size_t smem = (size_t)rb * 5 * sizeof(double);
  const bool ok = coop && smem <= 200 * 1024;
  if (rows_per_cta) *rows_per_cta = rb;
  if (n_cta) *n_cta = (int32_t)((n + rb - 1) / rb);
  return ok ? 1 : 0;
}


}  // extern "C"

namespace {
// Shared-memory plan of k_cg_resident_local: 0 = does not fit, else
// 1 + (x in shared memory) + 2 * (slice/ghost tables in shared memory).
int local_mode(int64_t rb, int32_t max_ghost, size_t* bytes) {
  int dev = 0, optin = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  const size_t static_smem = 1024;  // sred + bcast + slack
  const size_t cap = optin > (int)static_smem ? (size_t)optin - static_smem : 0;
  if (!coop || max_ghost < 0 || rb + max_ghost > 65536) return 0;
  const size_t xs = (size_t)(5 * rb + max_ghost) * sizeof(double);
  const size_t xg = (size_t)(4 * rb + max_ghost) * sizeof(double);
  const size_t tb = (size_t)(rb / 32 + 1) * 8 + (size_t)max_ghost * 4;
  int mode = 0;
  size_t b = 0;
  if (xs + tb <= cap) { mode = 4; b = xs + tb; }
  else if (xs <= cap) { mode = 2; b = xs; }
  else if (xg + tb <= cap) { mode = 3; b = xg + tb; }
  else if (xg <= cap) { mode = 1; b = xg; }
  if (bytes) *bytes = b;
  return mode;
}
}  // namespace

extern "C" {

int ab_debug_timeline(int64_t* buf) {
  if (cudaMemcpyToSymbol(g_timeline, &buf, sizeof(buf)) != cudaSuccess) return fail("ab_debug_timeline: copy failed");
  return AB_OK;
}

int ab_cg_resident_local_fits(int64_t rows_per_cta, int32_t max_ghost) {
  return local_mode(rows_per_cta, max_ghost, nullptr);
}


int ab_cg_resident_local(const ab_sell* a, const ab_cg_local* m, const double* b_in, double* b_zero,
                         const uint8_t* fixed, const double* dinv, double* x, double* z, int32_t maxit, double tol,
                         double* red, double* sc, double* part, void* stream) {
  if (!a || !m) return fail("ab_cg_resident_local: null matrix or map");
  if (!m->cols || !m->ghost_ptr || !m->ghost) return fail("ab_cg_resident_local: incomplete column map");
  int64_t n = a->n_rows, rb = 0;
  int32_t ncta = 0;
  ab_cg_resident_fits(n, &rb, &ncta);
  if (rb != m->rows_per_cta || ncta != m->n_cta)
    return fail("ab_cg_resident_local: column map built for another launch shape");
  const int64_t* sp = a->slice_ptr;
  const uint16_t* lcol = m->cols;
  const double* vals = a->vals;
  const int32_t* gp = m->ghost_ptr;
  const int32_t* gi = m->ghost;
  const int32_t* pm = m->perm;
  int mg = m->max_ghost;
  int depth = m->prefetch_depth;
  int mi = maxit;
  unsigned* bar = reinterpret_cast<unsigned*>(part + 5 * (size_t)ncta);
  if (cudaMemsetAsync(bar, 0, sizeof(unsigned), S(stream)) != cudaSuccess)
    return fail("ab_cg_resident_local: cannot reset the barrier counter");
  cudaError_t e;
  size_t smem = 0;
  {
    if (m->variant != 0) return fail("ab_cg_resident_local: unknown solver variant");
    int mode = local_mode(rb, mg, &smem);
    if (mode == 0) return fail("ab_cg_resident_local: system does not fit in shared memory");
    if (m->force_mode > 0) {  // a smaller plan than the best one (tests)
      if (m->force_mode > mode) return fail("ab_cg_resident_local: forced plan does not fit");
      mode = m->force_mode;
      const size_t xsb = (size_t)(5 * rb + mg) * 8, xgb = (size_t)(4 * rb + mg) * 8;
      const size_t tbb = (size_t)(rb / 32 + 1) * 8 + (size_t)mg * 4;
      smem = (mode == 2 || mode == 4 ? xsb : xgb) + (mode >= 3 ? tbb : 0);
    }
    const bool xs = mode == 2 || mode == 4, tb = mode >= 3;
    if (rb > (int64_t)kLocRowsPerThread * kResBlock) return fail("ab_cg_resident_local: too many rows per CTA");

    const void* fn = xs ? (tb ? (const void*)k_cg_resident_local<true, true> : (const void*)k_cg_resident_local<true, false>)
                        : (tb ? (const void*)k_cg_resident_local<false, true> : (const void*)k_cg_resident_local<false, false>);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return fail("ab_cg_resident_local: cannot reserve shared memory");
    void* args[] = {&n,           &rb,          &mg,  (void*)&sp, (void*)&lcol, (void*)&vals, (void*)&gp,
                    (void*)&gi,   (void*)&pm,   (void*)&b_in, &b_zero, (void*)&fixed, (void*)&dinv, &x, &z,
                    &mi,          &tol,         &red, &sc, &part, &bar, &depth};
    e = cudaLaunchCooperativeKernel(fn, dim3(ncta), dim3(kResBlock), args, smem, S(stream));
  }
  if (e != cudaSuccess) {
    set_error(std::string("ab_cg_resident_local: ") + cudaGetErrorString(e));
    return AB_ECUDA;
  }
  return check_launch("ab_cg_resident_local");
}


}  // extern "C"
