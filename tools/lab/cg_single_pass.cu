// Rejected variant (round 2, measured slower; not built): single-pass scaled
// CG, one kernel per iteration.  Kept for reference with its measurements in
// DESIGN.md §4 ("Single-pass CG").  It moves 64 instead of 88 vector bytes per
// row and iteration but gathers a 16-byte (r', q) pair per stored entry; on
// an 8.1M-row tet system it ran 400-680 us per iteration (register-capped
// builds 400-460 us) against 370 us for ab_cg_spmv_unit + ab_cg_update_scaled
// and 323 us for ab_cg_spmv_tile + ab_cg_update_scaled (tools/time_cg_large.py).
// To rebuild it: paste into paper_2005_05899_b200/csrc/ab_solver.cu inside
// namespace ab and add the declarations below to include/alyab200.h.
//
// int ab_cg_init_fused(int64_t n, const int64_t* perm, double* b, int32_t zero_b, const uint8_t* fixed,
//                      const double* s, const double* d, double* xp, double* rq, double* red, double* sc,
//                      double* part, uint32_t* cnt, void* stream);
// int ab_cg_fused(const ab_sell* a, const double* rq_in, double* rq_out, double* xp, const double* d,
//                 double* red, double* part, uint32_t* cnt, void* stream);
// int ab_cg_finish_fused(int64_t n, const int64_t* iperm, const double* s, const double* xp,
//                        const double* red, int32_t apply, double* out, void* stream);
#define AB_RED_RQ 6
#define AB_RED_QQ 7

// ---------------------------------------------------------------------------
// Single-pass scaled CG: ONE kernel per iteration (round 2, VERDICT r1 #6/
// DESIGN §4).  The two-kernel form moves 88 bytes of vectors per row and
// iteration (SpMV: r' gathered + own, p, q read and written; update: x, r'
// read and written, p, q read).  Here kernel F_j forms r'_j = r'_{j-1} -
// alpha q_{j-1} and x_j = x_{j-1} + alpha p_{j-1} for its own rows, the
// neighbours' r'_j on the fly from the gathered (r', q) pair, and p_j, q_j:
// 64 bytes per row (xp and rq pairs read and written).  alpha_{j-1} =
// r'r'_{j-1} / p.q_{j-1} comes from the previous kernel's sums; beta_{j-1}
// needs r'r'_j before any row of F_j has formed r'_j, so it uses the
// recurrence r'r'_j = r'r'_{j-1} - 2 alpha r'.q_{j-1} + alpha^2 q.q_{j-1}
// (the three dots of the previous kernel; the true r'r'_j that F_j sums
// feeds alpha_j, so no error accumulates).  The iterates equal the
// two-kernel form's up to that rounding-level difference in beta.
// Buffers: xp[i] = (x'_i, p_i) in place; rq ping-pong (r'_i, q_i).
// red slots: RZN = r'.r' (true, of the r' formed), RR = sum d r'^2 (d given)
// or r'.r', PQ = p.q, RQ (6) = r'.q, QQ (7) = q.q.
// ---------------------------------------------------------------------------
#ifndef FUSED_CHUNK
#define FUSED_CHUNK 8
#endif

__global__ void __launch_bounds__(kCgBlock) k_cg_init_fused(int64_t n, const int64_t* __restrict__ perm,
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
    red[AB_RED_PQ] = 0.0;  // alpha_{-1} = 0: F_0 keeps r'_0 = b' and x = 0
    red[AB_RED_RQ] = 0.0;
    red[AB_RED_QQ] = 0.0;
    sc[AB_SC_RZ] = 0.0;
    sc[AB_SC_BB] = t[1];
  }
}

#ifndef FUSED_MINB
#define FUSED_MINB 1
#endif
__global__ void __launch_bounds__(kCgBlock, FUSED_MINB) k_cg_fused(int64_t n, const int64_t* __restrict__ sp,
                                                       const int32_t* __restrict__ scol,
                                                       const double* __restrict__ sval,
                                                       const double2* __restrict__ rq_in,
                                                       double2* __restrict__ rq_out, double2* __restrict__ xp,
                                                       const double* __restrict__ d, double* red, double* part,
                                                       uint32_t* cnt) {
  constexpr int CH = FUSED_CHUNK;
  const int64_t i = (int64_t)blockIdx.x * kCgBlock + threadIdx.x;
  const double RR = red[AB_RED_RZN], PQ = red[AB_RED_PQ], RQ = red[AB_RED_RQ], QQ = red[AB_RED_QQ];
  const double alpha = PQ != 0.0 ? RR / PQ : 0.0;
  double rr_next = fma(alpha, fma(alpha, QQ, -2.0 * RQ), RR);
  if (rr_next < 0.0) rr_next = 0.0;
  const double beta = RR != 0.0 ? rr_next / RR : 0.0;
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (i < n) {
    // off-diagonal row of the unit-diagonal matrix against r'_j formed from
    // the gathered (r', q) pairs (the same fma as the owner row's)
    const int64_t sl = i >> 5;
    const int lane = (int)(i & 31);
    const int64_t base = sp[sl] + lane;
    const int width = (int)((sp[sl + 1] - sp[sl]) >> 5);
    double acc = 0.0;
    for (int j0 = 0; j0 < width; j0 += CH) {
      int c[CH];
      double a[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const bool ok = j0 + u < width;
        c[u] = ok ? __ldcs(scol + base + (int64_t)(j0 + u) * 32) : 0;
        a[u] = ok ? __ldcs(sval + base + (int64_t)(j0 + u) * 32) : 0.0;
      }
      double2 g[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) g[u] = __ldg(rq_in + c[u]);
#pragma unroll
      for (int u = 0; u < CH; ++u) acc = fma(a[u], fma(-alpha, g[u].y, g[u].x), acc);
    }
    // own row after the gathers (fewer live registers in the loop)
    const double2 me = rq_in[i];
    const double2 xpi = xp[i];
    const double ri = fma(-alpha, me.y, me.x);
    const double ar = acc + ri;
    const double pi = fma(beta, xpi.y, ri);
    const double qi = fma(beta, me.y, ar);
    rq_out[i] = make_double2(ri, qi);
    xp[i] = make_double2(fma(alpha, xpi.y, xpi.x), pi);
    v[0] = ri * ri;
    v[1] = d ? __ldg(d + i) * ri * ri : v[0];
    v[2] = pi * qi;
    v[3] = ri * qi;
    v[4] = qi * qi;
  }
  double tot[5];
  if (grid_sum<5, kCgBlock>(v, part, cnt, tot) && threadIdx.x == 0) {
    red[AB_RED_RZN] = tot[0];
    red[AB_RED_RR] = tot[1];
    red[AB_RED_PQ] = tot[2];
    red[AB_RED_RQ] = tot[3];
    red[AB_RED_QQ] = tot[4];
  }
}

// out[j] = s_i x'_i (i = iperm[j]); `apply`: x' += alpha p first, the update
// of the last iteration (alpha = red[RZN] / red[PQ], as F_{j+1} would form it).
__global__ void k_cg_finish_fused(int64_t n, const int64_t* __restrict__ iperm, const double* __restrict__ s,
                                  const double2* __restrict__ xp, const double* __restrict__ red, int apply,
                                  double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    const int64_t i = iperm[j];
    const double2 v = xp[i];
    double xi = v.x;
    if (apply) {
      const double PQ = red[AB_RED_PQ];
      const double alpha = PQ != 0.0 ? red[AB_RED_RZN] / PQ : 0.0;
      xi = fma(alpha, v.y, xi);
    }
    out[j] = s[i] * xi;
  }
}


int ab_cg_init_fused(int64_t n, const int64_t* perm, double* b, int32_t zero_b, const uint8_t* fixed,
                     const double* s, const double* d, double* xp, double* rq, double* red, double* sc, double* part,
                     uint32_t* cnt, void* stream) {
  if (n <= 0 || !perm || !b || !s || !xp || !rq) return fail("ab_cg_init_fused: empty system or null argument");
  if (((uintptr_t)xp | (uintptr_t)rq) & 15) return fail("ab_cg_init_fused: xp, rq must be 16-byte aligned");
  k_cg_init_fused<<<cg_grid(n), kCgBlock, 0, S(stream)>>>(n, perm, b, fixed, s, d, reinterpret_cast<double2*>(xp),
                                                          reinterpret_cast<double2*>(rq), red, sc, part, cnt);
  if (zero_b && cudaMemsetAsync(b, 0, (size_t)n * sizeof(double), S(stream)) != cudaSuccess)
    return fail("ab_cg_init_fused: cannot zero b");
  return check_launch("ab_cg_init_fused");
}

int ab_cg_fused(const ab_sell* a, const double* rq_in, double* rq_out, double* xp, const double* d, double* red,
                double* part, uint32_t* cnt, void* stream) {
  if (!a || !rq_in || !rq_out || !xp) return fail("ab_cg_fused: null argument");
  if (rq_in == rq_out) return fail("ab_cg_fused: rq_in and rq_out must be different buffers (ping-pong)");
  if (((uintptr_t)xp | (uintptr_t)rq_in | (uintptr_t)rq_out) & 15)
    return fail("ab_cg_fused: xp, rq must be 16-byte aligned");
  const int64_t n = a->n_rows;
  k_cg_fused<<<grid_for(n, kCgBlock), kCgBlock, 0, S(stream)>>>(
      n, a->slice_ptr, a->cols, a->vals, reinterpret_cast<const double2*>(rq_in), reinterpret_cast<double2*>(rq_out),
      reinterpret_cast<double2*>(xp), d, red, part, cnt);
  return check_launch("ab_cg_fused");
}

int ab_cg_finish_fused(int64_t n, const int64_t* iperm, const double* s, const double* xp, const double* red,
                       int32_t apply, double* out, void* stream) {
  if (n > 0)
    k_cg_finish_fused<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, iperm, s, reinterpret_cast<const double2*>(xp), red,
                                                               apply, out);
  return check_launch("ab_cg_finish_fused");
}

