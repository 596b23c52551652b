// Element-loop kernels: K1 mass/lumped mass, K2 momentum RHS, K4 divergence,
// K6 gradient, Laplacian values, centroids.
//
// One thread per element (the reference's pack lane, assembly.py:235-243;
// the CTA is the pack), gather -> Gauss loop -> scatter.
// Two scatter modes, chosen by measurement:
//   * direct: fp64 reductions to global memory (REDG.E.ADD.F64) per node;
//   * windowed: elements are processed in SFC-ordered blocks; each block
//     writes its element contributions into shared-memory slots and then
//     reduces them per unique node of the block's "node window" in a fixed
//     order, issuing one global reduction per (block, node) instead of one
//     per (element, node).
#include <cstdlib>

#include "ab_common.cuh"
#include "ab_tables.inc"

namespace ab {

template <int R> struct RuleT;
template <> struct RuleT<AB_RULE_TET1> { static constexpr int NN = 4, NG = 1; static constexpr bool TET = true; };
template <> struct RuleT<AB_RULE_TET4> { static constexpr int NN = 4, NG = 4; static constexpr bool TET = true; };
template <> struct RuleT<AB_RULE_PYR5> { static constexpr int NN = 5, NG = 5; static constexpr bool TET = false; };
template <> struct RuleT<AB_RULE_PRI6> { static constexpr int NN = 6, NG = 6; static constexpr bool TET = false; };
template <> struct RuleT<AB_RULE_HEX8> { static constexpr int NN = 8, NG = 8; static constexpr bool TET = false; };

// Kernel-side view of one category.
struct CatP {
  const double* __restrict__ coords;
  const int32_t* __restrict__ conn;
  int64_t n;
  double L0, L1, L2;  // periods (0 = none)
  int periodic;
  // Vreman filter width squared per element, Delta^2 = V_e^(2/3) (geometry
  // only: computed once by k_filter_width, ab_set_filter_width); nullable
  const double* __restrict__ delta2;
};

// Node windows of a category (windowed scatter), see DESIGN.md §4.2.
struct WinP {
  const int64_t* __restrict__ blk_ptr;   // [n_blocks+1] offsets into wnode
  const int32_t* __restrict__ wnode;     // window node ids
  const int32_t* __restrict__ wptr;      // [n_win+1] offsets into wslot
  const uint16_t* __restrict__ wslot;    // slot offset a*block + local_elem into the [NC][NN][block] slots
  const uint16_t* __restrict__ loc;      // [E][NN] window-local node index of each element node
  const int4* __restrict__ desc;         // per block {b0, b1, wptr[b0], wptr[b1]} (pipelined kernels)
  // pipelined kernels: the block's block*NN element-node references sorted by
  // window node, (slot offset | window index << 16); padding 0xffff0000
  const uint32_t* __restrict__ wref;
  int block;                             // elements per block (== blockDim.x)
  int wmax;                              // largest window (nodes) of any block
  // Colour mode (ab_set_window_colours; NULL corder = fp64-atomic scatter):
  // blocks grouped by colour, no two blocks of a colour share a window node,
  // colours processed in order behind a grid barrier, and every window
  // node's sum formed by one thread in a fixed order -> plain read-add-write,
  // bitwise reproducible results.
  const int32_t* __restrict__ corder;    // [n_blocks] logical -> physical block, grouped by colour
  const int64_t* __restrict__ cptr;      // [ncol+1] colour offsets into corder
  unsigned* gbar;                        // [ncol] colour-barrier counters (zeroed before every launch)
  int ncol;
};

template <int NN>
__device__ __forceinline__ void load_conn(const int32_t* __restrict__ conn, int64_t e, int (&nd)[NN]) {
  const int32_t* p = conn + e * NN;
  if constexpr (NN == 4) {
    int4 v = __ldg(reinterpret_cast<const int4*>(p));
    nd[0] = v.x; nd[1] = v.y; nd[2] = v.z; nd[3] = v.w;
  } else if constexpr (NN == 8) {
    int4 v = __ldg(reinterpret_cast<const int4*>(p));
    int4 w = __ldg(reinterpret_cast<const int4*>(p) + 1);
    nd[0] = v.x; nd[1] = v.y; nd[2] = v.z; nd[3] = v.w;
    nd[4] = w.x; nd[5] = w.y; nd[6] = w.z; nd[7] = w.w;
  } else if constexpr (NN == 6) {
    const int2* q = reinterpret_cast<const int2*>(p);
    int2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
    nd[0] = a.x; nd[1] = a.y; nd[2] = b.x; nd[3] = b.y; nd[4] = c.x; nd[5] = c.y;
  } else {
#pragma unroll
    for (int a = 0; a < NN; ++a) nd[a] = __ldg(p + a);
  }
}

template <int NN>
__device__ __forceinline__ void unwrap(const CatP& c, double (&x)[NN][3]) {
  if (c.periodic) {  // minimum-image unwrap relative to node 0
    const double L[3] = {c.L0, c.L1, c.L2};
#pragma unroll
    for (int a = 1; a < NN; ++a)
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (L[d] > 0.0) {
          double rel = x[a][d] - x[0][d];
          x[a][d] = x[0][d] + (rel - L[d] * rint(rel / L[d]));
        }
  }
}

template <int NN>
__device__ __forceinline__ void load_coords(const CatP& c, const int (&nd)[NN], double (&x)[NN][3]) {
#pragma unroll
  for (int a = 0; a < NN; ++a) {
    d4 v = ld4_nc(c.coords + 4 * (int64_t)nd[a]);
    x[a][0] = v.x; x[a][1] = v.y; x[a][2] = v.z;
  }
  unwrap<NN>(c, x);
}

template <int NN>
__device__ __forceinline__ void load_vec(const double* __restrict__ f4, const int (&nd)[NN], double (&u)[NN][3]) {
#pragma unroll
  for (int a = 0; a < NN; ++a) {
    d4 v = ld4_nc(f4 + 4 * (int64_t)nd[a]);
    u[a][0] = v.x; u[a][1] = v.y; u[a][2] = v.z;
  }
}

__device__ __forceinline__ double det3(const double (&m)[3][3]) {
  return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
         m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

// inv = J^-1 (cofactor form); returns det J.
__device__ __forceinline__ double inv3(const double (&m)[3][3], double (&iv)[3][3]) {
  double c00 = m[1][1] * m[2][2] - m[1][2] * m[2][1];
  double c01 = m[0][2] * m[2][1] - m[0][1] * m[2][2];
  double c02 = m[0][1] * m[1][2] - m[0][2] * m[1][1];
  double c10 = m[1][2] * m[2][0] - m[1][0] * m[2][2];
  double c11 = m[0][0] * m[2][2] - m[0][2] * m[2][0];
  double c12 = m[0][2] * m[1][0] - m[0][0] * m[1][2];
  double c20 = m[1][0] * m[2][1] - m[1][1] * m[2][0];
  double c21 = m[0][1] * m[2][0] - m[0][0] * m[2][1];
  double c22 = m[0][0] * m[1][1] - m[0][1] * m[1][0];
  double det = m[0][0] * c00 + m[0][1] * c10 + m[0][2] * c20;
  double id = 1.0 / det;
  iv[0][0] = c00 * id; iv[0][1] = c01 * id; iv[0][2] = c02 * id;
  iv[1][0] = c10 * id; iv[1][1] = c11 * id; iv[1][2] = c12 * id;
  iv[2][0] = c20 * id; iv[2][1] = c21 * id; iv[2][2] = c22 * id;
  return det;
}

// J[i][j] = sum_a x_a,i dN_a/dxi_j at Gauss point g.
template <int R, int NN>
__device__ __forceinline__ void jacobian(const double (&x)[NN][3], int g, double (&J)[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < NN; ++a) s = fma(x[a][i], c_dN[R][g][a][j], s);
      J[i][j] = s;
    }
}

// Physical gradients of the shape functions at Gauss point g; returns det J.
template <int R, int NN>
__device__ __forceinline__ double shape_grads(const double (&x)[NN][3], int g, double (&dNdx)[NN][3]) {
  double J[3][3], iv[3][3];
  if constexpr (RuleT<R>::TET) {
    // affine: J columns are the edges x_{j+1}-x_0; dN/dxi known in closed form
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) J[i][j] = x[j + 1][i] - x[0][i];
    double det = inv3(J, iv);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      dNdx[1][k] = iv[0][k];
      dNdx[2][k] = iv[1][k];
      dNdx[3][k] = iv[2][k];
      dNdx[0][k] = -(iv[0][k] + iv[1][k] + iv[2][k]);
    }
    return det;
  } else {
    jacobian<R, NN>(x, g, J);
    double det = inv3(J, iv);
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        dNdx[a][k] = c_dN[R][g][a][0] * iv[0][k] + c_dN[R][g][a][1] * iv[1][k] + c_dN[R][g][a][2] * iv[2][k];
    return det;
  }
}

// |det J| at Gauss point g with the reference's formulas (edge matrix for
// tets, assembly.py:131-133 / :276-277; trilinear J for others, :135-139).
template <int R, int NN>
__device__ __forceinline__ double abs_det(const double (&x)[NN][3], int g) {
  double J[3][3];
  if constexpr (RuleT<R>::TET) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) J[r][c] = x[r + 1][c] - x[0][c];
  } else {
    jacobian<R, NN>(x, g, J);
  }
  return fabs(det3(J));
}

// Vreman eddy viscosity: mu_t = rho c sqrt(B_beta / a:a),
// alpha_ij = du_j/dx_i = G_ji, beta = Delta^2 alpha^T alpha.
__device__ __forceinline__ double vreman(const double (&G)[3][3], double delta2, double rho, double c) {
  // S = alpha^T alpha (symmetric, S_ij = sum_m G_im G_jm); beta = Delta^2 S, so
  // B_beta = Delta^4 * (sum of the principal 2x2 minors of S) and a:a = tr S.
  double S[6];  // 00 11 22 01 02 12
  const int I[6] = {0, 1, 2, 0, 0, 1}, J[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double t = 0.0;
#pragma unroll
    for (int m = 0; m < 3; ++m) t = fma(G[I[k]][m], G[J[k]][m], t);
    S[k] = t;
  }
  const double aa = S[0] + S[1] + S[2];
  double Bm = S[0] * S[1] - S[3] * S[3] + S[0] * S[2] - S[4] * S[4] + S[1] * S[2] - S[5] * S[5];
  // sqrt(B / a:a) as B * rsqrt(B * a:a): one reciprocal square root instead
  // of an fp64 division and a square root (a few ulps from the quotient form)
  return (aa > 1e-30 && Bm > 0.0) ? rho * c * delta2 * (Bm * rsqrt(Bm * aa)) : 0.0;
}

// ---------------------------------------------------------------------------
// Scatter of per-element contributions r[NN][NC] to a [n][STRIDE] node array.
// ---------------------------------------------------------------------------
template <int NN, int NC, int STRIDE>
__device__ __forceinline__ void scatter_direct(double* __restrict__ out, const int (&nd)[NN],
                                               const double (&r)[NN][NC]) {
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int c = 0; c < NC; ++c) red_add(out + (int64_t)nd[a] * STRIDE + c, r[a][c]);
}

// Windowed scatter: every thread of the block must call it (contains
// __syncthreads); invalid lanes pass zeros.
// Per-thread window context, loaded once at kernel entry so that every
// independent global load of the three window phases (node ids and slot
// ranges of the thread's window node, the element's local node indices) is
// in flight together instead of one latency per phase.  Thread t owns window
// node b0 + t (and b0 + t + BLOCK, ... when a window exceeds the block).
template <int NN>
struct WinCtx {
  int64_t b0, b1;
  int node, s0, s1;
  bool has;
  int l[NN];
};

template <int NN, int BLOCK>
__device__ __forceinline__ WinCtx<NN> win_begin(const WinP& w, int64_t e, int64_t n_elem) {
  WinCtx<NN> x;
  x.b0 = __ldg(w.blk_ptr + blockIdx.x);
  x.b1 = __ldg(w.blk_ptr + blockIdx.x + 1);
  const int64_t k = x.b0 + threadIdx.x;
  x.has = k < x.b1;
  x.node = x.has ? __ldg(w.wnode + k) : 0;
  x.s0 = x.has ? __ldg(w.wptr + k) : 0;
  x.s1 = x.has ? __ldg(w.wptr + k + 1) : 0;
  if (e < n_elem) {
    const uint16_t* p = w.loc + e * NN;
    if constexpr (NN == 4) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
      x.l[0] = v.x & 0xffff; x.l[1] = v.x >> 16; x.l[2] = v.y & 0xffff; x.l[3] = v.y >> 16;
    } else {
#pragma unroll
      for (int a = 0; a < NN; ++a) x.l[a] = __ldg(p + a);
    }
  } else {
#pragma unroll
    for (int a = 0; a < NN; ++a) x.l[a] = 0;
  }
  return x;
}

// Phase C: element contributions -> shared slots SoA [NC][NN][BLOCK]
// (conflict-free), then the owner thread of each window node sums its slots
// in list order and issues one fp64 reduction per component.
template <int NN, int NC, int STRIDE, int BLOCK>
__device__ __forceinline__ void win_scatter(double* __restrict__ out, const WinP& w, const WinCtx<NN>& cx,
                                            double* slots, const double (&r)[NN][NC]) {
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int c = 0; c < NC; ++c) slots[(c * NN + a) * BLOCK + threadIdx.x] = r[a][c];
  __syncthreads();
  auto reduce = [&](int node, int s0, int s1) {
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    int s = s0;
    for (; s + 4 <= s1; s += 4) {
      int sl[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) sl[u] = __ldg(w.wslot + s + u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] += slots[c * NN * BLOCK + sl[u]];
      }
    }
    for (; s < s1; ++s) {
      const int sl = __ldg(w.wslot + s);
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] += slots[c * NN * BLOCK + sl];
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) red_add(out + (int64_t)node * STRIDE + c, acc[c]);
  };
  if (cx.has) reduce(cx.node, cx.s0, cx.s1);
  for (int64_t k = cx.b0 + threadIdx.x + BLOCK; k < cx.b1; k += BLOCK)
    reduce(__ldg(w.wnode + k), __ldg(w.wptr + k), __ldg(w.wptr + k + 1));
}

// Phase A: the block's unique nodes -> shared memory SoA [NV][wmax]
// (x, y, z, then NV-3 field components).
template <int NN, int NV, int BLOCK>
__device__ __forceinline__ void win_fill(const CatP& c, const WinP& w, const WinCtx<NN>& cx,
                                         const double* __restrict__ f, int fstride, double* nodes) {
  const int W = w.wmax;
  auto put = [&](int l, int64_t node) {
    const d4 X = ld4_nc(c.coords + 4 * node);
    double fv[3] = {0.0, 0.0, 0.0};
    if constexpr (NV == 6) {
      const d4 U = ld4_nc(f + 4 * node);
      fv[0] = U.x; fv[1] = U.y; fv[2] = U.z;
    } else if constexpr (NV == 4) {
      fv[0] = __ldg(f + node * fstride);
    }
    nodes[l] = X.x;
    nodes[W + l] = X.y;
    nodes[2 * W + l] = X.z;
#pragma unroll
    for (int q = 0; q < NV - 3; ++q) nodes[(3 + q) * W + l] = fv[q];
  };
  if (cx.has) put(threadIdx.x, cx.node);
  for (int64_t k = cx.b0 + threadIdx.x + BLOCK; k < cx.b1; k += BLOCK) put((int)(k - cx.b0), __ldg(w.wnode + k));
  __syncthreads();
}

// Phase B: element nodes from the window.
template <int NN, int NV>
__device__ __forceinline__ void win_element(const WinP& w, const WinCtx<NN>& cx, const double* nodes,
                                            double (&x)[NN][3], double (&f)[NN][NV == 6 ? 3 : 1]) {
  const int W = w.wmax;
#pragma unroll
  for (int a = 0; a < NN; ++a) {
    const int l = cx.l[a];
    x[a][0] = nodes[l];
    x[a][1] = nodes[W + l];
    x[a][2] = nodes[2 * W + l];
    if constexpr (NV == 6) {
      f[a][0] = nodes[3 * W + l];
      f[a][1] = nodes[4 * W + l];
      f[a][2] = nodes[5 * W + l];
    } else {
      f[a][0] = nodes[3 * W + l];
    }
  }
}

// (the pipelined engine needs the element bodies below; see after K6)

// ---------------------------------------------------------------------------
// K1: mass matrix / Jacobians / lumped mass
// ---------------------------------------------------------------------------
template <int R>
__global__ void k_mass(CatP c, double* __restrict__ ae, double* __restrict__ jdet, double* __restrict__ ml) {
  constexpr int NN = RuleT<R>::NN, NG = RuleT<R>::NG;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= c.n) return;
  int nd[NN];
  load_conn<NN>(c.conn, e, nd);
  double x[NN][3];
  load_coords<NN>(c, nd, x);
  double m[NN][NN];
#pragma unroll
  for (int i = 0; i < NN; ++i)
#pragma unroll
    for (int j = 0; j < NN; ++j) m[i][j] = 0.0;
  double dtet = RuleT<R>::TET ? abs_det<R, NN>(x, 0) : 0.0;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const double J = RuleT<R>::TET ? dtet : abs_det<R, NN>(x, g);
    if (jdet) jdet[e * NG + g] = J;
    const double jw = J * c_w[R][g];
#pragma unroll
    for (int i = 0; i < NN; ++i)
#pragma unroll
      for (int j = 0; j < NN; ++j) m[i][j] += jw * (c_N[R][g][i] * c_N[R][g][j]);
  }
  if (ae) {
    double* o = ae + e * NN * NN;
#pragma unroll
    for (int i = 0; i < NN; ++i)
#pragma unroll
      for (int j = 0; j < NN; ++j) o[i * NN + j] = m[i][j];
  }
  if (ml) {
#pragma unroll
    for (int i = 0; i < NN; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NN; ++j) s += m[i][j];
      red_add(ml + nd[i], s);
    }
  }
}

// ---------------------------------------------------------------------------
// K2: momentum RHS  R_a -= int rho N_a [2 eps(u) u + div(u) u] + 2 (mu+mu_t) eps : grad N_a
// ---------------------------------------------------------------------------
// d2: the element's precomputed Delta^2 (< 0: computed here from V_e)
template <int R, int NN, class Emit>
__device__ __forceinline__ void momentum_element(const ab_phys ph, const double (&x)[NN][3], const double (&u)[NN][3],
                                                 double d2, Emit emit) {
  constexpr int NG = RuleT<R>::NG;
  if constexpr (RuleT<R>::TET) {
    // Affine element: geometry, grad u and mu_t are constant, and the
    // convective Gauss sum is  sum_g w_g N_a(g) A u_g = A sum_b M_ab u_b with
    // the reference-element mass table M (c_M); each node's contribution is
    // emitted as soon as it is formed (no per-node accumulator registers).
    double dNdx[NN][3];
    const double det = shape_grads<R, NN>(x, 0, dNdx);
    const double adet = fabs(det);
    double wsum = 0.0;
#pragma unroll
    for (int g = 0; g < NG; ++g) wsum += c_w[R][g];
    const double vol = adet * wsum;
    double G[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < NN; ++a) s = fma(u[a][i], dNdx[a][j], s);
        G[i][j] = s;
      }
    const double div = G[0][0] + G[1][1] + G[2][2];
    double mu_eff = ph.mu;
    if (ph.c_vreman > 0.0) {
      if (d2 < 0.0) {
        const double d = cbrt(vol);
        d2 = d * d;
      }
      mu_eff += vreman(G, d2, ph.rho, ph.c_vreman);
    }
    // Symmetric A' = rho |J| (G + G^T + div I) and sigma = 2 mu_eff eps V,
    // 6 unique entries each (index k: 00 11 22 01 02 12).
    const double rdet = ph.rho * adet, mv = mu_eff * vol;
    double Ap[6], sg[6];
    {
      const double s00 = G[0][0] + G[0][0], s11 = G[1][1] + G[1][1], s22 = G[2][2] + G[2][2];
      const double s01 = G[0][1] + G[1][0], s02 = G[0][2] + G[2][0], s12 = G[1][2] + G[2][1];
      Ap[0] = rdet * (s00 + div); Ap[1] = rdet * (s11 + div); Ap[2] = rdet * (s22 + div);
      Ap[3] = rdet * s01; Ap[4] = rdet * s02; Ap[5] = rdet * s12;
      sg[0] = mv * s00; sg[1] = mv * s11; sg[2] = mv * s22;
      sg[3] = mv * s01; sg[4] = mv * s02; sg[5] = mv * s12;
    }
    // m_a = sum_b M_ab u_b; for the exactly integrated P1 mass (tet4),
    // M_ab = (1 + delta_ab) / 120, i.e. m_a = (u_a + sum_b u_b) / 120.
    double U[3] = {0.0, 0.0, 0.0};
    if constexpr (R == AB_RULE_TET4) {
#pragma unroll
      for (int b = 0; b < NN; ++b)
#pragma unroll
        for (int i = 0; i < 3; ++i) U[i] += u[b][i];
    }
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      double m[3];
      if constexpr (R == AB_RULE_TET4) {
#pragma unroll
        for (int i = 0; i < 3; ++i) m[i] = (u[a][i] + U[i]) * (1.0 / 120.0);
      } else {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double t = 0.0;
#pragma unroll
          for (int b = 0; b < NN; ++b) t = fma(c_M[R][a][b], u[b][i], t);
          m[i] = t;
        }
      }
      const double* d = dNdx[a];
      double r[3];
      r[0] = -(Ap[0] * m[0] + Ap[3] * m[1] + Ap[4] * m[2] + sg[0] * d[0] + sg[3] * d[1] + sg[4] * d[2]);
      r[1] = -(Ap[3] * m[0] + Ap[1] * m[1] + Ap[5] * m[2] + sg[3] * d[0] + sg[1] * d[1] + sg[5] * d[2]);
      r[2] = -(Ap[4] * m[0] + Ap[5] * m[1] + Ap[2] * m[2] + sg[4] * d[0] + sg[5] * d[1] + sg[2] * d[2]);
      emit(a, r);
    }
  } else {
    double r[NN][3];
#pragma unroll
    for (int a = 0; a < NN; ++a) r[a][0] = r[a][1] = r[a][2] = 0.0;
    double delta2 = d2;
    if (ph.c_vreman > 0.0 && d2 < 0.0) {
      double vol = 0.0;
#pragma unroll
      for (int g = 0; g < NG; ++g) vol += abs_det<R, NN>(x, g) * c_w[R][g];
      const double d = cbrt(vol);
      delta2 = d * d;
    }
#pragma unroll 1
    for (int g = 0; g < NG; ++g) {
      double dNdx[NN][3];
      const double dV = fabs(shape_grads<R, NN>(x, g, dNdx)) * c_w[R][g];
      double ug[3] = {0.0, 0.0, 0.0}, G[3][3];
#pragma unroll
      for (int b = 0; b < NN; ++b)
#pragma unroll
        for (int i = 0; i < 3; ++i) ug[i] = fma(c_N[R][g][b], u[b][i], ug[i]);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < NN; ++a) s = fma(u[a][i], dNdx[a][j], s);
          G[i][j] = s;
        }
      const double div = G[0][0] + G[1][1] + G[2][2];
      double mu_eff = ph.mu;
      if (ph.c_vreman > 0.0) mu_eff += vreman(G, delta2, ph.rho, ph.c_vreman);
      double cv[3], sg[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double s = div * ug[i];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double e2 = G[i][j] + G[j][i];
          s = fma(e2, ug[j], s);
          sg[i][j] = mu_eff * e2 * dV;
        }
        cv[i] = ph.rho * dV * s;
      }
#pragma unroll
      for (int a = 0; a < NN; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
          r[a][i] -= c_N[R][g][a] * cv[i] + sg[i][0] * dNdx[a][0] + sg[i][1] * dNdx[a][1] + sg[i][2] * dNdx[a][2];
    }
#pragma unroll
    for (int a = 0; a < NN; ++a) emit(a, r[a]);
  }
}

template <int R, int BLOCK, bool WIN>
__global__ void __launch_bounds__(BLOCK) k_momentum(CatP c, ab_phys ph, const double* __restrict__ u4,
                                                    double* __restrict__ rhs4, WinP w) {
  constexpr int NN = RuleT<R>::NN;
  extern __shared__ double sm[];
  const int64_t e = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  WinCtx<NN> cx;
  if constexpr (WIN) {
    cx = win_begin<NN, BLOCK>(w, e, c.n);
    win_fill<NN, 6, BLOCK>(c, w, cx, u4, 4, sm);
  }
  double r[NN][3];
#pragma unroll
  for (int a = 0; a < NN; ++a) r[a][0] = r[a][1] = r[a][2] = 0.0;
  if (e < c.n) {
    double x[NN][3], u[NN][3];
    if constexpr (WIN) {
      win_element<NN, 6>(w, cx, sm, x, u);
      unwrap<NN>(c, x);
      momentum_element<R, NN>(ph, x, u, c.delta2 ? __ldg(c.delta2 + e) : -1.0, [&](int a, const double (&v)[3]) {
        r[a][0] = v[0]; r[a][1] = v[1]; r[a][2] = v[2];
      });
    } else {
      int nd[NN];
      load_conn<NN>(c.conn, e, nd);
      load_coords<NN>(c, nd, x);
      load_vec<NN>(u4, nd, u);
      momentum_element<R, NN>(ph, x, u, c.delta2 ? __ldg(c.delta2 + e) : -1.0, [&](int a, const double (&v)[3]) {
#pragma unroll
        for (int i = 0; i < 3; ++i) red_add(rhs4 + 4 * (int64_t)nd[a] + i, v[i]);
      });
    }
  }
  if constexpr (WIN) win_scatter<NN, 3, 4, BLOCK>(rhs4, w, cx, sm + (size_t)w.wmax * 6, r);
}

// ---------------------------------------------------------------------------
// K4 divergence / K6 gradient  (int N_a div u, int N_a grad p)
// ---------------------------------------------------------------------------
template <int R, int NN>
__device__ __forceinline__ void divergence_element(double scale, const double (&x)[NN][3], const double (&u)[NN][3],
                                                   double (&r)[NN][1]) {
  constexpr int NG = RuleT<R>::NG;
#pragma unroll 1
  for (int g = 0; g < (RuleT<R>::TET ? 1 : NG); ++g) {
    double dNdx[NN][3];
    const double adet = fabs(shape_grads<R, NN>(x, g, dNdx));
    double div = 0.0;
#pragma unroll
    for (int a = 0; a < NN; ++a) div += u[a][0] * dNdx[a][0] + u[a][1] * dNdx[a][1] + u[a][2] * dNdx[a][2];
    if constexpr (RuleT<R>::TET) {
#pragma unroll
      for (int gg = 0; gg < NG; ++gg) {
        const double f = scale * adet * c_w[R][gg] * div;
#pragma unroll
        for (int a = 0; a < NN; ++a) r[a][0] = fma(c_N[R][gg][a], f, r[a][0]);
      }
    } else {
      const double f = scale * adet * c_w[R][g] * div;
#pragma unroll
      for (int a = 0; a < NN; ++a) r[a][0] = fma(c_N[R][g][a], f, r[a][0]);
    }
  }
}

template <int R, int NN>
__device__ __forceinline__ void gradient_element(double scale, const double (&x)[NN][3], const double (&pe)[NN][1],
                                                 double (&r)[NN][3]) {
  constexpr int NG = RuleT<R>::NG;
#pragma unroll 1
  for (int g = 0; g < (RuleT<R>::TET ? 1 : NG); ++g) {
    double dNdx[NN][3];
    const double adet = fabs(shape_grads<R, NN>(x, g, dNdx));
    double gp[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int k = 0; k < 3; ++k) gp[k] = fma(pe[a][0], dNdx[a][k], gp[k]);
#pragma unroll
    for (int gg = 0; gg < (RuleT<R>::TET ? NG : 1); ++gg) {
      const int gi = RuleT<R>::TET ? gg : g;
      const double f = scale * adet * c_w[R][gi];
#pragma unroll
      for (int a = 0; a < NN; ++a) {
        const double fn = f * c_N[R][gi][a];
#pragma unroll
        for (int k = 0; k < 3; ++k) r[a][k] = fma(fn, gp[k], r[a][k]);
      }
    }
  }
}

template <int R, int BLOCK, bool WIN>
__global__ void __launch_bounds__(BLOCK) k_divergence(CatP c, const double* __restrict__ u4, double scale,
                                                      double* __restrict__ out, WinP w) {
  constexpr int NN = RuleT<R>::NN;
  extern __shared__ double sm[];
  const int64_t e = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  WinCtx<NN> cx;
  if constexpr (WIN) {
    cx = win_begin<NN, BLOCK>(w, e, c.n);
    win_fill<NN, 6, BLOCK>(c, w, cx, u4, 4, sm);
  }
  double r[NN][1];
#pragma unroll
  for (int a = 0; a < NN; ++a) r[a][0] = 0.0;
  if (e < c.n) {
    double x[NN][3], u[NN][3];
    if constexpr (WIN) {
      win_element<NN, 6>(w, cx, sm, x, u);
      unwrap<NN>(c, x);
      divergence_element<R, NN>(scale, x, u, r);
    } else {
      int nd[NN];
      load_conn<NN>(c.conn, e, nd);
      load_coords<NN>(c, nd, x);
      load_vec<NN>(u4, nd, u);
      divergence_element<R, NN>(scale, x, u, r);
      scatter_direct<NN, 1, 1>(out, nd, r);
    }
  }
  if constexpr (WIN) win_scatter<NN, 1, 1, BLOCK>(out, w, cx, sm + (size_t)w.wmax * 6, r);
}

template <int R, int BLOCK, bool WIN>
__global__ void __launch_bounds__(BLOCK) k_gradient(CatP c, const double* __restrict__ p, double scale,
                                                    double* __restrict__ out4, WinP w) {
  constexpr int NN = RuleT<R>::NN;
  extern __shared__ double sm[];
  const int64_t e = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  WinCtx<NN> cx;
  if constexpr (WIN) {
    cx = win_begin<NN, BLOCK>(w, e, c.n);
    win_fill<NN, 4, BLOCK>(c, w, cx, p, 1, sm);
  }
  double r[NN][3];
#pragma unroll
  for (int a = 0; a < NN; ++a) r[a][0] = r[a][1] = r[a][2] = 0.0;
  if (e < c.n) {
    double x[NN][3], pe[NN][1];
    if constexpr (WIN) {
      win_element<NN, 4>(w, cx, sm, x, pe);
      unwrap<NN>(c, x);
      gradient_element<R, NN>(scale, x, pe, r);
    } else {
      int nd[NN];
      load_conn<NN>(c.conn, e, nd);
      load_coords<NN>(c, nd, x);
#pragma unroll
      for (int a = 0; a < NN; ++a) pe[a][0] = __ldg(p + nd[a]);
      gradient_element<R, NN>(scale, x, pe, r);
      scatter_direct<NN, 3, 4>(out4, nd, r);
    }
  }
  if constexpr (WIN) win_scatter<NN, 3, 4, BLOCK>(out4, w, cx, sm + (size_t)w.wmax * 4, r);
}


// ---------------------------------------------------------------------------
// Pipelined windowed element kernels.  Persistent CTAs walk the element
// blocks b = blockIdx.x, +gridDim.x, ... with a two-stage shared-memory
// pipeline:
//   * the block's window metadata (node ids, slot ranges, slot lists, the
//     elements' window-local indices) is contiguous in HBM and arrives by
//     bulk async copies (cp.async.bulk -> UBLKCP, mbarrier completion), two
//     blocks ahead;
//   * the window's node data (coordinates + field) is gathered with
//     cp.async (LDGSTS) one block ahead, straight into SoA shared memory;
//   * the current block is computed from shared memory and reduced per
//     window node into global memory (one fp64 RED per node and component).
// Latency of both loads is therefore hidden behind the FP64 work of the
// previous block instead of serialising the phases of every block.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "PW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra PW_%=;\n}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Byte range [lo, hi) of a global array, widened to 16-byte alignment for a
// bulk copy; returns the element offset of `lo` inside the copied chunk.
struct Chunk { const char* src; uint32_t bytes; uint32_t skip; };
__device__ __forceinline__ Chunk chunk16(const void* base, int64_t lo_elem, int64_t hi_elem, int es) {
  const uint64_t lo = (uint64_t)base + (uint64_t)lo_elem * es;
  const uint64_t hi = (uint64_t)base + (uint64_t)hi_elem * es;
  const uint64_t a = lo & ~(uint64_t)15;
  const uint64_t b = (hi + 15) & ~(uint64_t)15;
  return Chunk{reinterpret_cast<const char*>(a), (uint32_t)(b - a), (uint32_t)((lo - a) / es)};
}

// Shared-memory layout: 3 metadata stages (the descriptor of the CTA's next
// block, window node ids, sorted references, element window indices), 2
// node-data stages, 1 slot buffer.
template <int NN, int NV, int BLOCK>
struct PipeSmem {
  static __host__ __device__ size_t wcap(int wmax) { return ((size_t)wmax + 8 + 3) & ~(size_t)3; }
  static __host__ __device__ size_t meta_bytes(int wmax) {
    return 16 + wcap(wmax) * 4 + (size_t)BLOCK * NN * 4 + ((size_t)BLOCK * NN + 16) * 2;
  }
  static __host__ __device__ size_t node_bytes(int wmax) { return (size_t)NV * wmax * 8; }
  static __host__ __device__ size_t slot_bytes() { return sizeof(double) * 3 * NN * BLOCK; }
  static __host__ __device__ size_t total(int wmax) {
    return 3 * meta_bytes(wmax) + 2 * node_bytes(wmax) + slot_bytes();
  }
};

struct MetaPtr {
  int4* next;  // descriptor of the block after this one (bulk-copied with it)
  int32_t* wnode;
  uint32_t* wref;
  uint16_t* loc;
};

template <int NN, int NV, int BLOCK>
__device__ __forceinline__ MetaPtr meta_ptr(unsigned char* smem, int wmax, int q) {
  using L = PipeSmem<NN, NV, BLOCK>;
  unsigned char* base = smem + (size_t)q * L::meta_bytes(wmax);
  const size_t wn = L::wcap(wmax) * 4, wr = (size_t)BLOCK * NN * 4;
  MetaPtr m;
  m.next = reinterpret_cast<int4*>(base);
  base += 16;
  m.wnode = reinterpret_cast<int32_t*>(base);
  m.wref = reinterpret_cast<uint32_t*>(base + wn);
  m.loc = reinterpret_cast<uint16_t*>(base + wn + wr);
  return m;
}

// Offsets of a block's data inside its (16-byte widened) metadata chunks.
struct BlockView {
  int nw, skip_wnode;
};
__device__ __forceinline__ BlockView block_view(const WinP& w, int4 d) {
  BlockView v;
  v.nw = d.y - d.x;
  v.skip_wnode = (int)((((uint64_t)w.wnode + (uint64_t)d.x * 4) & 15) / 4);
  return v;
}

// Elected thread: bulk-copy the metadata of element block b, plus the
// descriptor of block bnext (the CTA's block after b; none if < 0), so no
// thread waits on a global descriptor load in the loop.
template <int NN>
__device__ __forceinline__ void issue_meta(const WinP& w, int64_t n_elem, int64_t b, int4 d, int64_t bnext,
                                           const MetaPtr& m, uint64_t* bar) {
  const int64_t e0 = b * w.block;
  const int64_t e1 = e0 + w.block < n_elem ? e0 + w.block : n_elem;
  const Chunk cw = chunk16(w.wnode, d.x, d.y, 4);
  const Chunk cr = chunk16(w.wref, e0 * NN, (e0 + w.block) * NN, 4);  // padded to whole blocks
  const Chunk cl = chunk16(w.loc, e0 * NN, e1 * NN, 2);
  mbar_arrive_tx(bar, cw.bytes + cr.bytes + cl.bytes + (bnext >= 0 ? 16u : 0u));
  if (bnext >= 0) bulk_copy(m.next, w.desc + bnext, 16, bar);
  bulk_copy(m.wnode, cw.src, cw.bytes, bar);
  bulk_copy(m.wref, cr.src, cr.bytes, bar);
  bulk_copy(m.loc, cl.src, cl.bytes, bar);
}

// All threads: cp.async gather of a block's window node data into shared
// memory as arrays of double2 pairs [NV/2][wmax] — (x,y),(z,u),(v,w) for
// NV = 6, (x,y),(z,p) for NV = 4 — so an element reads a node with NV/2
// 128-bit shared loads.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}

template <int NV, int BLOCK>
__device__ __forceinline__ void issue_nodes(const CatP& c, const double* __restrict__ f, int wmax, const MetaPtr& m,
                                            const BlockView& v, double* nodes) {
  double2* pr = reinterpret_cast<double2*>(nodes);
  for (int k = threadIdx.x; k < v.nw; k += BLOCK) {
    const int64_t node = m.wnode[v.skip_wnode + k];
    const double* xp = c.coords + 4 * node;
    cp_async16(pr + k, xp);                                  // (x, y)
    double* zu = reinterpret_cast<double*>(pr + wmax + k);   // (z, f0)
    cp_async8(zu, xp + 2);
    if constexpr (NV == 6) {
      const double* up = f + 4 * node;
      cp_async8(zu + 1, up);
      double* vw = reinterpret_cast<double*>(pr + 2 * wmax + k);  // (v, w)
      cp_async8(vw, up + 1);
      cp_async8(vw + 1, up + 2);
    } else {
      cp_async8(zu + 1, f + node);
    }
  }
  cp_async_commit();
}

enum { OP_MOMENTUM = 0, OP_DIVERGENCE = 1, OP_GRADIENT = 2 };

template <int R, int OP>
struct OpT;
template <int R> struct OpT<R, OP_MOMENTUM> { static constexpr int NV = 6, NC = 3, STRIDE = 4; };
template <int R> struct OpT<R, OP_DIVERGENCE> { static constexpr int NV = 6, NC = 1, STRIDE = 1; };
template <int R> struct OpT<R, OP_GRADIENT> { static constexpr int NV = 4, NC = 3, STRIDE = 4; };

#ifndef PIPE_OCC_K2
#define PIPE_OCC_K2 3  // register cap of the tet4 K2 (launch_bounds min CTAs); the compiler then uses 96 registers and 5 CTAs/SM are resident. C2 bench: 157.3 us vs 159.1 with the cap for 4 (94 regs)
#endif
#ifndef PIPE_D_BRANCHLESS
#define PIPE_D_BRANCHLESS 1
#endif
// minimum resident CTAs per SM requested from the register allocator
template <int R, int OP> struct PipeOcc { static constexpr int value = 1; };
template <> struct PipeOcc<AB_RULE_TET4, OP_MOMENTUM> { static constexpr int value = PIPE_OCC_K2; };

// Work sequence of a persistent CTA.  Atomic mode: blocks blockIdx.x,
// +gridDim.x, ... in SFC order.  Colour mode: the same walk inside each
// colour's slice of corder, colour after colour.  j = logical position
// (-1 = end), c = colour of that position (ncol at the end).
struct Pos {
  int64_t j;
  int c;
};
template <bool COL>
__device__ __forceinline__ Pos pos_first(const WinP& w, int64_t n_blocks) {
  Pos p{-1, 0};
  if constexpr (COL) {
    for (; p.c < w.ncol; ++p.c) {
      const int64_t j = __ldg(w.cptr + p.c) + blockIdx.x;
      if (j < __ldg(w.cptr + p.c + 1)) {
        p.j = j;
        return p;
      }
    }
  } else {
    if ((int64_t)blockIdx.x < n_blocks) p.j = blockIdx.x;
  }
  return p;
}
template <bool COL>
__device__ __forceinline__ Pos pos_next(const WinP& w, int64_t n_blocks, Pos p) {
  if (p.j < 0) return p;
  p.j += gridDim.x;
  if constexpr (COL) {
    while (p.j >= __ldg(w.cptr + p.c + 1)) {
      if (++p.c >= w.ncol) {
        p.j = -1;
        return p;
      }
      p.j = __ldg(w.cptr + p.c) + blockIdx.x;
    }
  } else {
    if (p.j >= n_blocks) p.j = -1;
  }
  return p;
}
template <bool COL>
__device__ __forceinline__ int64_t pos_block(const WinP& w, Pos p) {
  if constexpr (COL) return p.j >= 0 ? (int64_t)__ldg(w.corder + p.j) : -1;
  return p.j;
}

// Colour barrier: gbar[k] counts the CTAs that have finished colour k.  A
// CTA moving on from colour `done` to colour c announces done .. c-1 (one
// release-add each, in order), and before reducing into colour c it waits for
// gbar[c-1] == gridDim.x: every CTA has announced c-1, hence finished every
// colour <= c-1.  (One counter summed over all colours would let CTAs that
// skip ahead several colours satisfy the target for CTAs still behind.)
__device__ __forceinline__ void colour_arrive(unsigned* gbar, int from, int to) {
  for (int k = from; k < to; ++k) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar + k) : "memory");
}
__device__ __forceinline__ void colour_wait(const unsigned* gbar, int c) {
  if (c == 0) return;
  unsigned v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gbar + c - 1) : "memory");
  } while (v < gridDim.x);
}

// Colour-mode scratch behind the slot buffer: each thread's first window
// index (bit 31: the thread holds a single run), last window index and first
// run's partial sum.
template <int NC, int BLOCK>
struct ColSmem {
  static __host__ __device__ size_t bytes() { return (size_t)BLOCK * (8 + 8 * NC); }
};

// Persistent pipelined element kernel.  Iteration i (element block b_i):
//   A  wait metadata(b_{i+1}) [mbarrier], cp.async node data(b_{i+1})
//   B  wait node data(b_i) [cp.async group], __syncthreads; thread 0 then
//      bulk-copies metadata(b_{i+2}) into the stage of b_{i-1} (free: every
//      thread finished b_{i-1} before reaching this barrier)
//   C  elements of b_i -> shared slots, __syncthreads
//   D  window-node reductions of b_i -> global fp64 REDs
// Three metadata stages and two node stages make every buffer reuse safe
// with two CTA barriers per block.
// COL (mesh colouring, deterministic): before phase D of a block of colour c
// the CTA has announced every colour < c as finished and waits until all
// CTAs have (colour_arrive / colour_wait: one counter per colour); phase D
// then forms each window node's total in one thread (the references in
// sorted order, runs crossing lanes summed by the lane where they start) and
// issues ONE fp64 reduction per node: no two blocks of a colour share a
// node and the colours are ordered by the barrier (release/acquire, so the
// reductions of colour c happen before those of c+1 in every node's
// coherence order), hence every node's sum has a fixed order and the result
// is bitwise reproducible without paying for a read-add-write round trip.
// The prefetch pipeline runs across colour boundaries (it only reads).
template <int R, int OP, int BLOCK, bool COL>
__global__ void __launch_bounds__(BLOCK, PipeOcc<R, OP>::value) k_pipe(CatP c, WinP w, ab_phys ph, double scale,
                                                                       const double* __restrict__ f,
                                                                       double* __restrict__ out, int64_t n_blocks) {
  constexpr int NN = RuleT<R>::NN;
  constexpr int NV = OpT<R, OP>::NV, NC = OpT<R, OP>::NC, STRIDE = OpT<R, OP>::STRIDE;
  using L = PipeSmem<NN, NV, BLOCK>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[3];
  const int wmax = w.wmax;
  double* nodes0 = reinterpret_cast<double*>(smem + 3 * L::meta_bytes(wmax));
  double* slots = reinterpret_cast<double*>(smem + 3 * L::meta_bytes(wmax) + 2 * L::node_bytes(wmax));
  Pos p0 = pos_first<COL>(w, n_blocks);
  int done = 0;  // COL: colours this CTA has announced as finished
  if (p0.j < 0) {
    if constexpr (COL) {
      if (threadIdx.x == 0) colour_arrive(w.gbar, 0, w.ncol);
    }
    return;
  }
  if (threadIdx.x == 0) {
    mbar_init1(&bars[0]);
    mbar_init1(&bars[1]);
    mbar_init1(&bars[2]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // positions, physical blocks and descriptors (16 B each) of the current
  // and the next two blocks
  // (atomic mode derives the next blocks from b0 where they are used, so
  // only colour mode carries them across iterations)
  const int64_t stride = gridDim.x;
  auto nxt = [&](int64_t b) -> int64_t { return (b >= 0 && b + stride < n_blocks) ? b + stride : (int64_t)-1; };
  Pos p1 = pos_next<COL>(w, n_blocks, p0);
  Pos p2 = pos_next<COL>(w, n_blocks, p1);
  int64_t b0 = pos_block<COL>(w, p0);
  int64_t cb1 = COL ? pos_block<COL>(w, p1) : -1, cb2 = COL ? pos_block<COL>(w, p2) : -1;
  // d0, d1: descriptors of the current and the next block; the one after
  // arrives with the next block's metadata (MetaPtr::next)
  int4 d0, d1;
  {
    const int64_t b1 = COL ? cb1 : nxt(b0), b2 = COL ? cb2 : nxt(b1);
    d0 = __ldg(w.desc + b0);
    d1 = b1 >= 0 ? __ldg(w.desc + b1) : d0;
    if (threadIdx.x == 0) {
      issue_meta<NN>(w, c.n, b0, d0, b1, meta_ptr<NN, NV, BLOCK>(smem, wmax, 0), &bars[0]);
      if (b1 >= 0) issue_meta<NN>(w, c.n, b1, d1, b2, meta_ptr<NN, NV, BLOCK>(smem, wmax, 1), &bars[1]);
    }
  }
  mbar_wait_parity(&bars[0], 0);
  issue_nodes<NV, BLOCK>(c, f, wmax, meta_ptr<NN, NV, BLOCK>(smem, wmax, 0), block_view(w, d0), nodes0);

  int it = 0;
  for (; b0 >= 0; ++it) {
    const int mq = it % 3, mq1 = (it + 1) % 3, mq2 = (it + 2) % 3;
    double* nodes_cur = nodes0 + (size_t)(it & 1) * NV * wmax;
    double* nodes_nxt = nodes0 + (size_t)((it + 1) & 1) * NV * wmax;
    const int64_t b1 = COL ? cb1 : nxt(b0);
    const int64_t b2 = COL ? cb2 : nxt(b1);
    Pos p3{-1, 0};
    if constexpr (COL) p3 = pos_next<COL>(w, n_blocks, p2);
    const int64_t b3 = COL ? pos_block<COL>(w, p3) : nxt(b2);
    int4 d2 = d0;
    // precomputed filter width of this thread's element: in flight across the waits below
    double d2e = -1.0;
    if constexpr (OP == OP_MOMENTUM) {
      const int64_t ee = b0 * BLOCK + threadIdx.x;
      if (c.delta2 && ee < c.n) d2e = __ldg(c.delta2 + ee);
    }
    // A: node data of the next block
    if (b1 >= 0) {
      mbar_wait_parity(&bars[mq1], (uint32_t)(((it + 1) / 3) & 1));
      const MetaPtr m1 = meta_ptr<NN, NV, BLOCK>(smem, wmax, mq1);
      if (b2 >= 0) d2 = *m1.next;
      issue_nodes<NV, BLOCK>(c, f, wmax, m1, block_view(w, d1), nodes_nxt);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // B
    bool col_wait = false;
    if (threadIdx.x == 0) {
      if (b2 >= 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_meta<NN>(w, c.n, b2, d2, b3, meta_ptr<NN, NV, BLOCK>(smem, wmax, mq2), &bars[mq2]);
      }
      if constexpr (COL) {
        // every thread's phase D of the previous block is behind barrier B
        if (p0.c > done) {
          colour_arrive(w.gbar, done, p0.c);
          done = p0.c;
          col_wait = true;
        }
      }
    }
    // C: elements of this block
    const MetaPtr mc = meta_ptr<NN, NV, BLOCK>(smem, wmax, mq);
    const BlockView vc = block_view(w, d0);
    const int64_t e = b0 * BLOCK + threadIdx.x;
    if (e < c.n) {
      double x[NN][3], fv[NN][NV == 6 ? 3 : 1];
      int li[NN];
      if constexpr (NN == 4) {
        const uint2 lv = *reinterpret_cast<const uint2*>(mc.loc + threadIdx.x * NN);
        li[0] = lv.x & 0xffff; li[1] = lv.x >> 16; li[2] = lv.y & 0xffff; li[3] = lv.y >> 16;
      } else {
#pragma unroll
        for (int a = 0; a < NN; ++a) li[a] = mc.loc[threadIdx.x * NN + a];
      }
      const double2* pr = reinterpret_cast<const double2*>(nodes_cur);
#pragma unroll
      for (int a = 0; a < NN; ++a) {
        const int l = li[a];
        const double2 xy = pr[l], zf = pr[wmax + l];
        x[a][0] = xy.x;
        x[a][1] = xy.y;
        x[a][2] = zf.x;
        fv[a][0] = zf.y;
        if constexpr (NV == 6) {
          const double2 vw = pr[2 * wmax + l];
          fv[a][1] = vw.x;
          fv[a][2] = vw.y;
        }
      }
      unwrap<NN>(c, x);
      if constexpr (OP == OP_MOMENTUM) {
        momentum_element<R, NN>(ph, x, fv, d2e, [&](int a, const double (&v)[3]) {
#pragma unroll
          for (int k = 0; k < 3; ++k) slots[(k * NN + a) * BLOCK + threadIdx.x] = v[k];
        });
      } else {
        double r[NN][NC];
#pragma unroll
        for (int a = 0; a < NN; ++a)
#pragma unroll
          for (int k = 0; k < NC; ++k) r[a][k] = 0.0;
        if constexpr (OP == OP_DIVERGENCE) divergence_element<R, NN>(scale, x, fv, r);
        if constexpr (OP == OP_GRADIENT) gradient_element<R, NN>(scale, x, fv, r);
#pragma unroll
        for (int a = 0; a < NN; ++a)
#pragma unroll
          for (int k = 0; k < NC; ++k) slots[(k * NN + a) * BLOCK + threadIdx.x] = r[a][k];
      }
    } else {
#pragma unroll
      for (int a = 0; a < NN; ++a)
#pragma unroll
        for (int k = 0; k < NC; ++k) slots[(k * NN + a) * BLOCK + threadIdx.x] = 0.0;
    }
    if constexpr (COL) {
      if (col_wait) colour_wait(w.gbar, p0.c);
    }
    __syncthreads();
    // D: thread t sums the block's sorted references t*NN .. t*NN+NN-1 (the
    // block*NN element-node references ordered by window node), one fp64
    // reduction per (thread, window node) piece: every thread busy, no
    // variable-length list walks.
    {
      uint32_t rr[NN];
      const uint32_t* wr = mc.wref + threadIdx.x * NN;
      if constexpr (NN == 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(wr);
        rr[0] = v.x; rr[1] = v.y; rr[2] = v.z; rr[3] = v.w;
      } else if constexpr (NN == 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(wr), u = *reinterpret_cast<const uint4*>(wr + 4);
        rr[0] = v.x; rr[1] = v.y; rr[2] = v.z; rr[3] = v.w; rr[4] = u.x; rr[5] = u.y; rr[6] = u.z; rr[7] = u.w;
      } else {
#pragma unroll
        for (int k = 0; k < NN; ++k) rr[k] = wr[k];
      }
      double vq[NN][NC];
#pragma unroll
      for (int k = 0; k < NN; ++k)
#pragma unroll
        for (int q = 0; q < NC; ++q) vq[k][q] = slots[q * NN * BLOCK + (rr[k] & 0xffffu)];
      // pieces: maximal runs of equal window index.  Middle pieces are
      // reduced at once; the first (H) and last (T) may continue in the
      // neighbouring lanes: a lane with >= 2 pieces hands H to the lane
      // before it when that lane's last piece is the same window node (one
      // shuffle level; longer chains keep one reduction per lane).
      auto red_node = [&](uint32_t lw, const double (&v)[NC]) {
        const int node = mc.wnode[vc.skip_wnode + lw];
#pragma unroll
        for (int q = 0; q < NC; ++q) red_add(out + (int64_t)node * STRIDE + q, v[q]);
      };
#if PIPE_D_BRANCHLESS
      if constexpr (!COL) {
        // Branch-free form: segmented running sums a[k] over the runs of equal
        // window index, the first run's end kf found by selects, one shuffle
        // level of hand-over as below; only the reductions are predicated.
        uint32_t wv[NN];
#pragma unroll
        for (int k = 0; k < NN; ++k) wv[k] = rr[k] >> 16;
        double a[NN][NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) a[0][q] = vq[0][q];
#pragma unroll
        for (int k = 1; k < NN; ++k) {
          const bool e = wv[k] == wv[k - 1];
#pragma unroll
          for (int q = 0; q < NC; ++q) a[k][q] = e ? a[k - 1][q] + vq[k][q] : vq[k][q];
        }
        bool end[NN];
#pragma unroll
        for (int k = 0; k < NN - 1; ++k) end[k] = wv[k + 1] != wv[k];
        end[NN - 1] = true;
        int kf = NN - 1;
        double H[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) H[q] = a[NN - 1][q];
#pragma unroll
        for (int k = NN - 2; k >= 0; --k)
          if (end[k]) {
            kf = k;
#pragma unroll
            for (int q = 0; q < NC; ++q) H[q] = a[k][q];
          }
        const bool two = kf < NN - 1;
        const uint32_t f = wv[0], l = wv[NN - 1];
        const int lane = threadIdx.x & 31;
        const uint32_t mine = f | (two ? 0x80000000u : 0u);
        const uint32_t nxt = __shfl_down_sync(0xffffffffu, mine, 1);
        const uint32_t prv = __shfl_up_sync(0xffffffffu, l, 1);
        double hn[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) hn[q] = __shfl_down_sync(0xffffffffu, H[q], 1);
        const bool recv = lane != 31 && (nxt >> 31) && (nxt & 0xffffu) == l && l != 0xffffu;
        const bool give = lane != 0 && two && prv == f && f != 0xffffu;
#pragma unroll
        for (int k = 0; k < NN - 1; ++k)
          if (end[k] && wv[k] != 0xffffu && !(k == kf && give)) red_node(wv[k], a[k]);
        if (l != 0xffffu) {
          double t[NC];
#pragma unroll
          for (int q = 0; q < NC; ++q) t[q] = recv ? a[NN - 1][q] + hn[q] : a[NN - 1][q];
          red_node(l, t);
        }
      } else
#endif
      {
      double acc[NC], H[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) acc[q] = H[q] = vq[0][q];
      uint32_t cur = rr[0] >> 16;
      int np = 1;
#pragma unroll
      for (int k = 1; k < NN; ++k) {
        const uint32_t lw = rr[k] >> 16;
        if (lw != cur) {
          if (np == 1) {
#pragma unroll
            for (int q = 0; q < NC; ++q) H[q] = acc[q];
          } else if (cur != 0xffffu) {
            red_node(cur, acc);
          }
          ++np;
#pragma unroll
          for (int q = 0; q < NC; ++q) acc[q] = vq[k][q];
          cur = lw;
        } else {
#pragma unroll
          for (int q = 0; q < NC; ++q) acc[q] += vq[k][q];
        }
      }
      const uint32_t f = rr[0] >> 16, l = cur;
      if constexpr (COL) {
        // runs crossing lanes: summed in lane order by the lane holding
        // their start (its last piece), from the heads published here
        uint32_t* s_first = reinterpret_cast<uint32_t*>(slots + 3 * NN * BLOCK);
        uint32_t* s_last = s_first + BLOCK;
        double* s_head = reinterpret_cast<double*>(s_last + BLOCK);
        const int t = threadIdx.x;
        s_first[t] = f | (np == 1 ? 0x80000000u : 0u);
        s_last[t] = l;
#pragma unroll
        for (int q = 0; q < NC; ++q) s_head[q * BLOCK + t] = np == 1 ? acc[q] : H[q];
        __syncthreads();
        const bool cont_prev = t > 0 && s_last[t - 1] == f;
        if (np >= 2 && !cont_prev && f != 0xffffu) red_node(f, H);
        if (l != 0xffffu && (np >= 2 || !cont_prev)) {
          for (int u = t + 1; u < BLOCK; ++u) {
            const uint32_t fu = s_first[u];
            if ((fu & 0xffffu) != l) break;
#pragma unroll
            for (int q = 0; q < NC; ++q) acc[q] += s_head[q * BLOCK + u];
            if (!(fu >> 31)) break;
          }
          red_node(l, acc);
        }
      } else {
        const int lane = threadIdx.x & 31;
        const uint32_t mine = f | (np >= 2 ? 0x80000000u : 0u);
        const uint32_t nxt = __shfl_down_sync(0xffffffffu, mine, 1);
        const uint32_t prv = __shfl_up_sync(0xffffffffu, l, 1);
        double hn[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) hn[q] = __shfl_down_sync(0xffffffffu, H[q], 1);
        const bool recv = lane != 31 && (nxt >> 31) && (nxt & 0xffffu) == l && l != 0xffffu;
        const bool give = lane != 0 && np >= 2 && prv == f && f != 0xffffu;
        if (np >= 2 && !give && f != 0xffffu) red_node(f, H);
        if (l != 0xffffu) {
          if (recv) {
#pragma unroll
            for (int q = 0; q < NC; ++q) acc[q] += hn[q];
          }
          red_node(l, acc);
        }
      }
      }
    }
    if constexpr (COL) {
      p0 = p1;
      p1 = p2;
      p2 = p3;
      cb1 = b2;
      cb2 = b3;
    }
    b0 = b1;
    d0 = d1;
    d1 = d2;
  }
  if constexpr (COL) {
    __syncthreads();  // this CTA's last phase D is issued
    if (threadIdx.x == 0) colour_arrive(w.gbar, done, w.ncol);
  }
}

// Launch shape of the most recent pipelined element kernel (diagnostics:
// tests check that the persistent CTAs walk several blocks each).
static thread_local int64_t g_pipe_grid = 0, g_pipe_blocks = 0;

template <int R, int OP, int BLOCK, bool COL>
static int launch_pipe_impl(const CatP& c, const WinP& w, const ab_phys& ph, double scale, const double* f,
                            double* out, cudaStream_t stream) {
  constexpr int NN = RuleT<R>::NN;
  constexpr int NV = OpT<R, OP>::NV;
  using L = PipeSmem<NN, NV, BLOCK>;
  if (!w.wref) return fail("pipelined element kernel: sorted window references not registered (ab_set_window_refs)");
  const size_t smem = L::total(w.wmax) + (COL ? ColSmem<3, BLOCK>::bytes() : 0);
  auto kern = k_pipe<R, OP, BLOCK, COL>;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail("pipelined element kernel: shared memory request rejected");
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BLOCK, smem);
  if (per_sm < 1) return fail("pipelined element kernel does not fit on an SM");
  const int64_t n_blocks = (c.n + BLOCK - 1) / BLOCK;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > n_blocks) grid = n_blocks;
  g_pipe_grid = grid;
  g_pipe_blocks = n_blocks;
  if (COL) {
    // every CTA must be resident at once (colour barrier): grid <= sms * per_sm
    if (!w.gbar || !w.cptr || w.ncol < 1) return fail("k_pipe colour mode: colours not registered");
    static const bool split = getenv("AB_COLOUR_SPLIT") != nullptr;  // lab: one launch per colour
    if (split) {
      for (int cc = 0; cc < w.ncol; ++cc) {
        WinP w1 = w;
        w1.cptr = w.cptr + cc;
        w1.ncol = 1;
        kern<<<(unsigned)grid, BLOCK, smem, stream>>>(c, w1, ph, scale, f, out, n_blocks);
        if (int rc = check_launch("k_pipe")) return rc;
      }
      return AB_OK;
    }
    if (cudaMemsetAsync(w.gbar, 0, sizeof(unsigned) * w.ncol, stream) != cudaSuccess)
      return fail("k_pipe colour mode: barrier reset failed");
  }
  kern<<<(unsigned)grid, BLOCK, smem, stream>>>(c, w, ph, scale, f, out, n_blocks);
  return check_launch("k_pipe");
}

template <int R, int OP, int BLOCK>
static int launch_pipe(const CatP& c, const WinP& w, const ab_phys& ph, double scale, const double* f, double* out,
                       cudaStream_t stream) {
  if (w.corder) return launch_pipe_impl<R, OP, BLOCK, true>(c, w, ph, scale, f, out, stream);
  return launch_pipe_impl<R, OP, BLOCK, false>(c, w, ph, scale, f, out, stream);
}
// ---------------------------------------------------------------------------
// Vreman filter width Delta^2 = V_e^(2/3) per element (setup): the same
// operations as momentum_element's on-the-fly value, so K2 gives identical
// results with or without it, and K2 skips the fp64 cbrt.
// ---------------------------------------------------------------------------
template <int R>
__global__ void k_filter_width(CatP c, double* __restrict__ out) {
  constexpr int NN = RuleT<R>::NN, NG = RuleT<R>::NG;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= c.n) return;
  int nd[NN];
  load_conn<NN>(c.conn, e, nd);
  double x[NN][3];
  load_coords<NN>(c, nd, x);
  unwrap<NN>(c, x);
  double vol = 0.0;
  if constexpr (RuleT<R>::TET) {
    double dNdx[NN][3];
    const double adet = fabs(shape_grads<R, NN>(x, 0, dNdx));
    double wsum = 0.0;
#pragma unroll
    for (int g = 0; g < NG; ++g) wsum += c_w[R][g];
    vol = adet * wsum;
  } else {
#pragma unroll
    for (int g = 0; g < NG; ++g) vol += abs_det<R, NN>(x, g) * c_w[R][g];
  }
  const double d = cbrt(vol);
  out[e] = d * d;
}

// ---------------------------------------------------------------------------
// Laplacian values into a CSR pattern (setup)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t csr_find(const int64_t* __restrict__ rp, const int32_t* __restrict__ cols, int row,
                                            int col) {
  int64_t lo = rp[row], hi = rp[row + 1] - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) >> 1;
    int v = cols[mid];
    if (v == col) return mid;
    if (v < col) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

template <int R>
__global__ void k_laplacian(CatP c, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                            double* __restrict__ vals) {
  constexpr int NN = RuleT<R>::NN, NG = RuleT<R>::NG;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= c.n) return;
  int nd[NN];
  load_conn<NN>(c.conn, e, nd);
  double x[NN][3];
  load_coords<NN>(c, nd, x);
  double le[NN][NN];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) le[a][b] = 0.0;
#pragma unroll 1
  for (int g = 0; g < (RuleT<R>::TET ? 1 : NG); ++g) {
    double dNdx[NN][3];
    double dV = fabs(shape_grads<R, NN>(x, g, dNdx));
    if constexpr (RuleT<R>::TET) {
      double ws = 0.0;
      for (int gg = 0; gg < NG; ++gg) ws += c_w[R][gg];
      dV *= ws;
    } else {
      dV *= c_w[R][g];
    }
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int b = 0; b < NN; ++b)
        le[a][b] += dV * (dNdx[a][0] * dNdx[b][0] + dNdx[a][1] * dNdx[b][1] + dNdx[a][2] * dNdx[b][2]);
  }
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      int64_t pos = csr_find(rp, cols, nd[a], nd[b]);
      if (pos >= 0) red_add(vals + pos, le[a][b]);
    }
}

// Discrete gradient operator B_ab = int N_a grad N_b (3 planes) into the
// CSR pattern of the Laplacian (setup).  With it K4 is b = scale B . u and
// K6 is G p = B p as sparse products (ab_gradop_div / ab_gradop_grad); the
// Gauss sums are those of divergence_element / gradient_element.
template <int R>
__global__ void k_gradop(CatP c, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                         double* __restrict__ vx, double* __restrict__ vy, double* __restrict__ vz) {
  constexpr int NN = RuleT<R>::NN, NG = RuleT<R>::NG;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= c.n) return;
  int nd[NN];
  load_conn<NN>(c.conn, e, nd);
  double x[NN][3];
  load_coords<NN>(c, nd, x);
  double be[NN][NN][3];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) be[a][b][0] = be[a][b][1] = be[a][b][2] = 0.0;
#pragma unroll 1
  for (int g = 0; g < (RuleT<R>::TET ? 1 : NG); ++g) {
    double dNdx[NN][3];
    const double adet = fabs(shape_grads<R, NN>(x, g, dNdx));
#pragma unroll
    for (int gg = 0; gg < (RuleT<R>::TET ? NG : 1); ++gg) {
      const int gi = RuleT<R>::TET ? gg : g;
      const double f = adet * c_w[R][gi];
#pragma unroll
      for (int a = 0; a < NN; ++a) {
        const double fn = f * c_N[R][gi][a];
#pragma unroll
        for (int b = 0; b < NN; ++b)
#pragma unroll
          for (int k = 0; k < 3; ++k) be[a][b][k] = fma(fn, dNdx[b][k], be[a][b][k]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      const int64_t pos = csr_find(rp, cols, nd[a], nd[b]);
      if (pos >= 0) {
        red_add(vx + pos, be[a][b][0]);
        red_add(vy + pos, be[a][b][1]);
        red_add(vz + pos, be[a][b][2]);
      }
    }
}

// centroid = (sum_a x_a) / nnode, sequential in node order (numpy mean over
// axis 0 of the (nnode,3) gather, reference mesh.py:375).
template <int R>
__global__ void k_centroids(CatP c, double* __restrict__ out) {
  constexpr int NN = RuleT<R>::NN;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= c.n) return;
  int nd[NN];
  load_conn<NN>(c.conn, e, nd);
  double s[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 0; a < NN; ++a) {
    d4 v = ld4_nc(c.coords + 4 * (int64_t)nd[a]);
    s[0] = __dadd_rn(s[0], v.x);
    s[1] = __dadd_rn(s[1], v.y);
    s[2] = __dadd_rn(s[2], v.z);
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) out[e * 3 + d] = __ddiv_rn(s[d], (double)NN);
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
struct D2Entry { const int32_t* conn; const double* d2; int64_t n; };
static D2Entry g_d2[64];
static int g_nd2 = 0;

static const double* find_d2(const int32_t* conn, int64_t n) {
  for (int i = 0; i < g_nd2; ++i)
    if (g_d2[i].conn == conn && g_d2[i].n == n) return g_d2[i].d2;
  return nullptr;
}

static CatP cat_params(const ab_mesh* m, int k) {
  CatP c;
  c.coords = m->coords;
  c.conn = m->cat[k].conn;
  c.n = m->cat[k].n_elem;
  c.L0 = m->period[0];
  c.L1 = m->period[1];
  c.L2 = m->period[2];
  c.periodic = (c.L0 > 0.0 || c.L1 > 0.0 || c.L2 > 0.0) ? 1 : 0;
  c.delta2 = find_d2(c.conn, c.n);
  return c;
}

static int valid_mesh(const ab_mesh* m) {
  if (!m || !m->coords || m->n_cat < 0 || m->n_cat > 5) return fail("invalid ab_mesh");
  for (int k = 0; k < m->n_cat; ++k) {
    if (m->cat[k].rule < 0 || m->cat[k].rule > 4) return fail("invalid rule id in ab_mesh");
    if (m->cat[k].n_elem > 0 && !m->cat[k].conn) return fail("null connectivity");
  }
  return AB_OK;
}

// Dispatch a functor templated on the rule id.
template <class F>
static int dispatch_rule(int rule, F&& f) {
  switch (rule) {
    case AB_RULE_TET1: return f(std::integral_constant<int, AB_RULE_TET1>{});
    case AB_RULE_TET4: return f(std::integral_constant<int, AB_RULE_TET4>{});
    case AB_RULE_PYR5: return f(std::integral_constant<int, AB_RULE_PYR5>{});
    case AB_RULE_PRI6: return f(std::integral_constant<int, AB_RULE_PRI6>{});
    case AB_RULE_HEX8: return f(std::integral_constant<int, AB_RULE_HEX8>{});
  }
  return fail("unknown rule");
}

// ---------------------------------------------------------------------------
// Block colouring for the deterministic scatter (setup): Jones-Plassmann
// rounds with hashed priorities.  An uncoloured block whose uncoloured
// neighbours (blocks sharing a window node) all have lower priority takes the
// smallest colour none of its coloured neighbours has.  Two blocks coloured
// in the same round are never neighbours, so the result is a proper
// colouring, and it does not depend on thread scheduling.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t colour_prio(uint32_t b) {
  b ^= b >> 16; b *= 0x7feb352du; b ^= b >> 15; b *= 0x846ca68bu; b ^= b >> 16;
  return b;
}
__global__ void k_colour_round(int64_t nb, const int64_t* __restrict__ blk_ptr, const int32_t* __restrict__ wnode,
                               const int64_t* __restrict__ nptr, const int32_t* __restrict__ nblk, int32_t* colour,
                               int32_t* flags) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  volatile int32_t* col = colour;
  if (col[b] >= 0) return;
  const uint32_t pb = colour_prio((uint32_t)b);
  uint64_t mask = 0;
  for (int64_t k = blk_ptr[b]; k < blk_ptr[b + 1]; ++k) {
    const int n = wnode[k];
    for (int64_t m = nptr[n]; m < nptr[n + 1]; ++m) {
      const int32_t b2 = nblk[m];
      if (b2 == b) continue;
      const int32_t c2 = col[b2];
      if (c2 < 0) {
        const uint32_t p2 = colour_prio((uint32_t)b2);
        if (p2 > pb || (p2 == pb && b2 > b)) {
          flags[0] = 1;  // still work to do
          return;
        }
      } else {
        mask |= 1ull << c2;
      }
    }
  }
  const int c = __ffsll((long long)~mask) - 1;
  if (c < 0) {
    flags[1] = 1;  // more than 64 colours needed
    return;
  }
  col[b] = c;
}

static constexpr int kBlock = 128;

// Opt a kernel into > 48 KB of dynamic shared memory when a window needs it.
template <class K>
static int ensure_smem(K* kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return AB_OK;
  if (bytes > 227 * 1024) return fail("node window exceeds 227 KB of shared memory");
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return fail("cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed");
  return AB_OK;
}

// Windows are attached per category through ab_set_windows (host registry
// keyed by the connectivity pointer, so the ab_mesh struct stays plain).
struct WinEntry { const int32_t* conn; WinP w; };
static WinEntry g_win[64];
static int g_nwin = 0;

static bool find_win(const int32_t* conn, WinP* out) {
  for (int i = 0; i < g_nwin; ++i)
    if (g_win[i].conn == conn) { *out = g_win[i].w; return true; }
  return false;
}

}  // namespace ab

using namespace ab;

extern "C" {

// Register (or clear with blk_ptr == NULL) the node windows of a category.
int ab_set_windows(const int32_t* conn, int32_t block, const int64_t* blk_ptr, const int32_t* wnode,
                   const int32_t* wptr, const uint16_t* wslot, const uint16_t* loc, const int32_t* desc,
                   int32_t wmax) {
  const WinP wp{blk_ptr, wnode, wptr, wslot, loc, reinterpret_cast<const int4*>(desc), nullptr, block, wmax};
  for (int i = 0; i < g_nwin; ++i)
    if (g_win[i].conn == conn) {
      if (!blk_ptr) { g_win[i] = g_win[--g_nwin]; return AB_OK; }
      g_win[i].w = wp;
      return AB_OK;
    }
  if (!blk_ptr) return AB_OK;
  if (block != kBlock) return fail("ab_set_windows: block must be 128");
  if (wmax < 1 || wmax > 8 * kBlock) return fail("ab_set_windows: bad wmax");
  if (!wnode || !wptr || !wslot || !loc) return fail("ab_set_windows: null window array");
  if (g_nwin >= 64) return fail("ab_set_windows: registry full");
  g_win[g_nwin++] = WinEntry{conn, wp};
  return AB_OK;
}

// Sorted element-node references of a category's windows (pipelined kernels).
int ab_set_window_refs(const int32_t* conn, const uint32_t* wref) {
  for (int i = 0; i < g_nwin; ++i)
    if (g_win[i].conn == conn) {
      g_win[i].w.wref = wref;
      return AB_OK;
    }
  return fail("ab_set_window_refs: no windows registered for this connectivity");
}

// Colour mode of a category's pipelined kernels (NULL corder / ncol 0:
// back to fp64 atomics).  corder: blocks grouped by colour; cptr: [ncol+1];
// gbar: one device uint32 for the colour barrier.
int ab_set_window_colours(const int32_t* conn, int32_t ncol, const int32_t* corder, const int64_t* cptr,
                          uint32_t* gbar) {
  for (int i = 0; i < g_nwin; ++i)
    if (g_win[i].conn == conn) {
      if (!corder || ncol < 1) {
        g_win[i].w.corder = nullptr;
        g_win[i].w.cptr = nullptr;
        g_win[i].w.gbar = nullptr;
        g_win[i].w.ncol = 0;
        return AB_OK;
      }
      if (!cptr || !gbar) return fail("ab_set_window_colours: null cptr or barrier word");
      if (!g_win[i].w.desc) return fail("ab_set_window_colours: colour mode needs the pipelined windows (desc)");
      g_win[i].w.corder = corder;
      g_win[i].w.cptr = cptr;
      g_win[i].w.gbar = reinterpret_cast<unsigned*>(gbar);
      g_win[i].w.ncol = ncol;
      return AB_OK;
    }
  return fail("ab_set_window_colours: no windows registered for this connectivity");
}

// Jones-Plassmann colouring of n_blocks window blocks (device arrays;
// synchronises the stream once per round): colour[b] in [0, 64).
int ab_colour_blocks(int64_t n_blocks, const int64_t* blk_ptr, const int32_t* wnode, const int64_t* nptr,
                     const int32_t* nblk, int32_t* colour, int32_t* flags, void* stream) {
  if (n_blocks < 0 || !blk_ptr || !wnode || !nptr || !nblk || !colour || !flags)
    return fail("ab_colour_blocks: null argument");
  if (n_blocks == 0) return 0;
  cudaStream_t st = S(stream);
  if (cudaMemsetAsync(colour, 0xff, sizeof(int32_t) * n_blocks, st) != cudaSuccess)
    return fail("ab_colour_blocks: memset failed");
  for (int round = 0; round < 100000; ++round) {
    int32_t h[2] = {0, 0};
    cudaMemsetAsync(flags, 0, sizeof(int32_t) * 2, st);
    k_colour_round<<<grid_for(n_blocks, 256), 256, 0, st>>>(n_blocks, blk_ptr, wnode, nptr, nblk, colour, flags);
    if (int rc = check_launch("ab_colour_blocks")) return rc;
    cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail("ab_colour_blocks: round failed");
    if (h[1]) return fail("ab_colour_blocks: more than 64 colours needed");
    if (!h[0]) break;
  }
  return AB_OK;
}

int ab_filter_width(const ab_mesh* m, int32_t k, double* delta2, void* stream) {
  if (int rc = valid_mesh(m)) return rc;
  if (k < 0 || k >= m->n_cat) return fail("ab_filter_width: category out of range");
  if (!delta2) return fail("ab_filter_width: null output");
  CatP c = cat_params(m, k);
  c.delta2 = nullptr;
  if (c.n == 0) return AB_OK;
  return dispatch_rule(m->cat[k].rule, [&](auto r) {
    k_filter_width<decltype(r)::value><<<grid_for(c.n, 256), 256, 0, S(stream)>>>(c, delta2);
    return check_launch("ab_filter_width");
  });
}

int ab_set_filter_width(const int32_t* conn, int64_t n_elem, const double* delta2) {
  for (int i = 0; i < g_nd2; ++i)
    if (g_d2[i].conn == conn) {
      if (!delta2) { g_d2[i] = g_d2[--g_nd2]; return AB_OK; }
      g_d2[i].d2 = delta2;
      g_d2[i].n = n_elem;
      return AB_OK;
    }
  if (!delta2) return AB_OK;
  if (!conn || n_elem < 1) return fail("ab_set_filter_width: null connectivity");
  if (g_nd2 >= 64) return fail("ab_set_filter_width: registry full");
  g_d2[g_nd2++] = D2Entry{conn, delta2, n_elem};
  return AB_OK;
}

int ab_mass(const ab_mesh* m, int32_t k, double* ae, double* jdet, double* ml, int32_t tile, void* stream) {
  if (int rc = valid_mesh(m)) return rc;
  if (k < 0 || k >= m->n_cat) return fail("ab_mass: category out of range");
  if (tile < 1 || tile > 1024) return fail("ab_mass: tile must be in [1, 1024]");
  CatP c = cat_params(m, k);
  if (c.n == 0) return AB_OK;
  return dispatch_rule(m->cat[k].rule, [&](auto r) {
    // the pack (CTA tile) is capped by what the kernel's registers allow;
    // per-element results do not depend on it
    cudaFuncAttributes fa;
    int t = tile;
    if (cudaFuncGetAttributes(&fa, k_mass<decltype(r)::value>) == cudaSuccess && t > fa.maxThreadsPerBlock)
      t = fa.maxThreadsPerBlock & ~31;
    k_mass<decltype(r)::value><<<grid_for(c.n, t), t, 0, S(stream)>>>(c, ae, jdet, ml);
    return check_launch("ab_mass");
  });
}

int ab_last_pipe_shape(int64_t* grid, int64_t* n_blocks) {
  if (!grid || !n_blocks) return fail("ab_last_pipe_shape: null argument");
  *grid = g_pipe_grid;
  *n_blocks = g_pipe_blocks;
  return AB_OK;
}

int ab_momentum_rhs(const ab_mesh* m, const ab_phys* ph, const double* u4, double* rhs4, void* stream) {
  if (int rc = valid_mesh(m)) return rc;
  if (!ph || !u4 || !rhs4) return fail("ab_momentum_rhs: null argument");
  for (int k = 0; k < m->n_cat; ++k) {
    CatP c = cat_params(m, k);
    if (c.n == 0) continue;
    WinP w{};
    const bool win = find_win(c.conn, &w);
    int rc = dispatch_rule(m->cat[k].rule, [&](auto r) {
      constexpr int R = decltype(r)::value;
      constexpr int NN = RuleT<R>::NN;
      if (win && w.desc) {
        if (int rc = launch_pipe<R, OP_MOMENTUM, kBlock>(c, w, *ph, 1.0, u4, rhs4, S(stream))) return rc;
        return AB_OK;
      }
      if (win) {
        size_t sm = sizeof(double) * ((size_t)w.wmax * 6 + kBlock * NN * 3);
        if (int rc = ensure_smem(k_momentum<R, kBlock, true>, sm)) return rc;
        k_momentum<R, kBlock, true><<<grid_for(c.n, kBlock), kBlock, sm, S(stream)>>>(c, *ph, u4, rhs4, w);
      } else {
        k_momentum<R, kBlock, false><<<grid_for(c.n, kBlock), kBlock, 0, S(stream)>>>(c, *ph, u4, rhs4, w);
      }
      return check_launch("ab_momentum_rhs");
    });
    if (rc) return rc;
  }
  return AB_OK;
}

int ab_divergence(const ab_mesh* m, const double* u4, double scale, double* out, void* stream) {
  if (int rc = valid_mesh(m)) return rc;
  for (int k = 0; k < m->n_cat; ++k) {
    CatP c = cat_params(m, k);
    if (c.n == 0) continue;
    WinP w{};
    const bool win = find_win(c.conn, &w);
    int rc = dispatch_rule(m->cat[k].rule, [&](auto r) {
      constexpr int R = decltype(r)::value;
      constexpr int NN = RuleT<R>::NN;
      if (win && w.desc) {
        ab_phys ph{};
        if (int rc = launch_pipe<R, OP_DIVERGENCE, kBlock>(c, w, ph, scale, u4, out, S(stream))) return rc;
        return AB_OK;
      }
      if (win) {
        const size_t sm = sizeof(double) * ((size_t)w.wmax * 6 + kBlock * NN);
        if (int rc = ensure_smem(k_divergence<R, kBlock, true>, sm)) return rc;
        k_divergence<R, kBlock, true><<<grid_for(c.n, kBlock), kBlock, sm, S(stream)>>>(c, u4, scale, out, w);
      } else {
        k_divergence<R, kBlock, false><<<grid_for(c.n, kBlock), kBlock, 0, S(stream)>>>(c, u4, scale, out, w);
      }
      return check_launch("ab_divergence");
    });
    if (rc) return rc;
  }
  return AB_OK;
}

int ab_gradient(const ab_mesh* m, const double* p, double scale, double* out4, void* stream) {
  if (int rc = valid_mesh(m)) return rc;
  for (int k = 0; k < m->n_cat; ++k) {
    CatP c = cat_params(m, k);
    if (c.n == 0) continue;
    WinP w{};
    const bool win = find_win(c.conn, &w);
    int rc = dispatch_rule(m->cat[k].rule, [&](auto r) {
      constexpr int R = decltype(r)::value;
      constexpr int NN = RuleT<R>::NN;
      if (win && w.desc) {
        ab_phys ph{};
        if (int rc = launch_pipe<R, OP_GRADIENT, kBlock>(c, w, ph, scale, p, out4, S(stream))) return rc;
        return AB_OK;
      }
      if (win) {
        const size_t sm = sizeof(double) * ((size_t)w.wmax * 4 + kBlock * NN * 3);
        if (int rc = ensure_smem(k_gradient<R, kBlock, true>, sm)) return rc;
        k_gradient<R, kBlock, true><<<grid_for(c.n, kBlock), kBlock, sm, S(stream)>>>(c, p, scale, out4, w);
      } else {
        k_gradient<R, kBlock, false><<<grid_for(c.n, kBlock), kBlock, 0, S(stream)>>>(c, p, scale, out4, w);
      }
      return check_launch("ab_gradient");
    });
    if (rc) return rc;
  }
  return AB_OK;
}

int ab_laplacian_csr(const ab_mesh* m, const int64_t* rp, const int32_t* cols, double* vals, void* stream) {
  if (int rc = valid_mesh(m)) return rc;
  for (int k = 0; k < m->n_cat; ++k) {
    CatP c = cat_params(m, k);
    if (c.n == 0) continue;
    int rc = dispatch_rule(m->cat[k].rule, [&](auto r) {
      k_laplacian<decltype(r)::value><<<grid_for(c.n, 128), 128, 0, S(stream)>>>(c, rp, cols, vals);
      return check_launch("ab_laplacian_csr");
    });
    if (rc) return rc;
  }
  return AB_OK;
}

int ab_gradop_csr(const ab_mesh* m, const int64_t* rp, const int32_t* cols, double* vx, double* vy, double* vz,
                  void* stream) {
  if (int rc = valid_mesh(m)) return rc;
  if (!rp || !cols || !vx || !vy || !vz) return fail("ab_gradop_csr: null argument");
  for (int k = 0; k < m->n_cat; ++k) {
    CatP c = cat_params(m, k);
    if (c.n == 0) continue;
    int rc = dispatch_rule(m->cat[k].rule, [&](auto r) {
      k_gradop<decltype(r)::value><<<grid_for(c.n, 128), 128, 0, S(stream)>>>(c, rp, cols, vx, vy, vz);
      return check_launch("ab_gradop_csr");
    });
    if (rc) return rc;
  }
  return AB_OK;
}

int ab_centroids(const ab_mesh* m, int32_t k, double* out, void* stream) {
  if (int rc = valid_mesh(m)) return rc;
  if (k < 0 || k >= m->n_cat) return fail("ab_centroids: category out of range");
  CatP c = cat_params(m, k);
  c.periodic = 0;  // the reference averages raw node coordinates
  if (c.n == 0) return AB_OK;
  return dispatch_rule(m->cat[k].rule, [&](auto r) {
    k_centroids<decltype(r)::value><<<grid_for(c.n, 256), 256, 0, S(stream)>>>(c, out);
    return check_launch("ab_centroids");
  });
}

}  // extern "C"
