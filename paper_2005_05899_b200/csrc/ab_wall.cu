// K8: boundary assembly of the equilibrium wall model (Algorithm 1 line 4,
// PAPER.md:214, :228, :256-257; scheme of DESIGN.md §3, restated in
// oracle/fem.py:wall_traction).  One thread per wall face:
//   exchange point = mean of the owning element's off-face nodes (x_e, u_e),
//   n = outward unit normal of the (planar) face, y = |(x_e - x_c) . n|,
//   u_t = u_e - (u_e . n) n, u_tau from Reichardt's law (fixed Newton count),
//   every face node receives -rho u_tau^2 u_t/|u_t| * A / n_face_nodes
// accumulated into rhs4 (fp64 reductions: wall nodes are shared by faces),
// or, in the fixed-order form, stored per face and summed per wall node in
// ascending face order by k_wall_gather (bitwise reproducible).
#include "ab_common.cuh"

namespace ab {

constexpr double kKappa = 0.41;
constexpr int kReichardtIters = 12;

__device__ __forceinline__ void reichardt(double yp, double& up, double& dup) {
  const double e11 = exp(-yp / 11.0), e3 = exp(-yp / 3.0);
  up = log1p(kKappa * yp) / kKappa + 7.8 * (1.0 - e11 - (yp / 11.0) * e3);
  dup = 1.0 / (1.0 + kKappa * yp) + 7.8 * (e11 / 11.0 - e3 / 11.0 + (yp / 33.0) * e3);
}

__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

__global__ void k_wall(int64_t nfaces, const int32_t* __restrict__ face, const int32_t* __restrict__ off,
                       const double* __restrict__ coords4, const double* __restrict__ u4, double rho, double mu,
                       double* __restrict__ rhs4, double* __restrict__ ftrac) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nfaces) return;
  int fn[4], on[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    fn[k] = face[4 * f + k];
    on[k] = off[4 * f + k];
  }
  const int nf = fn[3] >= 0 ? 4 : 3;
  double fx[4][3];
  double xc[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < nf) {
      const d4 v = ld4_nc(coords4 + 4 * (int64_t)fn[k]);
      fx[k][0] = v.x; fx[k][1] = v.y; fx[k][2] = v.z;
    } else {
      fx[k][0] = fx[k][1] = fx[k][2] = 0.0;
    }
    xc[0] += fx[k][0]; xc[1] += fx[k][1]; xc[2] += fx[k][2];
  }
  double xe[3] = {0.0, 0.0, 0.0}, ue[3] = {0.0, 0.0, 0.0};
  int no = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (on[k] >= 0) {
      const d4 x = ld4_nc(coords4 + 4 * (int64_t)on[k]);
      const d4 u = ld4_nc(u4 + 4 * (int64_t)on[k]);
      xe[0] += x.x; xe[1] += x.y; xe[2] += x.z;
      ue[0] += u.x; ue[1] += u.y; ue[2] += u.z;
      ++no;
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    xc[d] /= nf;
    xe[d] /= no;
    ue[d] /= no;
  }
  double e1[3], e2[3], e3[3], a[3], b[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    e1[d] = fx[1][d] - fx[0][d];
    e2[d] = fx[2][d] - fx[0][d];
    e3[d] = fx[3][d] - fx[0][d];
  }
  cross3(e1, e2, a);
  if (nf == 4) cross3(e2, e3, b);
  const double area = 0.5 * sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]) +
                      (nf == 4 ? 0.5 * sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]) : 0.0);
  double nv[3] = {a[0] + b[0], a[1] + b[1], a[2] + b[2]};
  const double nl = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
  nv[0] /= nl; nv[1] /= nl; nv[2] /= nl;
  if (nv[0] * (xc[0] - xe[0]) + nv[1] * (xc[1] - xe[1]) + nv[2] * (xc[2] - xe[2]) < 0.0) {
    nv[0] = -nv[0]; nv[1] = -nv[1]; nv[2] = -nv[2];
  }
  const double y = fabs((xe[0] - xc[0]) * nv[0] + (xe[1] - xc[1]) * nv[1] + (xe[2] - xc[2]) * nv[2]);
  const double un = ue[0] * nv[0] + ue[1] * nv[1] + ue[2] * nv[2];
  const double ut[3] = {ue[0] - un * nv[0], ue[1] - un * nv[1], ue[2] - un * nv[2]};
  const double utm = sqrt(ut[0] * ut[0] + ut[1] * ut[1] + ut[2] * ut[2]);
  if (!(utm > 0.0)) {
    if (ftrac) ftrac[3 * f] = ftrac[3 * f + 1] = ftrac[3 * f + 2] = 0.0;
    return;
  }
  const double nu = mu / rho;
  double utau = sqrt(nu * utm / y);
  for (int it = 0; it < kReichardtIters; ++it) {
    const double yp = y * utau / nu;
    double up, dup;
    reichardt(yp, up, dup);
    const double fv = utau * up - utm;
    const double df = up + yp * dup;
    utau = fmax(utau - fv / df, 0.0);
  }
  const double coef = -rho * utau * utau / utm * area / nf;
  if (ftrac) {
    ftrac[3 * f] = coef * ut[0];
    ftrac[3 * f + 1] = coef * ut[1];
    ftrac[3 * f + 2] = coef * ut[2];
    return;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < nf) {
      double* r = rhs4 + 4 * (int64_t)fn[k];
      red_add(r + 0, coef * ut[0]);
      red_add(r + 1, coef * ut[1]);
      red_add(r + 2, coef * ut[2]);
    }
  }
}

// Fixed-order accumulation: wall node i adds its faces' tractions in
// ascending face order (one thread per node, plain read-add-write).
__global__ void k_wall_gather(int64_t n, const int32_t* __restrict__ node, const int64_t* __restrict__ ptr,
                              const int32_t* __restrict__ fref, const double* __restrict__ ftrac,
                              double* __restrict__ rhs4) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int64_t f = fref[k];
    s0 += ftrac[3 * f];
    s1 += ftrac[3 * f + 1];
    s2 += ftrac[3 * f + 2];
  }
  double* r = rhs4 + 4 * (int64_t)node[i];
  r[0] += s0;
  r[1] += s1;
  r[2] += s2;
}

}  // namespace ab

using namespace ab;

extern "C" {

int ab_wall_traction(const ab_wall* w, const ab_phys* phys, const double* coords4, const double* u4, double* rhs4,
                     void* stream) {
  if (!w || !phys || !coords4 || !u4 || !rhs4) return fail("ab_wall_traction: null argument");
  if (w->n_faces <= 0) return AB_OK;
  if (!w->face || !w->off) return fail("ab_wall_traction: null face lists");
  const bool ordered = w->node != nullptr;
  if (ordered && (!w->ptr || !w->fref || !w->ftrac || w->n_nodes <= 0))
    return fail("ab_wall_traction: incomplete fixed-order node lists");
  k_wall<<<grid_for(w->n_faces, 128), 128, 0, S(stream)>>>(w->n_faces, w->face, w->off, coords4, u4, phys->rho,
                                                          phys->mu, rhs4, ordered ? w->ftrac : nullptr);
  if (int rc = check_launch("ab_wall_traction")) return rc;
  if (!ordered) return AB_OK;
  k_wall_gather<<<grid_for(w->n_nodes, 128), 128, 0, S(stream)>>>(w->n_nodes, w->node, w->ptr, w->fref, w->ftrac,
                                                                 rhs4);
  return check_launch("ab_wall_traction(gather)");
}

}  // extern "C"
