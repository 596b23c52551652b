/* ORACLE (C restatement) — TEST INFRASTRUCTURE AND CPU BASELINE ONLY.
 *
 * The time step of oracle/fem.py (FlowOracle.step: SSP-RK3 momentum stages with
 * the EMAC + viscous + Vreman element RHS and the equilibrium wall model,
 * divergence, Jacobi-PCG on the assembled Laplacian, gradient correction;
 * PAPER.md:192-237 with the decisions of DESIGN.md §3) restated in C with
 * OpenMP so that bench.py's cpu_baseline / `--impl reference` legs time an
 * optimised multi-core CPU code instead of numpy.  Only tests/ and bench.py's
 * CPU legs load it (oracle/femc.py); the product package never does.
 *
 * PARITY UNPINNED by the reference (it has no Navier-Stokes code);
 * tests/test_oracle_c.py checks this restatement against oracle/fem.py on
 * tet, periodic hex and mixed tet/prism/pyramid/hex meshes (rel L2 <= 1e-12).
 *
 * Reference-element tables (N, dN/dxi, weights) are passed in from
 * oracle/fem.py's shape_tables / rule_points_weights, so both restatements use
 * the same numbers.  Affine tetrahedra take the closed form the GPU kernel uses
 * (constant geometry and grad u; convective Gauss sum = A sum_b M_ab u_b with
 * M_ab = sum_g w_g N_a(g) N_b(g) from the rule) — algebraically the oracle's
 * Gauss loop.  Scatters go to per-thread private arrays summed in thread order
 * (deterministic for a fixed thread count).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXN 8
#define MAXG 8

typedef struct {
  int nn, ng, tet;
  int64_t n_elem;
  const int32_t* conn; /* [n_elem][nn] */
  double N[MAXG][MAXN], dN[MAXG][MAXN][3], w[MAXG];
  double M[MAXN][MAXN]; /* sum_g w_g N_a N_b (affine tets) */
  double wsum;
} fc_cat;

typedef struct {
  int64_t n;
  const double* x; /* [n][3] */
  double period[3];
  int periodic;
  int ncat;
  fc_cat cat[5];
  int nthreads;
  double* priv; /* [nthreads][n][3] scratch */
} fc_mesh;

fc_mesh* fc_mesh_create(int64_t n, const double* x, const double* period, int nthreads) {
  fc_mesh* m = (fc_mesh*)calloc(1, sizeof(fc_mesh));
  m->n = n;
  m->x = x;
  for (int d = 0; d < 3; ++d) {
    m->period[d] = period ? period[d] : 0.0;
    if (m->period[d] > 0.0) m->periodic = 1;
  }
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
  m->nthreads = omp_get_max_threads();
#else
  m->nthreads = 1;
#endif
  m->priv = (double*)malloc(sizeof(double) * 3 * (size_t)n * (size_t)m->nthreads);
  return m;
}

int fc_nthreads(const fc_mesh* m) { return m->nthreads; }

/* N: [ng][nn], dN: [ng][nn][3], w: [ng] (oracle/fem.py tables, transposed to Gauss-major) */
int fc_add_category(fc_mesh* m, int nn, int ng, int tet, int64_t n_elem, const int32_t* conn, const double* N,
                    const double* dN, const double* w) {
  if (m->ncat >= 5 || nn > MAXN || ng > MAXG) return -1;
  fc_cat* c = &m->cat[m->ncat++];
  c->nn = nn;
  c->ng = ng;
  c->tet = tet;
  c->n_elem = n_elem;
  c->conn = conn;
  c->wsum = 0.0;
  for (int g = 0; g < ng; ++g) {
    c->w[g] = w[g];
    c->wsum += w[g];
    for (int a = 0; a < nn; ++a) {
      c->N[g][a] = N[g * nn + a];
      for (int k = 0; k < 3; ++k) c->dN[g][a][k] = dN[(g * nn + a) * 3 + k];
    }
  }
  for (int a = 0; a < nn; ++a)
    for (int b = 0; b < nn; ++b) {
      double s = 0.0;
      for (int g = 0; g < ng; ++g) s += c->w[g] * c->N[g][a] * c->N[g][b];
      c->M[a][b] = s;
    }
  return 0;
}

void fc_mesh_destroy(fc_mesh* m) {
  if (!m) return;
  free(m->priv);
  free(m);
}

static void gather_x(const fc_mesh* m, const fc_cat* c, int64_t e, double X[MAXN][3], int nd[MAXN]) {
  for (int a = 0; a < c->nn; ++a) {
    nd[a] = c->conn[e * c->nn + a];
    for (int k = 0; k < 3; ++k) X[a][k] = m->x[3 * (int64_t)nd[a] + k];
  }
  if (m->periodic)
    for (int k = 0; k < 3; ++k) {
      const double L = m->period[k];
      if (L > 0.0)
        for (int a = 1; a < c->nn; ++a) {
          const double rel = X[a][k] - X[0][k];
          X[a][k] = X[0][k] + rel - L * nearbyint(rel / L);
        }
    }
}

static double inv3(const double J[3][3], double iv[3][3]) {
  const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  const double c01 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  const double c02 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  const double c10 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  const double c11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  const double c12 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  const double c20 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  const double c21 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  const double c22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double det = J[0][0] * c00 + J[0][1] * c10 + J[0][2] * c20;
  const double id = 1.0 / det;
  iv[0][0] = c00 * id; iv[0][1] = c01 * id; iv[0][2] = c02 * id;
  iv[1][0] = c10 * id; iv[1][1] = c11 * id; iv[1][2] = c12 * id;
  iv[2][0] = c20 * id; iv[2][1] = c21 * id; iv[2][2] = c22 * id;
  return det;
}

/* dN/dx at Gauss point g; returns |det J| */
static double shape_grads(const fc_cat* c, const double X[MAXN][3], int g, double dNdx[MAXN][3]) {
  double J[3][3], iv[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int a = 0; a < c->nn; ++a) s += X[a][i] * c->dN[g][a][j];
      J[i][j] = s;
    }
  const double det = inv3(J, iv);
  for (int a = 0; a < c->nn; ++a)
    for (int k = 0; k < 3; ++k)
      dNdx[a][k] = c->dN[g][a][0] * iv[0][k] + c->dN[g][a][1] * iv[1][k] + c->dN[g][a][2] * iv[2][k];
  return fabs(det);
}

/* Vreman mu_t from G (G_ij = du_i/dx_j), Delta^2 */
static double vreman(const double G[3][3], double delta2, double rho, double cv) {
  double S[3][3];  /* alpha^T alpha with alpha_ij = G_ji: S_ij = sum_m G_im G_jm */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) S[i][j] = G[i][0] * G[j][0] + G[i][1] * G[j][1] + G[i][2] * G[j][2];
  const double aa = S[0][0] + S[1][1] + S[2][2];
  double B = delta2 * delta2 *
             (S[0][0] * S[1][1] - S[0][1] * S[0][1] + S[0][0] * S[2][2] - S[0][2] * S[0][2] + S[1][1] * S[2][2] -
              S[1][2] * S[1][2]);
  if (B < 0.0) B = 0.0;
  return aa > 1e-30 ? rho * cv * sqrt(B / aa) : 0.0;
}

static void zero_priv(fc_mesh* m, int nc) {
  const int64_t tot = (int64_t)m->nthreads * m->n * nc;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < tot; ++i) m->priv[i] = 0.0;
}

/* out[i*nc + k] (+)= sum over threads in thread order */
static void reduce_priv(fc_mesh* m, int nc, double* out, int accumulate) {
  const int64_t len = m->n * nc;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < len; ++i) {
    double s = accumulate ? out[i] : 0.0;
    for (int t = 0; t < m->nthreads; ++t) s += m->priv[(int64_t)t * len + i];
    out[i] = s;
  }
}

static int tid(void) {
#ifdef _OPENMP
  return omp_get_thread_num();
#else
  return 0;
#endif
}

/* R (N,3) = momentum RHS of u (N,3) (overwrites R) */
void fc_momentum(fc_mesh* m, const double* u, double rho, double mu, double cvr, double* R) {
  zero_priv(m, 3);
  for (int k = 0; k < m->ncat; ++k) {
    const fc_cat* c = &m->cat[k];
    const int nn = c->nn, ng = c->ng;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < c->n_elem; ++e) {
      double* P = m->priv + (int64_t)tid() * m->n * 3;
      double X[MAXN][3], U[MAXN][3], r[MAXN][3];
      int nd[MAXN];
      gather_x(m, c, e, X, nd);
      for (int a = 0; a < nn; ++a)
        for (int i = 0; i < 3; ++i) {
          U[a][i] = u[3 * (int64_t)nd[a] + i];
          r[a][i] = 0.0;
        }
      if (c->tet) {
        double dNdx[MAXN][3];
        const double adet = shape_grads(c, X, 0, dNdx);
        const double vol = adet * c->wsum;
        double G[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int a = 0; a < nn; ++a) s += U[a][i] * dNdx[a][j];
            G[i][j] = s;
          }
        const double div = G[0][0] + G[1][1] + G[2][2];
        double mue = mu;
        if (cvr > 0.0) {
          const double d = cbrt(vol);
          mue += vreman(G, d * d, rho, cvr);
        }
        double A[3][3], sg[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            const double e2 = G[i][j] + G[j][i];
            A[i][j] = rho * adet * (e2 + (i == j ? div : 0.0));
            sg[i][j] = mue * e2 * vol;
          }
        for (int a = 0; a < nn; ++a) {
          double mm[3] = {0.0, 0.0, 0.0};
          for (int b = 0; b < nn; ++b)
            for (int i = 0; i < 3; ++i) mm[i] += c->M[a][b] * U[b][i];
          for (int i = 0; i < 3; ++i)
            r[a][i] = -(A[i][0] * mm[0] + A[i][1] * mm[1] + A[i][2] * mm[2] + sg[i][0] * dNdx[a][0] +
                        sg[i][1] * dNdx[a][1] + sg[i][2] * dNdx[a][2]);
        }
      } else {
        double delta2 = 0.0;
        if (cvr > 0.0) {
          double vol = 0.0, dtmp[MAXN][3];
          for (int g = 0; g < ng; ++g) vol += shape_grads(c, X, g, dtmp) * c->w[g];
          const double d = cbrt(vol);
          delta2 = d * d;
        }
        for (int g = 0; g < ng; ++g) {
          double dNdx[MAXN][3];
          const double dV = shape_grads(c, X, g, dNdx) * c->w[g];
          double ug[3] = {0.0, 0.0, 0.0}, G[3][3];
          for (int b = 0; b < nn; ++b)
            for (int i = 0; i < 3; ++i) ug[i] += c->N[g][b] * U[b][i];
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
              double s = 0.0;
              for (int a = 0; a < nn; ++a) s += U[a][i] * dNdx[a][j];
              G[i][j] = s;
            }
          const double div = G[0][0] + G[1][1] + G[2][2];
          const double mue = mu + (cvr > 0.0 ? vreman(G, delta2, rho, cvr) : 0.0);
          double cv[3], sg[3][3];
          for (int i = 0; i < 3; ++i) {
            double s = div * ug[i];
            for (int j = 0; j < 3; ++j) {
              const double e2 = G[i][j] + G[j][i];
              s += e2 * ug[j];
              sg[i][j] = mue * e2 * dV;
            }
            cv[i] = rho * dV * s;
          }
          for (int a = 0; a < nn; ++a)
            for (int i = 0; i < 3; ++i)
              r[a][i] -= c->N[g][a] * cv[i] + sg[i][0] * dNdx[a][0] + sg[i][1] * dNdx[a][1] + sg[i][2] * dNdx[a][2];
        }
      }
      for (int a = 0; a < nn; ++a)
        for (int i = 0; i < 3; ++i) P[3 * (int64_t)nd[a] + i] += r[a][i];
    }
  }
  reduce_priv(m, 3, R, 0);
}

/* out (N) (overwritten) = scale * sum_e int N_a div(u) */
void fc_divergence(fc_mesh* m, const double* u, double scale, double* out) {
  zero_priv(m, 1);
  for (int k = 0; k < m->ncat; ++k) {
    const fc_cat* c = &m->cat[k];
    const int nn = c->nn, ng = c->ng;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < c->n_elem; ++e) {
      double* P = m->priv + (int64_t)tid() * m->n;
      double X[MAXN][3], r[MAXN];
      int nd[MAXN];
      gather_x(m, c, e, X, nd);
      for (int a = 0; a < nn; ++a) r[a] = 0.0;
      for (int g = 0; g < (c->tet ? 1 : ng); ++g) {
        double dNdx[MAXN][3];
        const double adet = shape_grads(c, X, g, dNdx);
        double div = 0.0;
        for (int a = 0; a < nn; ++a)
          for (int i = 0; i < 3; ++i) div += u[3 * (int64_t)nd[a] + i] * dNdx[a][i];
        if (c->tet) {
          for (int gg = 0; gg < ng; ++gg)
            for (int a = 0; a < nn; ++a) r[a] += c->N[gg][a] * adet * c->w[gg] * div;
        } else {
          for (int a = 0; a < nn; ++a) r[a] += c->N[g][a] * adet * c->w[g] * div;
        }
      }
      for (int a = 0; a < nn; ++a) P[nd[a]] += scale * r[a];
    }
  }
  reduce_priv(m, 1, out, 0);
}

/* out (N,3) (overwritten) = sum_e int N_a grad(p) */
void fc_gradient(fc_mesh* m, const double* p, double* out) {
  zero_priv(m, 3);
  for (int k = 0; k < m->ncat; ++k) {
    const fc_cat* c = &m->cat[k];
    const int nn = c->nn, ng = c->ng;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < c->n_elem; ++e) {
      double* P = m->priv + (int64_t)tid() * m->n * 3;
      double X[MAXN][3], r[MAXN][3];
      int nd[MAXN];
      gather_x(m, c, e, X, nd);
      for (int a = 0; a < nn; ++a) r[a][0] = r[a][1] = r[a][2] = 0.0;
      for (int g = 0; g < (c->tet ? 1 : ng); ++g) {
        double dNdx[MAXN][3];
        const double adet = shape_grads(c, X, g, dNdx);
        double gp[3] = {0.0, 0.0, 0.0};
        for (int a = 0; a < nn; ++a)
          for (int i = 0; i < 3; ++i) gp[i] += p[nd[a]] * dNdx[a][i];
        for (int gg = (c->tet ? 0 : g); gg < (c->tet ? ng : g + 1); ++gg)
          for (int a = 0; a < nn; ++a)
            for (int i = 0; i < 3; ++i) r[a][i] += c->N[gg][a] * adet * c->w[gg] * gp[i];
      }
      for (int a = 0; a < nn; ++a)
        for (int i = 0; i < 3; ++i) P[3 * (int64_t)nd[a] + i] += r[a][i];
    }
  }
  reduce_priv(m, 3, out, 0);
}

/* R (N,3) += wall-model traction (faces/off: [F][4], -1 padded) */
void fc_wall(fc_mesh* m, int64_t nf, const int32_t* face, const int32_t* off, const double* u, double rho, double mu,
             double* R) {
  const double kappa = 0.41, nu = mu / rho;
  for (int64_t f = 0; f < nf; ++f) {
    double fx[4][3], xc[3] = {0, 0, 0}, xe[3] = {0, 0, 0}, ue[3] = {0, 0, 0};
    int n_f = 0, n_o = 0;
    for (int k = 0; k < 4; ++k) {
      const int a = face[4 * f + k];
      for (int d = 0; d < 3; ++d) fx[k][d] = a >= 0 ? m->x[3 * (int64_t)a + d] : 0.0;
      if (a >= 0) {
        ++n_f;
        for (int d = 0; d < 3; ++d) xc[d] += fx[k][d];
      }
      const int o = off[4 * f + k];
      if (o >= 0) {
        ++n_o;
        for (int d = 0; d < 3; ++d) {
          xe[d] += m->x[3 * (int64_t)o + d];
          ue[d] += u[3 * (int64_t)o + d];
        }
      }
    }
    for (int d = 0; d < 3; ++d) {
      xc[d] /= n_f;
      xe[d] /= n_o;
      ue[d] /= n_o;
    }
    double e1[3], e2[3], e3[3], a[3], b[3] = {0, 0, 0};
    for (int d = 0; d < 3; ++d) {
      e1[d] = fx[1][d] - fx[0][d];
      e2[d] = fx[2][d] - fx[0][d];
      e3[d] = fx[3][d] - fx[0][d];
    }
    a[0] = e1[1] * e2[2] - e1[2] * e2[1];
    a[1] = e1[2] * e2[0] - e1[0] * e2[2];
    a[2] = e1[0] * e2[1] - e1[1] * e2[0];
    if (n_f == 4) {
      b[0] = e2[1] * e3[2] - e2[2] * e3[1];
      b[1] = e2[2] * e3[0] - e2[0] * e3[2];
      b[2] = e2[0] * e3[1] - e2[1] * e3[0];
    }
    const double area = 0.5 * sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]) +
                        (n_f == 4 ? 0.5 * sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]) : 0.0);
    double nv[3] = {a[0] + b[0], a[1] + b[1], a[2] + b[2]};
    const double nl = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
    for (int d = 0; d < 3; ++d) nv[d] /= nl;
    if (nv[0] * (xc[0] - xe[0]) + nv[1] * (xc[1] - xe[1]) + nv[2] * (xc[2] - xe[2]) < 0.0)
      for (int d = 0; d < 3; ++d) nv[d] = -nv[d];
    const double y = fabs((xe[0] - xc[0]) * nv[0] + (xe[1] - xc[1]) * nv[1] + (xe[2] - xc[2]) * nv[2]);
    const double un = ue[0] * nv[0] + ue[1] * nv[1] + ue[2] * nv[2];
    const double ut[3] = {ue[0] - un * nv[0], ue[1] - un * nv[1], ue[2] - un * nv[2]};
    const double utm = sqrt(ut[0] * ut[0] + ut[1] * ut[1] + ut[2] * ut[2]);
    if (!(utm > 0.0)) continue;
    double utau = sqrt(nu * utm / y);
    for (int it = 0; it < 12; ++it) {
      const double yp = y * utau / nu;
      const double e11 = exp(-yp / 11.0), e3v = exp(-yp / 3.0);
      const double up = log1p(kappa * yp) / kappa + 7.8 * (1.0 - e11 - (yp / 11.0) * e3v);
      const double dup = 1.0 / (1.0 + kappa * yp) + 7.8 * (e11 / 11.0 - e3v / 11.0 + (yp / 33.0) * e3v);
      const double fv = utau * up - utm, df = up + yp * dup;
      utau = fmax(utau - fv / df, 0.0);
    }
    const double coef = -rho * utau * utau / utm * area / n_f;
    for (int k = 0; k < 4; ++k) {
      const int a2 = face[4 * f + k];
      if (a2 >= 0)
        for (int d = 0; d < 3; ++d) R[3 * (int64_t)a2 + d] += coef * ut[d];
    }
  }
}

/* Jacobi-PCG in the operation order of oracle/fem.py:pcg (x0 = 0, fixed
 * iteration count unless tol > 0); CSR int64 row pointers, int32 columns.
 * scratch: 5 * n doubles.  Returns the iteration count. */
int fc_pcg(int64_t n, const int64_t* rp, const int32_t* ci, const double* av, const double* b, const double* dinv,
           int maxit, double tol, double* x, double* scratch) {
  double *r = scratch, *z = scratch + n, *p = scratch + 2 * n, *q = scratch + 3 * n, *t = scratch + 4 * n;
  double rz = 0.0, bb = 0.0, rr;
#pragma omp parallel for schedule(static) reduction(+ : rz, bb)
  for (int64_t i = 0; i < n; ++i) {
    x[i] = 0.0;
    r[i] = b[i];
    z[i] = dinv[i] * b[i];
    p[i] = q[i] = 0.0;
    rz += r[i] * z[i];
    bb += b[i] * b[i];
  }
  rr = bb;
  double beta = 0.0;
  int it = 0;
  while (it < maxit) {
    if (tol > 0.0 && bb > 0.0 && sqrt(rr / bb) <= tol) break;
    double pq = 0.0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += av[k] * z[ci[k]];
      t[i] = s;
    }
#pragma omp parallel for schedule(static) reduction(+ : pq)
    for (int64_t i = 0; i < n; ++i) {
      p[i] = z[i] + beta * p[i];
      q[i] = t[i] + beta * q[i];
      pq += p[i] * q[i];
    }
    const double alpha = pq != 0.0 ? rz / pq : 0.0;
    double rz_new = 0.0, rr_new = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : rz_new, rr_new)
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
      z[i] = dinv[i] * r[i];
      rz_new += r[i] * z[i];
      rr_new += r[i] * r[i];
    }
    rr = rr_new;
    beta = rz != 0.0 ? rz_new / rz : 0.0;
    rz = rz_new;
    ++it;
  }
  return it;
}

/* One fractional step (FlowOracle.step).  State u (N,3), p (N), gp (N,3)
 * updated in place.  minv: 1/M_L; ufix: per-component mask (N,3 uint8) with
 * values ufv (N,3); pfix (N uint8).  work: 11 N doubles. */
int fc_step(fc_mesh* m, double rho, double mu, double cvr, double dt, int cg_iters, double cg_tol, double* u,
            double* p, double* gp, const double* minv, const uint8_t* ufix, const double* ufv, const uint8_t* pfix,
            int64_t nf, const int32_t* face, const int32_t* off, const int64_t* rp, const int32_t* ci,
            const double* av, const double* dinv, double* work) {
  const int64_t n = m->n;
  double *u0 = work, *us = work + 3 * n, *R = work + 6 * n, *b = work + 9 * n, *dp = work + 10 * n;
  double* gd = R;  /* reused after the stages */
  double* pcg_scr = (double*)malloc(sizeof(double) * 5 * (size_t)n);
  const double k = dt / rho;
  static const double A[3] = {0.0, 0.75, 1.0 / 3.0}, B[3] = {1.0, 0.25, 2.0 / 3.0};
  memcpy(u0, u, sizeof(double) * 3 * n);
  memcpy(us, u, sizeof(double) * 3 * n);
  for (int s = 0; s < 3; ++s) {
    fc_momentum(m, us, rho, mu, cvr, R);
    if (nf > 0) fc_wall(m, nf, face, off, us, rho, mu, R);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) {
        const int64_t j = 3 * i + d;
        double v = A[s] * u0[j] + B[s] * (us[j] + k * minv[i] * (R[j] - gp[j]));
        if (ufix && ufix[j]) v = ufv[j];
        us[j] = v;
      }
  }
  fc_divergence(m, us, -(rho / dt), b);
  if (pfix)
    for (int64_t i = 0; i < n; ++i)
      if (pfix[i]) b[i] = 0.0;
  const int it = fc_pcg(n, rp, ci, av, b, dinv, cg_iters, cg_tol, dp, pcg_scr);
  fc_gradient(m, dp, gd);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < 3; ++d) {
      const int64_t j = 3 * i + d;
      double v = us[j] - k * minv[i] * gd[j];
      if (ufix && ufix[j]) v = ufv[j];
      u[j] = v;
      gp[j] += gd[j];
    }
    p[i] += dp[i];
  }
  free(pcg_scr);
  return it;
}
