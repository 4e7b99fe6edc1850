/*
 * oracle/sumfact_oracle.c — CPU restatement of the reference's per-cell
 * kernels.  TEST INFRASTRUCTURE ONLY: imported by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * legs as the CHECKER or the CPU baseline, never by the product path.
 *
 * What it restates (reference = /root/reference/pkg/src/sumfact):
 *   - geometry: J[a][b] = sum_v coords[3v+a] dPhi_v/dxhat_b (geometry.py:42-64)
 *     with the P1 tables Bc/Dc; det by cofactor expansion along row 0 and
 *     G[a][b] = cof(b,a)/det, (a+b) odd negated (geometry.py:71-99);
 *     S = |det| (geometry.py:102-108);
 *   - physical gradient (grad f)_k = sum_l G[l][k] d_l f (forms.py:181-183);
 *   - integrands: _mass v*u (forms.py:173), _laplace sum_k (grad v)_k
 *     (grad u)_k (forms.py:186-189), _weighted_laplace kappa*laplace
 *     (forms.py:192-193), scaled by w_q * S_q and summed over the points
 *     (forms.py:392-395);
 *   - coefficient evaluation by per-axis 1D contractions, i.e. the
 *     spectral-mode sum-factorised schedule of passes.py:672-743 (x, then y,
 *     then z, transposed in reverse);
 *   - the neo-Hookean residual of SURVEY.md §8(a) row a17 (no reference
 *     form exists; SPEC.md:8, 387 declare it out of scope).
 * Layouts: SURVEY.md Appendix A (dof (ix*n+iy)*n+iz, vector dof *3+comp,
 * coords v = 4a+2b+c, A zero-filled then accumulated, scheduling.py:372).
 * Tables are basis-major T[i*m + q] exactly as the emitted C indexes them.
 *
 * Cell loops are OpenMP-parallel (static schedule); each cell is independent
 * (the emitted kernels are reentrant).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXN 17
#define MAXM 18

typedef struct {
  int n, m;
  const double *B, *D, *w, *Bc, *Dc;
} tabs_t;

/* ---- geometry (reference geometry.py:42-99) -------------------------- */
static void hex_jacobian(const tabs_t *t, const double *X, int qx, int qy, int qz,
                         double J[3][3]) {
  const int m = t->m;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) J[a][b] = 0.0;
  for (int va = 0; va < 2; ++va)
    for (int vb = 0; vb < 2; ++vb)
      for (int vc = 0; vc < 2; ++vc) {
        const int v = 4 * va + 2 * vb + vc;
        const double bx = t->Bc[va * m + qx], by = t->Bc[vb * m + qy], bz = t->Bc[vc * m + qz];
        const double dx = t->Dc[va * m + qx], dy = t->Dc[vb * m + qy], dz = t->Dc[vc * m + qz];
        const double dphi[3] = {dx * by * bz, bx * dy * bz, bx * by * dz};
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) J[a][b] += X[3 * v + a] * dphi[b];
      }
}

static double minor3(const double J[3][3], int r, int c) {
  int rs[2], cs[2], k = 0, l = 0;
  for (int i = 0; i < 3; ++i) {
    if (i != r) rs[k++] = i;
    if (i != c) cs[l++] = i;
  }
  return J[rs[0]][cs[0]] * J[rs[1]][cs[1]] - J[rs[0]][cs[1]] * J[rs[1]][cs[0]];
}

/* G = J^-1 by the adjugate; returns det (reference geometry.py:71-99). */
static double inverse_and_det3(const double J[3][3], double G[3][3]) {
  const double det = (J[0][0] * minor3(J, 0, 0) - J[0][1] * minor3(J, 0, 1)) +
                     J[0][2] * minor3(J, 0, 2);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double cof = minor3(J, b, a);
      if ((a + b) % 2) cof = -cof;
      G[a][b] = cof / det;
    }
  return det;
}

/* ---- 1D contraction helpers ------------------------------------------ */
/* out[..q..] = sum_i T[i*m+q] in[..i..] along one axis of a 3D box.
 * in has extents (e0,e1,e2) with `axis` of extent n, out the same with m. */
static void contract3(const double *T, int n, int m, int axis, const int ein[3],
                      const double *in, double *out, int transpose) {
  /* transpose=0: in extent n -> out extent m using T[i*m+q]
   * transpose=1: in extent m -> out extent n using T[i*m+q] (sum over q) */
  int eo[3] = {ein[0], ein[1], ein[2]};
  eo[axis] = transpose ? n : m;
  const int so[3] = {eo[1] * eo[2], eo[2], 1};
  const int si[3] = {ein[1] * ein[2], ein[2], 1};
  for (int a = 0; a < eo[0]; ++a)
    for (int b = 0; b < eo[1]; ++b)
      for (int c = 0; c < eo[2]; ++c) {
        const int idx[3] = {a, b, c};
        double s = 0.0;
        const int kext = ein[axis];
        for (int k = 0; k < kext; ++k) {
          int ii[3] = {a, b, c};
          ii[axis] = k;
          const double tv = transpose ? T[idx[axis] * m + k] : T[k * m + idx[axis]];
          s += tv * in[ii[0] * si[0] + ii[1] * si[1] + ii[2] * si[2]];
        }
        out[a * so[0] + b * so[1] + c * so[2]] = s;
      }
}

/* reference gradient of a scalar field at the m^3 points:
 * g[l][q] = d_l u(q), via x -> y -> z contractions (8 nests). */
static void ref_gradient(const tabs_t *t, const double *u, double *g /* 3*m^3 */,
                         double *w1, double *w2, double *w3) {
  const int n = t->n, m = t->m;
  const int e0[3] = {n, n, n};
  const int e1[3] = {m, n, n};
  const int e2[3] = {m, m, n};
  const int M3 = m * m * m;
  double *bx = w1, *dx = w1 + m * n * n;
  contract3(t->B, n, m, 0, e0, u, bx, 0);
  contract3(t->D, n, m, 0, e0, u, dx, 0);
  double *bb = w2, *bd = w2 + m * m * n, *db = w2 + 2 * m * m * n;
  contract3(t->B, n, m, 1, e1, bx, bb, 0);
  contract3(t->D, n, m, 1, e1, bx, bd, 0);
  contract3(t->B, n, m, 1, e1, dx, db, 0);
  contract3(t->B, n, m, 2, e2, db, g + 0 * M3, 0);
  contract3(t->B, n, m, 2, e2, bd, g + 1 * M3, 0);
  contract3(t->D, n, m, 2, e2, bb, g + 2 * M3, 0);
  (void)w3;
}

/* A += sum_q sum_l d_l phi_i(q) f[l][q]  (transposed schedule). */
static void ref_gradient_transpose(const tabs_t *t, const double *f /* 3*m^3 */, double *A,
                                   double *w1, double *w2, double *w3) {
  const int n = t->n, m = t->m;
  const int M3 = m * m * m;
  const int eq[3] = {m, m, m};
  const int e2[3] = {m, m, n};
  const int e1[3] = {m, n, n};
  double *sx = w2, *sy = w2 + m * m * n, *sz = w2 + 2 * m * m * n;
  contract3(t->B, n, m, 2, eq, f + 0 * M3, sx, 1);
  contract3(t->B, n, m, 2, eq, f + 1 * M3, sy, 1);
  contract3(t->D, n, m, 2, eq, f + 2 * M3, sz, 1);
  double *r1 = w1, *r2 = w1 + m * n * n, *tmp = w3;
  contract3(t->B, n, m, 1, e2, sx, r1, 1);
  contract3(t->D, n, m, 1, e2, sy, r2, 1);
  contract3(t->B, n, m, 1, e2, sz, tmp, 1);
  for (int i = 0; i < m * n * n; ++i) r2[i] += tmp[i];
  double *a1 = w3, *a2 = w3 + n * n * n;
  contract3(t->D, n, m, 0, e1, r1, a1, 1);
  contract3(t->B, n, m, 0, e1, r2, a2, 1);
  for (int i = 0; i < n * n * n; ++i) A[i] += a1[i] + a2[i];
}

/* ---- C2: hex Laplace action (forms.py:186-189 via action_form) -------- */
void oracle_hex_laplace_action(int n, int m, const double *B, const double *D,
                               const double *w, const double *Bc, const double *Dc,
                               int64_t ncells, const double *coords, const double *u,
                               double *A) {
  const tabs_t t = {n, m, B, D, w, Bc, Dc};
  const int N3 = n * n * n, M3 = m * m * m;
#pragma omp parallel
  {
    const size_t wsz = (size_t)3 * MAXM * MAXM * MAXM;
    double *g = (double *)malloc(sizeof(double) * 3 * M3);
    double *w1 = (double *)malloc(sizeof(double) * wsz);
    double *w2 = (double *)malloc(sizeof(double) * wsz);
    double *w3 = (double *)malloc(sizeof(double) * wsz);
#pragma omp for schedule(static)
    for (int64_t c = 0; c < ncells; ++c) {
      const double *X = coords + 24 * c;
      double *a = A + N3 * c;
      memset(a, 0, sizeof(double) * N3);
      ref_gradient(&t, u + N3 * c, g, w1, w2, w3);
      for (int qx = 0; qx < m; ++qx)
        for (int qy = 0; qy < m; ++qy)
          for (int qz = 0; qz < m; ++qz) {
            const int q = (qx * m + qy) * m + qz;
            double J[3][3], G[3][3];
            hex_jacobian(&t, X, qx, qy, qz, J);
            const double det = inverse_and_det3(J, G);
            const double scale = (w[qx] * w[qy] * w[qz]) * fabs(det);
            double gu[3];
            for (int k = 0; k < 3; ++k)
              gu[k] = G[0][k] * g[q] + G[1][k] * g[M3 + q] + G[2][k] * g[2 * M3 + q];
            for (int l = 0; l < 3; ++l)
              g[l * M3 + q] = scale * (G[l][0] * gu[0] + G[l][1] * gu[1] + G[l][2] * gu[2]);
          }
      ref_gradient_transpose(&t, g, a, w1, w2, w3);
    }
    free(g);
    free(w1);
    free(w2);
    free(w3);
  }
}

/* ---- C3: GLL-collocated (weighted) Laplace action --------------------- */
/* B = I (Delta tabulation, elements.py:214-216): d_l u needs one
 * D-contraction along axis l; kappa at point q is w1[q] (Delta property). */
void oracle_hex_colloc_action(int n, const double *D, const double *w, const double *Bc,
                              const double *Dc, int64_t ncells, const double *coords,
                              const double *u, const double *kappa, double *A) {
  const tabs_t t = {n, n, NULL, D, w, Bc, Dc};
  const int N3 = n * n * n;
  const int e[3] = {n, n, n};
#pragma omp parallel
  {
    double *g = (double *)malloc(sizeof(double) * 3 * N3);
    double *tmp = (double *)malloc(sizeof(double) * N3);
#pragma omp for schedule(static)
    for (int64_t c = 0; c < ncells; ++c) {
      const double *X = coords + 24 * c;
      const double *uc = u + N3 * c;
      double *a = A + N3 * c;
      memset(a, 0, sizeof(double) * N3);
      for (int l = 0; l < 3; ++l) contract3(D, n, n, l, e, uc, g + l * N3, 0);
      for (int qx = 0; qx < n; ++qx)
        for (int qy = 0; qy < n; ++qy)
          for (int qz = 0; qz < n; ++qz) {
            const int q = (qx * n + qy) * n + qz;
            double J[3][3], G[3][3];
            hex_jacobian(&t, X, qx, qy, qz, J);
            const double det = inverse_and_det3(J, G);
            double scale = (w[qx] * w[qy] * w[qz]) * fabs(det);
            if (kappa) scale *= kappa[N3 * c + q];
            double gu[3];
            for (int k = 0; k < 3; ++k)
              gu[k] = G[0][k] * g[q] + G[1][k] * g[N3 + q] + G[2][k] * g[2 * N3 + q];
            for (int l = 0; l < 3; ++l)
              g[l * N3 + q] = scale * (G[l][0] * gu[0] + G[l][1] * gu[1] + G[l][2] * gu[2]);
          }
      for (int l = 0; l < 3; ++l) {
        contract3(D, n, n, l, e, g + l * N3, tmp, 1);
        for (int i = 0; i < N3; ++i) a[i] += tmp[i];
      }
    }
    free(g);
    free(tmp);
  }
}

/* ---- C1: quad mass / Laplace action ----------------------------------- */
static void quad_geometry(const tabs_t *t, const double *X, int qx, int qy, double G[2][2],
                          double *det) {
  const int m = t->m;
  double J[2][2] = {{0, 0}, {0, 0}};
  for (int va = 0; va < 2; ++va)
    for (int vb = 0; vb < 2; ++vb) {
      const int v = 2 * va + vb;
      const double dphi[2] = {t->Dc[va * m + qx] * t->Bc[vb * m + qy],
                              t->Bc[va * m + qx] * t->Dc[vb * m + qy]};
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) J[a][b] += X[2 * v + a] * dphi[b];
    }
  /* reference geometry.py:83-87 */
  const double d = J[0][0] * J[1][1] + -(J[0][1] * J[1][0]);
  G[0][0] = J[1][1] / d;
  G[0][1] = -J[0][1] / d;
  G[1][0] = -J[1][0] / d;
  G[1][1] = J[0][0] / d;
  *det = d;
}

/* which: 0 = mass (forms.py:173), 1 = Laplace (forms.py:186-189) */
void oracle_quad_action(int which, int n, int m, const double *B, const double *D,
                        const double *w, const double *Bc, const double *Dc, int64_t ncells,
                        const double *coords, const double *u, double *A) {
  const tabs_t t = {n, m, B, D, w, Bc, Dc};
  const int N2 = n * n;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < ncells; ++c) {
    const double *X = coords + 8 * c;
    const double *uc = u + N2 * c;
    double *a = A + N2 * c;
    memset(a, 0, sizeof(double) * N2);
    for (int qx = 0; qx < m; ++qx)
      for (int qy = 0; qy < m; ++qy) {
        double G[2][2], det;
        quad_geometry(&t, X, qx, qy, G, &det);
        const double scale = (w[qx] * w[qy]) * fabs(det);
        double val = 0, g0 = 0, g1 = 0;
        for (int ix = 0; ix < n; ++ix)
          for (int iy = 0; iy < n; ++iy) {
            const double ui = uc[ix * n + iy];
            val += B[ix * m + qx] * B[iy * m + qy] * ui;
            g0 += D[ix * m + qx] * B[iy * m + qy] * ui;
            g1 += B[ix * m + qx] * D[iy * m + qy] * ui;
          }
        double f0 = 0, f1 = 0;
        if (which == 1) {
          const double gu0 = G[0][0] * g0 + G[1][0] * g1;
          const double gu1 = G[0][1] * g0 + G[1][1] * g1;
          f0 = scale * (G[0][0] * gu0 + G[0][1] * gu1);
          f1 = scale * (G[1][0] * gu0 + G[1][1] * gu1);
        }
        for (int ix = 0; ix < n; ++ix)
          for (int iy = 0; iy < n; ++iy) {
            if (which == 0)
              a[ix * n + iy] += scale * B[ix * m + qx] * B[iy * m + qy] * val;
            else
              a[ix * n + iy] += D[ix * m + qx] * B[iy * m + qy] * f0 +
                                B[ix * m + qx] * D[iy * m + qy] * f1;
          }
      }
  }
}

/* ---- C5: hex Laplace local matrix (registry `laplace`) ---------------- */
/* A[i*N3 + j] = sum_q w S sum_k (grad phi_i)_k (grad phi_j)_k, test-major
 * (forms.py:402-408).  Per point: K = w S G G^T, then rank-3 updates. */
void oracle_hex_laplace_matrix(int n, int m, const double *B, const double *D,
                               const double *w, const double *Bc, const double *Dc,
                               int64_t ncells, const double *coords, double *A) {
  const tabs_t t = {n, m, B, D, w, Bc, Dc};
  const int N3 = n * n * n;
#pragma omp parallel
  {
    double *dphi = (double *)malloc(sizeof(double) * 3 * N3);
    double *kd = (double *)malloc(sizeof(double) * 3 * N3);
#pragma omp for schedule(static)
    for (int64_t c = 0; c < ncells; ++c) {
      const double *X = coords + 24 * c;
      double *a = A + (int64_t)N3 * N3 * c;
      memset(a, 0, sizeof(double) * (size_t)N3 * N3);
      for (int qx = 0; qx < m; ++qx)
        for (int qy = 0; qy < m; ++qy)
          for (int qz = 0; qz < m; ++qz) {
            double J[3][3], G[3][3];
            hex_jacobian(&t, X, qx, qy, qz, J);
            const double det = inverse_and_det3(J, G);
            const double scale = (w[qx] * w[qy] * w[qz]) * fabs(det);
            double K[3][3];
            for (int l = 0; l < 3; ++l)
              for (int r = 0; r < 3; ++r)
                K[l][r] = scale * (G[l][0] * G[r][0] + G[l][1] * G[r][1] + G[l][2] * G[r][2]);
            for (int ix = 0; ix < n; ++ix)
              for (int iy = 0; iy < n; ++iy)
                for (int iz = 0; iz < n; ++iz) {
                  const int i = (ix * n + iy) * n + iz;
                  dphi[i] = D[ix * m + qx] * B[iy * m + qy] * B[iz * m + qz];
                  dphi[N3 + i] = B[ix * m + qx] * D[iy * m + qy] * B[iz * m + qz];
                  dphi[2 * N3 + i] = B[ix * m + qx] * B[iy * m + qy] * D[iz * m + qz];
                }
            for (int l = 0; l < 3; ++l)
              for (int i = 0; i < N3; ++i)
                kd[l * N3 + i] = K[l][0] * dphi[i] + K[l][1] * dphi[N3 + i] +
                                 K[l][2] * dphi[2 * N3 + i];
            for (int i = 0; i < N3; ++i) {
              const double d0 = dphi[i], d1 = dphi[N3 + i], d2 = dphi[2 * N3 + i];
              double *row = a + (int64_t)i * N3;
              for (int j = 0; j < N3; ++j)
                row[j] += d0 * kd[j] + d1 * kd[N3 + j] + d2 * kd[2 * N3 + j];
            }
          }
    }
    free(dphi);
    free(kd);
  }
}

/* ---- C4: neo-Hookean residual --------------- */
/* F = I + grad u (physical), J = det F, F^-T = cof(F)/J,
 * P = mu (F - F^-T) + lambda ln(J) F^-T,
 * r_(i,a) = sum_q w S sum_k P[a][k] (grad phi_i)_k. */
void oracle_hex_neohookean(int n, int m, const double *B, const double *D, const double *w,
                           const double *Bc, const double *Dc, double mu, double lam,
                           int64_t ncells, const double *coords, const double *u, double *A) {
  const tabs_t t = {n, m, B, D, w, Bc, Dc};
  const int N3 = n * n * n, M3 = m * m * m;
#pragma omp parallel
  {
    const size_t wsz = (size_t)3 * MAXM * MAXM * MAXM;
    double *uc = (double *)malloc(sizeof(double) * N3);
    double *g = (double *)malloc(sizeof(double) * 3 * 3 * M3);
    double *ac = (double *)malloc(sizeof(double) * N3);
    double *w1 = (double *)malloc(sizeof(double) * wsz);
    double *w2 = (double *)malloc(sizeof(double) * wsz);
    double *w3 = (double *)malloc(sizeof(double) * wsz);
#pragma omp for schedule(static)
    for (int64_t c = 0; c < ncells; ++c) {
      const double *X = coords + 24 * c;
      double *a = A + 3 * N3 * c;
      memset(a, 0, sizeof(double) * 3 * N3);
      for (int comp = 0; comp < 3; ++comp) {
        for (int i = 0; i < N3; ++i) uc[i] = u[3 * N3 * c + 3 * i + comp];
        ref_gradient(&t, uc, g + comp * 3 * M3, w1, w2, w3);
      }
      for (int qx = 0; qx < m; ++qx)
        for (int qy = 0; qy < m; ++qy)
          for (int qz = 0; qz < m; ++qz) {
            const int q = (qx * m + qy) * m + qz;
            double J[3][3], G[3][3];
            hex_jacobian(&t, X, qx, qy, qz, J);
            const double det = inverse_and_det3(J, G);
            const double scale = (w[qx] * w[qy] * w[qz]) * fabs(det);
            double F[3][3];
            for (int aa = 0; aa < 3; ++aa)
              for (int k = 0; k < 3; ++k) {
                const double *ga = g + aa * 3 * M3;
                const double gk = G[0][k] * ga[q] + G[1][k] * ga[M3 + q] + G[2][k] * ga[2 * M3 + q];
                F[aa][k] = (aa == k ? 1.0 : 0.0) + gk;
              }
            double Jf = (F[0][0] * minor3(F, 0, 0) - F[0][1] * minor3(F, 0, 1)) +
                        F[0][2] * minor3(F, 0, 2);
            const double lnJ = log(Jf);
            for (int aa = 0; aa < 3; ++aa) {
              double P[3];
              for (int k = 0; k < 3; ++k) {
                double cof = minor3(F, aa, k);
                if ((aa + k) % 2) cof = -cof;
                const double finvT = cof / Jf;
                P[k] = mu * (F[aa][k] - finvT) + (lam * lnJ) * finvT;
              }
              /* flux for test component aa: f_l = scale sum_k G[l][k] P[k] */
              double *ga = g + aa * 3 * M3;
              for (int l = 0; l < 3; ++l)
                ga[l * M3 + q] = scale * (G[l][0] * P[0] + G[l][1] * P[1] + G[l][2] * P[2]);
            }
          }
      for (int comp = 0; comp < 3; ++comp) {
        memset(ac, 0, sizeof(double) * N3);
        ref_gradient_transpose(&t, g + comp * 3 * M3, ac, w1, w2, w3);
        for (int i = 0; i < N3; ++i) a[3 * i + comp] = ac[i];
      }
    }
    free(uc);
    free(g);
    free(ac);
    free(w1);
    free(w2);
    free(w3);
  }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
