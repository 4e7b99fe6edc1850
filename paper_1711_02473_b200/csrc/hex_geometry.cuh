// Trilinear hex geometry evaluated on the fly per quadrature point.
//
// Reference semantics:
//   J[a][b] = sum_v coords[3v+a] * dPhi_v/dxhat_b(xi_q)  (geometry.py:42-64)
//   with Phi_v the P1 tensor basis, v = 4*ix + 2*iy + iz, P1 values
//   Bc[k][q] = (1-xi_q, xi_q) and derivatives Dc = (-1, +1) (exact);
//   G = J^-1 by the adjugate, S = |det J|            (geometry.py:71-108).
//
// Tensor structure used here: column b of J (dx/dxhat_b) does not depend on
// xi_b.  A thread that owns the quadrature line (qx, qy, *) therefore keeps
//   col2            constant along the line, and
//   col0, col1      affine in the P1 values at qz
// and forms each J in 12 FMAs instead of the 9 x 8-term sums of the
// reference loop nest.  The inverse is never formed: with rows
//   r0 = col1 x col2, r1 = col2 x col0, r2 = col0 x col1  (adj(J) rows),
// G = [r0; r1; r2] / det, and the Laplace flux is
//   f = (w/|det|) R R^T g ,  g = reference gradient,
// evaluated as two 3x3 mat-vecs.
#pragma once

#include "sfk_internal.cuh"

namespace sfk {

struct HexLineGeom {
  double al0[2][3];  // col0(qz) = al0[0]*Bc0[qz] + al0[1]*Bc1[qz]
  double al1[2][3];  // col1(qz) = al1[0]*Bc0[qz] + al1[1]*Bc1[qz]
  double c2[3];      // col2 (constant along z)

  // X: 24 coords of the cell (v = 4a+2b+c, comp inner); (bx0,bx1), (by0,by1)
  // the P1 values at the line's qx, qy.
  __device__ __forceinline__ void setup(const double* X, double bx0, double bx1,
                                        double by0, double by1) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
      for (int cz = 0; cz < 2; ++cz) {
        // d/dxhat_x: vertex pairs (1,b,cz) - (0,b,cz)
        const double e00 = X[3 * (4 + cz) + k] - X[3 * cz + k];
        const double e01 = X[3 * (6 + cz) + k] - X[3 * (2 + cz) + k];
        al0[cz][k] = fma(e01, by1, e00 * by0);
        // d/dxhat_y: (a,1,cz) - (a,0,cz)
        const double e10 = X[3 * (2 + cz) + k] - X[3 * cz + k];
        const double e11 = X[3 * (6 + cz) + k] - X[3 * (4 + cz) + k];
        al1[cz][k] = fma(e11, bx1, e10 * bx0);
      }
      // d/dxhat_z: (a,b,1) - (a,b,0)
      const double f00 = X[3 * 1 + k] - X[3 * 0 + k];
      const double f01 = X[3 * 3 + k] - X[3 * 2 + k];
      const double f10 = X[3 * 5 + k] - X[3 * 4 + k];
      const double f11 = X[3 * 7 + k] - X[3 * 6 + k];
      c2[k] = fma(fma(f11, by1, f10 * by0), bx1, fma(f01, by1, f00 * by0) * bx0);
    }
  }

    // Same from the cell's 36 edge differences precomputed once per cell by
  // hex_cell_edges (every line of the cell shares them): identical roundings.
  __device__ __forceinline__ void setup_edges(const double* E, double bx0, double bx1,
                                              double by0, double by1) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
      for (int cz = 0; cz < 2; ++cz) {
        const double* e = E + 4 * (3 * cz + k);
        al0[cz][k] = fma(e[1], by1, e[0] * by0);
        al1[cz][k] = fma(e[3], bx1, e[2] * bx0);
      }
      const double* f = E + 24 + 4 * k;
      c2[k] = fma(fma(f[3], by1, f[2] * by0), bx1, fma(f[1], by1, f[0] * by0) * bx0);
    }
  }

  // Same from the cell's per-line-family table (hex_cell_lg): al0 depends on
  // qy only, al1 on qx only, c2 = g1 bx1 + g0 bx0 with g depending on qy
  // only — identical operations and roundings, 6 FP64 ops instead of 78.
  __device__ __forceinline__ void setup_lg(const double* LG, int n, int qx, int qy, double bx0,
                                           double bx1) {
    const double* a0 = LG + 6 * qy;
    const double* a1 = LG + 6 * n + 6 * qx;
    const double* g = LG + 12 * n + 6 * qy;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
      for (int cz = 0; cz < 2; ++cz) {
        al0[cz][k] = a0[3 * cz + k];
        al1[cz][k] = a1[3 * cz + k];
      }
      c2[k] = fma(g[3 + k], bx1, g[k] * bx0);
    }
  }

  // Adjugate rows and determinant at the point with P1 z-values (b0, b1).
  __device__ __forceinline__ double adj(double b0, double b1, double r0[3],
                                        double r1[3], double r2[3]) const {
    double c0[3], c1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      c0[k] = fma(al0[1][k], b1, al0[0][k] * b0);
      c1[k] = fma(al1[1][k], b1, al1[0][k] * b0);
    }
    cross(c1, c2, r0);
    cross(c2, c0, r1);
    cross(c0, c1, r2);
    return fma(c0[2], r0[2], fma(c0[1], r0[1], c0[0] * r0[0]));
  }

  static __device__ __forceinline__ void cross(const double a[3], const double b[3],
                                               double o[3]) {
    o[0] = fma(a[1], b[2], -(a[2] * b[1]));
    o[1] = fma(a[2], b[0], -(a[0] * b[2]));
    o[2] = fma(a[0], b[1], -(a[1] * b[0]));
  }
};

// Same geometry with the adjugate rows precomputed as polynomials in the z
// point t = xi_z (= the P1 table value Bc1[qz]) along the line:
//   col0 = A + t dA,  col1 = B + t dB  (A = al0[0], dA = al0[1] - al0[0], ...)
//   r0 = col1 x col2 = P0 + t Q0          (col2 constant along the line)
//   r1 = col2 x col0 = P1 + t Q1
//   r2 = col0 x col1 = S0 + t (S1 + t S2)
//   det = col2 . r2
// 15 FP64 ops per point instead of 33 (the setup's 7 cross products are
// shared by the line's m points).  The affine form uses 1 - t for the table
// value Bc0[qz]; they differ by at most an ulp (a 1e-16 relative change of J).
struct HexLineAdj {
  double P0[3], Q0[3], P1[3], Q1[3], S0[3], S1[3], S2[3], c2[3];

  __device__ __forceinline__ void setup(const double* X, double bx0, double bx1, double by0,
                                        double by1) {
    HexLineGeom g;
    g.setup(X, bx0, bx1, by0, by1);
    from_geom(g);
  }
  __device__ __forceinline__ void setup_edges(const double* E, double bx0, double bx1,
                                              double by0, double by1) {
    HexLineGeom g;
    g.setup_edges(E, bx0, bx1, by0, by1);
    from_geom(g);
  }
  __device__ __forceinline__ void setup_lg(const double* LG, int n, int qx, int qy, double bx0,
                                           double bx1) {
    HexLineGeom g;
    g.setup_lg(LG, n, qx, qy, bx0, bx1);
    from_geom(g);
  }
  __device__ __forceinline__ void from_geom(const HexLineGeom& g) {
    double A[3], dA[3], B[3], dB[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      A[k] = g.al0[0][k];
      dA[k] = g.al0[1][k] - g.al0[0][k];
      B[k] = g.al1[0][k];
      dB[k] = g.al1[1][k] - g.al1[0][k];
    }
    from_parts(A, dA, B, dB, g.c2);
  }
  // From the line's column polynomials: col0 = A + t dA (A, dA depend on qy
  // only), col1 = B + t dB (qx only), col2 = cc — callers that share A, dA
  // (or B, dB) between the lines of a cell form them once (identical roundings).
  __device__ __forceinline__ void from_parts(const double A[3], const double dA[3],
                                             const double B[3], const double dB[3],
                                             const double cc[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) c2[k] = cc[k];
    HexLineGeom::cross(B, c2, P0);
    HexLineGeom::cross(dB, c2, Q0);
    HexLineGeom::cross(c2, A, P1);
    HexLineGeom::cross(c2, dA, Q1);
    double u[3], v[3];
    HexLineGeom::cross(A, B, S0);
    HexLineGeom::cross(A, dB, u);
    HexLineGeom::cross(dA, B, v);
    HexLineGeom::cross(dA, dB, S2);
#pragma unroll
    for (int k = 0; k < 3; ++k) S1[k] = u[k] + v[k];
  }

  __device__ __forceinline__ double adj(double t, double r0[3], double r1[3],
                                        double r2[3]) const {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      r0[k] = fma(t, Q0[k], P0[k]);
      r1[k] = fma(t, Q1[k], P1[k]);
      r2[k] = fma(t, fma(t, S2[k], S1[k]), S0[k]);
    }
    return fma(c2[2], r2[2], fma(c2[1], r2[1], c2[0] * r2[0]));
  }
};

// The 36 edge differences of a cell's vertices that HexLineGeom::setup forms
// (X: 24 coords, v = 4a+2b+c, component inner), in setup_edges' order:
//   E[4*(3*cz+k) + 0..3] = x-edges (b = 0, 1) and y-edges (a = 0, 1) at z = cz
//   E[24 + 4*k + 0..3]   = z-edges (a, b) = (0,0), (0,1), (1,0), (1,1)
// Entry e of the 36 (callers spread e over threads).
__device__ __forceinline__ double hex_cell_edge(const double* X, int e) {
  if (e < 24) {
    const int g = e >> 2, w = e & 3, cz = g / 3, k = g - 3 * cz;
    switch (w) {
      case 0: return X[3 * (4 + cz) + k] - X[3 * cz + k];        // e00
      case 1: return X[3 * (6 + cz) + k] - X[3 * (2 + cz) + k];  // e01
      case 2: return X[3 * (2 + cz) + k] - X[3 * cz + k];        // e10
      default: return X[3 * (6 + cz) + k] - X[3 * (4 + cz) + k]; // e11
    }
  }
  const int k = (e - 24) >> 2, w = (e - 24) & 3;   // f00, f01, f10, f11
  const int v0 = 2 * w;                             // (a, b) = (w >> 1, w & 1), c = 0
  return X[3 * (v0 + 1) + k] - X[3 * v0 + k];
}

// Per-cell line-geometry table (18 n doubles), entry e:
//   [0, 6n)    al0[qy][cz][k]  = e01 by1(qy) + e00 by0(qy)   (x-edges, b = 0 / 1)
//   [6n, 12n)  al1[qx][cz][k]  = e11 bx1(qx) + e10 bx0(qx)   (y-edges, a = 0 / 1)
//   [12n, 18n) g[qy][w][k]     w = 0: f01 by1 + f00 by0, w = 1: f11 by1 + f10 by0
// with exactly HexLineGeom::setup's operations; Bc[q], Bc[n + q] = P1 values.
__device__ __forceinline__ double hex_cell_lg(const double* X, const double* Bc, int n, int e) {
  const int part = e / (6 * n), r = e - part * 6 * n;
  const int q = r / 6, j = r - 6 * q, hi = j / 3, k = j - 3 * hi;   // hi = cz or w
  const double b0 = Bc[q], b1 = Bc[n + q];
  if (part == 0) {
    const double e00 = X[3 * (4 + hi) + k] - X[3 * hi + k];
    const double e01 = X[3 * (6 + hi) + k] - X[3 * (2 + hi) + k];
    return fma(e01, b1, e00 * b0);
  }
  if (part == 1) {
    const double e10 = X[3 * (2 + hi) + k] - X[3 * hi + k];
    const double e11 = X[3 * (6 + hi) + k] - X[3 * (4 + hi) + k];
    return fma(e11, b1, e10 * b0);
  }
  // w = hi: (a = hi) z-edges (hi, 0) and (hi, 1)
  const double fl = X[3 * (4 * hi + 1) + k] - X[3 * (4 * hi) + k];       // f(a,0)
  const double fh = X[3 * (4 * hi + 3) + k] - X[3 * (4 * hi + 2) + k];   // f(a,1)
  return fma(fh, b1, fl * b0);
}

// f = s * R R^T g  (R rows r0, r1, r2).  In place on (g0, g1, g2).
__device__ __forceinline__ void laplace_flux(const double r0[3], const double r1[3],
                                             const double r2[3], double s,
                                             double& g0, double& g1, double& g2) {
  const double h0 = g0 * s, h1 = g1 * s, h2 = g2 * s;
  double v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = fma(h2, r2[k], fma(h1, r1[k], h0 * r0[k]));
  g0 = fma(r0[2], v[2], fma(r0[1], v[1], r0[0] * v[0]));
  g1 = fma(r1[2], v[2], fma(r1[1], v[1], r1[0] * v[0]));
  g2 = fma(r2[2], v[2], fma(r2[1], v[1], r2[0] * v[0]));
}

}  // namespace sfk
