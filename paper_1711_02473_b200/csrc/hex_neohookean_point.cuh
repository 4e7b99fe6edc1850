// Pointwise part of the neo-Hookean residual (BASELINE config C4), shared by
// hex_neohookean.cu and hex_neohookean3.cu: from the nine reference-gradient
// values of the displacement at one quadrature point to the nine flux values
// the transposed contractions consume:
//   F = I + grad u,  J = det F,  F^-T = cof(F) / J,
//   P = mu (F - F^-T) + lambda ln(J) F^-T,
//   flux[a][l] = w sign(det Jg) sum_k adj(Jg)[l][k] P[a][k].
#pragma once

#include "hex_geometry.cuh"

#ifndef SFK_NEO_FASTLOG
#define SFK_NEO_FASTLOG 0   // measured slower (p = 4 0.657 -> 0.689 ms, r01di_*)
#endif

namespace sfk {

// ln J for the volumetric term.  Near J = 1 (every finite BASELINE point:
// |J - 1| is a few 1e-2) ln J = 2 atanh(z), z = (J - 1)/(J + 1), summed as
// 2z (1 + z^2/3 + ... + z^14/15): for |J - 1| < 1/16, |z| < 0.0323 and the
// truncation is below 1e-23 relative; the rounding of z and the Horner sum
// is a few ulp — far inside the 1e-12 gate.  Elsewhere (and for J <= 0,
// NaN as in the reference) the libm log.  Meant to replace a ~40-instruction
// dependent chain that was 13% of C4's stall samples
// (profiles/r01cn_C4_p4.md), but the branch and the extra code measured
// 2-5% slower than libm alone (profiles/r01di_*.jsonl): off by default.
__device__ __forceinline__ double neo_log(double J) {
  const double d = J - 1.0;
  if (SFK_NEO_FASTLOG && fabs(d) < 0.0625) {
    const double z = d * rcp64(J + 1.0);
    const double z2 = z * z;
    double t = 1.0 / 15.0;
    t = fma(t, z2, 1.0 / 13.0);
    t = fma(t, z2, 1.0 / 11.0);
    t = fma(t, z2, 1.0 / 9.0);
    t = fma(t, z2, 1.0 / 7.0);
    t = fma(t, z2, 1.0 / 5.0);
    t = fma(t, z2, 1.0 / 3.0);
    t = fma(t, z2, 1.0);
    return 2.0 * z * t;
  }
  return log(J);
}

// g[3a + l]: reference derivative l (0 x, 1 y, 2 z) of component a at the
// point with z-coordinate table value t = Bc[1][q]; w = w_qx w_qy w_qz.
// Overwrites g with the nine fluxes.
__device__ __forceinline__ void neo_point_flux(const HexLineAdj& geo, double t, double w,
                                               double mu, double lam, double g[9]) {
  double rr[3][3];
  const double det = geo.adj(t, rr[0], rr[1], rr[2]);
  const double idet = rcp64(det);
  // grad u_a [k] = (1/det) sum_l r_l[k] d_l u_a ;  F = I + grad u
  double F[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double g0 = g[3 * a];      // d_x
    const double g1 = g[3 * a + 1];  // d_y
    const double g2 = g[3 * a + 2];  // d_z
#pragma unroll
    for (int k = 0; k < 3; ++k)
      F[a][k] = fma(fma(g2, rr[2][k], fma(g1, rr[1][k], g0 * rr[0][k])), idet,
                    a == k ? 1.0 : 0.0);
  }
  double cof[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int a1 = (a + 1) % 3, a2 = (a + 2) % 3, k1 = (k + 1) % 3, k2 = (k + 2) % 3;
      cof[a][k] = fma(F[a1][k1], F[a2][k2], -(F[a1][k2] * F[a2][k1]));
    }
  const double Jf = fma(F[0][2], cof[0][2], fma(F[0][1], cof[0][1], F[0][0] * cof[0][0]));
  const double iJ = rcp64(Jf);
  // P = mu F + (lambda ln J - mu) / J * cof(F)
  const double beta = (lam * neo_log(Jf) - mu) * iJ;
  // flux f_a[l] = w sign(det) sum_k r_l[k] P[a][k]
  const double s = w * (det < 0.0 ? -1.0 : 1.0);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double P[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) P[k] = fma(mu, F[a][k], beta * cof[a][k]);
#pragma unroll
    for (int l = 0; l < 3; ++l)
      g[3 * a + l] = s * fma(rr[l][2], P[2], fma(rr[l][1], P[1], rr[l][0] * P[0]));
  }
}

}  // namespace sfk
