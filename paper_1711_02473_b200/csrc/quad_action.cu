// Quad Q_p mass and Laplace actions, fused over shared inputs — BASELINE
// config C1 (Q3, GL(4)^2, 1024 cells: b_M = M u and b_K = K u).
//
// Reference: registry `action_mass` / `action_laplace` on `quad`
// (forms.py:173, 186-189, 261-263), 2D geometry geometry.py:80-87
// (J from the P1 coordinate element, closed-form 2x2 inverse, S = |det|).
// Spectral schedule: x stage {B, D} u; y stage B(Bx u) [value],
// D(Bx u) [d_y], B(Dx u) [d_x]; pointwise; transposed y then x.
//
// B200 mapping: thread per (cell, line); x-lines -> smem -> y-lines (which
// also run the pointwise transform and the transposed y contraction in
// registers) -> smem -> x-lines write A.  Both outputs come from one pass
// over (coords, u): the mass and Laplace kernels share the x/y forward
// contractions.  C1 is launch-bound (1024 cells = 16 KB of dofs), so the
// CTA is one warp of 8 cells to spread the batch over many SMs.
#include "hex_geometry.cuh"

namespace sfk {

template <int N, int M, int CPB, bool MASS, bool LAP>
__global__ void __launch_bounds__(round_up(CPB * (M > N ? M : N), 32))
quad_action_kernel(const __grid_constant__ Tabs<N, M> T, int64_t ncells,
                   const double* __restrict__ coords, const double* __restrict__ u,
                   double* __restrict__ Amass, double* __restrict__ Alap) {
  constexpr int L = M > N ? M : N;
  constexpr int PL = N | 1;  // padded line length
  // per cell: X0, X1 [M][PL]  then  Sm, Sx, Sy [M][PL]
  constexpr int CS = 3 * M * PL;
  __shared__ double sbuf[CPB * CS];
  __shared__ double sC[CPB * 8];
  const int tid = threadIdx.x;
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int64_t rem = ncells - cell0;
  const int ncb = rem < CPB ? (int)rem : CPB;
  for (int i = tid; i < CPB * 8; i += blockDim.x)
    sC[i] = i < ncb * 8 ? __ldg(coords + cell0 * 8 + i) : 0.0;
  const int c = tid / L, line = tid - (tid / L) * L;
  const bool on = c < CPB;
  double* cb = sbuf + c * CS;

  // ---- x-lines (iy = line): X0 = Bx u, X1 = Dx u --------------------
  if (on && line < N) {
    double ul[N];
#pragma unroll
    for (int i = 0; i < N; ++i)
      ul[i] = c < ncb ? __ldg(u + (cell0 + c) * (N * N) + i * N + line) : 0.0;
#pragma unroll
    for (int q = 0; q < M; ++q) {
      double b = T.B[q] * ul[0], d = T.D[q] * ul[0];
#pragma unroll
      for (int i = 1; i < N; ++i) {
        b = fma(T.B[i * M + q], ul[i], b);
        d = fma(T.D[i * M + q], ul[i], d);
      }
      cb[q * PL + line] = b;
      cb[M * PL + q * PL + line] = d;
    }
  }
  __syncthreads();

  // ---- y-lines (qx = line): values/gradients, flux, transposed y ------
  double sm[N], sx[N], sy[N];
  if (on && line < M) {
    const int qx = line;
    double x0[N], x1[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      x0[i] = cb[qx * PL + i];
      x1[i] = cb[M * PL + qx * PL + i];
      sm[i] = sx[i] = sy[i] = 0.0;
    }
    const double* X = sC + c * 8;
    // col1 = d x / d eta: constant along the line; col0 affine in Bc(qy)
    const double bx0 = T.Bc[qx], bx1 = T.Bc[M + qx];
    double c1[2], e0[2][2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      c1[k] = fma(X[2 * 3 + k] - X[2 * 2 + k], bx1, (X[2 * 1 + k] - X[k]) * bx0);
      e0[0][k] = X[2 * 2 + k] - X[k];          // (1,0) - (0,0)
      e0[1][k] = X[2 * 3 + k] - X[2 * 1 + k];  // (1,1) - (0,1)
    }
#pragma unroll
    for (int q = 0; q < M; ++q) {
      double val = T.B[q] * x0[0], gy = T.D[q] * x0[0], gx = T.B[q] * x1[0];
#pragma unroll
      for (int i = 1; i < N; ++i) {
        val = fma(T.B[i * M + q], x0[i], val);
        gy = fma(T.D[i * M + q], x0[i], gy);
        gx = fma(T.B[i * M + q], x1[i], gx);
      }
      double c0[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) c0[k] = fma(e0[1][k], T.Bc[M + q], e0[0][k] * T.Bc[q]);
      const double det = fma(c0[0], c1[1], -(c1[0] * c0[1]));
      const double w = T.W[qx] * T.W[q];
      double fm = 0, fx = 0, fy = 0;
      if (MASS) fm = (w * fabs(det)) * val;
      if (LAP) {
        // adjugate rows r0 = (c1y, -c1x), r1 = (-c0y, c0x); f = w/|det| R R^T g
        const double s = w * rcp64(fabs(det));
        const double h0 = gx * s, h1 = gy * s;
        const double v0 = fma(h1, -c0[1], h0 * c1[1]);
        const double v1 = fma(h1, c0[0], -(h0 * c1[0]));
        fx = fma(-c1[0], v1, c1[1] * v0);
        fy = fma(c0[0], v1, -(c0[1] * v0));
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if (MASS) sm[i] = fma(T.B[i * M + q], fm, sm[i]);
        if (LAP) {
          sx[i] = fma(T.B[i * M + q], fx, sx[i]);
          sy[i] = fma(T.D[i * M + q], fy, sy[i]);
        }
      }
    }
  }
  __syncthreads();
  if (on && line < M) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (MASS) cb[line * PL + i] = sm[i];
      if (LAP) {
        cb[M * PL + line * PL + i] = sx[i];
        cb[2 * M * PL + line * PL + i] = sy[i];
      }
    }
  }
  __syncthreads();

  // ---- x-lines (iy = line): transposed x, write A -------------------
  if (on && line < N && c < ncb) {
    const int64_t off = (cell0 + c) * (N * N) + line;
    if (MASS) {
      double v[M];
#pragma unroll
      for (int q = 0; q < M; ++q) v[q] = cb[q * PL + line];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double a = T.B[i * M] * v[0];
#pragma unroll
        for (int q = 1; q < M; ++q) a = fma(T.B[i * M + q], v[q], a);
        Amass[off + i * N] = a;
      }
    }
    if (LAP) {
      double vx[M], vy[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        vx[q] = cb[M * PL + q * PL + line];
        vy[q] = cb[2 * M * PL + q * PL + line];
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double a = fma(T.D[i * M], vx[0], T.B[i * M] * vy[0]);
#pragma unroll
        for (int q = 1; q < M; ++q) {
          a = fma(T.D[i * M + q], vx[q], a);
          a = fma(T.B[i * M + q], vy[q], a);
        }
        Alap[off + i * N] = a;
      }
    }
  }
}

template <int N, int M>
static int launch_quad_nm(const sfk_plan* pm, const sfk_plan* pl, int64_t ncells, double* Am,
                          double* Al, const double* coords, const double* u, cudaStream_t s) {
  constexpr int L = M > N ? M : N;
  constexpr int CPB = (32 / L) > 0 ? 32 / L : 1;
  constexpr int THREADS = round_up(CPB * L, 32);
  const sfk_plan* src = pm ? pm : pl;
  const Tabs<N, M> T = make_tabs<N, M>(src);
  const unsigned grid = (unsigned)((ncells + CPB - 1) / CPB);
  if (pm && pl)
    quad_action_kernel<N, M, CPB, true, true><<<grid, THREADS, 0, s>>>(T, ncells, coords, u, Am, Al);
  else if (pm)
    quad_action_kernel<N, M, CPB, true, false><<<grid, THREADS, 0, s>>>(T, ncells, coords, u, Am, nullptr);
  else
    quad_action_kernel<N, M, CPB, false, true><<<grid, THREADS, 0, s>>>(T, ncells, coords, u, nullptr, Al);
  note_launch();
  return cuda_status(cudaGetLastError(), "quad_action_kernel launch");
}

// p0/p1: any of {action_mass, action_laplace} quad plans with equal tables;
// p1 may be NULL (single kernel).  A0/A1 follow p0/p1.
int launch_quad_action(const sfk_plan* p0, const sfk_plan* p1, int64_t ncells, double* A0,
                       double* A1, const double* coords, const double* u, cudaStream_t s) {
  const sfk_plan* pm = nullptr;
  const sfk_plan* pl = nullptr;
  double *Am = nullptr, *Al = nullptr;
  if (p0->kind == SFK_KIND_ACTION_MASS) { pm = p0; Am = A0; } else { pl = p0; Al = A0; }
  if (p1) {
    if (p1->kind == SFK_KIND_ACTION_MASS) {
      if (pm) return fail(SFK_EINVAL, "two mass plans in one fused quad launch");
      pm = p1; Am = A1;
    } else {
      if (pl) return fail(SFK_EINVAL, "two Laplace plans in one fused quad launch");
      pl = p1; Al = A1;
    }
  }
  if (p0->collocated)
    return fail(SFK_EUNSUPPORTED, "quad actions: collocated GLL variant not instantiated");
  const int n = p0->n, m = p0->m;
  if (n == m) {
    switch (n) {
      case 2: return launch_quad_nm<2, 2>(pm, pl, ncells, Am, Al, coords, u, s);
      case 3: return launch_quad_nm<3, 3>(pm, pl, ncells, Am, Al, coords, u, s);
      case 4: return launch_quad_nm<4, 4>(pm, pl, ncells, Am, Al, coords, u, s);
      case 5: return launch_quad_nm<5, 5>(pm, pl, ncells, Am, Al, coords, u, s);
      case 6: return launch_quad_nm<6, 6>(pm, pl, ncells, Am, Al, coords, u, s);
      case 7: return launch_quad_nm<7, 7>(pm, pl, ncells, Am, Al, coords, u, s);
      case 8: return launch_quad_nm<8, 8>(pm, pl, ncells, Am, Al, coords, u, s);
      case 9: return launch_quad_nm<9, 9>(pm, pl, ncells, Am, Al, coords, u, s);
      case 10: return launch_quad_nm<10, 10>(pm, pl, ncells, Am, Al, coords, u, s);
      case 11: return launch_quad_nm<11, 11>(pm, pl, ncells, Am, Al, coords, u, s);
      case 12: return launch_quad_nm<12, 12>(pm, pl, ncells, Am, Al, coords, u, s);
      case 13: return launch_quad_nm<13, 13>(pm, pl, ncells, Am, Al, coords, u, s);
      case 14: return launch_quad_nm<14, 14>(pm, pl, ncells, Am, Al, coords, u, s);
      case 15: return launch_quad_nm<15, 15>(pm, pl, ncells, Am, Al, coords, u, s);
      case 16: return launch_quad_nm<16, 16>(pm, pl, ncells, Am, Al, coords, u, s);
      case 17: return launch_quad_nm<17, 17>(pm, pl, ncells, Am, Al, coords, u, s);
      default: break;
    }
  }
  return fail(SFK_EUNSUPPORTED, "quad actions: no kernel for n=%d, m=%d (n==m in 2..17)", n, m);
}

}  // namespace sfk
