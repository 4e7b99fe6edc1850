// Hex Q_1 local stiffness matrices, one thread per cell — BASELINE C5 at p=1.
//
// Same math and reference mapping as hex_matrix.cu (registry `laplace` on
// `hex`, forms.py:186-189; test index outermost A[i*8 + j], forms.py:402-408):
//   A[i][j] = sum_q g_i(q)^T K_q g_j(q),  K_q = (w_q/|det J|) R R^T,
// g_i^l = reference gradient of basis i = 4a+2b+c (D on axis l, B elsewhere).
// At n = m = 2 a cell has 8 points and 8 basis functions, so one thread holds
// the whole symmetric matrix (36 accumulators) and walks the 8 points:
// per point 24 basis gradients, 6 K entries (adjugate rows, hex_geometry.cuh),
// h_j = K g_j, then A_ij += g_i . h_j for j >= i.  No shared-memory phases
// and no barriers (the CTA-phase kernel of hex_matrix.cu spent most of its
// time there at p = 1: frac 0.20).  Coords arrive through padded shared
// memory (16-byte cp.async); each warp stages its 32 finished matrices in
// shared memory (stride 65 doubles: conflict-free) and writes them out as
// contiguous 512-byte rows.
#include <cstdlib>

#include "async_copy.cuh"
#include "hex_geometry.cuh"

namespace sfk {

namespace m1 {
constexpr int CPB = 128;   // cells (= threads) per CTA
constexpr int CS = 26;     // padded coords stride
constexpr int AS = 65;     // padded matrix stride (64 used)
constexpr size_t SMEM = (size_t)CPB * (CS + AS) * sizeof(double);
}  // namespace m1

template <int MINB>
__global__ void __launch_bounds__(m1::CPB, MINB)
hex_laplace_matrix_p1(const __grid_constant__ Tabs<2, 2> T, int64_t ncells,
                      const double* __restrict__ coords, double* __restrict__ A) {
  using namespace m1;
  extern __shared__ __align__(16) double smem[];
  double* sC = smem;
  double* sA = smem + CPB * CS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
  {
    const double* cg = coords + cell0 * 24;
    if ((reinterpret_cast<uintptr_t>(cg) & 15) == 0) {
      for (int ch = tid; ch < ncb * 12; ch += CPB) {
        const int c = ch / 12, k = ch - c * 12;
        cp_async16(sC + c * CS + 2 * k, cg + 2 * ch);
      }
    } else {
      for (int e = tid; e < ncb * 24; e += CPB) cp_async8(sC + (e / 24) * CS + e % 24, cg + e);
    }
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();

  double acc[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) acc[k] = 0.0;
  if (tid < ncb) {
    const double* X = sC + tid * CS;   // read per line from shared memory (saves 24 registers)
#pragma unroll 1
    for (int line = 0; line < 4; ++line) {          // (qx, qy)
      const int qx = line >> 1, qy = line & 1;
      HexLineGeom geo;
      geo.setup(X, T.Bc[qx], T.Bc[2 + qx], T.Bc[qy], T.Bc[2 + qy]);
      const double wxy = T.W[qx] * T.W[qy];
      // x/y factors of the 8 basis gradients on this line: [a][b]
      double fxD[4], fyD[4], fBB[4];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          fxD[2 * a + b] = T.D[2 * a + qx] * T.B[2 * b + qy];   // d/dx: Dx By
          fyD[2 * a + b] = T.B[2 * a + qx] * T.D[2 * b + qy];   // d/dy: Bx Dy
          fBB[2 * a + b] = T.B[2 * a + qx] * T.B[2 * b + qy];   // d/dz: Bx By (Dz below)
        }
#pragma unroll 1
      for (int qz = 0; qz < 2; ++qz) {
        double r0[3], r1[3], r2[3];
        const double det = geo.adj(T.Bc[qz], T.Bc[2 + qz], r0, r1, r2);
        const double s = (wxy * T.W[qz]) * rcp64(fabs(det));
        // K = s R R^T (symmetric)
        const double k00 = s * fma(r0[2], r0[2], fma(r0[1], r0[1], r0[0] * r0[0]));
        const double k11 = s * fma(r1[2], r1[2], fma(r1[1], r1[1], r1[0] * r1[0]));
        const double k22 = s * fma(r2[2], r2[2], fma(r2[1], r2[1], r2[0] * r2[0]));
        const double k01 = s * fma(r0[2], r1[2], fma(r0[1], r1[1], r0[0] * r1[0]));
        const double k02 = s * fma(r0[2], r2[2], fma(r0[1], r2[1], r0[0] * r2[0]));
        const double k12 = s * fma(r1[2], r2[2], fma(r1[1], r2[1], r1[0] * r2[0]));
        double g0[8], g1[8], g2[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int ab = i >> 1, c = i & 1;
          const double bz = T.B[2 * c + qz], dz = T.D[2 * c + qz];
          g0[i] = fxD[ab] * bz;
          g1[i] = fyD[ab] * bz;
          g2[i] = fBB[ab] * dz;
        }
        // column j: h = K g_j, then A_ij += g_i . h for i <= j
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double h0 = fma(k02, g2[j], fma(k01, g1[j], k00 * g0[j]));
          const double h1 = fma(k12, g2[j], fma(k11, g1[j], k01 * g0[j]));
          const double h2 = fma(k22, g2[j], fma(k12, g1[j], k02 * g0[j]));
#pragma unroll
          for (int i = 0; i <= j; ++i) {
            const int k = i * 8 - i * (i - 1) / 2 + (j - i);   // upper-triangle index
            acc[k] = fma(g2[i], h2, fma(g1[i], h1, fma(g0[i], h0, acc[k])));
          }
        }
      }
    }
  }
  // stage the warp's 32 matrices (full, mirrored) and write contiguous rows
  double* sw = sA + warp * 32 * AS;
  {
    int k = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = i; j < 8; ++j, ++k) {
        sw[lane * AS + i * 8 + j] = acc[k];
        sw[lane * AS + j * 8 + i] = acc[k];
      }
  }
  __syncwarp();
  const int wc0 = warp * 32;
  const int nw = ncb - wc0 < 32 ? ncb - wc0 : 32;
  if (nw > 0) {
    double* out = A + (cell0 + wc0) * 64;
    for (int e = lane; e < nw * 64; e += 32) out[e] = sw[(e >> 6) * AS + (e & 63)];
  }
}

int launch_hex_matrix_p1(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         cudaStream_t s) {
  if (p->n != 2 || p->m != 2) return SFK_EUNSUPPORTED;
  // register budget: MINB=2 -> no spills (254 regs unconstrained); MINB=3
  // spills ~300 B.  option c5_p1_minb = 3 selects the latter for A/B runs.
  const int minb = option(OPT_C5_P1_MINB) == 3 ? 3 : 2;
  auto kern = minb == 3 ? hex_laplace_matrix_p1<3> : hex_laplace_matrix_p1<2>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, m1::CPB, m1::SMEM, "hex_matrix_p1", &sh))
    return rc_;
  const Tabs<2, 2> T = make_tabs<2, 2>(p);
  const unsigned grid = (unsigned)((ncells + m1::CPB - 1) / m1::CPB);
  kern<<<grid, m1::CPB, m1::SMEM, s>>>(T, ncells, coords, A);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_matrix_p1 launch");
}

}  // namespace sfk
