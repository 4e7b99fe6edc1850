// Hex Q_p mass action b = M u (registry `action_mass` on `hex`).
//
// Reference: forms.py:173 (_mass: v * u), :235-243 action_form,
// :261-263 REGISTRY; scaled by w_q |det J_q| (forms.py:393-394,
// geometry.py:107).  Its spectral-mode schedule is the B-only half of the
// Laplace action's: 3 forward contractions (x, y, z with B), the pointwise
// scale, 3 transposed contractions (z, y, x with B^T).
//
// Same line-kernel mapping as hex_action.cu (one CTA per CPB cells, thread
// per 1D line, lines re-dealt between axes through shared memory); the z
// stage, the scale by w |det J| (geometry on the fly, hex_geometry.cuh) and
// the transposed z stage run back to back in registers.
#include "hex_geometry.cuh"

namespace sfk {

template <int N, int M, int CPB>
struct HexMassCfg {
  static constexpr int NN = N * N;
  static constexpr int MN = M * N;
  static constexpr int MM = M * M;
  static constexpr int LINES = MM > NN ? MM : NN;
  static constexpr int THREADS = round_up(CPB * LINES, 32);
  static constexpr int PX = NN | 1;            // x-plane stride of X[q][iy][iz]
  static constexpr int LZ = N | 1;             // z-line stride of Y[qx][qy][iz]
  static constexpr int XSZ = M * PX;
  static constexpr int YSZ = MM * LZ;
  static constexpr size_t SMEM = (size_t)CPB * (XSZ + YSZ + 24) * sizeof(double);
};

template <int N, int M, int CPB>
__global__ void __launch_bounds__(HexMassCfg<N, M, CPB>::THREADS)
hex_mass_action_kernel(const __grid_constant__ Tabs<N, M> T, int64_t ncells,
                       const double* __restrict__ coords, const double* __restrict__ u,
                       double* __restrict__ A) {
  using C = HexMassCfg<N, M, CPB>;
  constexpr int NN = C::NN, MN = C::MN, MM = C::MM, PX = C::PX, LZ = C::LZ;
  extern __shared__ double smem[];
  double* sX = smem;                    // [CPB][M][PX]
  double* sY = sX + CPB * C::XSZ;       // [CPB][M*M][LZ]
  double* sC = sY + CPB * C::YSZ;       // [CPB][24]

  const int tid = threadIdx.x;
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int64_t rem = ncells - cell0;
  const int ncb = rem < CPB ? (int)rem : CPB;

  for (int i = tid; i < CPB * 24; i += C::THREADS)
    sC[i] = i < ncb * 24 ? __ldg(coords + cell0 * 24 + i) : 0.0;

  // x stage: line (iy, iz)
  if (tid < CPB * NN) {
    const int c = tid / NN, r = tid - c * NN;
    double uu[N];
#pragma unroll
    for (int i = 0; i < N; ++i)
      uu[i] = c < ncb ? __ldg(u + (cell0 + c) * (N * NN) + r + i * NN) : 0.0;
    double* xo = sX + c * C::XSZ + r;
#pragma unroll
    for (int q = 0; q < M; ++q) {
      double b = T.B[q] * uu[0];
#pragma unroll
      for (int i = 1; i < N; ++i) b = fma(T.B[i * M + q], uu[i], b);
      xo[q * PX] = b;
    }
  }
  __syncthreads();

  // y stage: line (qx, iz)
  if (tid < CPB * MN) {
    const int c = tid / MN, r = tid - c * MN;
    const int qx = r / N, iz = r - qx * N;
    const double* xi = sX + c * C::XSZ + qx * PX + iz;
    double a[N];
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = xi[i * N];
    double* yo = sY + c * C::YSZ + qx * M * LZ + iz;
#pragma unroll
    for (int q = 0; q < M; ++q) {
      double b = T.B[q] * a[0];
#pragma unroll
      for (int i = 1; i < N; ++i) b = fma(T.B[i * M + q], a[i], b);
      yo[q * LZ] = b;
    }
  }
  __syncthreads();

  // z stage, scale by w |det J|, transposed z stage: line (qx, qy)
  if (tid < CPB * MM) {
    const int c = tid / MM, r = tid - c * MM;
    const int qx = r / M, qy = r - qx * M;
    double* yl = sY + c * C::YSZ + r * LZ;
    double y[N], s[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      y[i] = yl[i];
      s[i] = 0.0;
    }
    HexLineGeom geo;
    geo.setup(sC + c * 24, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
    const double wxy = T.W[qx] * T.W[qy];
#pragma unroll
    for (int q = 0; q < M; ++q) {
      double v = T.B[q] * y[0];
#pragma unroll
      for (int i = 1; i < N; ++i) v = fma(T.B[i * M + q], y[i], v);
      double r0[3], r1[3], r2[3];
      const double det = geo.adj(T.Bc[q], T.Bc[M + q], r0, r1, r2);
      v *= (wxy * T.W[q]) * fabs(det);
#pragma unroll
      for (int i = 0; i < N; ++i) s[i] = fma(T.B[i * M + q], v, s[i]);
    }
    // each thread rewrites only its own line: no barrier needed before
#pragma unroll
    for (int i = 0; i < N; ++i) yl[i] = s[i];
  }
  __syncthreads();

  // transposed y stage: line (qx, iz)
  if (tid < CPB * MN) {
    const int c = tid / MN, r = tid - c * MN;
    const int qx = r / N, iz = r - qx * N;
    const double* yi = sY + c * C::YSZ + qx * M * LZ + iz;
    double p[M];
#pragma unroll
    for (int q = 0; q < M; ++q) p[q] = yi[q * LZ];
    double* xo = sX + c * C::XSZ + qx * PX + iz;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double a = T.B[i * M] * p[0];
#pragma unroll
      for (int q = 1; q < M; ++q) a = fma(T.B[i * M + q], p[q], a);
      xo[i * N] = a;
    }
  }
  __syncthreads();

  // transposed x stage: line (iy, iz) -> A (overwritten)
  if (tid < CPB * NN) {
    const int c = tid / NN, r = tid - c * NN;
    if (c < ncb) {
      const double* xi = sX + c * C::XSZ + r;
      double p[M];
#pragma unroll
      for (int q = 0; q < M; ++q) p[q] = xi[q * PX];
      double* ap = A + (cell0 + c) * (N * NN) + r;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double a = T.B[i * M] * p[0];
#pragma unroll
        for (int q = 1; q < M; ++q) a = fma(T.B[i * M + q], p[q], a);
        ap[i * NN] = a;
      }
    }
  }
}

template <int N, int M, int CPB>
static int launch_mass(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                       const double* u, cudaStream_t s) {
  using C = HexMassCfg<N, M, CPB>;
  auto kern = hex_mass_action_kernel<N, M, CPB>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_mass", &sh))
    return rc_;
  const Tabs<N, M> T = make_tabs<N, M>(p);
  const int64_t grid = (ncells + CPB - 1) / CPB;
  kern<<<(unsigned)grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, u, A);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_mass_action_kernel launch");
}

bool hex_mass_supported(int n, int m) {
  return (n == m && n >= 2 && n <= 10) || (m == n + 1 && n >= 2 && n <= 8);
}

int launch_hex_mass(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                    const double* w0, cudaStream_t s) {
  const int n = p->n, m = p->m;
  if (n == m) {
    switch (n) {
      case 2: return launch_mass<2, 2, 32>(p, ncells, A, coords, w0, s);
      case 3: return launch_mass<3, 3, 16>(p, ncells, A, coords, w0, s);
      case 4: return launch_mass<4, 4, 8>(p, ncells, A, coords, w0, s);
      case 5: return launch_mass<5, 5, 5>(p, ncells, A, coords, w0, s);
      case 6: return launch_mass<6, 6, 4>(p, ncells, A, coords, w0, s);
      case 7: return launch_mass<7, 7, 3>(p, ncells, A, coords, w0, s);
      case 8: return launch_mass<8, 8, 2>(p, ncells, A, coords, w0, s);
      case 9: return launch_mass<9, 9, 2>(p, ncells, A, coords, w0, s);
      case 10: return launch_mass<10, 10, 1>(p, ncells, A, coords, w0, s);
      default: break;
    }
  } else if (m == n + 1) {
    switch (n) {
      case 2: return launch_mass<2, 3, 16>(p, ncells, A, coords, w0, s);
      case 3: return launch_mass<3, 4, 8>(p, ncells, A, coords, w0, s);
      case 4: return launch_mass<4, 5, 5>(p, ncells, A, coords, w0, s);
      case 5: return launch_mass<5, 6, 4>(p, ncells, A, coords, w0, s);
      case 6: return launch_mass<6, 7, 3>(p, ncells, A, coords, w0, s);
      case 7: return launch_mass<7, 8, 2>(p, ncells, A, coords, w0, s);
      case 8: return launch_mass<8, 9, 2>(p, ncells, A, coords, w0, s);
      default: break;
    }
  }
  return fail(SFK_EUNSUPPORTED,
              "hex action_mass: no kernel for n=%d, m=%d (m==n in 2..10, m==n+1 in 2..8)", n, m);
}

}  // namespace sfk
