// Hex Q_p Laplace action b = K u, Gauss-Legendre (or any non-collocated)
// quadrature with M points per axis — BASELINE config C2 (the headline).
//
// Reference: the spectral-mode program of `action_laplace` on `hex`
// (forms.py:186-189 _laplace, :235-243 action_form, passes.py:672-743
// run_pipeline, scheduling.py:617-738 emit_c).  Its contraction schedule
// is 8 forward 1D contractions
//     x: {B, D} u          y: {B, D} (Bx u), B (Dx u)
//     z: D (ByBx u), B (DyBx u), B (ByDx u)      -> reference gradient g
// a pointwise flux f = w|J| G G^T g, and 8 transposed contractions
//     z: Bz^T fx, Bz^T fy, Dz^T fz
//     y: By^T (.x), Dy^T (.y) + By^T (.z)
//     x: Dx^T (.x) + Bx^T (.yz)                  -> A (overwritten)
//
// B200 mapping ("line" kernel).  A CTA owns CPB consecutive cells.  Every
// stage is a set of independent 1D contractions along one axis; each thread
// owns one LINE of that axis in registers (N inputs -> M outputs, N*M DFMA
// per table, the table entry a constant-bank operand of the DFMA because the
// tables are a __grid_constant__ parameter and the loops are fully
// unrolled).  Between stages the lines are re-dealt through shared memory
// (one STS + one LDS per value per stage), which keeps the smem:DFMA ratio
// at ~2/N.  The z stage, the pointwise flux (geometry recomputed per point
// from the 8 vertices, hex_geometry.cuh) and the transposed z stage run
// back-to-back in registers.  u is read straight from HBM by the x-stage
// threads (each warp load is a run of contiguous dofs) and A is written the
// same way; nothing but the cell's coords, u and A touches HBM.
#include "hex_geometry.cuh"

namespace sfk {

template <int N, int M, int CPB>
struct HexActionCfg {
  static constexpr int NN = N * N;
  static constexpr int MN = M * N;
  static constexpr int MM = M * M;
  static constexpr int LINES = MM > NN ? MM : NN;
  static constexpr int THREADS = round_up(CPB * LINES, 32);
  // x-plane stride in the X/R arrays (X[q][iy][iz]); padded so the y-stage
  // reads (lanes over (qx, iz)) fall in distinct banks.
  static constexpr int PX = (N >= 4) ? NN + (((N - NN) % 16) + 16) % 16 : NN;
  // z-line stride in the Y/S arrays (odd => conflict-free z-stage reads).
  static constexpr int LZ = N | 1;
  static constexpr int XSZ = 2 * M * PX;        // two arrays [M][N][N] (padded)
  static constexpr int YSZ = 3 * MM * LZ;       // three arrays [M][M][N] (padded)
  static constexpr size_t SMEM = (size_t)CPB * (XSZ + YSZ + 24) * sizeof(double);
};

template <int N, int M, int CPB>
__global__ void __launch_bounds__(HexActionCfg<N, M, CPB>::THREADS)
hex_laplace_action_kernel(const __grid_constant__ Tabs<N, M> T, int64_t ncells,
                          const double* __restrict__ coords,
                          const double* __restrict__ u,
                          double* __restrict__ A) {
  using C = HexActionCfg<N, M, CPB>;
  constexpr int NN = C::NN, MN = C::MN, MM = C::MM, PX = C::PX, LZ = C::LZ;
  constexpr int YA = MM * LZ;  // one Y/S array
  constexpr int XA = M * PX;   // one X/R array
  extern __shared__ double smem[];
  double* sX = smem;                    // [CPB][2][M][PX]
  double* sY = sX + CPB * C::XSZ;       // [CPB][3][M*M][LZ]
  double* sC = sY + CPB * C::YSZ;       // [CPB][24]

  const int tid = threadIdx.x;
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int64_t rem = ncells - cell0;
  const int ncb = rem < CPB ? (int)rem : CPB;

  for (int i = tid; i < CPB * 24; i += C::THREADS)
    sC[i] = i < ncb * 24 ? __ldg(coords + cell0 * 24 + i) : 0.0;

  // ---- x stage: line (iy, iz); X0 = Bx u, X1 = Dx u --------------------
  if (tid < CPB * NN) {
    const int c = tid / NN, r = tid - c * NN;
    double uu[N];
    if (c < ncb) {
      const double* up = u + (cell0 + c) * (N * NN) + r;
#pragma unroll
      for (int i = 0; i < N; ++i) uu[i] = __ldg(up + i * NN);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) uu[i] = 0.0;
    }
    double* xo = sX + c * C::XSZ + r;
#pragma unroll
    for (int q = 0; q < M; ++q) {
      double b = T.B[q] * uu[0], d = T.D[q] * uu[0];
#pragma unroll
      for (int i = 1; i < N; ++i) {
        b = fma(T.B[i * M + q], uu[i], b);
        d = fma(T.D[i * M + q], uu[i], d);
      }
      xo[q * PX] = b;
      xo[XA + q * PX] = d;
    }
  }
  __syncthreads();

  // ---- y stage: line (qx, iz); BB = By X0, BD = Dy X0, DB = By X1 -------
  if (tid < CPB * MN) {
    const int c = tid / MN, r = tid - c * MN;
    const int qx = r / N, iz = r - qx * N;
    const double* xi = sX + c * C::XSZ + qx * PX + iz;
    double a0[N], a1[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      a0[i] = xi[i * N];
      a1[i] = xi[XA + i * N];
    }
    double* yo = sY + c * C::YSZ + qx * M * LZ + iz;
#pragma unroll
    for (int q = 0; q < M; ++q) {
      double bb = T.B[q] * a0[0], bd = T.D[q] * a0[0], db = T.B[q] * a1[0];
#pragma unroll
      for (int i = 1; i < N; ++i) {
        bb = fma(T.B[i * M + q], a0[i], bb);
        bd = fma(T.D[i * M + q], a0[i], bd);
        db = fma(T.B[i * M + q], a1[i], db);
      }
      yo[q * LZ] = bb;
      yo[YA + q * LZ] = bd;
      yo[2 * YA + q * LZ] = db;
    }
  }
  __syncthreads();

  // ---- z stage + pointwise flux + transposed z stage: line (qx, qy) -----
  const bool zact = tid < CPB * MM;
  double sx[N], sy[N], sz[N];
  int zoff = 0;
  if (zact) {
    const int c = tid / MM, r = tid - c * MM;
    const int qx = r / M, qy = r - qx * M;
    zoff = c * C::YSZ + r * LZ;
    const double* yi = sY + zoff;
    double bb[N], bd[N], db[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      bb[i] = yi[i];
      bd[i] = yi[YA + i];
      db[i] = yi[2 * YA + i];
    }
    HexLineGeom geo;
    geo.setup(sC + c * 24, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
    const double wxy = T.W[qx] * T.W[qy];
#pragma unroll
    for (int i = 0; i < N; ++i) sx[i] = sy[i] = sz[i] = 0.0;
#pragma unroll
    for (int q = 0; q < M; ++q) {
      double gz = T.D[q] * bb[0], gy = T.B[q] * bd[0], gx = T.B[q] * db[0];
#pragma unroll
      for (int i = 1; i < N; ++i) {
        gz = fma(T.D[i * M + q], bb[i], gz);
        gy = fma(T.B[i * M + q], bd[i], gy);
        gx = fma(T.B[i * M + q], db[i], gx);
      }
      double r0[3], r1[3], r2[3];
      const double det = geo.adj(T.Bc[q], T.Bc[M + q], r0, r1, r2);
      const double s = (wxy * T.W[q]) * rcp64(fabs(det));
      laplace_flux(r0, r1, r2, s, gx, gy, gz);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        sx[i] = fma(T.B[i * M + q], gx, sx[i]);
        sy[i] = fma(T.B[i * M + q], gy, sy[i]);
        sz[i] = fma(T.D[i * M + q], gz, sz[i]);
      }
    }
  }
  __syncthreads();
  if (zact) {
    double* yo = sY + zoff;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      yo[i] = sx[i];
      yo[YA + i] = sy[i];
      yo[2 * YA + i] = sz[i];
    }
  }
  __syncthreads();

  // ---- transposed y stage: line (qx, iz) --------------------------------
  if (tid < CPB * MN) {
    const int c = tid / MN, r = tid - c * MN;
    const int qx = r / N, iz = r - qx * N;
    const double* yi = sY + c * C::YSZ + qx * M * LZ + iz;
    double px[M], py[M], pz[M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
      px[q] = yi[q * LZ];
      py[q] = yi[YA + q * LZ];
      pz[q] = yi[2 * YA + q * LZ];
    }
    double* xo = sX + c * C::XSZ + qx * PX + iz;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double r1 = T.B[i * M] * px[0];
      double r2 = fma(T.D[i * M], py[0], T.B[i * M] * pz[0]);
#pragma unroll
      for (int q = 1; q < M; ++q) {
        r1 = fma(T.B[i * M + q], px[q], r1);
        r2 = fma(T.D[i * M + q], py[q], r2);
        r2 = fma(T.B[i * M + q], pz[q], r2);
      }
      xo[i * N] = r1;
      xo[XA + i * N] = r2;
    }
  }
  __syncthreads();

  // ---- transposed x stage: line (iy, iz) -> A ----------------------------
  if (tid < CPB * NN) {
    const int c = tid / NN, r = tid - c * NN;
    if (c < ncb) {
      const double* xi = sX + c * C::XSZ + r;
      double p1[M], p2[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        p1[q] = xi[q * PX];
        p2[q] = xi[XA + q * PX];
      }
      double* ap = A + (cell0 + c) * (N * NN) + r;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double a = fma(T.D[i * M], p1[0], T.B[i * M] * p2[0]);
#pragma unroll
        for (int q = 1; q < M; ++q) {
          a = fma(T.D[i * M + q], p1[q], a);
          a = fma(T.B[i * M + q], p2[q], a);
        }
        ap[i * NN] = a;
      }
    }
  }
}

template <int N, int M, int CPB>
static int launch_nm(const sfk_plan* p, int64_t ncells, double* A,
                     const double* coords, const double* u, cudaStream_t s) {
  using C = HexActionCfg<N, M, CPB>;
  auto kern = hex_laplace_action_kernel<N, M, CPB>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_action", &sh))
    return rc_;
  const Tabs<N, M> T = make_tabs<N, M>(p);
  const int64_t grid = (ncells + CPB - 1) / CPB;
  kern<<<(unsigned)grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, u, A);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_kernel launch");
}

// cells per CTA for n = m: ~256-288 threads, ~95-100% lane use.
int launch_hex_action(const sfk_plan* p, int64_t ncells, double* A,
                      const double* coords, const double* w0, const double*,
                      cudaStream_t s) {
  const int n = p->n, m = p->m;
  if (n == m) {
    switch (n) {
      case 2: return launch_nm<2, 2, 64>(p, ncells, A, coords, w0, s);
      case 3: return launch_nm<3, 3, 32>(p, ncells, A, coords, w0, s);
      case 4: return launch_nm<4, 4, 16>(p, ncells, A, coords, w0, s);
      case 5: return launch_nm<5, 5, 10>(p, ncells, A, coords, w0, s);
      case 6: return launch_nm<6, 6, 8>(p, ncells, A, coords, w0, s);
      case 7: return launch_nm<7, 7, 5>(p, ncells, A, coords, w0, s);
      case 8: return launch_nm<8, 8, 4>(p, ncells, A, coords, w0, s);
      case 9: return launch_nm<9, 9, 3>(p, ncells, A, coords, w0, s);
      case 10: return launch_nm<10, 10, 2>(p, ncells, A, coords, w0, s);
      default: break;
    }
  } else if (m == n + 1) {
    switch (n) {
      case 2: return launch_nm<2, 3, 32>(p, ncells, A, coords, w0, s);
      case 3: return launch_nm<3, 4, 16>(p, ncells, A, coords, w0, s);
      case 4: return launch_nm<4, 5, 10>(p, ncells, A, coords, w0, s);
      case 5: return launch_nm<5, 6, 8>(p, ncells, A, coords, w0, s);
      case 6: return launch_nm<6, 7, 5>(p, ncells, A, coords, w0, s);
      case 7: return launch_nm<7, 8, 4>(p, ncells, A, coords, w0, s);
      case 8: return launch_nm<8, 9, 3>(p, ncells, A, coords, w0, s);
      default: break;
    }
  }
  return fail(SFK_EUNSUPPORTED,
              "hex action_laplace: no kernel instantiated for n=%d dofs/axis, "
              "m=%d points/axis (supported: m==n in 2..10, m==n+1 in 2..8)", n, m);
}

}  // namespace sfk
