// Hex Q_p Laplace action, v6 schedule with R lines per thread — C2 at the
// high degrees.
//
// Same operator, reference mapping, stages A..I, tables, shared layouts
// (hex_action6_layout.cuh), per-cell line-geometry table and bulk staging
// as v6 (hex_action6.cu).  The difference: a thread owns R lines of every
// stage (line t and t + THREADS, ...) and contracts them together, so each
// table entry — a uniform constant load (LDCU) feeding the DFMAs — is
// loaded once per R lines, and every thread carries R x n independent FMA
// chains.  At n = 9 the one-line kernel issues 560 LDCU against 1480 FP64
// instructions per thread and batch (profiles/r02_sass_mix.md): the issue
// port, not the FP64 pipe, was the first limit.
#include "async_copy.cuh"
#include "hex_action6_layout.cuh"
#include "hex_colloc_deriv.cuh"
#include "hex_geometry.cuh"

namespace sfk {

// out[r][o] = sum_i T[i*LD + o] in[r][i] for R lines: each table entry is
// read once for all R lines.
template <int NI, int NO, int LD, int R>
__device__ __forceinline__ void v6r_contract(const double* T, const double (*in)[NI],
                                             double (*out)[NO]) {
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    const double t = T[o];
#pragma unroll
    for (int r = 0; r < R; ++r) out[r][o] = t * in[r][0];
  }
#pragma unroll
  for (int i = 1; i < NI; ++i)
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      const double t = T[i * LD + o];
#pragma unroll
      for (int r = 0; r < R; ++r) out[r][o] = fma(t, in[r][i], out[r][o]);
    }
}

__host__ __device__ constexpr int v6r_slot(int n) {
  int s = 0;
  for (int r = V6_P1; r <= V6_P2; ++r) s = v6_role(n, r).cs > s ? v6_role(n, r).cs : s;
  return s;
}

template <int N, int CPB, int R>
struct V6RCfg {
  static constexpr int NN = N * N, N3 = N * N * N;
  static constexpr int L = CPB * NN;                        // lines per stage
  static constexpr int THREADS = round_up((L + R - 1) / R, 32);
  static constexpr int S = CPB * v6r_slot(N);
  static constexpr int USZ = round_up(CPB * N3 + 1, 2);
  static constexpr int CSZ = CPB * 24;
  static constexpr int GSZ = CPB * 18 * N;
  static constexpr size_t SMEM = (size_t)(4 * S + USZ + 2 * CSZ + GSZ + 4) * sizeof(double);
};

template <int N, int CPB, int R, int MINB>
__global__ void __launch_bounds__(V6RCfg<N, CPB, R>::THREADS, MINB)
hex_laplace_action_v6r(const __grid_constant__ TabsV6<N> T, int64_t ncells,
                       const double* __restrict__ coords, const double* __restrict__ u,
                       double* __restrict__ A) {
  using C = V6RCfg<N, CPB, R>;
  constexpr int NN = C::NN, N3 = C::N3, TH = C::THREADS, L = C::L, LD = TabsV6<N>::LD;
  constexpr V6Arr P1 = v6_role(N, V6_P1), Qr = v6_role(N, V6_Q), Vr = v6_role(N, V6_V),
                  GZr = v6_role(N, V6_GZ), GXr = v6_role(N, V6_GX), GYr = v6_role(N, V6_GY),
                  Rr = v6_role(N, V6_R), P2 = v6_role(N, V6_P2);
  extern __shared__ __align__(16) double smem[];
  double* S1 = smem;
  double* S2 = S1 + C::S;
  double* S3 = S2 + C::S;
  double* S4 = S3 + C::S;
  double* sU = S4 + C::S;
  double* sCo = sU + C::USZ;               // [2][CPB*24]
  double* sLG = sCo + 2 * C::CSZ;          // [CPB][18 N]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sLG + C::GSZ + 2);
  const int tid = threadIdx.x;
  const int64_t nbatch = (ncells + CPB - 1) / CPB;

  // lines of this thread: l = tid + j*TH; idle ones alias line 0
  bool on[R];
  int cc[R], ra[R], rb[R], rr[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int l = tid + j * TH;
    on[j] = l < L;
    const int lt = on[j] ? l : 0;
    cc[j] = lt / NN;
    rr[j] = lt - cc[j] * NN;
    ra[j] = rr[j] / N;
    rb[j] = rr[j] - ra[j] * N;
  }

  auto prefetch = [&](int64_t bt, int buf) {
    if (tid == 0) {
      const int64_t c0 = bt * CPB;
      const int nc = (int)((ncells - c0) < CPB ? (ncells - c0) : CPB);
      fence_proxy_async_smem();
      unsigned bytes = bulk_copy_phase(sU, u + c0 * N3, nc * N3, bar);
      bulk_g2s(sCo + buf * C::CSZ, coords + c0 * 24, (unsigned)nc * 192u, bar);
      mbar_arrive_expect_tx(bar, bytes + (unsigned)nc * 192u);
    }
  };

  if (tid == 0) mbar_init(bar, 1);
  __syncthreads();
  int64_t b = blockIdx.x;
  if (b < nbatch) prefetch(b, 0);
  for (int k = 0; b < nbatch; b += gridDim.x, ++k) {
    const int cur = k & 1;
    const int64_t cell0 = b * CPB;
    const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
    cp_async_wait<0>();
    mbar_wait(bar, (unsigned)(k & 1));
    __syncthreads();
    const double* su = sU + dst_shift(u + cell0 * N3);

    // ---- A: x-lines (y, z): P = B_x u -> S1; line-geometry tables ----------
    {
      double in[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i)
          in[j][i] = (on[j] && cc[j] < ncb) ? su[cc[j] * N3 + i * NN + rr[j]] : 0.0;
      v6r_contract<N, N, LD, R>(T.B, in, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* p = S1 + cc[j] * P1.cs + ra[j] * P1.sy + rb[j];
#pragma unroll
          for (int q = 0; q < N; ++q) p[q * P1.sx] = o[j][q];
        }
      for (int e = tid; e < CPB * 18 * N; e += TH) {
        const int c = e / (18 * N);
        sLG[e] = hex_cell_lg(sCo + cur * C::CSZ + c * 24, T.Bc, N, e - c * 18 * N);
      }
    }
    __syncthreads();
    if (b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- B: y-lines (x, z): Q = B_y P -> S2 ---------------------------------
    {
      double in[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* p = S1 + cc[j] * P1.cs + ra[j] * P1.sx + rb[j];
#pragma unroll
        for (int i = 0; i < N; ++i) in[j][i] = p[i * P1.sy];
      }
      v6r_contract<N, N, LD, R>(T.B, in, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* q = S2 + cc[j] * Qr.cs + ra[j] * Qr.sx + rb[j];
#pragma unroll
          for (int jj = 0; jj < N; ++jj) q[jj * Qr.sy] = o[j][jj];
        }
    }
    __syncthreads();

    // ---- C: z-lines (y, x): V = B_z Q -> S1, gz = C_z V -> S4 ---------------
    {
      double in[R][N], v[R][N], g[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* q = S2 + cc[j] * Qr.cs + ra[j] * Qr.sy + rb[j] * Qr.sx;
#pragma unroll
        for (int i = 0; i < N; ++i) in[j][i] = q[i];
      }
      v6r_contract<N, N, LD, R>(T.B, in, v);
      v6r_contract<N, N, LD, R>(T.C, v, g);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* w = S1 + cc[j] * Vr.cs + ra[j] * Vr.sy + rb[j] * Vr.sx;
          double* wz = S4 + cc[j] * GZr.cs + ra[j] * GZr.sy + rb[j] * GZr.sx;
#pragma unroll
          for (int jj = 0; jj < N; ++jj) {
            w[jj] = v[j][jj];
            wz[jj] = g[j][jj];
          }
        }
    }
    __syncthreads();

    // ---- D: gx = C_x V -> S2 (x-lines); gy = C_y V -> S3 (y-lines) ---------
    {
      double in[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* v = S1 + cc[j] * Vr.cs + ra[j] * Vr.sy + rb[j];
#pragma unroll
        for (int i = 0; i < N; ++i) in[j][i] = v[i * Vr.sx];
      }
      v6r_contract<N, N, LD, R>(T.C, in, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* g = S2 + cc[j] * GXr.cs + ra[j] * GXr.sy + rb[j];
#pragma unroll
          for (int jj = 0; jj < N; ++jj) g[jj * GXr.sx] = o[j][jj];
        }
    }
    __syncwarp();
    {
      double in[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* v = S1 + cc[j] * Vr.cs + ra[j] * Vr.sx + rb[j];
#pragma unroll
        for (int i = 0; i < N; ++i) in[j][i] = v[i * Vr.sy];
      }
      v6r_contract<N, N, LD, R>(T.C, in, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* g = S3 + cc[j] * GYr.cs + ra[j] * GYr.sx + rb[j];
#pragma unroll
          for (int jj = 0; jj < N; ++jj) g[jj * GYr.sy] = o[j][jj];
        }
    }
    __syncthreads();

    // ---- E: z-lines: geometry + flux in place, one line at a time ----------
#pragma unroll 1
    for (int j = 0; j < R; ++j) {
      if (!on[j]) continue;
      const int c = cc[j], qy = ra[j], qx = rb[j];
      double* gxl = S2 + c * GXr.cs + qx * GXr.sx + qy * GXr.sy;
      double* gyl = S3 + c * GYr.cs + qy * GYr.sy + qx * GYr.sx;
      double* gzl = S4 + c * GZr.cs + qy * GZr.sy + qx * GZr.sx;
      HexLineAdj geo;
      geo.setup_lg(sLG + c * 18 * N, N, qx, qy, T.Bc[qx], T.Bc[N + qx]);
      const double wxy = T.W[qx] * T.W[qy];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        double gx = gxl[q], gy = gyl[q], g2 = gzl[q];
        double r0[3], r1[3], r2[3];
        const double det = geo.adj(T.Bc[N + q], r0, r1, r2);
        const double s = (wxy * T.W[q]) * rcp64(fabs(det));
        laplace_flux(r0, r1, r2, s, gx, gy, g2);
        gxl[q] = gx;
        gyl[q] = gy;
        gzl[q] = g2;
      }
    }
    __syncthreads();

    // ---- F: tx = C_x^T fx, ty = C_y^T fy, tz = C_z^T fz (in place) ---------
    {
      double in[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* g = S2 + cc[j] * GXr.cs + ra[j] * GXr.sy + rb[j];
#pragma unroll
        for (int i = 0; i < N; ++i) in[j][i] = on[j] ? g[i * GXr.sx] : 0.0;
      }
      v6r_contract<N, N, LD, R>(T.CT, in, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* g = S2 + cc[j] * GXr.cs + ra[j] * GXr.sy + rb[j];
#pragma unroll
          for (int jj = 0; jj < N; ++jj) g[jj * GXr.sx] = o[j][jj];
        }
    }
    __syncwarp();
    {
      double in[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* g = S3 + cc[j] * GYr.cs + ra[j] * GYr.sx + rb[j];
#pragma unroll
        for (int i = 0; i < N; ++i) in[j][i] = on[j] ? g[i * GYr.sy] : 0.0;
      }
      v6r_contract<N, N, LD, R>(T.CT, in, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* g = S3 + cc[j] * GYr.cs + ra[j] * GYr.sx + rb[j];
#pragma unroll
          for (int jj = 0; jj < N; ++jj) g[jj * GYr.sy] = o[j][jj];
        }
    }
    __syncwarp();
    {
      double in[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* g = S4 + cc[j] * GZr.cs + ra[j] * GZr.sy + rb[j] * GZr.sx;
#pragma unroll
        for (int i = 0; i < N; ++i) in[j][i] = on[j] ? g[i] : 0.0;
      }
      v6r_contract<N, N, LD, R>(T.CT, in, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* g = S4 + cc[j] * GZr.cs + ra[j] * GZr.sy + rb[j] * GZr.sx;
#pragma unroll
          for (int jj = 0; jj < N; ++jj) g[jj] = o[j][jj];
        }
    }
    __syncthreads();

    // ---- G: z-lines: t = tx + ty + tz, R = B_z^T t -> S1 --------------------
    {
      double t[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int c = cc[j], qy = ra[j], qx = rb[j];
        const double* gxl = S2 + c * GXr.cs + qx * GXr.sx + qy * GXr.sy;
        const double* gyl = S3 + c * GYr.cs + qy * GYr.sy + qx * GYr.sx;
        const double* tzl = S4 + c * GZr.cs + qy * GZr.sy + qx * GZr.sx;
#pragma unroll
        for (int q = 0; q < N; ++q) t[j][q] = (gxl[q] + gyl[q]) + tzl[q];
      }
      v6r_contract<N, N, LD, R>(T.BT, t, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* w = S1 + cc[j] * Rr.cs + ra[j] * Rr.sy + rb[j] * Rr.sx;
#pragma unroll
          for (int i = 0; i < N; ++i) w[i] = o[j][i];
        }
    }
    __syncthreads();

    // ---- H: y-lines: B_y^T R -> S2 (P2) -------------------------------------
    {
      double in[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* q = S1 + cc[j] * Rr.cs + ra[j] * Rr.sx + rb[j];
#pragma unroll
        for (int jj = 0; jj < N; ++jj) in[j][jj] = q[jj * Rr.sy];
      }
      v6r_contract<N, N, LD, R>(T.BT, in, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j]) {
          double* p = S2 + cc[j] * P2.cs + ra[j] * P2.sx + rb[j];
#pragma unroll
          for (int i = 0; i < N; ++i) p[i * P2.sy] = o[j][i];
        }
    }
    __syncthreads();

    // ---- I: x-lines: A = B_x^T (.) -> HBM ----------------------------------
    {
      double in[R][N], o[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* p = S2 + cc[j] * P2.cs + ra[j] * P2.sy + rb[j];
#pragma unroll
        for (int q = 0; q < N; ++q) in[j][q] = p[q * P2.sx];
      }
      v6r_contract<N, N, LD, R>(T.BT, in, o);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (on[j] && cc[j] < ncb) {
          double* ap = A + (cell0 + cc[j]) * N3 + rr[j];
#pragma unroll
          for (int i = 0; i < N; ++i) ap[i * NN] = o[j][i];
        }
    }
  }
}

template <int N, int CPB, int R, int MINB>
static int launch_v6r(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                      const double* u, cudaStream_t s) {
  using C = V6RCfg<N, CPB, R>;
  if (((reinterpret_cast<uintptr_t>(coords)) & 15) != 0) return SFK_EUNSUPPORTED;
  auto kern = hex_laplace_action_v6r<N, CPB, R, MINB>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_action_v6r", &sh, true))
    return rc_;
  const TabsV6<N> T = make_tabs_v6<N>(p);
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, u, A);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_v6r launch");
}

// (cells per CTA, lines per thread, min CTAs per SM) per n; v6_cfg = 1, 2
// select the A/B alternatives
int launch_hex_action_v6r(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          const double* w0, cudaStream_t s) {
  if (p->n != p->m || !p->has_ct) return SFK_EUNSUPPORTED;
  const int alt = (int)option(OPT_V6_CFG);
  switch (p->n) {
    case 7:
      if (alt == 1) return launch_v6r<7, 5, 2, 3>(p, ncells, A, coords, w0, s);
      return launch_v6r<7, 5, 2, 2>(p, ncells, A, coords, w0, s);
    case 9:
      if (alt == 1) return launch_v6r<9, 3, 2, 3>(p, ncells, A, coords, w0, s);
      if (alt == 2) return launch_v6r<9, 4, 2, 2>(p, ncells, A, coords, w0, s);
      return launch_v6r<9, 3, 2, 2>(p, ncells, A, coords, w0, s);
    default: return SFK_EUNSUPPORTED;
  }
}

}  // namespace sfk
