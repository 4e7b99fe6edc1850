// Hex Q_p Laplace action, line kernel v3 — BASELINE config C2 (headline).
//
// Math and reference mapping as in hex_action.cu (forms.py:186-189 _laplace,
// :235-243 action_form, passes.py:672-743 spectral schedule,
// scheduling.py:617-738 emitted kernel): 8 forward 1D contractions, the
// pointwise flux w|J| G G^T grad u with J recomputed per point from the
// 8 vertices, 8 transposed contractions; A overwritten.
//
// Mapping (one thread per line and stage; r01 ncu captures in profiles/):
//  * persistent CTAs; u and coords of the next cell batch stream HBM ->
//    shared memory with cp.async while the current batch computes (u right
//    after the x stage consumed it, coords double-buffered);
//  * every contraction streams its input line ("i outer"): each input value
//    is read once and feeds M independent accumulator chains, so DFMA
//    latency is covered by ILP within the thread, and the table entry of
//    each DFMA is a constant-bank operand (fully unrolled, __grid_constant__
//    tables);
//  * the z stage runs as three passes over thread-private shared lines
//    (gradients in place, pointwise flux in place — a rolled loop, the
//    per-point geometry being identical code for every point — then the
//    transposed z contraction in place);
//  * shared strides from tools/smem_pads_action.py (bank-conflict search).
#include <cstdlib>
// 128-bit (B, D) table pairs measured slower here (p=5 1.03 -> 1.6 ms):
// separate B / D tables
#define SFK_TAB_PAIRS 0
#ifndef SFK_V3_MINB5
#define SFK_V3_MINB5 2   // min CTAs/SM at n = 5 (A/B builds; 3 spills: 0.508 -> 0.615 ms, r01da_*)
#endif
#ifndef SFK_V3_YT
#define SFK_V3_YT 1
#endif
#include "async_copy.cuh"
#include "hex_geometry.cuh"

namespace sfk {

// Layout per cell (doubles):
//   X/R [2][M][N][N]  index k*XA + q*PX + iy*XY + iz       XA = M*PX
//   Y/S [3][M][M][N]  index k*YA + qx*YX + qy*LZ + iz      YA = M*YX
template <int N_, int M_, int CPB_, int XY_, int PX_, int XC_, int LZ_, int YX_, int YC_>
struct Act3Layout {
  static constexpr int N = N_, M = M_, CPB = CPB_;
  static constexpr int XY = XY_, PX = PX_, XC = XC_, LZ = LZ_, YX = YX_, YC = YC_;
  static constexpr int NN = N * N, MN = M * N, MM = M * M, N3 = N * N * N;
  static constexpr int XA = M * PX, YA = M * YX;
  static constexpr int THREADS = round_up(CPB * (MM > NN ? MM : NN), 32);
  static constexpr int USZ = round_up(CPB * N3 + 1, 2);
  static constexpr int CSZ = CPB * 24;
  static constexpr size_t SMEM = (size_t)(round_up(CPB * XC + CPB * YC, 2) + USZ + 2 * CSZ) * sizeof(double);
  static_assert(XC >= 2 * XA && YC >= 3 * YA && LZ >= M && LZ >= N, "layout too small");
};

// GS = false: batched E-vector action, A[c] = A_c u[c] (BASELINE C2).
// GS = true : global operator y += sum_c P_c^T A_c P_c x (SURVEY.md §8(f)
//             item 1): `u` is the global vector x, `A` the global vector y,
//             cmap[c][i] the global dof of local dof i of cell c.  The gather
//             is fused into the x stage (x[cmap] read through L1/L2, the map
//             block itself streamed with cp.async), the scatter into the
//             transposed x stage (fp64 atomicAdd; neighbouring cells share
//             face/edge/vertex dofs).
template <class L, int MINB, bool GS = false>
__global__ void __launch_bounds__(L::THREADS, MINB)
hex_laplace_action_v3(const __grid_constant__ Tabs<L::N, L::M> T, int64_t ncells,
                      const double* __restrict__ coords, const double* __restrict__ u,
                      double* __restrict__ A, const int* __restrict__ cmap = nullptr) {
  constexpr int N = L::N, M = L::M, CPB = L::CPB, NN = L::NN, MN = L::MN, MM = L::MM;
  constexpr int N3 = L::N3, XY = L::XY, PX = L::PX, XC = L::XC, LZ = L::LZ, YX = L::YX;
  constexpr int YC = L::YC, XA = L::XA, YA = L::YA, TH = L::THREADS;
  // YT: Y/S lines qy-major (element (qx, qy, z) at qy*YX + qx*LZ + z), so
  // the y / y^T stages (thread (qx, iz), iz fastest) touch consecutive
  // addresses; the z stage sees the same line slots in another order.  On at
  // n = 5 only (tools/smem_pads_yt.py: y-stage wavefronts 31 -> 25 per
  // access at the z-optimal cell stride 381; the other n keep their
  // searched qx-major strides).
  constexpr bool YT = SFK_V3_YT && N == 5 && YX == M * LZ;
  constexpr int QS = YT ? YX : LZ;
  extern __shared__ __align__(16) double smem[];
  double* sX = smem;
  double* sY = sX + CPB * XC;
  double* sU = smem + round_up(CPB * XC + CPB * YC, 2);
  double* sCo = sU + L::USZ;
  const int tid = threadIdx.x;
  const int64_t nbatch = (ncells + CPB - 1) / CPB;

  int* sMap = reinterpret_cast<int*>(sU);   // GS: [2][CPB*N3] in the u buffer
  auto prefetch = [&](int64_t bb, int buf) {
    const int64_t c0 = bb * CPB;
    const int nc = (int)((ncells - c0) < CPB ? (ncells - c0) : CPB);
    if (GS) {
      for (int i = tid; i < nc * N3; i += TH) cp_async4(sMap + buf * CPB * N3 + i, cmap + c0 * N3 + i);
    } else {
      async_copy_phase<TH>(sU + dst_shift(u + c0 * N3), u + c0 * N3, nc * N3, tid);
    }
    async_copy<TH>(sCo + buf * L::CSZ, coords + c0 * 24, nc * 24, tid);
    cp_async_commit();
  };

  int64_t b = blockIdx.x;
  if (b < nbatch) prefetch(b, 0);
  for (int k = 0; b < nbatch; b += gridDim.x, ++k) {
    const int cur = k & 1;
    const int64_t cell0 = b * CPB;
    const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
    cp_async_wait<0>();
    __syncthreads();
    const double* sC = sCo + cur * L::CSZ;

    // ---- x stage: line (c, iy, iz) -> X0 = Bx u, X1 = Dx u ---------------
    if (tid < CPB * NN) {
      const int c = tid / NN, r = tid - c * NN;
      const int iy = r / N, iz = r - iy * N;
      const double* ui = sU + (GS ? 0 : dst_shift(u + cell0 * N3)) + c * N3 + r;
      const int* mi = sMap + cur * CPB * N3 + c * N3 + r;
      const bool live = c < ncb;
      auto uval = [&](int i) { return GS ? __ldg(u + mi[i * NN]) : ui[i * NN]; };
      double xb[M], xd[M];
      {
        const double v = live ? uval(0) : 0.0;
#pragma unroll
        for (int q = 0; q < M; ++q) {
          xb[q] = TB(q) * v;
          xd[q] = TD(q) * v;
        }
      }
#pragma unroll
      for (int i = 1; i < N; ++i) {
        const double v = live ? uval(i) : 0.0;
#pragma unroll
        for (int q = 0; q < M; ++q) {
          xb[q] = fma(TB(i * M + q), v, xb[q]);
          xd[q] = fma(TD(i * M + q), v, xd[q]);
        }
      }
      double* xo = sX + c * XC + iy * XY + iz;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        xo[q * PX] = xb[q];
        xo[XA + q * PX] = xd[q];
      }
    }
    __syncthreads();
    if (b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- y stage: line (c, qx, iz) -> BB = By X0, BD = Dy X0, DB = By X1 --
    if (tid < CPB * MN) {
      const int c = tid / MN, r = tid - c * MN;
      const int qx = r / N, iz = r - qx * N;
      const double* xi = sX + c * XC + qx * PX + iz;
      double bb[M], bd[M], db[M];
      {
        const double v0 = xi[0], v1 = xi[XA];
#pragma unroll
        for (int q = 0; q < M; ++q) {
          bb[q] = TB(q) * v0;
          bd[q] = TD(q) * v0;
          db[q] = TB(q) * v1;
        }
      }
#pragma unroll
      for (int i = 1; i < N; ++i) {
        const double v0 = xi[i * XY], v1 = xi[XA + i * XY];
#pragma unroll
        for (int q = 0; q < M; ++q) {
          bb[q] = fma(TB(i * M + q), v0, bb[q]);
          bd[q] = fma(TD(i * M + q), v0, bd[q]);
          db[q] = fma(TB(i * M + q), v1, db[q]);
        }
      }
      double* yo = sY + c * YC + (YT ? qx * LZ : qx * YX) + iz;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        yo[q * QS] = bb[q];
        yo[YA + q * QS] = bd[q];
        yo[2 * YA + q * QS] = db[q];
      }
    }
    __syncthreads();

    // ---- z stage: line (c, qx, qy), three in-place passes ------------------
    if (tid < CPB * MM) {
      const int c = tid / MM, r = tid - c * MM;
      const int r0 = r / M, r1 = r - r0 * M;
      const int qx = YT ? r1 : r0, qy = YT ? r0 : r1;
      double* yl = sY + c * YC + r0 * YX + r1 * LZ;
      // (1) reference gradient: slot0 <- Dz BB (d_z), slot1 <- Bz BD (d_y),
      //     slot2 <- Bz DB (d_x)
      {
        double gz[M], gy[M], gx[M];
        {
          const double v0 = yl[0], v1 = yl[YA], v2 = yl[2 * YA];
#pragma unroll
          for (int q = 0; q < M; ++q) {
            gz[q] = TD(q) * v0;
            gy[q] = TB(q) * v1;
            gx[q] = TB(q) * v2;
          }
        }
#pragma unroll
        for (int i = 1; i < N; ++i) {
          const double v0 = yl[i], v1 = yl[YA + i], v2 = yl[2 * YA + i];
#pragma unroll
          for (int q = 0; q < M; ++q) {
            gz[q] = fma(TD(i * M + q), v0, gz[q]);
            gy[q] = fma(TB(i * M + q), v1, gy[q]);
            gx[q] = fma(TB(i * M + q), v2, gx[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < M; ++q) {
          yl[q] = gz[q];
          yl[YA + q] = gy[q];
          yl[2 * YA + q] = gx[q];
        }
      }
      // (2) pointwise geometry + flux, rolled (identical code per point)
      {
        HexLineAdj geo;
        geo.setup(sC + c * 24, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
        const double wxy = T.W[qx] * T.W[qy];
#pragma unroll 1
        for (int q = 0; q < M; ++q) {
          double gz = yl[q], gy = yl[YA + q], gx = yl[2 * YA + q];
          double r0[3], r1[3], r2[3];
          const double det = geo.adj(T.Bc[M + q], r0, r1, r2);
          const double s = (wxy * T.W[q]) * rcp64(fabs(det));
          laplace_flux(r0, r1, r2, s, gx, gy, gz);
          yl[q] = gz;
          yl[YA + q] = gy;
          yl[2 * YA + q] = gx;
        }
      }
      // (3) transposed z: slot0 <- Dz^T f_z, slot1 <- Bz^T f_y, slot2 <- Bz^T f_x
      {
        double sz[N], sy[N], sx[N];
        {
          const double f0 = yl[0], f1 = yl[YA], f2 = yl[2 * YA];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            sz[i] = TD(i * M) * f0;
            sy[i] = TB(i * M) * f1;
            sx[i] = TB(i * M) * f2;
          }
        }
#pragma unroll
        for (int q = 1; q < M; ++q) {
          const double f0 = yl[q], f1 = yl[YA + q], f2 = yl[2 * YA + q];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            sz[i] = fma(TD(i * M + q), f0, sz[i]);
            sy[i] = fma(TB(i * M + q), f1, sy[i]);
            sx[i] = fma(TB(i * M + q), f2, sx[i]);
          }
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
          yl[i] = sz[i];
          yl[YA + i] = sy[i];
          yl[2 * YA + i] = sx[i];
        }
      }
    }
    __syncthreads();

    // ---- transposed y: line (c, qx, iz) -> R1 = By^T Sx, R2 = Dy^T Sy + By^T Sz
    if (tid < CPB * MN) {
      const int c = tid / MN, r = tid - c * MN;
      const int qx = r / N, iz = r - qx * N;
      const double* yi = sY + c * YC + (YT ? qx * LZ : qx * YX) + iz;
      double r1[N], r2[N];
      {
        const double pz = yi[0], py = yi[YA], px = yi[2 * YA];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          r1[i] = TB(i * M) * px;
          r2[i] = fma(TD(i * M), py, TB(i * M) * pz);
        }
      }
#pragma unroll
      for (int q = 1; q < M; ++q) {
        const double pz = yi[q * QS], py = yi[YA + q * QS], px = yi[2 * YA + q * QS];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          r1[i] = fma(TB(i * M + q), px, r1[i]);
          r2[i] = fma(TD(i * M + q), py, r2[i]);
          r2[i] = fma(TB(i * M + q), pz, r2[i]);
        }
      }
      double* xo = sX + c * XC + qx * PX + iz;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        xo[i * XY] = r1[i];
        xo[XA + i * XY] = r2[i];
      }
    }
    __syncthreads();

    // ---- transposed x: line (c, iy, iz) -> A = Dx^T R1 + Bx^T R2 -----------
    if (tid < CPB * NN) {
      const int c = tid / NN, r = tid - c * NN;
      if (c < ncb) {
        const int iy = r / N, iz = r - iy * N;
        const double* xi = sX + c * XC + iy * XY + iz;
        double a[N];
        {
          const double p1 = xi[0], p2 = xi[XA];
#pragma unroll
          for (int i = 0; i < N; ++i) a[i] = fma(TD(i * M), p1, TB(i * M) * p2);
        }
#pragma unroll
        for (int q = 1; q < M; ++q) {
          const double p1 = xi[q * PX], p2 = xi[XA + q * PX];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            a[i] = fma(TD(i * M + q), p1, a[i]);
            a[i] = fma(TB(i * M + q), p2, a[i]);
          }
        }
        if (GS) {
          const int* mi = sMap + cur * CPB * N3 + c * N3 + r;
#pragma unroll
          for (int i = 0; i < N; ++i) atomicAdd(A + mi[i * NN], a[i]);
        } else {
          double* ap = A + (cell0 + c) * N3 + r;
#pragma unroll
          for (int i = 0; i < N; ++i) ap[i * NN] = a[i];
        }
      }
    }
    __syncthreads();   // X/R is rewritten by the next batch's x stage
  }
}

template <class L, int MINB, bool GS = false>
static int launch_v3(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* u, cudaStream_t s, const int* cmap = nullptr) {
  auto kern = hex_laplace_action_v3<L, MINB, GS>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, L::THREADS, L::SMEM, "hex_action_v3", &sh, true))
    return rc_;
  const Tabs<L::N, L::M> T = make_tabs<L::N, L::M>(p);
  const int64_t nbatch = (ncells + L::CPB - 1) / L::CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, L::THREADS, L::SMEM, s>>>(T, ncells, coords, u, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_v3 launch");
}

// (N, M, CPB, XY, PX, XC, LZ, YX, YC) from tools/smem_pads_action.py
template <bool GS>
static int dispatch_v3(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                       const double* w0, cudaStream_t s, const int* cmap) {
  if (p->n != p->m) return SFK_EUNSUPPORTED;
  switch (p->n) {
    case 2: return launch_v3<Act3Layout<2, 2, 64, 2, 6, 28, 3, 6, 36>, 2, GS>(p, ncells, A, coords, w0, s, cmap);
    case 3: return launch_v3<Act3Layout<3, 3, 32, 3, 19, 121, 3, 9, 91>, 2, GS>(p, ncells, A, coords, w0, s, cmap);
    case 4: return launch_v3<Act3Layout<4, 4, 16, 4, 20, 160, 5, 20, 240>, 2, GS>(p, ncells, A, coords, w0, s, cmap);
    case 5: return launch_v3<Act3Layout<5, 5, 10, 5, 37, 377, 5, 25, 381>, SFK_V3_MINB5, GS>(p, ncells, A, coords, w0, s, cmap);
    case 6: return launch_v3<Act3Layout<6, 6, 8, 6, 38, 468, 9, 54, 980>, 2, GS>(p, ncells, A, coords, w0, s, cmap);
    case 7: return launch_v3<Act3Layout<7, 7, 5, 7, 55, 785, 9, 63, 1337>, 2, GS>(p, ncells, A, coords, w0, s, cmap);
    case 8: return launch_v3<Act3Layout<8, 8, 4, 8, 72, 1152, 9, 72, 1728>, 2, GS>(p, ncells, A, coords, w0, s, cmap);
    case 9: return launch_v3<Act3Layout<9, 9, 3, 9, 89, 1617, 9, 81, 2201>, 2, GS>(p, ncells, A, coords, w0, s, cmap);
    default: return SFK_EUNSUPPORTED;
  }
}

int launch_hex_action_v3(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s) {
  return dispatch_v3<false>(p, ncells, A, coords, w0, s, nullptr);
}

static bool force_v3_small() { return option(OPT_C2G_SMALL) == 3; }   // A/B of the p = 2, 3 path

// Same generation as the E-vector action per degree (sfk_api.cu c2_auto):
// p = 1 cell kernel, p = 2, 3 v4, p = 5, 6, 8 v2, p = 7 DMMA, p = 4 v3.
// option c2g_kernel = 3 forces v3 (A/B runs).
int launch_hex_action_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                         double* y, const double* coords, cudaStream_t s) {
  const bool force_v3 = option(OPT_C2G_KERNEL) == 3;
  const bool force_v2 = option(OPT_C2G_KERNEL) == 2;
  // round 2: the collocation-derivative kernels with fused gather / scatter
  // (v6 at n = 4..7, 9; tc8c at n = 8) unless option c2g_kernel picks a
  // round-1 generation (1 = round 1 selection below)
  if (option(OPT_C2G_KERNEL) == 0 && p->n == p->m) {
    int rc = p->n == 8 ? launch_hex_action_tc8c_gs(p, ncells, cmap, x, y, coords, s)
                       : launch_hex_action_v6_gs(p, ncells, cmap, x, y, coords, s);
    if (rc != SFK_EUNSUPPORTED) return rc;
  }
  if (!force_v3 && p->n == p->m) {
    if (p->n == 2 && (reinterpret_cast<uintptr_t>(cmap) & 15) == 0)   // int4 map loads
      return launch_hex_action_p1_gs(p, ncells, cmap, x, y, coords, s);
    if (p->n == 3 && !force_v3_small() && !force_v2)
      return launch_hex_action_cell_gs(p, ncells, cmap, x, y, coords, s);
    if ((p->n == 3 || p->n == 4) && !force_v3_small())
      return launch_hex_action_v4_gs(p, ncells, cmap, x, y, coords, s);
    if ((p->n == 6 || p->n == 7 || p->n == 9) && !force_v2)
      return launch_hex_action_v5_gs(p, ncells, cmap, x, y, coords, s);
    if (p->n == 6 || p->n == 7 || p->n == 9 || (p->n == 4 && force_v3_small()))
      return launch_hex_action_v2_gs(p, ncells, cmap, x, y, coords, s);
    if (p->n == 8) return launch_hex_action_tc_gs(p, ncells, cmap, x, y, coords, s);
  }
  return dispatch_v3<true>(p, ncells, y, coords, x, s, cmap);
}

}  // namespace sfk
