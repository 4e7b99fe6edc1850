// Hex Q_p Laplace action, warp-synchronous line kernel v4 — BASELINE C2,
// small degrees (n = m in 3..5, p = 2..4).
//
// Same math, reference mapping and stage bodies as v3 (hex_action3.cu; its
// header cites forms.py / passes.py / scheduling.py).  What changes is the
// ownership: for n = m every stage of a cell has exactly n^2 lines, so a
// warp can own floor(32 / n^2) whole cells (3 at n = 3, 2 at n = 4, 1 at
// n = 5) through all five stages.  Every exchange between stages then stays
// inside the warp (__syncwarp), and each warp prefetches its own cells' u
// and coords with cp.async — the CTA has no __syncthreads at all.  The v3
// capture at p = 2 spent 23% of its stall samples in barriers
// (profiles/r01ay_C2_p2.md).
#include <cstdlib>

#include "async_copy.cuh"
#include "hex_geometry.cuh"

namespace sfk {

template <int N_, int WARPS_, int XY_, int PX_, int XC_, int LZ_, int YX_, int YC_>
struct Act4Layout {
  static constexpr int N = N_, M = N_, WARPS = WARPS_;
  static constexpr int XY = XY_, PX = PX_, XC = XC_, LZ = LZ_, YX = YX_, YC = YC_;
  static constexpr int NN = N * N, N3 = N * N * N;
  static constexpr int CPW = 32 / NN;              // cells per warp
  static constexpr int CPB = CPW * WARPS;          // cells per CTA batch
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int XA = M * PX, YA = M * YX;
  static constexpr int CELLS = CPW * (XC + YC);    // per-warp X/R + Y/S
  static constexpr int UW = round_up(CPW * N3 + 1, 2);   // per-warp u (16B multiple)
  static constexpr int CW = CPW * 24;              // per-warp coords (one buffer)
  static constexpr int WS = round_up(CELLS, 2) + UW + 2 * CW;   // per-warp doubles
  static constexpr size_t SMEM = (size_t)WARPS * WS * sizeof(double);
  static_assert(XC >= 2 * XA && YC >= 3 * YA && LZ >= M, "layout too small");
  static_assert(CPW >= 1, "n^2 > 32");
};

// GS = true: global operator y += sum_c P_c^T A_c P_c x (SURVEY.md §8(f)
// item 1), as in v3: each warp double-buffers its cells' map (int32) in its
// u slot, gathers x through it in the x stage and scatter-adds y with fp64
// atomics in the transposed x stage.
template <class L, int MINB, bool GS = false>
__global__ void __launch_bounds__(L::THREADS, MINB)
hex_laplace_action_v4(const __grid_constant__ TabsBD<L::N, L::M> T, int64_t ncells,
                      const double* __restrict__ coords, const double* __restrict__ u,
                      double* __restrict__ A, const int* __restrict__ cmap = nullptr) {
  constexpr int N = L::N, M = L::M, NN = L::NN, N3 = L::N3, CPW = L::CPW, CPB = L::CPB;
  constexpr int XY = L::XY, PX = L::PX, XC = L::XC, LZ = L::LZ, YX = L::YX, YC = L::YC;
  constexpr int XA = L::XA, YA = L::YA, MN = M * N, MM = M * M;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* base = smem + warp * L::WS;
  double* sX = base;                               // [CPW][XC]
  double* sY = base + CPW * XC;                    // [CPW][YC]
  double* sU = base + round_up(L::CELLS, 2);       // [CPW*N3 + 1]
  double* sCo = sU + L::UW;                        // [2][CPW*24]
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  int* sMap = reinterpret_cast<int*>(sU);            // GS: [2][CPW*N3] int32
  static_assert(!GS || CPW * N3 <= L::UW, "map double buffer does not fit");

  auto prefetch = [&](int64_t bb, int buf) {
    const int64_t c0 = bb * CPB + warp * CPW;
    const int nc = (int)((ncells - c0) < CPW ? (ncells - c0) : CPW);
    if (nc > 0) {
      if (GS) {
        for (int e = lane; e < nc * N3; e += 32) cp_async4(sMap + buf * CPW * N3 + e, cmap + c0 * N3 + e);
      } else {
        async_copy_phase<32>(sU + dst_shift(u + c0 * N3), u + c0 * N3, nc * N3, lane);
      }
      async_copy<32>(sCo + buf * L::CW, coords + c0 * 24, nc * 24, lane);
    }
    cp_async_commit();
  };

  int64_t b = blockIdx.x;
  if (b < nbatch) prefetch(b, 0);
  for (int k = 0; b < nbatch; b += gridDim.x, ++k) {
    const int cur = k & 1;
    const int64_t cell0 = b * CPB + warp * CPW;   // this warp's first cell
    const int ncw = (int)((ncells - cell0) < CPW ? (ncells - cell0) : CPW);
    cp_async_wait<0>();
    __syncwarp();
    const double* sC = sCo + cur * L::CW;
    const bool act = lane < CPW * NN;              // n = m: every stage has NN lines/cell
    const int c = act ? lane / NN : 0, r = act ? lane - (lane / NN) * NN : 0;
    const bool live = act && c < ncw;
    const int* smap = sMap + cur * CPW * N3;

    // ---- x stage: line (c, iy, iz) -> X0 = Bx u, X1 = Dx u ---------------
    if (act) {
      const int iy = r / N, iz = r - iy * N;
      const double* ui = sU + (GS ? 0 : dst_shift(u + cell0 * N3)) + c * N3 + r;
      const int* mi = smap + c * N3 + r;
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
    __syncwarp();
    if (b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- y stage: line (c, qx, iz) -> BB = By X0, BD = Dy X0, DB = By X1 --
    if (act) {
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
      double* yo = sY + c * YC + qx * YX + iz;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        yo[q * LZ] = bb[q];
        yo[YA + q * LZ] = bd[q];
        yo[2 * YA + q * LZ] = db[q];
      }
    }
    __syncwarp();

    // ---- z stage: line (c, qx, qy), three in-place passes ------------------
    if (act) {
      const int qx = r / M, qy = r - qx * M;
      double* yl = sY + c * YC + qx * YX + qy * LZ;
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
    __syncwarp();

    // ---- transposed y: line (c, qx, iz) -> R1 = By^T Sx, R2 = Dy^T Sy + By^T Sz
    if (act) {
      const int qx = r / N, iz = r - qx * N;
      const double* yi = sY + c * YC + qx * YX + iz;
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
        const double pz = yi[q * LZ], py = yi[YA + q * LZ], px = yi[2 * YA + q * LZ];
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
    __syncwarp();

    // ---- transposed x: line (c, iy, iz) -> A = Dx^T R1 + Bx^T R2 -----------
    if (live) {
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
        const int* mi = smap + c * N3 + r;
#pragma unroll
        for (int i = 0; i < N; ++i) atomicAdd(A + mi[i * NN], a[i]);
      } else {
        double* ap = A + (cell0 + c) * N3 + r;
#pragma unroll
        for (int i = 0; i < N; ++i) ap[i * NN] = a[i];
      }
    }
    __syncwarp();   // X/R is rewritten by this warp's next x stage
  }
}

template <class L, int MINB, bool GS = false>
static int launch_v4(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* u, cudaStream_t s, const int* cmap = nullptr) {
  auto kern = hex_laplace_action_v4<L, MINB, GS>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, L::THREADS, L::SMEM, "hex_action_v4", &sh, true))
    return rc_;
  const TabsBD<L::N, L::M> T = make_tabs_bd<L::N, L::M>(p);
  const int64_t nbatch = (ncells + L::CPB - 1) / L::CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, L::THREADS, L::SMEM, s>>>(T, ncells, coords, u, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_v4 launch");
}

// 16 warps per CTA, no min-blocks cap: measured best of 4 / 8 / 12 / 16 / 24 /
// 32 warps and caps 1-3 (profiles/r01ba_c2_v4.jsonl)
#ifndef SFK_V4_WARPS
#define SFK_V4_WARPS 16
#endif
#ifndef SFK_V4_MINB
#define SFK_V4_MINB 1
#endif

// per-n shared strides: v3's searched paddings (tools/smem_pads_action.py)
int launch_hex_action_v4(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s) {
  if (p->n != p->m) return SFK_EUNSUPPORTED;
  constexpr int W = SFK_V4_WARPS, MB = SFK_V4_MINB;
  switch (p->n) {
    case 3: return launch_v4<Act4Layout<3, W, 3, 19, 121, 3, 9, 91>, MB>(p, ncells, A, coords, w0, s);
    case 4: return launch_v4<Act4Layout<4, W, 4, 20, 160, 5, 20, 240>, MB>(p, ncells, A, coords, w0, s);
    case 5: return launch_v4<Act4Layout<5, W, 5, 37, 377, 5, 25, 381>, MB>(p, ncells, A, coords, w0, s);
    default: return SFK_EUNSUPPORTED;
  }
}

int launch_hex_action_v4_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s) {
  if (p->n != p->m) return SFK_EUNSUPPORTED;
  constexpr int W = SFK_V4_WARPS, MB = SFK_V4_MINB;
  switch (p->n) {
    case 3: return launch_v4<Act4Layout<3, W, 3, 19, 121, 3, 9, 91>, MB, true>(p, ncells, y, coords, x, s, cmap);
    case 4: return launch_v4<Act4Layout<4, W, 4, 20, 160, 5, 20, 240>, MB, true>(p, ncells, y, coords, x, s, cmap);
    default: return SFK_EUNSUPPORTED;
  }
}

}  // namespace sfk
