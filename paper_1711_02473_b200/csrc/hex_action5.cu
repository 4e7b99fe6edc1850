// Hex Q_p Laplace action, line kernel v5 — BASELINE C2 (headline) at the
// high degrees.
//
// Same math, reference mapping, shared-memory layout and pipeline as v2
// (hex_action2.cu: forms.py:186-189, 235-243; passes.py:672-743;
// scheduling.py:617-738), one line per thread.  What changes is the
// instruction schedule inside a stage.  v2 stores each output right after
// its accumulation behind an `if (line is live)` branch; the branch fences
// the compiler's scheduler, so a warp only ever had the 2-3 chains of ONE
// output in flight (x^T: a single 2M-deep chain).  The DFMA latency on B200
// is 8 cycles and the FP64 pipe takes one warp-DFMA per 2 cycles per SMSP
// (tools/fp64_lat.cu, profiles/r01bt_fp64_lat.txt), so with 4 resident
// warps per SMSP every stall elsewhere (LDS, barrier, LDCU) left the pipe
// idle: "wait" was the top stall reason (27%) of v2 at p = 8.
//
// Here every stage computes its outputs in groups of G: the G x (2 or 3)
// accumulator chains of a group are independent, the stores of a group sit
// behind one branch, and the transposed stages keep one chain per table
// (summed at the end).  G trades registers for ILP; it is chosen per degree
// from measurements (launch_hex_action_v5).
#include <cstdlib>

// pointwise loop unroll factor (0 = per degree; A/B builds)
#ifndef SFK_V5_UP
#define SFK_V5_UP 0
#endif
// Y/S line order (1 = qy-major; A/B builds)
#ifndef SFK_V5_YT
#define SFK_V5_YT 1
#endif

#include "async_copy.cuh"
#include "hex_geometry.cuh"
#include "hex_line_cfg.cuh"

namespace sfk {

constexpr int V5_UP = SFK_V5_UP;

// Per-cell Y/S stride padding for the qy-major layout (tools/smem_pads_yt.py:
// modelled wavefronts of the y-stage and z-stage accesses, cell boundaries
// included, z weighted 3x as it is accessed 3x as often; n = 9: 2201,
// n = 7: 1031, n = 6: 764 doubles per cell).
__host__ __device__ constexpr int v5_ypad(int n) {
#ifdef SFK_V5_YPAD
  if (SFK_V5_YPAD >= 0) return SFK_V5_YPAD;
#endif
  return SFK_V5_YT ? (n == 9 ? 14 : n == 7 ? 2 : n == 6 ? 8 : n == 5 ? 6 : 0) : 0;
}

// GS = true: global operator y += sum_c P_c^T A_c P_c x (SURVEY.md §8(f)
// item 1), as in v2: `u` is x, `A` is y, cmap[c][i] the global dof of local
// dof i; the map (int32) is double-buffered in the u buffer, x is gathered
// through it in the x stage and y scattered with fp64 atomics in x^T.
template <int N, int CPB, int G, int MINB, bool PAIRS, bool GS = false>
__global__ void __launch_bounds__(HexAction2Cfg<N, N, CPB, 1, v5_ypad(N)>::THREADS, MINB)
hex_laplace_action_v5(const __grid_constant__ TabsBD<N, N> T, int64_t ncells,
                      const double* __restrict__ coords, const double* __restrict__ u,
                      double* __restrict__ A, const int* __restrict__ cmap = nullptr) {
  using C = HexAction2Cfg<N, N, CPB, 1, v5_ypad(N)>;
  constexpr int M = N;
  constexpr int NN = C::NN, MN = C::MN, MM = C::MM, N3 = C::N3, PX = C::PX, LZ = C::LZ;
  constexpr int XA = C::XA, YA = C::YA, TH = C::THREADS;
  // YT: Y/S lines stored qy-major ([qy][qx][z]) instead of qx-major: the y
  // and y^T stages (thread (qx, iz), iz fastest) then touch consecutive
  // addresses LZ*qx + iz — conflict-free — while the z stage (thread = line
  // slot, stride LZ odd) stays conflict-free; qx-major cost 2-3-way
  // conflicts there (profiles/r01bv_p6.md: 34% excess wavefronts).
  constexpr bool YT = SFK_V5_YT;
  constexpr int QS = YT ? M * LZ : LZ;      // stride of q (= qy) in the y stages
  // pointwise loop: 3-way unrolled at n = 9 (126 registers, p = 8 3.51 ->
  // 3.46 ms, profiles/r01by_*.jsonl), rolled elsewhere (no gain / spills)
  constexpr int UPN = V5_UP > 0 ? V5_UP : (N == 9 ? 3 : 1);
  extern __shared__ __align__(16) double smem[];
  double* sX = smem;                        // [CPB][2][M][PX]
  double* sY = sX + CPB * C::XSZ;           // [CPB][3][M*M][LZ]
  double* sU = smem + round_up(CPB * C::XSZ + CPB * C::YSZ, 2);  // [CPB*N3+1]
  double* sCo = sU + C::USZ;                // [2][CPB*24]
  const int tid = threadIdx.x;
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  int* sMap = reinterpret_cast<int*>(sU);   // GS: [2][CPB*N3] int32 in the u buffer
  static_assert(!GS || 2 * CPB * N3 <= 2 * C::USZ, "map double buffer does not fit");

  auto prefetch = [&](int64_t b, int buf) {
    const int64_t c0 = b * CPB;
    const int nc = (int)((ncells - c0) < CPB ? (ncells - c0) : CPB);
    if (GS) {
      for (int i = tid; i < nc * N3; i += TH)
        cp_async4(sMap + buf * CPB * N3 + i, cmap + c0 * N3 + i);
    } else {
      async_copy_phase<TH>(sU + dst_shift(u + c0 * N3), u + c0 * N3, nc * N3, tid);
    }
    async_copy<TH>(sCo + buf * C::CSZ, coords + c0 * 24, nc * 24, tid);
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
    const double* su = sU + (GS ? 0 : dst_shift(u + cell0 * N3));
    const int* smap = sMap + cur * CPB * N3;
    const double* sC = sCo + cur * C::CSZ;

    // ---- x stage: line (c, iy, iz): X0 = Bx u, X1 = Dx u ----------------
    {
      constexpr int L = CPB * NN;
      const bool on = tid < L;
      const int lc = on ? tid : 0;
      const int c = lc / NN, r = lc - c * NN;
      const bool live = on && c < ncb;
      double uu[N];
#pragma unroll
      for (int i = 0; i < N; ++i)
        uu[i] = live ? (GS ? __ldg(u + smap[c * N3 + i * NN + r]) : su[c * N3 + i * NN + r]) : 0.0;
      double* xo = sX + c * C::XSZ + r;
#pragma unroll
      for (int q0 = 0; q0 < M; q0 += G) {
        double bq[G], dq[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (q0 + g < M) {
            bq[g] = TBP(q0 + g) * uu[0];
            dq[g] = TDP(q0 + g) * uu[0];
          }
#pragma unroll
        for (int i = 1; i < N; ++i)
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (q0 + g < M) {
              bq[g] = fma(TBP(i * M + q0 + g), uu[i], bq[g]);
              dq[g] = fma(TDP(i * M + q0 + g), uu[i], dq[g]);
            }
        if (on) {
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (q0 + g < M) {
              xo[(q0 + g) * PX] = bq[g];
              xo[XA + (q0 + g) * PX] = dq[g];
            }
        }
      }
    }
    __syncthreads();
    if (b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- y stage: line (c, qx, iz): BB = By X0, BD = Dy X0, DB = By X1 ---
    {
      constexpr int L = CPB * MN;
      const bool on = tid < L;
      const int lc = on ? tid : 0;
      const int c = lc / MN, r = lc - c * MN;
      const int qx = r / N, iz = r - qx * N;
      const double* xi = sX + c * C::XSZ + qx * PX + iz;
      double a0[N], a1[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        a0[i] = xi[i * N];
        a1[i] = xi[XA + i * N];
      }
      double* yo = sY + c * C::YSZ + (YT ? qx * LZ : qx * M * LZ) + iz;
#pragma unroll
      for (int q0 = 0; q0 < M; q0 += G) {
        double bb[G], bd[G], db[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (q0 + g < M) {
            bb[g] = TBP(q0 + g) * a0[0];
            bd[g] = TDP(q0 + g) * a0[0];
            db[g] = TBP(q0 + g) * a1[0];
          }
#pragma unroll
        for (int i = 1; i < N; ++i)
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (q0 + g < M) {
              bb[g] = fma(TBP(i * M + q0 + g), a0[i], bb[g]);
              bd[g] = fma(TDP(i * M + q0 + g), a0[i], bd[g]);
              db[g] = fma(TBP(i * M + q0 + g), a1[i], db[g]);
            }
        if (on) {
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (q0 + g < M) {
              yo[(q0 + g) * QS] = bb[g];
              yo[YA + (q0 + g) * QS] = bd[g];
              yo[2 * YA + (q0 + g) * QS] = db[g];
            }
        }
      }
    }
    __syncthreads();

    // ---- z stage: line (c, qx, qy), three in-place passes ----------------
    {
      constexpr int L = CPB * MM;
      const bool on = tid < L;
      const int lc = on ? tid : 0;
      const int c = lc / MM, r = lc - c * MM;
      double* yl = sY + c * C::YSZ + r * LZ;
      // (1) reference gradient lines: slot 0 <- Dz BB, 1 <- Bz BD, 2 <- Bz DB
      {
        double bb[N], bd[N], db[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          bb[i] = yl[i];
          bd[i] = yl[YA + i];
          db[i] = yl[2 * YA + i];
        }
#pragma unroll
        for (int q0 = 0; q0 < M; q0 += G) {
          double gz[G], gy[G], gx[G];
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (q0 + g < M) {
              gz[g] = TDP(q0 + g) * bb[0];
              gy[g] = TBP(q0 + g) * bd[0];
              gx[g] = TBP(q0 + g) * db[0];
            }
#pragma unroll
          for (int i = 1; i < N; ++i)
#pragma unroll
            for (int g = 0; g < G; ++g)
              if (q0 + g < M) {
                gz[g] = fma(TDP(i * M + q0 + g), bb[i], gz[g]);
                gy[g] = fma(TBP(i * M + q0 + g), bd[i], gy[g]);
                gx[g] = fma(TBP(i * M + q0 + g), db[i], gx[g]);
              }
          if (on) {
#pragma unroll
            for (int g = 0; g < G; ++g)
              if (q0 + g < M) {
                yl[q0 + g] = gz[g];
                yl[YA + q0 + g] = gy[g];
                yl[2 * YA + q0 + g] = gx[g];
              }
          }
        }
      }
      // (2) pointwise: geometry per point + Laplace flux, in place
      {
        const int r0 = r / M, r1 = r - r0 * M;
        const int qx = YT ? r1 : r0, qy = YT ? r0 : r1;
        HexLineAdj geo;
        geo.setup(sC + c * 24, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
        const double wxy = T.W[qx] * T.W[qy];
#pragma unroll (UPN)
        for (int q = 0; q < M; ++q) {
          double gz = yl[q], gy = yl[YA + q], gx = yl[2 * YA + q];
          double r0[3], r1[3], r2[3];
          const double det = geo.adj(T.Bc[M + q], r0, r1, r2);
          const double s = (wxy * T.W[q]) * rcp64(fabs(det));
          laplace_flux(r0, r1, r2, s, gx, gy, gz);
          if (on) {
            yl[q] = gz;
            yl[YA + q] = gy;
            yl[2 * YA + q] = gx;
          }
        }
      }
      // (3) transposed z, in place: slot 0 <- Dz^T f_z, 1 <- Bz^T f_y,
      //     2 <- Bz^T f_x
      {
        double fz[M], fy[M], fx[M];
#pragma unroll
        for (int q = 0; q < M; ++q) {
          fz[q] = yl[q];
          fy[q] = yl[YA + q];
          fx[q] = yl[2 * YA + q];
        }
#pragma unroll
        for (int i0 = 0; i0 < N; i0 += G) {
          double sz[G], sy[G], sx[G];
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (i0 + g < N) {
              sz[g] = TDP((i0 + g) * M) * fz[0];
              sy[g] = TBP((i0 + g) * M) * fy[0];
              sx[g] = TBP((i0 + g) * M) * fx[0];
            }
#pragma unroll
          for (int q = 1; q < M; ++q)
#pragma unroll
            for (int g = 0; g < G; ++g)
              if (i0 + g < N) {
                sz[g] = fma(TDP((i0 + g) * M + q), fz[q], sz[g]);
                sy[g] = fma(TBP((i0 + g) * M + q), fy[q], sy[g]);
                sx[g] = fma(TBP((i0 + g) * M + q), fx[q], sx[g]);
              }
          if (on) {
#pragma unroll
            for (int g = 0; g < G; ++g)
              if (i0 + g < N) {
                yl[i0 + g] = sz[g];
                yl[YA + i0 + g] = sy[g];
                yl[2 * YA + i0 + g] = sx[g];
              }
          }
        }
      }
    }
    __syncthreads();

    // ---- transposed y: line (c, qx, iz): R1 = By^T Sx,
    //      R2 = Dy^T Sy + By^T Sz (two chains, summed last) ------------------
    {
      constexpr int L = CPB * MN;
      const bool on = tid < L;
      const int lc = on ? tid : 0;
      const int c = lc / MN, r = lc - c * MN;
      const int qx = r / N, iz = r - qx * N;
      const double* yi = sY + c * C::YSZ + (YT ? qx * LZ : qx * M * LZ) + iz;
      double pz[M], py[M], px[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        pz[q] = yi[q * QS];
        py[q] = yi[YA + q * QS];
        px[q] = yi[2 * YA + q * QS];
      }
      double* xo = sX + c * C::XSZ + qx * PX + iz;
#pragma unroll
      for (int i0 = 0; i0 < N; i0 += G) {
        double r1[G], r2[G], r3[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (i0 + g < N) {
            r1[g] = TBP((i0 + g) * M) * px[0];
            r2[g] = TDP((i0 + g) * M) * py[0];
            r3[g] = TBP((i0 + g) * M) * pz[0];
          }
#pragma unroll
        for (int q = 1; q < M; ++q)
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (i0 + g < N) {
              r1[g] = fma(TBP((i0 + g) * M + q), px[q], r1[g]);
              r2[g] = fma(TDP((i0 + g) * M + q), py[q], r2[g]);
              r3[g] = fma(TBP((i0 + g) * M + q), pz[q], r3[g]);
            }
        if (on) {
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (i0 + g < N) {
              xo[(i0 + g) * N] = r1[g];
              xo[XA + (i0 + g) * N] = r2[g] + r3[g];
            }
        }
      }
    }
    __syncthreads();

    // ---- transposed x: line (c, iy, iz) -> A = Dx^T R1 + Bx^T R2 -----------
    {
      constexpr int L = CPB * NN;
      const bool on = tid < L && tid / NN < ncb;
      const int lc = on ? tid : 0;
      const int c = lc / NN, r = lc - c * NN;
      const double* xi = sX + c * C::XSZ + r;
      double p1[M], p2[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        p1[q] = xi[q * PX];
        p2[q] = xi[XA + q * PX];
      }
      double* ap = A + (cell0 + c) * N3 + r;
#pragma unroll
      for (int i0 = 0; i0 < N; i0 += G) {
        double a1[G], a2[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (i0 + g < N) {
            a1[g] = TDP((i0 + g) * M) * p1[0];
            a2[g] = TBP((i0 + g) * M) * p2[0];
          }
#pragma unroll
        for (int q = 1; q < M; ++q)
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (i0 + g < N) {
              a1[g] = fma(TDP((i0 + g) * M + q), p1[q], a1[g]);
              a2[g] = fma(TBP((i0 + g) * M + q), p2[q], a2[g]);
            }
        if (on) {
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (i0 + g < N) {
              if (GS) atomicAdd(A + smap[c * N3 + (i0 + g) * NN + r], a1[g] + a2[g]);
              else ap[(i0 + g) * NN] = a1[g] + a2[g];
            }
        }
      }
    }
    __syncthreads();   // X/R is rewritten by the next batch's x stage
  }
}

template <int N, int CPB, int G, int MINB, bool PAIRS, bool GS = false>
static int launch_v5(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* u, cudaStream_t s, const int* cmap = nullptr) {
  using C = HexAction2Cfg<N, N, CPB, 1, v5_ypad(N)>;
  auto kern = hex_laplace_action_v5<N, CPB, G, MINB, PAIRS, GS>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_action_v5", &sh, true))
    return rc_;
  const TabsBD<N, N> T = make_tabs_bd<N, N>(p);
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, u, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_v5 launch");
}

// Output group size per degree: option c2_g overrides (tuning runs only).
template <int N, int CPB, int G0, bool PAIRS = true>
static int pick_v5(int g, const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                   const double* w0, cudaStream_t s) {
  switch (g ? g : G0) {
    case 1: return launch_v5<N, CPB, 1, 2, PAIRS>(p, ncells, A, coords, w0, s);
    case 2: return launch_v5<N, CPB, 2, 2, PAIRS>(p, ncells, A, coords, w0, s);
    default: return launch_v5<N, CPB, 3, 2, PAIRS>(p, ncells, A, coords, w0, s);
  }
}

int launch_hex_action_v5(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s) {
  if (p->n != p->m) return SFK_EUNSUPPORTED;
  const int g_env = (int)option(OPT_C2_G);
  const int cpb6_env = (int)option(OPT_V5_CPB6);
  switch (p->n) {
    // profiles/r01bu_*.jsonl (same box, ms at 2^18 cells; G = 1 / 2 / 3):
    //   n = 5: 0.592 / 0.590 / 0.588 (v3 0.531 stays)   n = 6: 0.985 / 1.87 (spills) / 1.10
    //   n = 7: 1.676 / 1.621 / 1.667                     n = 9: 3.642 / 3.513 / 4.33 (spills)
    case 5: return pick_v5<5, 10, 2>(g_env, p, ncells, A, coords, w0, s);
    case 6:
      // CPB 7 = 256 threads (register cap 128: (B, D) pairs fit) over CPB 8
      // = 288 threads (cap 96: no pairs): 0.995 -> 0.947 ms with G = 1
      // (profiles/r01cb_*.jsonl); option v5_cpb6 = 8 selects the latter.  6 cells
      // per CTA at 3 CTAs/SM spill (80-register cap): 1.07 ms (r01cz_*)
      if (cpb6_env == 8) return pick_v5<6, 8, 1, false>(g_env, p, ncells, A, coords, w0, s);
      return pick_v5<6, 7, 1>(g_env, p, ncells, A, coords, w0, s);
    case 7: return pick_v5<7, 5, 2>(g_env, p, ncells, A, coords, w0, s);
    case 9: return pick_v5<9, 3, 2>(g_env, p, ncells, A, coords, w0, s);
    default: return SFK_EUNSUPPORTED;
  }
}

// Global operator (fused gather / scatter) through v5 at n = 6, 7, 9.
int launch_hex_action_v5_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s) {
  if (p->n != p->m) return SFK_EUNSUPPORTED;
  switch (p->n) {
    case 6: return launch_v5<6, 7, 1, 2, true, true>(p, ncells, y, coords, x, s, cmap);
    case 7: return launch_v5<7, 5, 2, 2, true, true>(p, ncells, y, coords, x, s, cmap);
    case 9: return launch_v5<9, 3, 2, 2, true, true>(p, ncells, y, coords, x, s, cmap);
    default: return SFK_EUNSUPPORTED;
  }
}

}  // namespace sfk
