// Hex Q_p Laplace action, line kernel v2 — BASELINE config C2 (headline).
//
// Same math and reference mapping as hex_action.cu (v1; see its header:
// forms.py:186-189, 235-243; passes.py:672-743 schedule; scheduling.py:617-738
// emitted kernel).  What changes is the B200 mapping, driven by the r01 ncu
// capture of v1 at p=8 (profiles/r01a_prof_p8.md): FP64 pipe 53% busy, one
// 8-warp CTA per SM (254 registers), 14% of stalls on the HBM loads of u,
// 7% on barriers, and one LDCU (constant -> uniform register) per DFMA in
// the contractions.
//
//  * R lines per thread and stage: every table entry fetched into a uniform
//    register feeds R DFMAs (R independent accumulator sets = R-fold ILP).
//  * Persistent CTAs, double-buffered: u and coords of the NEXT cell batch
//    are copied HBM -> shared memory with cp.async (LDGSTS) while the
//    current batch computes; the x stage reads u from shared memory.
//  * z stage in three register-light passes over thread-private shared
//    lines: (1) reference gradient lines written in place, (2) pointwise
//    geometry + flux in place, (3) transposed z in place — no barrier
//    between them and no 6N-wide register working set.
//  * Small CTAs (2+ per SM) so barrier waits of one CTA overlap with the
//    other's work.
#include <cstdlib>

#include "async_copy.cuh"
#include "hex_geometry.cuh"
#include "hex_line_cfg.cuh"

// SFK_V2_CLAMP=1: threads past a stage's last line redo that line instead of
// skipping it, so every store is unconditional (no branch between the
// unrolled output iterations: the compiler can interleave the accumulator
// chains of different outputs; with the branches the transposed stages ran
// as one 2M-deep DFMA chain at a time).
#ifndef SFK_V2_CLAMP
#define SFK_V2_CLAMP 0
#endif

namespace sfk {

constexpr bool CLAMP = SFK_V2_CLAMP;
// SFK_V2_SPLIT=1: the transposed y/x stages accumulate each table's sum in
// its own chain (2-3 independent M-deep DFMA chains per output instead of one
// 2M/3M-deep chain); summation order changes, within the 1e-12 gate.
#ifndef SFK_V2_SPLIT
#define SFK_V2_SPLIT 1
#endif
constexpr bool SPLIT = SFK_V2_SPLIT;

__device__ __forceinline__ int clamp_line(int ln, int L) {
  return CLAMP ? (ln < L ? ln : L - 1) : ln;
}


// ROLL: 0 = everything unrolled; 1 = pointwise loop rolled; 2 = also the
// outer (output-index) loop of every contraction rolled (table entries then
// come from warp-uniform constant loads; code size drops ~M-fold).
// GS = true: global operator y += sum_c P_c^T A_c P_c x (SURVEY.md §8(f)
// item 1), as in hex_action3.cu: `u` is x, `A` is y, cmap[c][i] the global
// dof of local dof i; the map (int32) is double-buffered in the u buffer, x
// is gathered through it in the x stage and y scattered with fp64 atomics
// in the transposed x stage.
template <int N, int M, int CPB, int R, int MINB, int ROLL, bool GS = false>
__global__ void __launch_bounds__(HexAction2Cfg<N, M, CPB, R>::THREADS, MINB)
hex_laplace_action_v2(const __grid_constant__ TabsBD<N, M> T, int64_t ncells,
                      const double* __restrict__ coords, const double* __restrict__ u,
                      double* __restrict__ A, const int* __restrict__ cmap = nullptr) {
  using C = HexAction2Cfg<N, M, CPB, R>;
  // (B, D) pairs spill at n = 6 (96-register cap at CPB 8): separate tables there
  constexpr bool PAIRS = SFK_TAB_PAIRS && N != 6;
  constexpr int NN = C::NN, MN = C::MN, MM = C::MM, N3 = C::N3, PX = C::PX, LZ = C::LZ;
  constexpr int XA = C::XA, YA = C::YA, TH = C::THREADS;
  constexpr int UQ = ROLL >= 2 ? 1 : M, UI = ROLL >= 2 ? 1 : N, UP = ROLL >= 1 ? 1 : M;
  extern __shared__ __align__(16) double smem[];
  double* sX = smem;                        // [CPB][2][M][PX]
  double* sY = sX + CPB * C::XSZ;           // [CPB][3][M*M][LZ]
  double* sU = smem + round_up(CPB * C::XSZ + CPB * C::YSZ, 2);  // [CPB*N3+1]
  double* sCo = sU + C::USZ;                // [2][CPB*24] (double buffer)
  const int tid = threadIdx.x;
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  int* sMap = reinterpret_cast<int*>(sU);   // GS: [2][CPB*N3] int32 in the u buffer
  static_assert(!GS || 2 * CPB * N3 <= 2 * C::USZ, "map double buffer does not fit");

  // u of the next batch streams into the single u buffer as soon as the
  // current x stage has consumed it (overlapping the y, z, y^T, x^T stages);
  // coords are double-buffered because the z stage still needs them.
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

    // ---- x stage: lines (c, iy, iz): X0 = Bx u, X1 = Dx u -------------
    {
      constexpr int L = CPB * NN;
      int ln[R];
      bool on[R];
      double uu[R][N];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        ln[j] = clamp_line(tid + j * TH, L);
        on[j] = CLAMP || tid + j * TH < L;
        const int lc = on[j] ? ln[j] : 0;
        const int c = lc / NN, r = lc - c * NN;
        const bool live = on[j] && c < ncb;
#pragma unroll
        for (int i = 0; i < N; ++i)
          uu[j][i] = GS ? (live ? __ldg(u + smap[c * N3 + i * NN + r]) : 0.0)
                        : su[c * N3 + i * NN + r];
        if (!live) {
#pragma unroll
          for (int i = 0; i < N; ++i) uu[j][i] = 0.0;
        }
      }
#pragma unroll (UQ)
      for (int q = 0; q < M; ++q) {
        double bq[R], dq[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          bq[j] = TBP(q) * uu[j][0];
          dq[j] = TDP(q) * uu[j][0];
        }
#pragma unroll
        for (int i = 1; i < N; ++i)
#pragma unroll
          for (int j = 0; j < R; ++j) {
            bq[j] = fma(TBP(i * M + q), uu[j][i], bq[j]);
            dq[j] = fma(TDP(i * M + q), uu[j][i], dq[j]);
          }
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (CLAMP || on[j]) {
            const int c = ln[j] / NN, r = ln[j] - c * NN;
            double* xo = sX + c * C::XSZ + r;
            xo[q * PX] = bq[j];
            xo[XA + q * PX] = dq[j];
          }
      }
    }
    __syncthreads();
    if (b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- y stage: lines (c, qx, iz): BB = By X0, BD = Dy X0, DB = By X1 --
    {
      constexpr int L = CPB * MN;
      double a0[R][N], a1[R][N];
      int ln[R];
      bool on[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        ln[j] = clamp_line(tid + j * TH, L);
        on[j] = CLAMP || tid + j * TH < L;
        const int lc = on[j] ? ln[j] : 0;
        const int c = lc / MN, r = lc - c * MN;
        const int qx = r / N, iz = r - qx * N;
        const double* xi = sX + c * C::XSZ + qx * PX + iz;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          a0[j][i] = xi[i * N];
          a1[j][i] = xi[XA + i * N];
        }
      }
#pragma unroll (UQ)
      for (int q = 0; q < M; ++q) {
        double bb[R], bd[R], db[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          bb[j] = TBP(q) * a0[j][0];
          bd[j] = TDP(q) * a0[j][0];
          db[j] = TBP(q) * a1[j][0];
        }
#pragma unroll
        for (int i = 1; i < N; ++i)
#pragma unroll
          for (int j = 0; j < R; ++j) {
            bb[j] = fma(TBP(i * M + q), a0[j][i], bb[j]);
            bd[j] = fma(TDP(i * M + q), a0[j][i], bd[j]);
            db[j] = fma(TBP(i * M + q), a1[j][i], db[j]);
          }
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (CLAMP || on[j]) {
            const int c = ln[j] / MN, r = ln[j] - c * MN;
            const int qx = r / N, iz = r - qx * N;
            double* yo = sY + c * C::YSZ + (qx * M + q) * LZ + iz;
            yo[0] = bb[j];
            yo[YA] = bd[j];
            yo[2 * YA] = db[j];
          }
      }
    }
    __syncthreads();

    // ---- z stage: lines (c, qx, qy), three in-place passes ---------------
    {
      constexpr int L = CPB * MM;
      int ln[R];
      bool on[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        ln[j] = clamp_line(tid + j * TH, L);
        on[j] = CLAMP || tid + j * TH < L;
      }
      // (1) reference gradient lines: slot 0 <- Dz BB (d_z), 1 <- Bz BD (d_y),
      //     2 <- Bz DB (d_x)
      {
        double bb[R][N], bd[R][N], db[R][N];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int c = on[j] ? ln[j] / MM : 0, r = on[j] ? ln[j] - c * MM : 0;
          const double* yi = sY + c * C::YSZ + r * LZ;
#pragma unroll (UQ)
          for (int i = 0; i < N; ++i) {
            bb[j][i] = yi[i];
            bd[j][i] = yi[YA + i];
            db[j][i] = yi[2 * YA + i];
          }
        }
#pragma unroll
        for (int q = 0; q < M; ++q) {
          double gz[R], gy[R], gx[R];
#pragma unroll
          for (int j = 0; j < R; ++j) {
            gz[j] = TDP(q) * bb[j][0];
            gy[j] = TBP(q) * bd[j][0];
            gx[j] = TBP(q) * db[j][0];
          }
#pragma unroll
          for (int i = 1; i < N; ++i)
#pragma unroll
            for (int j = 0; j < R; ++j) {
              gz[j] = fma(TDP(i * M + q), bb[j][i], gz[j]);
              gy[j] = fma(TBP(i * M + q), bd[j][i], gy[j]);
              gx[j] = fma(TBP(i * M + q), db[j][i], gx[j]);
            }
          if (M > N) {
            // in place is only safe once every input entry was read: for
            // M > N the outputs q >= N go beyond the inputs, q < N overwrite
            // inputs already consumed (all inputs are in registers)
          }
#pragma unroll
          for (int j = 0; j < R; ++j)
            if (CLAMP || on[j]) {
              const int c = ln[j] / MM, r = ln[j] - c * MM;
              double* yo = sY + c * C::YSZ + r * LZ + q;
              yo[0] = gz[j];
              yo[YA] = gy[j];
              yo[2 * YA] = gx[j];
            }
        }
      }
      // (2) pointwise: geometry per point + Laplace flux, in place
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int lc = on[j] ? ln[j] : 0;
        const int c = lc / MM, r = lc - c * MM;
        const int qx = r / M, qy = r - qx * M;
        double* yl = sY + c * C::YSZ + r * LZ;
        HexLineAdj geo;
        geo.setup(sC + c * 24, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
        const double wxy = T.W[qx] * T.W[qy];
#pragma unroll (UP)
        for (int q = 0; q < M; ++q) {
          double gz = yl[q], gy = yl[YA + q], gx = yl[2 * YA + q];
          double r0[3], r1[3], r2[3];
          const double det = geo.adj(T.Bc[M + q], r0, r1, r2);
          const double s = (wxy * T.W[q]) * rcp64(fabs(det));
          laplace_flux(r0, r1, r2, s, gx, gy, gz);
          if (CLAMP || on[j]) {
            yl[q] = gz;
            yl[YA + q] = gy;
            yl[2 * YA + q] = gx;
          }
        }
      }
      // (3) transposed z, in place: slot 0 <- Dz^T f_z, 1 <- Bz^T f_y,
      //     2 <- Bz^T f_x
      {
        double fz[R][M], fy[R][M], fx[R][M];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int c = on[j] ? ln[j] / MM : 0, r = on[j] ? ln[j] - c * MM : 0;
          const double* yi = sY + c * C::YSZ + r * LZ;
#pragma unroll
          for (int q = 0; q < M; ++q) {
            fz[j][q] = yi[q];
            fy[j][q] = yi[YA + q];
            fx[j][q] = yi[2 * YA + q];
          }
        }
#pragma unroll (UI)
        for (int i = 0; i < N; ++i) {
          double sz[R], sy[R], sx[R];
#pragma unroll
          for (int j = 0; j < R; ++j) {
            sz[j] = TDP(i * M) * fz[j][0];
            sy[j] = TBP(i * M) * fy[j][0];
            sx[j] = TBP(i * M) * fx[j][0];
          }
#pragma unroll
          for (int q = 1; q < M; ++q)
#pragma unroll
            for (int j = 0; j < R; ++j) {
              sz[j] = fma(TDP(i * M + q), fz[j][q], sz[j]);
              sy[j] = fma(TBP(i * M + q), fy[j][q], sy[j]);
              sx[j] = fma(TBP(i * M + q), fx[j][q], sx[j]);
            }
#pragma unroll
          for (int j = 0; j < R; ++j)
            if (CLAMP || on[j]) {
              const int c = ln[j] / MM, r = ln[j] - c * MM;
              double* yo = sY + c * C::YSZ + r * LZ + i;
              yo[0] = sz[j];
              yo[YA] = sy[j];
              yo[2 * YA] = sx[j];
            }
        }
      }
    }
    __syncthreads();

    // ---- transposed y stage: lines (c, qx, iz) ----------------------------
    {
      constexpr int L = CPB * MN;
      double pz[R][M], py[R][M], px[R][M];
      int ln[R];
      bool on[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        ln[j] = clamp_line(tid + j * TH, L);
        on[j] = CLAMP || tid + j * TH < L;
        const int lc = on[j] ? ln[j] : 0;
        const int c = lc / MN, r = lc - c * MN;
        const int qx = r / N, iz = r - qx * N;
        const double* yi = sY + c * C::YSZ + qx * M * LZ + iz;
#pragma unroll
        for (int q = 0; q < M; ++q) {
          pz[j][q] = yi[q * LZ];
          py[j][q] = yi[YA + q * LZ];
          px[j][q] = yi[2 * YA + q * LZ];
        }
      }
#pragma unroll (UI)
      for (int i = 0; i < N; ++i) {
        double r1[R], r2[R];
        if (SPLIT) {
          // three independent M-deep chains (Dy^T Sy and By^T Sz summed last)
          double r3[R];
#pragma unroll
          for (int j = 0; j < R; ++j) {
            r1[j] = TBP(i * M) * px[j][0];
            r2[j] = TDP(i * M) * py[j][0];
            r3[j] = TBP(i * M) * pz[j][0];
          }
#pragma unroll
          for (int q = 1; q < M; ++q)
#pragma unroll
            for (int j = 0; j < R; ++j) {
              r1[j] = fma(TBP(i * M + q), px[j][q], r1[j]);
              r2[j] = fma(TDP(i * M + q), py[j][q], r2[j]);
              r3[j] = fma(TBP(i * M + q), pz[j][q], r3[j]);
            }
#pragma unroll
          for (int j = 0; j < R; ++j) r2[j] += r3[j];
        } else {
#pragma unroll
          for (int j = 0; j < R; ++j) {
            r1[j] = TBP(i * M) * px[j][0];
            r2[j] = fma(TDP(i * M), py[j][0], TBP(i * M) * pz[j][0]);
          }
#pragma unroll
          for (int q = 1; q < M; ++q)
#pragma unroll
            for (int j = 0; j < R; ++j) {
              r1[j] = fma(TBP(i * M + q), px[j][q], r1[j]);
              r2[j] = fma(TDP(i * M + q), py[j][q], r2[j]);
              r2[j] = fma(TBP(i * M + q), pz[j][q], r2[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (CLAMP || on[j]) {
            const int c = ln[j] / MN, r = ln[j] - c * MN;
            const int qx = r / N, iz = r - qx * N;
            double* xo = sX + c * C::XSZ + qx * PX + iz;
            xo[i * N] = r1[j];
            xo[XA + i * N] = r2[j];
          }
      }
    }
    __syncthreads();

    // ---- transposed x stage: lines (c, iy, iz) -> A ------------------------
    {
      constexpr int L = CPB * NN;
      double p1[R][M], p2[R][M];
      int ln[R];
      bool on[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        // CLAMP: lines past the live cells redo the last live line (same
        // inputs, same instructions: bit-identical duplicate stores)
        ln[j] = CLAMP ? clamp_line(tid + j * TH, ncb * NN) : tid + j * TH;
        on[j] = tid + j * TH < L && ((tid + j * TH) / NN) < ncb;
        const int c = (CLAMP || on[j]) ? ln[j] / NN : 0, r = (CLAMP || on[j]) ? ln[j] - c * NN : 0;
        const double* xi = sX + c * C::XSZ + r;
#pragma unroll
        for (int q = 0; q < M; ++q) {
          p1[j][q] = xi[q * PX];
          p2[j][q] = xi[XA + q * PX];
        }
      }
#pragma unroll (UI)
      for (int i = 0; i < N; ++i) {
        double a[R];
        if (SPLIT) {
          // two independent M-deep chains (Dx^T R1 and Bx^T R2 summed last)
          double a2[R];
#pragma unroll
          for (int j = 0; j < R; ++j) {
            a[j] = TDP(i * M) * p1[j][0];
            a2[j] = TBP(i * M) * p2[j][0];
          }
#pragma unroll
          for (int q = 1; q < M; ++q)
#pragma unroll
            for (int j = 0; j < R; ++j) {
              a[j] = fma(TDP(i * M + q), p1[j][q], a[j]);
              a2[j] = fma(TBP(i * M + q), p2[j][q], a2[j]);
            }
#pragma unroll
          for (int j = 0; j < R; ++j) a[j] += a2[j];
        } else {
#pragma unroll
          for (int j = 0; j < R; ++j) a[j] = fma(TDP(i * M), p1[j][0], TBP(i * M) * p2[j][0]);
#pragma unroll
          for (int q = 1; q < M; ++q)
#pragma unroll
            for (int j = 0; j < R; ++j) {
              a[j] = fma(TDP(i * M + q), p1[j][q], a[j]);
              a[j] = fma(TBP(i * M + q), p2[j][q], a[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (CLAMP || on[j]) {
            const int c = ln[j] / NN, r = ln[j] - c * NN;
            if (GS) atomicAdd(A + smap[c * N3 + i * NN + r], on[j] ? a[j] : 0.0);
            else A[(cell0 + c) * N3 + i * NN + r] = a[j];
          }
      }
    }
    __syncthreads();   // X/R region is rewritten by the next batch's x stage
  }
}

template <int N, int M, int CPB, int R, int MINB, int ROLL = 1, bool GS = false>
static int launch_v2(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* u, cudaStream_t s, const int* cmap = nullptr) {
  using C = HexAction2Cfg<N, M, CPB, R>;
  auto kern = hex_laplace_action_v2<N, M, CPB, R, MINB, ROLL, GS>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_action_v2", &sh, true))
    return rc_;
  const TabsBD<N, M> T = make_tabs_bd<N, M>(p);
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, u, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_v2 launch");
}

// Per-degree configuration (cells per CTA, lines per thread, min CTAs/SM,
// loop rolling).  options c2_r = 1|2 and c2_roll = 1|2 override the defaults
// (tuning runs only).

template <int N, int CPB, int MINB1, int MINB2>
static int pick(int r, int roll, const sfk_plan* p, int64_t ncells, double* A,
                const double* coords, const double* w0, cudaStream_t s) {
  if (r == 2) return launch_v2<N, N, CPB, 2, MINB2, 1>(p, ncells, A, coords, w0, s);
  if (roll == 2) return launch_v2<N, N, CPB, 1, MINB1, 2>(p, ncells, A, coords, w0, s);
  return launch_v2<N, N, CPB, 1, MINB1, 1>(p, ncells, A, coords, w0, s);
}

int launch_hex_action_v2(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s) {
  if (p->n != p->m) return SFK_EUNSUPPORTED;   // caller falls back to v1
  const int r_env = (int)option(OPT_C2_R), roll_env = (int)option(OPT_C2_ROLL);
  const int r = r_env ? r_env : 1, roll = roll_env ? roll_env : 1;
  switch (p->n) {
    case 2: return pick<2, 64, 2, 2>(r, roll, p, ncells, A, coords, w0, s);
    case 3: return pick<3, 32, 2, 2>(r, roll, p, ncells, A, coords, w0, s);
    case 4: return pick<4, 16, 2, 2>(r, roll, p, ncells, A, coords, w0, s);
    case 5: return pick<5, 10, 2, 2>(r, roll, p, ncells, A, coords, w0, s);
    case 6: return pick<6, 8, 2, 2>(r, roll, p, ncells, A, coords, w0, s);
    case 7: return pick<7, 5, 2, 2>(r, roll, p, ncells, A, coords, w0, s);
    case 8: return pick<8, 4, 2, 2>(r, roll, p, ncells, A, coords, w0, s);
    case 9: return pick<9, 3, 2, 2>(r, roll, p, ncells, A, coords, w0, s);
    default: return SFK_EUNSUPPORTED;
  }
}

int launch_hex_action_v2_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s) {
  if (p->n != p->m) return SFK_EUNSUPPORTED;
  switch (p->n) {
    case 4: return launch_v2<4, 4, 16, 1, 2, 1, true>(p, ncells, y, coords, x, s, cmap);
    case 6: return launch_v2<6, 6, 8, 1, 2, 1, true>(p, ncells, y, coords, x, s, cmap);
    case 7: return launch_v2<7, 7, 5, 1, 2, 1, true>(p, ncells, y, coords, x, s, cmap);
    case 9: return launch_v2<9, 9, 3, 1, 2, 1, true>(p, ncells, y, coords, x, s, cmap);
    default: return SFK_EUNSUPPORTED;
  }
}

}  // namespace sfk
