// Hex Q_p Laplace action, one thread per cell at small n — BASELINE C2 at
// p = 2 (n = m = 3); also the p = 2 global operator (GS).
//
// Same math and reference mapping as the other C2 kernels (forms.py:186-189,
// 235-243; passes.py:672-743 schedule; scheduling.py:617-738 emitted
// kernel).  The line kernels (v4 at p = 2) give each lane one 1D line per
// stage: 3 cells x 9 lines = 27 of 32 lanes busy, lines re-dealt through
// shared memory between stages.  Here a thread owns a whole cell and runs the
// pipeline in slices, so nothing is exchanged between threads (no barrier in
// the pipeline, every lane busy):
//   (A) per iz-slice: the x contraction of the n x n (ix, iy) dofs (in
//       registers) feeds the y contraction at once; the 3 y-outputs
//       (BB, BD, DB) of the slice go to this thread's private shared-memory
//       block Y[3][qx][qy][iz] (3 n^3 doubles, odd stride: the per-thread
//       64-bit accesses of a warp are conflict-free);
//   (B) per z-line (qx, qy): z contraction, per-point geometry + Laplace
//       flux (HexLineAdj), transposed z — written back in place;
//   (C) per iz-slice: transposed y (registers) feeding transposed x.
// The CTA's u block (contiguous in HBM) arrives through shared memory with
// coalesced 16-byte cp.async and A leaves the same way (per-thread scattered
// 8-byte loads / stores were 0.101 vs 0.081 ms, profiles/r01cu_*.jsonl);
// coords are read as 16-byte vectors straight into registers.  Occupancy is
// bounded by the per-thread shared block (4 CTAs of 64 threads per SM).
#include <cstdint>
#include <cstdlib>

#include "async_copy.cuh"
#include "hex_geometry.cuh"

#ifndef SFK_CELL_STAGE
#define SFK_CELL_STAGE 1
#endif

namespace sfk {

// TabsBD plus the collocation derivative C = B^-1 D (CD variant)
template <int N>
struct TabsCell : TabsBD<N, N> {
  double C[N * N];   // C[q'*N + q]
};

template <int N>
struct CellCfg {
  static constexpr int N3 = N * N * N;
  static constexpr int YS = (3 * N3) | 1;        // per-thread Y block (odd stride)
};

// GS = true: global operator y += sum_c P_c^T A_c P_c x (SURVEY.md §8(f)
// item 1): `u` is x, `A` is y; the CTA's block of the cell -> dof map
// (int32, contiguous) is staged in the u area, each thread gathers its
// cell's x values through it and scatter-adds its results with fp64 atomics.
// CD: the collocation-derivative form of phases (A) and (C) (v6's schedule
// inside the slice loops): per slice Bx, By, then C_x, C_y on the interpolated
// slice (108 instead of 135 FMA per slice and direction); phase (B) is
// unchanged (gz = D_z BB etc., since C_y B_y = D_y).
// LG: phase (B) runs qy-outer and forms the line-geometry parts that depend
// on one of qx, qy only once per cell instead of once per line (STAGE only:
// the qx parts live in the thread's sU row, free between (A) and (C)).
template <int N, int TH, int MINB, bool GS = false, bool CD = false, bool LG = false>
__global__ void __launch_bounds__(TH, MINB)
hex_laplace_action_cell(const __grid_constant__ TabsCell<N> T, int64_t ncells,
                        const double* __restrict__ coords, const double* __restrict__ u,
                        double* __restrict__ A, const int* __restrict__ cmap = nullptr) {
  constexpr bool PAIRS = true;
  constexpr bool STAGE = SFK_CELL_STAGE || GS;
  constexpr bool LGS = LG && STAGE && !GS;
  constexpr int M = N, N3 = CellCfg<N>::N3, YS = CellCfg<N>::YS;
  constexpr int S1 = N3;                           // slot stride in Y
  extern __shared__ double smem[];
  double* Y = smem + threadIdx.x * YS;             // [3][qx][qy][iz] at ((qx*M+qy)*N+iz)
  // STAGE: the CTA's u block (TH cells x N^3, contiguous in HBM) is copied
  // to shared memory with coalesced 16-byte cp.async, and A leaves the same
  // way; per-thread rows of N^3 doubles (odd for n = 3: conflict-free reads)
  double* sU = smem + TH * YS;
  const int64_t cell0 = (int64_t)blockIdx.x * TH;
  const int64_t cell = cell0 + threadIdx.x;
  const int ncb = (int)((ncells - cell0) < TH ? (ncells - cell0) : TH);
  int* sMap = reinterpret_cast<int*>(sU);          // GS: [thread][N3] int32
  if (GS) {
    for (int i = threadIdx.x; i < ncb * N3; i += TH) cp_async4(sMap + i, cmap + cell0 * N3 + i);
    cp_async_commit();
  } else if (STAGE) {
    async_copy<TH>(sU, u + cell0 * N3, ncb * N3, threadIdx.x);
    cp_async_commit();
  }
  double X[24];   // this cell's coords, in registers (the geometry setup runs per z-line)
  auto cell_pipeline = [&]() {
    const double* uc = u + cell * N3;
    // the whole cell's dofs in flight at once (the slice order would touch
    // every sector of the cell's 8 N^3 bytes N times)
    double ua[N3];
    if (GS) {
#pragma unroll
      for (int k = 0; k < N3; ++k) ua[k] = __ldg(u + sMap[threadIdx.x * N3 + k]);
    } else if (STAGE) {
#pragma unroll
      for (int k = 0; k < N3; ++k) ua[k] = sU[threadIdx.x * N3 + k];
    } else {
#pragma unroll
      for (int k = 0; k < N3; ++k) ua[k] = __ldg(uc + k);
    }

    // (A) forward x + y, one iz-slice at a time
#pragma unroll
    for (int iz = 0; CD && iz < N; ++iz) {
      double x0[M][N], q[M][M];   // Bx u [qx][iy];  By Bx u [qx][qy]
#pragma unroll
      for (int qx = 0; qx < M; ++qx)
#pragma unroll
        for (int iy = 0; iy < N; ++iy) {
          double b = TBP(qx) * ua[iy * N + iz];
#pragma unroll
          for (int ix = 1; ix < N; ++ix) b = fma(TBP(ix * M + qx), ua[(ix * N + iy) * N + iz], b);
          x0[qx][iy] = b;
        }
#pragma unroll
      for (int qx = 0; qx < M; ++qx)
#pragma unroll
        for (int qy = 0; qy < M; ++qy) {
          double b = TBP(qy) * x0[qx][0];
#pragma unroll
          for (int iy = 1; iy < N; ++iy) b = fma(TBP(iy * M + qy), x0[qx][iy], b);
          q[qx][qy] = b;
        }
#pragma unroll
      for (int qx = 0; qx < M; ++qx)
#pragma unroll
        for (int qy = 0; qy < M; ++qy) {
          double gy = T.C[qy] * q[qx][0], gx = T.C[qx] * q[0][qy];
#pragma unroll
          for (int k = 1; k < M; ++k) {
            gy = fma(T.C[k * M + qy], q[qx][k], gy);
            gx = fma(T.C[k * M + qx], q[k][qy], gx);
          }
          const int o = (qx * M + qy) * N + iz;
          Y[o] = q[qx][qy];      // BB
          Y[S1 + o] = gy;        // BD = D_y B_x u
          Y[2 * S1 + o] = gx;    // DB = B_y D_x u
        }
    }
#pragma unroll
    for (int iz = 0; !CD && iz < N; ++iz) {
      double ux[N][N];   // [ix][iy]
#pragma unroll
      for (int ix = 0; ix < N; ++ix)
#pragma unroll
        for (int iy = 0; iy < N; ++iy) ux[ix][iy] = ua[(ix * N + iy) * N + iz];
      double x0[M][N], x1[M][N];   // [qx][iy]: Bx u, Dx u
#pragma unroll
      for (int qx = 0; qx < M; ++qx)
#pragma unroll
        for (int iy = 0; iy < N; ++iy) {
          double b = TBP(qx) * ux[0][iy], d = TDP(qx) * ux[0][iy];
#pragma unroll
          for (int ix = 1; ix < N; ++ix) {
            b = fma(TBP(ix * M + qx), ux[ix][iy], b);
            d = fma(TDP(ix * M + qx), ux[ix][iy], d);
          }
          x0[qx][iy] = b;
          x1[qx][iy] = d;
        }
#pragma unroll
      for (int qx = 0; qx < M; ++qx)
#pragma unroll
        for (int qy = 0; qy < M; ++qy) {
          double bb = TBP(qy) * x0[qx][0], bd = TDP(qy) * x0[qx][0], db = TBP(qy) * x1[qx][0];
#pragma unroll
          for (int iy = 1; iy < N; ++iy) {
            bb = fma(TBP(iy * M + qy), x0[qx][iy], bb);
            bd = fma(TDP(iy * M + qy), x0[qx][iy], bd);
            db = fma(TBP(iy * M + qy), x1[qx][iy], db);
          }
          const int o = (qx * M + qy) * N + iz;
          Y[o] = bb;
          Y[S1 + o] = bd;
          Y[2 * S1 + o] = db;
        }
    }

    // (B) z-lines: gradients, pointwise flux, transposed z, in place
    auto z_line = [&](int qx, int qy, const HexLineAdj& geo) {
      double* yl = Y + (qx * M + qy) * N;
      double bb[N], bd[N], db[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        bb[i] = yl[i];
        bd[i] = yl[S1 + i];
        db[i] = yl[2 * S1 + i];
      }
      double gz[M], gy[M], gx[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        gz[q] = TDP(q) * bb[0];
        gy[q] = TBP(q) * bd[0];
        gx[q] = TBP(q) * db[0];
#pragma unroll
        for (int i = 1; i < N; ++i) {
          gz[q] = fma(TDP(i * M + q), bb[i], gz[q]);
          gy[q] = fma(TBP(i * M + q), bd[i], gy[q]);
          gx[q] = fma(TBP(i * M + q), db[i], gx[q]);
        }
      }
      const double wxy = T.W[qx] * T.W[qy];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        double r0[3], r1[3], r2[3];
        const double det = geo.adj(T.Bc[M + q], r0, r1, r2);
        const double s = (wxy * T.W[q]) * rcp64(fabs(det));
        laplace_flux(r0, r1, r2, s, gx[q], gy[q], gz[q]);
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double sz = TDP(i * M) * gz[0], sy = TBP(i * M) * gy[0], sx = TBP(i * M) * gx[0];
#pragma unroll
        for (int q = 1; q < M; ++q) {
          sz = fma(TDP(i * M + q), gz[q], sz);
          sy = fma(TBP(i * M + q), gy[q], sy);
          sx = fma(TBP(i * M + q), gx[q], sx);
        }
        yl[i] = sz;
        yl[S1 + i] = sy;
        yl[2 * S1 + i] = sx;
      }
    };
    if (LGS) {
      // line geometry shared between lines: col1's polynomial (B, dB) per qx
      // in this thread's free sU row, col0's (A, dA) and col2's partial sums
      // per qy in registers — the operations of HexLineAdj::setup, formed 3
      // instead of 9 times (bit-identical)
      double* lgx = sU + threadIdx.x * N3;
#pragma unroll
      for (int qx = 0; qx < M; ++qx) {
        const double bx0 = T.Bc[qx], bx1 = T.Bc[M + qx];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double a0 = fma(X[3 * 6 + k] - X[3 * 4 + k], bx1, (X[3 * 2 + k] - X[k]) * bx0);
          const double a1 = fma(X[3 * 7 + k] - X[3 * 5 + k], bx1, (X[3 * 3 + k] - X[3 + k]) * bx0);
          lgx[6 * qx + k] = a0;
          lgx[6 * qx + 3 + k] = a1 - a0;
        }
      }
#pragma unroll 1
      for (int qy = 0; qy < M; ++qy) {
        const double by0 = T.Bc[qy], by1 = T.Bc[M + qy];
        double Ay[3], dAy[3], g0[3], g1[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double a0 = fma(X[3 * 6 + k] - X[3 * 2 + k], by1, (X[3 * 4 + k] - X[k]) * by0);
          const double a1 = fma(X[3 * 7 + k] - X[3 * 3 + k], by1, (X[3 * 5 + k] - X[3 + k]) * by0);
          Ay[k] = a0;
          dAy[k] = a1 - a0;
          g0[k] = fma(X[3 * 3 + k] - X[3 * 2 + k], by1, (X[3 * 1 + k] - X[k]) * by0);
          g1[k] = fma(X[3 * 7 + k] - X[3 * 6 + k], by1, (X[3 * 5 + k] - X[3 * 4 + k]) * by0);
        }
#pragma unroll 1
        for (int qx = 0; qx < M; ++qx) {
          const double bx0 = T.Bc[qx], bx1 = T.Bc[M + qx];
          double Bx[3], dBx[3], cc[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            Bx[k] = lgx[6 * qx + k];
            dBx[k] = lgx[6 * qx + 3 + k];
            cc[k] = fma(g1[k], bx1, g0[k] * bx0);
          }
          HexLineAdj geo;
          geo.from_parts(Ay, dAy, Bx, dBx, cc);
          z_line(qx, qy, geo);
        }
      }
    } else {
#pragma unroll 1
      for (int l = 0; l < M * M; ++l) {
        const int qx = l / M, qy = l - qx * M;
        HexLineAdj geo;
        geo.setup(X, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
        z_line(qx, qy, geo);
      }
    }

    // (C) transposed y + x, one iz-slice at a time
    double* ac = A + cell * N3;
#pragma unroll 1
    for (int iz = 0; CD && iz < N; ++iz) {
      // t = C_x^T Sx + C_y^T Sy + Sz on the slice, then B_y^T, B_x^T
      double sx[M][M], sy[M][M], t[M][M], r[M][N];
#pragma unroll
      for (int qx = 0; qx < M; ++qx)
#pragma unroll
        for (int qy = 0; qy < M; ++qy) {
          const int o = (qx * M + qy) * N + iz;
          t[qx][qy] = Y[o];
          sy[qx][qy] = Y[S1 + o];
          sx[qx][qy] = Y[2 * S1 + o];
        }
#pragma unroll
      for (int qx = 0; qx < M; ++qx)
#pragma unroll
        for (int qy = 0; qy < M; ++qy) {
          double v = t[qx][qy];
#pragma unroll
          for (int k = 0; k < M; ++k) {
            v = fma(T.C[qx * M + k], sx[k][qy], v);
            v = fma(T.C[qy * M + k], sy[qx][k], v);
          }
          t[qx][qy] = v;
        }
#pragma unroll
      for (int qx = 0; qx < M; ++qx)
#pragma unroll
        for (int iy = 0; iy < N; ++iy) {
          double a = TBP(iy * M) * t[qx][0];
#pragma unroll
          for (int qy = 1; qy < M; ++qy) a = fma(TBP(iy * M + qy), t[qx][qy], a);
          r[qx][iy] = a;
        }
#pragma unroll
      for (int ix = 0; ix < N; ++ix)
#pragma unroll
        for (int iy = 0; iy < N; ++iy) {
          double a = TBP(ix * M) * r[0][iy];
#pragma unroll
          for (int qx = 1; qx < M; ++qx) a = fma(TBP(ix * M + qx), r[qx][iy], a);
          if (GS) atomicAdd(A + sMap[threadIdx.x * N3 + (ix * N + iy) * N + iz], a);
          else if (STAGE) sU[threadIdx.x * N3 + (ix * N + iy) * N + iz] = a;
          else ac[(ix * N + iy) * N + iz] = a;
        }
    }
#pragma unroll 1
    for (int iz = 0; !CD && iz < N; ++iz) {
      double r1[M][N], r2[M][N];   // [qx][iy]: By^T Sx, Dy^T Sy + By^T Sz
#pragma unroll
      for (int qx = 0; qx < M; ++qx) {
        double pz[M], py[M], px[M];
#pragma unroll
        for (int qy = 0; qy < M; ++qy) {
          const int o = (qx * M + qy) * N + iz;
          pz[qy] = Y[o];
          py[qy] = Y[S1 + o];
          px[qy] = Y[2 * S1 + o];
        }
#pragma unroll
        for (int iy = 0; iy < N; ++iy) {
          double a = TBP(iy * M) * px[0], b = TDP(iy * M) * py[0], c = TBP(iy * M) * pz[0];
#pragma unroll
          for (int qy = 1; qy < M; ++qy) {
            a = fma(TBP(iy * M + qy), px[qy], a);
            b = fma(TDP(iy * M + qy), py[qy], b);
            c = fma(TBP(iy * M + qy), pz[qy], c);
          }
          r1[qx][iy] = a;
          r2[qx][iy] = b + c;
        }
      }
#pragma unroll
      for (int ix = 0; ix < N; ++ix)
#pragma unroll
        for (int iy = 0; iy < N; ++iy) {
          double a = TDP(ix * M) * r1[0][iy], b = TBP(ix * M) * r2[0][iy];
#pragma unroll
          for (int qx = 1; qx < M; ++qx) {
            a = fma(TDP(ix * M + qx), r1[qx][iy], a);
            b = fma(TBP(ix * M + qx), r2[qx][iy], b);
          }
          if (GS) atomicAdd(A + sMap[threadIdx.x * N3 + (ix * N + iy) * N + iz], a + b);
          else if (STAGE) sU[threadIdx.x * N3 + (ix * N + iy) * N + iz] = a + b;
          else ac[(ix * N + iy) * N + iz] = a + b;
        }
    }
  };
  // (coords staged like u through the Y region measured slower: 0.081 ->
  // 0.090 ms, profiles/r01cv_*.jsonl — they are read as 16-byte vectors)
  if (STAGE) {
    cp_async_wait<0>();
    __syncthreads();
  }
  if (cell < ncells) {
    const double* cg = coords + cell * 24;
    if ((reinterpret_cast<uintptr_t>(cg) & 15) == 0) {
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(cg) + k);
        X[2 * k] = v.x;
        X[2 * k + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 24; ++k) X[k] = __ldg(cg + k);
    }
  }
  if (cell < ncells) cell_pipeline();
  if (STAGE && !GS) {
    __syncthreads();   // every live thread's row is in sU
    double* ag = A + cell0 * N3;
    const bool al = ((reinterpret_cast<uintptr_t>(ag)) & 15) == 0;
    const int n = ncb * N3;
    if (al) {
      for (int i = threadIdx.x; i < n / 2; i += TH)
        reinterpret_cast<double2*>(ag)[i] = reinterpret_cast<const double2*>(sU)[i];
      if ((n & 1) && threadIdx.x == 0) ag[n - 1] = sU[n - 1];
    } else {
      for (int i = threadIdx.x; i < n; i += TH) ag[i] = sU[i];
    }
  }
}

template <int N, int TH, int MINB, bool GS = false, bool CD = false, bool LG = false>
static int launch_cell(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                       const double* u, cudaStream_t s, const int* cmap = nullptr) {
  constexpr size_t SMEM =
      (size_t)TH * (CellCfg<N>::YS + (SFK_CELL_STAGE || GS ? CellCfg<N>::N3 : 0)) * sizeof(double);
  if (CD && !p->has_ct) return SFK_EUNSUPPORTED;
  auto kern = hex_laplace_action_cell<N, TH, MINB, GS, CD, LG>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, TH, SMEM, "hex_action_cell", &sh, true))
    return rc_;
  TabsCell<N> T;
  static_cast<TabsBD<N, N>&>(T) = make_tabs_bd<N, N>(p);
  for (int k = 0; k < N * N; ++k) T.C[k] = p->has_ct ? p->Ct[k] : 0.0;
  const int64_t grid = (ncells + TH - 1) / TH;
  if (grid > 0) kern<<<(unsigned)grid, TH, SMEM, s>>>(T, ncells, coords, u, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_cell launch");
}

#ifdef SFK_CELL_ONLY_N
// probe builds (tools/kernel_sweep.py): one instantiation instead of the dispatch
}  // namespace sfk
extern "C" int SFK_CELL_PROBE_ENTRY(const sfk_plan* p, int64_t ncells, double* A,
                                    const double* coords, const double* w0, void* stream) {
  if (p->n != SFK_CELL_ONLY_N || p->n != p->m)
    return sfk::fail(SFK_EUNSUPPORTED, "probe build: n = m = %d only", SFK_CELL_ONLY_N);
  return sfk::launch_cell<SFK_CELL_ONLY_N, SFK_CELLP_TH, SFK_CELLP_MINB, false, SFK_CELLP_CD != 0,
                          SFK_CELLP_LG != 0>(p, ncells, A, coords, w0, (cudaStream_t)stream);
}
namespace sfk {
#else
// Threads per CTA: option cell_th overrides (tuning runs only).
int launch_hex_action_cell(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, cudaStream_t s) {
  if (p->n != p->m) return SFK_EUNSUPPORTED;
  const int th = (int)option(OPT_CELL_TH);
  const int minb = (int)option(OPT_CELL_MINB);
  switch (p->n) {
    case 3:
      // 64 threads per CTA (profiles/r01cs_*.jsonl: 0.1008 ms vs 0.1071 / 0.1032
      // at 96 / 128); option cell_minb = 5 caps registers for a 5th CTA per SM
      if (th == 128) return launch_cell<3, 128, 1>(p, ncells, A, coords, w0, s);
      if (th == 96) return launch_cell<3, 96, 1>(p, ncells, A, coords, w0, s);
      if (minb == 5) return launch_cell<3, 64, 5>(p, ncells, A, coords, w0, s);
      // collocation-derivative slices (CD): 0.0760 -> 0.0740 ms
      // (profiles/r02ae_cfg*.json); option v6_cfg = 6 selects the round-1 form
      if (option(OPT_V6_CFG) == 6) return launch_cell<3, 64, 1>(p, ncells, A, coords, w0, s);
      // line geometry shared between the cell's z-lines (LG): 0.0740 -> 0.0723 ms,
      // bit-identical (profiles/r02am_p2_lgs*.json*); option v6_cfg = 7 drops it
      if (option(OPT_V6_CFG) == 7) return launch_cell<3, 64, 1, false, true>(p, ncells, A, coords, w0, s);
      if (th == 64) return launch_cell<3, 64, 1, false, true, true>(p, ncells, A, coords, w0, s);
      // one warp per CTA (tools/kernel_sweep.py cell, profiles/r02cn_cell_sweep.jsonl):
      // 0.0778 -> 0.0758 ms
      return launch_cell<3, 32, 1, false, true, true>(p, ncells, A, coords, w0, s);
    case 4:
      if (th == 64) return launch_cell<4, 64, 1>(p, ncells, A, coords, w0, s);
      return launch_cell<4, 32, 1>(p, ncells, A, coords, w0, s);
    default: return SFK_EUNSUPPORTED;
  }
}

// Global operator through the thread-per-cell kernel at n = 3.
int launch_hex_action_cell_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                              double* y, const double* coords, cudaStream_t s) {
  if (p->n != 3 || p->m != 3) return SFK_EUNSUPPORTED;
  return launch_cell<3, 64, 1, true>(p, ncells, y, coords, x, s, cmap);
}

#endif  // SFK_CELL_ONLY_N

}  // namespace sfk
