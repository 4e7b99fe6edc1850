// Hex Q_p Laplace action, collocation-derivative schedule with ONE WARP PER
// CELL — BASELINE C2 at the high degrees (n^2 > 32 lines per direction).
//
// Same operator, reference mapping, schedule (stages A..I), tables and
// shared layouts as v6 (hex_action6.cu, hex_action6_layout.cuh): C = B^-1 D,
// 12 n^4 FMA per cell.  What changes is ownership.  v6 gives each of the
// CTA's threads one line of a cell and separates the nine stages by CTA
// barriers, so every warp of the CTA is in the same stage at the same time.
// Here a warp owns a whole cell: lane l runs lines l, l + 32, l + 64, ... of
// every stage (ceil(n^2 / 32) passes; the loads of all passes first, then
// their contractions — up to 3 n independent chains — then the stores), the
// stages are separated by __syncwarp only, and the warp stages its own u
// (into slot S4, free from stage G to the next stage C) and coordinates.
// No CTA barrier at all: the warps of an SM drift through different stages,
// so the shared-memory stages of one overlap the FP64 stages of another.
// The DMMA kernel at n = 8 gained 1.49x from exactly this (tc8c,
// profiles/r02l_*, r02m_*).
#include "async_copy.cuh"
#include "hex_action6_layout.cuh"
#include "hex_colloc_deriv.cuh"
#include "hex_geometry.cuh"

namespace sfk {

__host__ __device__ constexpr int v7_slot(int n) {
  int s = 0;
  for (int r = V6_P1; r <= V6_P2; ++r) s = v6_role(n, r).cs > s ? v6_role(n, r).cs : s;
  return s;
}

template <int N, int WARPS>
struct V7Cfg {
  static constexpr int NN = N * N, N3 = N * N * N;
  static constexpr int NP = (NN + 31) / 32;                 // line passes per stage
  static constexpr int SLOT = (v7_slot(N) + 1) & ~1;        // doubles per cell and slot
  static constexpr int CELL = 4 * SLOT + 2 * 24 + 36 + 2;   // slots, coords x2, edges
  static constexpr int THREADS = 32 * WARPS;
  static constexpr size_t SMEM = (size_t)WARPS * CELL * sizeof(double);
  static_assert(N3 + 1 <= SLOT, "u fits slot S4");
};

template <int N, int WARPS, int MINB>
__global__ void __launch_bounds__(V7Cfg<N, WARPS>::THREADS, MINB)
hex_laplace_action_v7(const __grid_constant__ TabsV6<N> T, int64_t ncells,
                      const double* __restrict__ coords, const double* __restrict__ u,
                      double* __restrict__ A) {
  using C = V7Cfg<N, WARPS>;
  constexpr int NN = C::NN, N3 = C::N3, NP = C::NP, SL = C::SLOT, LD = TabsV6<N>::LD;
  // one cell per warp: every role at the cell's slot base (cell stride unused)
  constexpr V6Arr P1 = v6_role(N, V6_P1), Qr = v6_role(N, V6_Q), Vr = v6_role(N, V6_V),
                  GZr = v6_role(N, V6_GZ), GXr = v6_role(N, V6_GX), GYr = v6_role(N, V6_GY),
                  Rr = v6_role(N, V6_R), P2 = v6_role(N, V6_P2);
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* base = smem + warp * C::CELL;
  double* S1 = base;
  double* S2 = S1 + SL;
  double* S3 = S2 + SL;
  double* S4 = S3 + SL;                    // gz / fz / tz, and u between G and C
  double* sCo = S4 + SL;                   // [2][24]
  double* sGE = sCo + 48;                  // [36]
  const int64_t nbatch = (ncells + WARPS - 1) / WARPS;

  // lane -> line of pass ps: l = lane + 32 ps, (a, b) = (l / N, l % N)
  int la[NP], lb[NP];
  bool ok[NP];
#pragma unroll
  for (int ps = 0; ps < NP; ++ps) {
    const int l = lane + 32 * ps;
    ok[ps] = l < NN;
    const int lc = ok[ps] ? l : 0;
    la[ps] = lc / N;
    lb[ps] = lc - la[ps] * N;
  }

  auto prefetch = [&](int64_t bt, int buf) {
    const int64_t cg = bt * WARPS + warp;
    if (cg < ncells) {
      async_copy_phase<32>(S4 + dst_shift(u + cg * N3), u + cg * N3, N3, lane);
      if (lane < 24) cp_async8(sCo + buf * 24 + lane, coords + cg * 24 + lane);
    }
    cp_async_commit();
  };

  int64_t b = blockIdx.x;
  if (b < nbatch) prefetch(b, 0);
  for (int k = 0; b < nbatch; b += gridDim.x, ++k) {
    const int cur = k & 1;
    const int64_t cell = b * WARPS + warp;
    const bool live = cell < ncells;           // warp-uniform
    cp_async_wait<0>();
    __syncwarp();
    const double* su = S4 + dst_shift(u + cell * N3);
    const double* X = sCo + cur * 24;

    // ---- A: x-lines (y, z): P = B_x u -> S1; edges of the cell -> sGE ------
    {
      double in[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int i = 0; i < N; ++i) in[ps][i] = (live && ok[ps]) ? su[i * NN + la[ps] * N + lb[ps]] : 0.0;
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.B, in[ps], o[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int q = 0; q < N; ++q) S1[q * P1.sx + la[ps] * P1.sy + lb[ps]] = o[ps][q];
        }
      if (lane < 36 - 32) sGE[32 + lane] = hex_cell_edge(X, 32 + lane);
      sGE[lane] = hex_cell_edge(X, lane);
    }
    __syncwarp();

    // ---- B: y-lines (x, z): Q = B_y P -> S2 ---------------------------------
    {
      double in[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int i = 0; i < N; ++i) in[ps][i] = S1[la[ps] * P1.sx + i * P1.sy + lb[ps]];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.B, in[ps], o[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int j = 0; j < N; ++j) S2[la[ps] * Qr.sx + j * Qr.sy + lb[ps]] = o[ps][j];
        }
    }
    __syncwarp();

    // ---- C: z-lines (y, x): V = B_z Q -> S1, gz = C_z V -> S4 ---------------
    {
      double in[NP][N], v[NP][N], g[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int i = 0; i < N; ++i) in[ps][i] = S2[la[ps] * Qr.sy + lb[ps] * Qr.sx + i];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.B, in[ps], v[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.C, v[ps], g[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int j = 0; j < N; ++j) {
            S1[la[ps] * Vr.sy + lb[ps] * Vr.sx + j] = v[ps][j];
            S4[la[ps] * GZr.sy + lb[ps] * GZr.sx + j] = g[ps][j];
          }
        }
    }
    __syncwarp();

    // ---- D: x-lines (y, z): gx = C_x V -> S2; y-lines (x, z): gy -> S3 ------
    {
      double in[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int i = 0; i < N; ++i) in[ps][i] = S1[la[ps] * Vr.sy + i * Vr.sx + lb[ps]];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.C, in[ps], o[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int j = 0; j < N; ++j) S2[j * GXr.sx + la[ps] * GXr.sy + lb[ps]] = o[ps][j];
        }
    }
    {
      double in[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int i = 0; i < N; ++i) in[ps][i] = S1[la[ps] * Vr.sx + i * Vr.sy + lb[ps]];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.C, in[ps], o[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int j = 0; j < N; ++j) S3[la[ps] * GYr.sx + j * GYr.sy + lb[ps]] = o[ps][j];
        }
    }
    __syncwarp();

    // ---- E: z-lines (y, x): geometry + flux in place (S2, S3, S4) -----------
#pragma unroll 1
    for (int ps = 0; ps < NP; ++ps) {
      if (!ok[ps]) continue;
      const int qy = la[ps], qx = lb[ps];
      double* gxl = S2 + qx * GXr.sx + qy * GXr.sy;
      double* gyl = S3 + qy * GYr.sy + qx * GYr.sx;
      double* gzl = S4 + qy * GZr.sy + qx * GZr.sx;
      HexLineAdj geo;
      geo.setup_edges(sGE, T.Bc[qx], T.Bc[N + qx], T.Bc[qy], T.Bc[N + qy]);
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
    __syncwarp();

    // ---- F: x-lines tx = C_x^T fx; y-lines ty = C_y^T fy; z-lines tz = C_z^T
    //      fz, each in place (every lane loads all its lines first) ----------
    {
      double in[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int i = 0; i < N; ++i) in[ps][i] = ok[ps] ? S2[i * GXr.sx + la[ps] * GXr.sy + lb[ps]] : 0.0;
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.CT, in[ps], o[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int j = 0; j < N; ++j) S2[j * GXr.sx + la[ps] * GXr.sy + lb[ps]] = o[ps][j];
        }
    }
    {
      double in[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int i = 0; i < N; ++i) in[ps][i] = ok[ps] ? S3[la[ps] * GYr.sx + i * GYr.sy + lb[ps]] : 0.0;
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.CT, in[ps], o[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int j = 0; j < N; ++j) S3[la[ps] * GYr.sx + j * GYr.sy + lb[ps]] = o[ps][j];
        }
    }
    {
      double in[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int i = 0; i < N; ++i) in[ps][i] = ok[ps] ? S4[la[ps] * GZr.sy + lb[ps] * GZr.sx + i] : 0.0;
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.CT, in[ps], o[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int j = 0; j < N; ++j) S4[la[ps] * GZr.sy + lb[ps] * GZr.sx + j] = o[ps][j];
        }
    }
    __syncwarp();

    // ---- G: z-lines (y, x): t = tx + ty + tz; R = B_z^T t -> S1 -------------
    {
      double t[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) {
        const int qy = la[ps], qx = lb[ps];
#pragma unroll
        for (int q = 0; q < N; ++q)
          t[ps][q] = (S2[qx * GXr.sx + qy * GXr.sy + q] + S3[qy * GYr.sy + qx * GYr.sx + q]) +
                     S4[qy * GZr.sy + qx * GZr.sx + q];
      }
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.BT, t[ps], o[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int i = 0; i < N; ++i) S1[la[ps] * Rr.sy + lb[ps] * Rr.sx + i] = o[ps][i];
        }
    }
    __syncwarp();
    // S4 is free until the next stage C: stage the next batch's u there
    if (b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- H: y-lines (x, z): B_y^T R -> S2 (layout P2) -----------------------
    {
      double in[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int j = 0; j < N; ++j) in[ps][j] = S1[la[ps] * Rr.sx + j * Rr.sy + lb[ps]];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.BT, in[ps], o[ps]);
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
        if (ok[ps]) {
#pragma unroll
          for (int i = 0; i < N; ++i) S2[la[ps] * P2.sx + i * P2.sy + lb[ps]] = o[ps][i];
        }
    }
    __syncwarp();

    // ---- I: x-lines (y, z): A = B_x^T (.) -> HBM ----------------------------
    {
      double in[NP][N], o[NP][N];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps)
#pragma unroll
        for (int q = 0; q < N; ++q) in[ps][q] = S2[q * P2.sx + la[ps] * P2.sy + lb[ps]];
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) v6_contract<N, N, LD>(T.BT, in[ps], o[ps]);
      if (live) {
        double* ap = A + cell * N3;
#pragma unroll
        for (int ps = 0; ps < NP; ++ps)
          if (ok[ps]) {
#pragma unroll
            for (int i = 0; i < N; ++i) ap[i * NN + la[ps] * N + lb[ps]] = o[ps][i];
          }
      }
    }
    // next batch: its stage A writes S1 (read by H above) and reads S4 (u),
    // both after this warp's own program order + the __syncwarp at the top
  }
}

template <int N, int WARPS, int MINB>
static int launch_v7(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* u, cudaStream_t s) {
  using C = V7Cfg<N, WARPS>;
  auto kern = hex_laplace_action_v7<N, WARPS, MINB>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_action_v7", &sh, true))
    return rc_;
  const TabsV6<N> T = make_tabs_v6<N>(p);
  const int64_t nbatch = (ncells + WARPS - 1) / WARPS;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, u, A);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_v7 launch");
}

// (warps per CTA, min CTAs per SM) per n; option v6_cfg = 1, 2 select A/B
// alternatives.
int launch_hex_action_v7(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s) {
  if (p->n != p->m || !p->has_ct) return SFK_EUNSUPPORTED;
  const int alt = (int)option(OPT_V6_CFG);
  switch (p->n) {
    case 6:
      if (alt == 1) return launch_v7<6, 4, 4>(p, ncells, A, coords, w0, s);
      return launch_v7<6, 4, 3>(p, ncells, A, coords, w0, s);
    case 7:
      if (alt == 1) return launch_v7<7, 4, 4>(p, ncells, A, coords, w0, s);
      return launch_v7<7, 4, 3>(p, ncells, A, coords, w0, s);
    case 9:
      if (alt == 1) return launch_v7<9, 2, 4>(p, ncells, A, coords, w0, s);
      if (alt == 2) return launch_v7<9, 8, 1>(p, ncells, A, coords, w0, s);
      return launch_v7<9, 4, 2>(p, ncells, A, coords, w0, s);
    default: return SFK_EUNSUPPORTED;
  }
}

}  // namespace sfk
