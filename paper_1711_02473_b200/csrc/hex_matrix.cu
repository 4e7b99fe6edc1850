// Hex Q_p local stiffness matrices — BASELINE config C5 (p = 1..4).
//
// Reference: registry `laplace` on `hex` (forms.py:186-189), rank 2, test
// index outermost: A[i*N3 + j] (forms.py:402-408); the
// spectral-mode program is sum-factorised to O(n^7) (SURVEY.md §8(a),
// reference count 15n^7 + 27n^6 + ...).
//
//   A[i][j] = sum_q sum_{l,l'} dphi_i^l(q) K_q[l][l'] dphi_j^l'(q),
//   K_q = w_q |J| G G^T = (w_q/|det|) R R^T  (R = adjugate rows),
//   dphi^l = T^l_x (x) T^l_y (x) T^l_z, T^l_d = D if d == l else B.
//
// Factorisation used here, for every quadrature plane qx (outer loop):
//   Z_ll'[qy][iz][jz]      = sum_qz T^l_z[iz][qz] T^l'_z[jz][qz] K_ll'(qx,qy,qz)
//   Y_g[iy][jy][iz][jz]    = sum_{(l,l') in g} sum_qy T^l_y[iy][qy] T^l'_y[jy][qy] Z_ll'
//   A[ix,jx][...]         += sum_g T^l_x[ix][qx] T^l'_x[jx][qx] Y_g
// where g groups the 9 (l,l') pairs by their x-table pattern (BB, BD, DB,
// DD): 4 x-contractions instead of 9.  Per cell ~ 9 m^3 n^2 + 9 m^2 n^4 +
// 4 m n^6 FMA (p=4: 0.48 M FMA vs the reference's 1.69 M flops).
//
// B200 mapping: one CTA per cell (n^4 threads; several cells for n <= 3).
// K at all points, Z for all planes and Y_g for all planes live in shared
// memory (150 KB at p=4), each produced by one CTA-wide phase; every thread
// r = (iy, iz, jy, jz) contracts Z over qy into its 4 Y_g values per plane.  A final pass gives each
// thread its n^2 outputs A[(ix,iy,iz),(jx,jy,jz)] from 4m shared loads and
// 4 m n^2 register FMAs — no register array lives across the plane loop (the
// r01 version spilled it).  Output rows are written straight from registers:
// for fixed (ix, jx) a warp stores runs of n^2 contiguous doubles; the 125 KB
// (p=4) of a cell is complete in L2 before eviction, so DRAM sees full lines.
#include <cstdlib>

#include "hex_geometry.cuh"

#ifndef SFK_MAT_ZB
#define SFK_MAT_ZB 1   // batched-pair Z phase at n <= 3 (A/B builds: 0)
#endif
#ifndef SFK_MAT_YB
#define SFK_MAT_YB 1   // all-jy Y phase at n <= 3 (A/B builds: 0)
#endif
#ifndef SFK_MAT_MINB3
#define SFK_MAT_MINB3 6   // min CTAs/SM of the n = 3 kernel (one-cell CTAs; A/B builds)
#endif

namespace sfk {

#ifdef SFK_MAT_ONLY_N
namespace {   // probe objects differ in macros, not template arguments: keep instances apart
#endif

template <int N, int M>
struct TabsMat {
  double B[N * M];
  double D[N * M];
  double W[M];
  double Bc[2 * M];
};

template <int N, int M, int CPB>
struct MatCfg {
  static constexpr int N2 = N * N, N3 = N * N * N, N4 = N * N * N * N, M3 = M * M * M;
  static constexpr int THREADS = round_up(CPB * N4, 32);
  static constexpr int ZS = 9 * M * M * N2;  // Z[pair][qx][qy][iz][jz] for one cell
  static constexpr int KS = 6 * M3;          // K (6 unique entries) at every point
  static constexpr int TS = 2 * N * M;       // B and D copies (runtime-indexed reads)
  static constexpr int YS = 4 * M * N4;      // Y_g[qx][r] for one cell, all planes
  static constexpr int DS = (CPB * N3 + 1) / 2;  // the cells' dof lists (int32, CSR mode)
  static constexpr size_t SMEM =
      (size_t)(CPB * (ZS + KS + YS + 24) + TS + DS) * sizeof(double);
};

// pair (l, l') -> symmetric K index: 00 11 22 01 02 12
__host__ __device__ constexpr int ksym(int l, int r) {
  return l == r ? l : (l + r == 1 ? 3 : (l + r == 2 ? 4 : 5));
}

// Four phases per CTA, each over all quadrature planes at once (3 barriers):
//  K  at every point (threads over points),
//  Z_ll'[qx][qy][iz][jz] = sum_qz Tz Tz' K_ll'   (threads over (pair, qx, qy, iz, jz)),
//  Y_g[qx][r]            = sum over pairs in g, qy (thread r = (iy, iz, jy, jz)),
//  A[(ix,..),(jx,..)]    = sum_{g,qx} Tx Tx' Y_g[qx][r]   (thread r, then stores).
// Position of column `col` in the sorted CSR row [lo, hi) (lower bound).
__device__ __forceinline__ int64_t csr_find(const int32_t* __restrict__ col_idx, int64_t lo,
                                            int64_t hi, int32_t col) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(col_idx + mid) < col) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// CSR = false: A[cell][N3*N3] is written (the reference's per-cell output).
// CSR = true : the cell matrices are scatter-added into the assembled CSR
//              matrix (values A, pattern row_ptr / col_idx from sfk_csr_create)
//              through cell_dofs — the local matrix never reaches HBM.
template <int N, int M, int CPB, bool CSR, bool YMAP = false>
__global__ void __launch_bounds__(MatCfg<N, M, CPB>::THREADS, (N == 3 && CPB == 1) ? SFK_MAT_MINB3 : 0)
hex_laplace_matrix_kernel(const __grid_constant__ TabsMat<N, M> T, int64_t ncells,
                          const double* __restrict__ coords, double* __restrict__ A,
                          const int32_t* __restrict__ dofs, const int64_t* __restrict__ row_ptr,
                          const int32_t* __restrict__ col_idx, const int32_t* __restrict__ emap) {
  using C = MatCfg<N, M, CPB>;
  constexpr int N2 = C::N2, N3 = C::N3, N4 = C::N4, M3 = C::M3;
  constexpr bool ZB = SFK_MAT_ZB && N <= 3;
  constexpr bool YB = SFK_MAT_YB && N <= 3 && !YMAP;
  extern __shared__ double smem[];
  double* sZ = smem;                       // [CPB][9][M][M][N2]
  double* sK = sZ + CPB * C::ZS;           // [CPB][6][M3]
  double* sY = sK + CPB * C::KS;           // [CPB][4][M][N4]
  double* sC = sY + CPB * C::YS;           // [CPB][24]
  double* sT = sC + CPB * 24;              // B, D
  int32_t* sD = reinterpret_cast<int32_t*>(sT + C::TS);  // [CPB][N3] (CSR)
  const int tid = threadIdx.x;
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int64_t rem = ncells - cell0;
  const int ncb = rem < CPB ? (int)rem : CPB;
  for (int i = tid; i < CPB * 24; i += C::THREADS)
    sC[i] = i < ncb * 24 ? __ldg(coords + cell0 * 24 + i) : 0.0;
  if (CSR)
    for (int i = tid; i < ncb * N3; i += C::THREADS) sD[i] = __ldg(dofs + cell0 * N3 + i);
  for (int i = tid; i < N * M; i += C::THREADS) {
    sT[i] = T.B[i];
    sT[N * M + i] = T.D[i];
  }
  // thread -> (cell, iy, iz, jy, jz)
  const bool act = tid < CPB * N4;
  const int c = act ? tid / N4 : 0, r = tid - c * N4;
  // YMAP: (jy, iy) fastest, so the lanes of a warp share (iz, jz) and the
  // Y-stage Z loads are broadcasts — faster at n = 4, slower at n = 3, 5
  // where the less contiguous output stores cost more (A/B:
  // profiles/r01bh_c5_ymap.jsonl)
  const int iy = YMAP ? (r / N) % N : r / (N * N2);
  const int iz = YMAP ? r / (N * N2) : (r / N2) % N;
  const int jy = YMAP ? r % N : (r / N) % N;
  const int jz = YMAP ? (r / N2) % N : r % N;
  __syncthreads();

  // ---- K at every point: threads over (cell, qx, qy, qz) -------------------
  for (int t = tid; t < CPB * M3; t += C::THREADS) {
    const int cc = t / M3, rr = t - cc * M3;
    const int qx = rr / (M * M), qy = (rr / M) % M, qz = rr % M;
    HexLineGeom geo;
    geo.setup(sC + cc * 24, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
    double r0[3], r1[3], r2[3];
    const double det = geo.adj(T.Bc[qz], T.Bc[M + qz], r0, r1, r2);
    const double s = ((T.W[qx] * T.W[qy]) * T.W[qz]) * rcp64(fabs(det));
    double* k = sK + cc * C::KS + rr;
    const double* rows[3] = {r0, r1, r2};
#pragma unroll
    for (int l = 0; l < 3; ++l)
#pragma unroll
      for (int m2 = l; m2 < 3; ++m2) {
        const double* a = rows[l];
        const double* b = rows[m2];
        k[ksym(l, m2) * M3] = s * fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
      }
  }
  __syncthreads();
  // ---- Z_ll'[qx][qy][iz][jz]: threads over (cell, pair, qx, qy, iz, jz) -----
  // ZB (small n): threads over (cell, qx, qy, iz, jz), all 9 pairs per
  // thread — the index arithmetic and the K / table loads are shared by the
  // pairs (at n = 3 the per-entry form was issue-bound on integer work:
  // FP64 pipe 29%, profiles/r01cj_C5_p2.md).  Same products, same order.
  if (ZB) {
    constexpr int PL = M * M * N2;   // one pair's plane block
    for (int t = tid; t < CPB * PL; t += C::THREADS) {
      const int cc = t / PL, q2 = t - cc * PL;
      const int qxy = q2 / N2, zz = q2 - qxy * N2;
      const int a = zz / N, b = zz - a * N;
      double ta[2][M], tb[2][M], kk[6][M];
#pragma unroll
      for (int qz = 0; qz < M; ++qz) {
        ta[0][qz] = sT[a * M + qz];
        ta[1][qz] = sT[N * M + a * M + qz];
        tb[0][qz] = sT[b * M + qz];
        tb[1][qz] = sT[N * M + b * M + qz];
      }
      const double* k = sK + cc * C::KS + qxy * M;
#pragma unroll
      for (int e = 0; e < 6; ++e)
#pragma unroll
        for (int qz = 0; qz < M; ++qz) kk[e][qz] = k[e * M3 + qz];
      double* zo = sZ + cc * C::ZS + q2;
#pragma unroll
      for (int pair = 0; pair < 9; ++pair) {
        const int l = pair / 3, lp = pair - 3 * l;
        double z = 0.0;
#pragma unroll
        for (int qz = 0; qz < M; ++qz)
          z = fma(ta[l == 2][qz] * tb[lp == 2][qz], kk[ksym(l, lp)][qz], z);
        zo[pair * PL] = z;
      }
    }
  }
  for (int t = tid; !ZB && t < CPB * C::ZS; t += C::THREADS) {
    const int cc = t / C::ZS, rr = t - cc * C::ZS;
    const int pair = rr / (M * M * N2), q2 = rr - pair * (M * M * N2);
    const int qxy = q2 / N2, zz = q2 - qxy * N2;
    const int a = zz / N, b = zz - a * N;
    const int l = pair / 3, lp = pair - 3 * l;
    const double* ta = sT + (l == 2 ? N * M : 0) + a * M;
    const double* tb = sT + (lp == 2 ? N * M : 0) + b * M;
    const double* k = sK + cc * C::KS + ksym(l, lp) * M3 + qxy * M;
    double z = 0.0;
#pragma unroll
    for (int qz = 0; qz < M; ++qz) z = fma(ta[qz] * tb[qz], k[qz], z);
    sZ[cc * C::ZS + rr] = z;
  }
  __syncthreads();
  // ---- y contraction into the 4 x-pattern groups, every plane ---------------
  // ZB (small n): threads over (cell, qx, iy, iz, jz), every jy per thread:
  // the 9 M z-values of (qx, iz, jz) are loaded once for the N jy outputs
  // (the per-(iy,iz,jy,jz) form issued one shared load per FMA).  Same
  // accumulation order per output.
  if (YB) {
    constexpr int YT = M * N3;   // work items per cell
    for (int t = tid; t < CPB * YT; t += C::THREADS) {
      const int cc = t / YT, w = t - cc * YT;
      const int qx = w / N3, w2 = w - qx * N3;
      const int yi = w2 / N2, w3 = w2 - yi * N2;
      const int zi = w3 / N, zj = w3 - zi * N;
      const double* z = sZ + cc * C::ZS + qx * M * N2 + zi * N + zj;
      double zv[9][M];
#pragma unroll
      for (int pr = 0; pr < 9; ++pr)
#pragma unroll
        for (int qy = 0; qy < M; ++qy) zv[pr][qy] = z[pr * M * M * N2 + qy * N2];
      double bi[M], di[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        bi[q] = sT[yi * M + q];
        di[q] = sT[N * M + yi * M + q];
      }
#pragma unroll
      for (int yj = 0; yj < N; ++yj) {
        double pyj[4][M];
#pragma unroll
        for (int q = 0; q < M; ++q) {
          const double bj = sT[yj * M + q], dj = sT[N * M + yj * M + q];
          pyj[0][q] = bi[q] * bj;
          pyj[1][q] = bi[q] * dj;
          pyj[2][q] = di[q] * bj;
          pyj[3][q] = di[q] * dj;
        }
        double yg[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int l = 0; l < 3; ++l)
#pragma unroll
          for (int lp = 0; lp < 3; ++lp) {
            const int pat = (l == 1 ? 2 : 0) + (lp == 1 ? 1 : 0);
            const int grp = (l == 0 ? 2 : 0) + (lp == 0 ? 1 : 0);
#pragma unroll
            for (int qy = 0; qy < M; ++qy)
              yg[grp] = fma(pyj[pat][qy], zv[l * 3 + lp][qy], yg[grp]);
          }
        // r = (iy, iz, jy, jz) in the non-YMAP thread order of phase B
        double* y = sY + cc * C::YS + qx * N4 + ((yi * N + zi) * N + yj) * N + zj;
#pragma unroll
        for (int g = 0; g < 4; ++g) y[g * M * N4] = yg[g];
      }
    }
  }
  if (!YB && act) {
    double py[4][M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
      const double bi = sT[iy * M + q], di = sT[N * M + iy * M + q];
      const double bj = sT[jy * M + q], dj = sT[N * M + jy * M + q];
      py[0][q] = bi * bj;
      py[1][q] = bi * dj;
      py[2][q] = di * bj;
      py[3][q] = di * dj;
    }
#pragma unroll 1
    for (int qx = 0; qx < M; ++qx) {
      const double* z = sZ + c * C::ZS + qx * M * N2 + iz * N + jz;
      double yg[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int lp = 0; lp < 3; ++lp) {
          const int pat = (l == 1 ? 2 : 0) + (lp == 1 ? 1 : 0);
          const int grp = (l == 0 ? 2 : 0) + (lp == 0 ? 1 : 0);
          const double* zp = z + (l * 3 + lp) * M * M * N2;
#pragma unroll
          for (int qy = 0; qy < M; ++qy) yg[grp] = fma(py[pat][qy], zp[qy * N2], yg[grp]);
        }
      double* y = sY + c * C::YS + qx * N4 + r;
#pragma unroll
      for (int g = 0; g < 4; ++g) y[g * M * N4] = yg[g];
    }
  }
  __syncthreads();

  // ---- phase B: x contraction and store --------------------------------------
  if (act && c < ncb) {
    double acc[N][N];
#pragma unroll
    for (int ix = 0; ix < N; ++ix)
#pragma unroll
      for (int jx = 0; jx < N; ++jx) acc[ix][jx] = 0.0;
    const double* y = sY + c * C::YS + r;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const double* ta = (g & 2) ? T.D : T.B;  // test  (row) x-table
      const double* tb = (g & 1) ? T.D : T.B;  // trial (col) x-table
#pragma unroll
      for (int qx = 0; qx < M; ++qx) {
        const double v = y[(g * M + qx) * N4];
#pragma unroll
        for (int jx = 0; jx < N; ++jx) {
          const double t = tb[jx * M + qx] * v;
#pragma unroll
          for (int ix = 0; ix < N; ++ix) acc[ix][jx] = fma(ta[ix * M + qx], t, acc[ix][jx]);
        }
      }
    }
    const int rowoff = iy * N + iz;   // + ix * N2  -> test index
    const int coloff = jy * N + jz;   // + jx * N2  -> trial index
    if (CSR && emap) {
      // positions precomputed per pattern (sfk_csr_entry_map): one load each
      const int32_t* mp = emap + (cell0 + c) * (int64_t)(N3 * N3);
#pragma unroll
      for (int ix = 0; ix < N; ++ix)
#pragma unroll
        for (int jx = 0; jx < N; ++jx)
          atomicAdd(A + __ldg(mp + (ix * N2 + rowoff) * N3 + jx * N2 + coloff), acc[ix][jx]);
    } else if (CSR) {
      const int32_t* cd = sD + c * N3;
      int32_t cols[N];
#pragma unroll
      for (int jx = 0; jx < N; ++jx) cols[jx] = cd[jx * N2 + coloff];
#pragma unroll
      for (int ix = 0; ix < N; ++ix) {
        const int32_t row = cd[ix * N2 + rowoff];
        const int64_t lo = __ldg(row_ptr + row), hi = __ldg(row_ptr + row + 1);
#pragma unroll
        for (int jx = 0; jx < N; ++jx)
          atomicAdd(A + csr_find(col_idx, lo, hi, cols[jx]), acc[ix][jx]);
      }
    } else {
      double* out = A + (cell0 + c) * (int64_t)(N3 * N3);
#pragma unroll
      for (int ix = 0; ix < N; ++ix)
#pragma unroll
        for (int jx = 0; jx < N; ++jx)
          out[(int64_t)(ix * N2 + rowoff) * N3 + jx * N2 + coloff] = acc[ix][jx];
    }
  }
}

template <int N, int M, int CPB, bool CSR = false, bool YMAP = false>
static int launch_mat(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                      cudaStream_t s, const int32_t* dofs = nullptr,
                      const int64_t* row_ptr = nullptr, const int32_t* col_idx = nullptr,
                      const int32_t* emap = nullptr) {
  using C = MatCfg<N, M, CPB>;
  TabsMat<N, M> T;
  for (int i = 0; i < N; ++i)
    for (int q = 0; q < M; ++q) {
      T.B[i * M + q] = p->B[i * p->m + q];
      T.D[i * M + q] = p->D[i * p->m + q];
    }
  for (int q = 0; q < M; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[M + q] = p->Bc[p->m + q];
  }
  const unsigned grid = (unsigned)((ncells + CPB - 1) / CPB);
  auto kern = hex_laplace_matrix_kernel<N, M, CPB, CSR, YMAP>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_matrix", &sh))
    return rc_;
  kern<<<grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, A, dofs, row_ptr, col_idx, emap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_matrix_kernel launch");
}

#ifdef SFK_MAT_ONLY_N
// probe builds (tools/kernel_sweep.py c5): one instantiation of the FMA kernel
}  // anonymous namespace
}  // namespace sfk
extern "C" int SFK_MAT_PROBE_ENTRY(const sfk_plan* p, int64_t ncells, double* A,
                                   const double* coords, const double* w0, void* stream) {
  (void)w0;
  if (p->n != SFK_MAT_ONLY_N || p->m != SFK_MAT_ONLY_N)
    return sfk::fail(SFK_EUNSUPPORTED, "probe build: n = m = %d only", SFK_MAT_ONLY_N);
  return sfk::launch_mat<SFK_MAT_ONLY_N, SFK_MAT_ONLY_N, SFK_MATP_CPB>(p, ncells, A, coords,
                                                                      (cudaStream_t)stream);
}
namespace sfk {
#else
int launch_hex_matrix(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                      cudaStream_t s) {
  if (p->collocated)
    return fail(SFK_EUNSUPPORTED, "hex laplace matrix: collocated variant not instantiated");
  if (p->n == p->m) {
    switch (p->n) {
      case 2: {
        // thread-per-cell kernel (hex_matrix_p1.cu); option c5_p1 = 1 selects
        // the CTA-phase kernel below for A/B runs
        const bool phase = option(OPT_C5_P1) == 1;
        if (!phase) return launch_hex_matrix_p1(p, ncells, A, coords, s);
        return launch_mat<2, 2, 16>(p, ncells, A, coords, s);
      }
      // (a DMMA version at n = 3 measured slower, 0.54 vs 0.37 ms: too little
      // work per cell for the padded tiles, profiles/r01bl_c5_p2_dmma.jsonl)
      // one cell per 96-thread CTA at 6 CTAs per SM (tools/kernel_sweep.py c5,
      // profiles/r02cs_c5_sweep.jsonl: 0.2908 -> 0.2499 ms; 3 cells per CTA before)
      case 3: return launch_mat<3, 3, 1>(p, ncells, A, coords, s);
      case 4: {
        // DMMA kernel (hex_matrix_tc.cu); option c5_p3 = 1 selects the FMA one,
        // c5_hi_cfg = 3, 4 the chunked DMMA kernel of hex_matrix_tcn.cu (slower
        // here: 0.98 vs 1.08 / 1.18 ms, profiles/r02bc_c5.jsonl)
        if (option(OPT_C5_HI_CFG) >= 3) return launch_hex_matrix_tcn(p, ncells, A, coords, s);
        const bool phase = option(OPT_C5_P3) == 1;
        if (!phase) {
          const int rc = launch_hex_matrix_tc4(p, ncells, A, coords, s);
          if (rc != SFK_EUNSUPPORTED) return rc;
        }
        return launch_mat<4, 4, 1, false, true>(p, ncells, A, coords, s);
      }
      case 5: {
        // chunked DMMA kernel (hex_matrix_tcn.cu): 5.01 -> 4.41 ms against
        // tc5 (profiles/r02bc_c5.jsonl); option c5_p4 = 1 selects the FMA
        // kernel, c5_p4 = 2 tc5 (hex_matrix_tc.cu)
        const int64_t v = option(OPT_C5_P4);
        if (v == 1) return launch_mat<5, 5, 1>(p, ncells, A, coords, s);
        if (v == 2) {
          const int rc = launch_hex_matrix_tc5(p, ncells, A, coords, s);
          if (rc != SFK_EUNSUPPORTED) return rc;
          return launch_mat<5, 5, 1>(p, ncells, A, coords, s);
        }
        return launch_hex_matrix_tcn(p, ncells, A, coords, s);
      }
      default:
        // p = 5..8: chunked DMMA kernel (hex_matrix_tcn.cu)
        if (hex_matrix_tcn_supported(p->n, p->m))
          return launch_hex_matrix_tcn(p, ncells, A, coords, s);
        break;
    }
  }
  return fail(SFK_EUNSUPPORTED,
              "hex laplace matrix: no kernel for n=%d, m=%d (n==m in 2..9, p<=8)", p->n, p->m);
}

int launch_hex_matrix_csr(const sfk_plan* p, int64_t ncells, const int32_t* dofs,
                          const double* coords, const int64_t* row_ptr, const int32_t* col_idx,
                          const int32_t* emap, double* values, cudaStream_t s) {
  if (p->collocated || p->n != p->m)
    return fail(SFK_EUNSUPPORTED, "CSR assembly: hex laplace with m == n only");
  // (the DMMA kernels of hex_matrix_tc.cu have an entry-map epilogue too, but
  // their fragment-order map loads and atomics scatter: p = 3 1.74 -> 1.88 ms,
  // p = 4 8.7 -> 10.9 ms, profiles/r01bk_csr_dmma.jsonl; option csr_dmma = 1 uses them)
  const bool csr_dmma = option(OPT_CSR_DMMA) == 1;
  if (csr_dmma && emap && (p->n == 4 || p->n == 5)) {
    const int rc = p->n == 4 ? launch_hex_matrix_tc4(p, ncells, values, coords, s, emap)
                             : launch_hex_matrix_tc5(p, ncells, values, coords, s, emap);
    if (rc != SFK_EUNSUPPORTED) return rc;
  }
  switch (p->n) {
    case 2:
      return launch_mat<2, 2, 16, true>(p, ncells, values, coords, s, dofs, row_ptr, col_idx,
                                        emap);
    case 3:
      return launch_mat<3, 3, 3, true>(p, ncells, values, coords, s, dofs, row_ptr, col_idx,
                                        emap);
    case 4:
      return launch_mat<4, 4, 1, true>(p, ncells, values, coords, s, dofs, row_ptr, col_idx,
                                        emap);
    case 5:
      return launch_mat<5, 5, 1, true>(p, ncells, values, coords, s, dofs, row_ptr, col_idx,
                                        emap);
    default:
      // p = 5..8: the chunked DMMA kernel with its entry-map epilogue
      if (hex_matrix_tcn_supported(p->n, p->m)) {
        if (!emap)
          return fail(SFK_EUNSUPPORTED,
                      "CSR assembly at p >= 5 needs the entry map (sfk_csr_entry_map)");
        return launch_hex_matrix_tcn(p, ncells, values, coords, s, emap);
      }
      break;
  }
  return fail(SFK_EUNSUPPORTED, "CSR assembly: no kernel for n=%d (p<=8)", p->n);
}

#endif  // SFK_MAT_ONLY_N

}  // namespace sfk
