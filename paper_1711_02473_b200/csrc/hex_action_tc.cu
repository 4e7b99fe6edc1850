// Hex Q_7 Laplace action on the FP64 tensor cores (DMMA) — BASELINE C2 at
// p = 7 (n = m = 8 dofs / GL points per axis).
//
// Same math, reference mapping and stage structure as hex_action3.cu
// (forms.py:186-189, 235-243; passes.py:672-743; scheduling.py:617-738);
// the difference is WHO computes a contraction stage.  In the line kernels
// each thread owns a 1D line and issues n*m DFMA (+ a constant load per two
// DFMA) per table.  Here a warp owns tiles of 8 lines and every stage is a
// batched 8x8x8 GEMM on `mma.sync.m8n8k4.f64` (SASS DMMA): for n = m = 8
//   out[q][line] = sum_i T[i][q] in[i][line]
// is exactly two m8n8k4 steps per table and tile, no padding.  DMMA and DFMA
// share the FP64 throughput on B200 (profiles/r01_fp64_mix.txt), so the gain
// is issue bandwidth: one DMMA does the work of 8 DFMA + 4 constant loads and
// leaves the issue slots to the per-point geometry/flux (DFMA).
//
// Two fragment forms:
//  * D-form (x, y, y^T, x^T stages): lines are the MMA n-dimension, the
//    contraction index k = kq + 4*ks; outputs D[q][line pair] are stored as
//    128-bit words (lines are contiguous in memory along iz).
//  * D'-form (z and z^T, contraction along the contiguous z axis): lines are
//    the MMA m-dimension, k = 2*kq + ks, so a lane's two k-step operands are
//    adjacent (one 128-bit load) and its two outputs too (one 128-bit store,
//    in place).
// Shared layouts use an XOR swizzle of the fastest index (bit 2, driven by
// bit 1 of the slower indices) instead of padding, which makes every
// fragment load/store and the pointwise pass bank-conflict free with ~2%
// padding.
#include <type_traits>

#include "async_copy.cuh"
#include "hex_geometry.cuh"

namespace sfk {

// Pointwise geometry of the tc8 kernel: the direct HexLineGeom form (33
// FP64 ops per point).  SFK_TC8_GEOM=0 selects HexLineAdj (adjugate rows as
// polynomials in xi_z, 15 ops per point), which the line kernels use but
// which measured slower here: p = 7 2.10 -> 2.35 ms (profiles/r01ch_*.jsonl).
#ifndef SFK_TC8_GEOM
#define SFK_TC8_GEOM 1
#endif
using TC8Geo = std::conditional<SFK_TC8_GEOM == 1, HexLineGeom, HexLineAdj>::type;
template <class TT>
__device__ __forceinline__ double tc8_adj(const HexLineGeom& g, const TT& T, int q, double r0[3],
                                          double r1[3], double r2[3]) {
  return g.adj(T.Bc[q], T.Bc[8 + q], r0, r1, r2);
}
template <class TT>
__device__ __forceinline__ double tc8_adj(const HexLineAdj& g, const TT& T, int q, double r0[3],
                                          double r1[3], double r2[3]) {
  return g.adj(T.Bc[8 + q], r0, r1, r2);
}

__device__ __forceinline__ void dmma_acc(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

#ifndef SFK_TC8_CPB
#define SFK_TC8_CPB 4   // 2 cells / 4 warps per CTA at 4 CTAs/SM measured slower: 2.09 -> 2.57 ms (r01dj_*)
#endif
namespace tc8 {
constexpr int N = 8, M = 8, NN = 64, N3 = 512;
constexpr int CPB = SFK_TC8_CPB;         // cells per CTA (4: 8 warps; 2: 4 warps)
constexpr int THREADS = CPB * NN;        // 256: one thread per z-line in the pointwise pass
constexpr int WARPS = THREADS / 32;
constexpr int TILES = CPB * 8;           // 8-line tiles per stage (8 per cell)
constexpr int TPW = TILES / WARPS;       // tiles per warp
constexpr int UPL = 68, UC = N * UPL;    // u   [c][ix][iy*8+iz], plane stride 68
constexpr int PX = 72, XA = M * PX;      // X/R [c][k][q][iy][iz] (swizzled iz)
constexpr int XC = 2 * XA;
constexpr int YX = 66, YA = M * YX;      // Y/S [c][k][qx][qy][z]  (swizzled z)
constexpr int YC = 3 * YA + 8;
constexpr int CSZ = CPB * 24;
constexpr size_t SMEM = (size_t)(CPB * XC + CPB * YC + CPB * UC + 2 * CSZ) * sizeof(double);

__device__ __forceinline__ int sw(int a) { return ((a >> 1) & 1) << 2; }
// X/R element (q, iy, iz) of one array
__device__ __forceinline__ int xaddr(int q, int iy, int iz) {
  return q * PX + iy * 8 + (iz ^ sw(q) ^ sw(iy));
}
// Y/S element (qx, qy, z) of one array
__device__ __forceinline__ int yaddr(int qx, int qy, int z) { return qx * YX + qy * 8 + (z ^ sw(qy)); }
}  // namespace tc8

// GS = true: global operator y += sum_c P_c^T A_c P_c x (SURVEY.md §8(f)
// item 1): the map cmap[c][0..511] (int32) is double-buffered in the u area,
// x is gathered through it by the x stage, y scattered with fp64 atomics by
// the transposed x stage.
template <bool GS>
__global__ void __launch_bounds__(tc8::THREADS, 8 / tc8::CPB)
hex_laplace_action_tc8(const __grid_constant__ Tabs<8, 8> T, int64_t ncells,
                       const double* __restrict__ coords, const double* __restrict__ u,
                       double* __restrict__ A, const int* __restrict__ cmap) {
  using namespace tc8;
  extern __shared__ __align__(16) double smem[];
  double* sX = smem;
  double* sY = sX + CPB * XC;
  double* sU = sY + CPB * YC;
  double* sCo = sU + CPB * UC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, gq = lane >> 2;   // fragment coordinates
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  int* sMap = reinterpret_cast<int*>(sU);   // GS: [2][CPB*512] int32
  static_assert(2 * CPB * N3 <= 2 * CPB * UC, "map double buffer does not fit");

  // table fragments
  //  D-form fwd  A[m=q][k=i]  : T[4ks+kq][gq]      (bf, df)
  //  D-form bwd  A[m=i][k=q]  : T[gq][4ks+kq]      (bb, db)
  //  D'-form fwd B[k=i][n=q]  : T[2kq+ks][gq]      (zbf, zdf)
  //  D'-form bwd B[k=q][n=i]  : T[gq][2kq+ks]      (zbb, zdb)
  double bf[2], df[2], bb[2], db[2], zbf[2], zdf[2], zbb[2], zdb[2];
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    bf[ks] = T.B[(4 * ks + kq) * M + gq];
    df[ks] = T.D[(4 * ks + kq) * M + gq];
    bb[ks] = T.B[gq * M + 4 * ks + kq];
    db[ks] = T.D[gq * M + 4 * ks + kq];
    zbf[ks] = T.B[(2 * kq + ks) * M + gq];
    zdf[ks] = T.D[(2 * kq + ks) * M + gq];
    zbb[ks] = T.B[gq * M + 2 * kq + ks];
    zdb[ks] = T.D[gq * M + 2 * kq + ks];
  }

  // u: 64 doubles per ix-plane -> plane stride UPL (16B chunks when aligned)
  auto prefetch = [&](int64_t bt, int buf) {
    const int64_t c0 = bt * CPB;
    const int nc = (int)((ncells - c0) < CPB ? (ncells - c0) : CPB);
    const double* src = u + c0 * N3;
    if (GS) {
      for (int e = tid; e < nc * N3; e += THREADS)
        cp_async4(sMap + buf * CPB * N3 + e, cmap + c0 * N3 + e);
    } else if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      for (int ch = tid; ch < nc * (N3 / 2); ch += THREADS) {
        const int c = ch >> 8, r = ch & 255;
        cp_async16(sU + c * UC + (r >> 5) * UPL + 2 * (r & 31), src + 2 * ch);
      }
    } else {
      for (int e = tid; e < nc * N3; e += THREADS) {
        const int c = e >> 9, r = e & 511;
        cp_async8(sU + c * UC + (r >> 6) * UPL + (r & 63), src + e);
      }
    }
    async_copy<THREADS>(sCo + buf * CSZ, coords + c0 * 24, nc * 24, tid);
    cp_async_commit();
  };

  int64_t b = blockIdx.x;
  if (b < nbatch) prefetch(b, 0);
  for (int it = 0; b < nbatch; b += gridDim.x, ++it) {
    const int cur = it & 1;
    const int64_t cell0 = b * CPB;
    const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
    cp_async_wait<0>();
    __syncthreads();
    const double* sC = sCo + cur * CSZ;
    const int* smap = sMap + cur * CPB * N3;

    // Each warp owns tiles t = warp + WARPS*j (the same in-cell tile index for
    // TPW cells): all fragment loads first, then the DMMAs (TPW independent
    // accumulator chains), then the stores.
    // ---- x stage (D-form): tile (c, iy), lines iz; X0 = Bx u, X1 = Dx u ----
    {
      double f[TPW][2], o[TPW][4];
      // in-cell tile index of this warp's j-th tile: (warp + WARPS*j) & 7
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        if (GS) {
          const int* mp = smap + c * N3 + ((warp + WARPS * j) & 7) * 8 + gq;   // (ix, iy, iz = gq)
          f[j][0] = c < ncb ? __ldg(u + mp[kq * NN]) : 0.0;
          f[j][1] = c < ncb ? __ldg(u + mp[(4 + kq) * NN]) : 0.0;
        } else {
          const double* in = sU + c * UC + ((warp + WARPS * j) & 7) * 8 + gq;
          f[j][0] = in[kq * UPL];
          f[j][1] = in[(4 + kq) * UPL];
        }
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          if (ks == 0) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.0;
          dmma_acc(o[j][0], o[j][1], bf[ks], f[j][ks]);
          dmma_acc(o[j][2], o[j][3], df[ks], f[j][ks]);
        }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        double* out = sX + c * XC + xaddr(gq, ((warp + WARPS * j) & 7), 2 * kq);
        *reinterpret_cast<double2*>(out) = make_double2(o[j][0], o[j][1]);
        *reinterpret_cast<double2*>(out + XA) = make_double2(o[j][2], o[j][3]);
      }
    }
    __syncthreads();
    if (b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- y stage (D-form): tile (c, qx), lines iz; BB, BD <- X0, DB <- X1 --
    {
      double f[TPW][4], o[TPW][6];
      // in-cell tile index of this warp's j-th tile: (warp + WARPS*j) & 7
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        const double* x = sX + c * XC;
        f[j][0] = x[xaddr(((warp + WARPS * j) & 7), kq, gq)];
        f[j][1] = x[xaddr(((warp + WARPS * j) & 7), 4 + kq, gq)];
        f[j][2] = x[XA + xaddr(((warp + WARPS * j) & 7), kq, gq)];
        f[j][3] = x[XA + xaddr(((warp + WARPS * j) & 7), 4 + kq, gq)];
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          if (ks == 0) o[j][0] = o[j][1] = o[j][2] = o[j][3] = o[j][4] = o[j][5] = 0.0;
          dmma_acc(o[j][0], o[j][1], bf[ks], f[j][ks]);
          dmma_acc(o[j][2], o[j][3], df[ks], f[j][ks]);
          dmma_acc(o[j][4], o[j][5], bf[ks], f[j][2 + ks]);
        }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        double* out = sY + c * YC + yaddr(((warp + WARPS * j) & 7), gq, 2 * kq);
        *reinterpret_cast<double2*>(out) = make_double2(o[j][0], o[j][1]);           // BB
        *reinterpret_cast<double2*>(out + YA) = make_double2(o[j][2], o[j][3]);      // BD
        *reinterpret_cast<double2*>(out + 2 * YA) = make_double2(o[j][4], o[j][5]);  // DB
      }
    }
    __syncthreads();

    // ---- z forward (D'-form, in place): tile (c, qx), lines qy --------------
    //  slot0 <- Dz BB (d_z), slot1 <- Bz BD (d_y), slot2 <- Bz DB (d_x)
    {
      double2 f[TPW][3];
      double o[TPW][6];
      // in-cell tile index of this warp's j-th tile: (warp + WARPS*j) & 7
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        const double* y = sY + c * YC + yaddr(((warp + WARPS * j) & 7), gq, 2 * kq);
#pragma unroll
        for (int s = 0; s < 3; ++s) f[j][s] = *reinterpret_cast<const double2*>(y + s * YA);
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        o[j][0] = o[j][1] = o[j][2] = o[j][3] = o[j][4] = o[j][5] = 0.0;
        dmma_acc(o[j][0], o[j][1], f[j][0].x, zdf[0]);
        dmma_acc(o[j][2], o[j][3], f[j][1].x, zbf[0]);
        dmma_acc(o[j][4], o[j][5], f[j][2].x, zbf[0]);
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        dmma_acc(o[j][0], o[j][1], f[j][0].y, zdf[1]);
        dmma_acc(o[j][2], o[j][3], f[j][1].y, zbf[1]);
        dmma_acc(o[j][4], o[j][5], f[j][2].y, zbf[1]);
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        double* y = sY + c * YC + yaddr(((warp + WARPS * j) & 7), gq, 2 * kq);
#pragma unroll
        for (int s = 0; s < 3; ++s)
          *reinterpret_cast<double2*>(y + s * YA) = make_double2(o[j][2 * s], o[j][2 * s + 1]);
      }
    }
    __syncthreads();

    // ---- pointwise: thread per z-line (c, qx, qy), two points per step ------
    {
      const int c = tid >> 6, r = tid & 63;
      const int qx = r & 7, qy = r >> 3;
      double* yl = sY + c * YC;
      TC8Geo geo;
      geo.setup(sC + c * 24, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
      const double wxy = T.W[qx] * T.W[qy];
#pragma unroll 1
      for (int q = 0; q < M; q += 2) {
        double* p = yl + yaddr(qx, qy, q);
        double2 gz = *reinterpret_cast<double2*>(p);
        double2 gy = *reinterpret_cast<double2*>(p + YA);
        double2 gx = *reinterpret_cast<double2*>(p + 2 * YA);
        {
          double r0[3], r1[3], r2[3];
          const double det = tc8_adj(geo, T, q, r0, r1, r2);
          const double s = (wxy * T.W[q]) * rcp64(fabs(det));
          laplace_flux(r0, r1, r2, s, gx.x, gy.x, gz.x);
        }
        {
          double r0[3], r1[3], r2[3];
          const double det = tc8_adj(geo, T, q + 1, r0, r1, r2);
          const double s = (wxy * T.W[q + 1]) * rcp64(fabs(det));
          laplace_flux(r0, r1, r2, s, gx.y, gy.y, gz.y);
        }
        *reinterpret_cast<double2*>(p) = gz;
        *reinterpret_cast<double2*>(p + YA) = gy;
        *reinterpret_cast<double2*>(p + 2 * YA) = gx;
      }
    }
    __syncthreads();

    // ---- z backward (D'-form, in place): slot0 <- Dz^T fz, 1 <- Bz^T fy,
    //      2 <- Bz^T fx --------------------------------------------------------
    {
      double2 f[TPW][3];
      double o[TPW][6];
      // in-cell tile index of this warp's j-th tile: (warp + WARPS*j) & 7
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        const double* y = sY + c * YC + yaddr(((warp + WARPS * j) & 7), gq, 2 * kq);
#pragma unroll
        for (int s = 0; s < 3; ++s) f[j][s] = *reinterpret_cast<const double2*>(y + s * YA);
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        o[j][0] = o[j][1] = o[j][2] = o[j][3] = o[j][4] = o[j][5] = 0.0;
        dmma_acc(o[j][0], o[j][1], f[j][0].x, zdb[0]);
        dmma_acc(o[j][2], o[j][3], f[j][1].x, zbb[0]);
        dmma_acc(o[j][4], o[j][5], f[j][2].x, zbb[0]);
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        dmma_acc(o[j][0], o[j][1], f[j][0].y, zdb[1]);
        dmma_acc(o[j][2], o[j][3], f[j][1].y, zbb[1]);
        dmma_acc(o[j][4], o[j][5], f[j][2].y, zbb[1]);
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        double* y = sY + c * YC + yaddr(((warp + WARPS * j) & 7), gq, 2 * kq);
#pragma unroll
        for (int s = 0; s < 3; ++s)
          *reinterpret_cast<double2*>(y + s * YA) = make_double2(o[j][2 * s], o[j][2 * s + 1]);
      }
    }
    __syncthreads();

    // ---- y backward (D-form): tile (c, qx), lines iz;
    //      R1 = By^T Sx, R2 = Dy^T Sy + By^T Sz ---------------------------------
    {
      double f[TPW][6], o[TPW][4];
      // in-cell tile index of this warp's j-th tile: (warp + WARPS*j) & 7
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        const double* y = sY + c * YC;
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          f[j][2 * s] = y[s * YA + yaddr(((warp + WARPS * j) & 7), kq, gq)];
          f[j][2 * s + 1] = y[s * YA + yaddr(((warp + WARPS * j) & 7), 4 + kq, gq)];
        }
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          if (ks == 0) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.0;
          dmma_acc(o[j][0], o[j][1], bb[ks], f[j][4 + ks]);   // By^T Sx
          dmma_acc(o[j][2], o[j][3], db[ks], f[j][2 + ks]);   // Dy^T Sy
          dmma_acc(o[j][2], o[j][3], bb[ks], f[j][ks]);       // By^T Sz
        }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        double* out = sX + c * XC + xaddr(((warp + WARPS * j) & 7), gq, 2 * kq);
        *reinterpret_cast<double2*>(out) = make_double2(o[j][0], o[j][1]);
        *reinterpret_cast<double2*>(out + XA) = make_double2(o[j][2], o[j][3]);
      }
    }
    __syncthreads();

    // ---- x backward (D-form): tile (c, iy), lines iz; A = Dx^T R1 + Bx^T R2 -
    {
      double f[TPW][4], o[TPW][2];
      // in-cell tile index of this warp's j-th tile: (warp + WARPS*j) & 7
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        const double* x = sX + c * XC;
        f[j][0] = x[xaddr(kq, ((warp + WARPS * j) & 7), gq)];
        f[j][1] = x[xaddr(4 + kq, ((warp + WARPS * j) & 7), gq)];
        f[j][2] = x[XA + xaddr(kq, ((warp + WARPS * j) & 7), gq)];
        f[j][3] = x[XA + xaddr(4 + kq, ((warp + WARPS * j) & 7), gq)];
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          if (ks == 0) o[j][0] = o[j][1] = 0.0;
          dmma_acc(o[j][0], o[j][1], db[ks], f[j][ks]);
          dmma_acc(o[j][0], o[j][1], bb[ks], f[j][2 + ks]);
        }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int c = (warp + WARPS * j) >> 3;
        if (GS && c < ncb) {
          const int* mp = smap + c * N3 + gq * NN + ((warp + WARPS * j) & 7) * 8 + 2 * kq;
          atomicAdd(A + mp[0], o[j][0]);
          atomicAdd(A + mp[1], o[j][1]);
        } else if (c < ncb) {
          // D: ix = gq, iz = 2kq + h -> A[cell][ix*64 + iy*8 + iz]
          double* ap = A + (cell0 + c) * N3 + gq * NN + ((warp + WARPS * j) & 7) * 8 + 2 * kq;
          if ((reinterpret_cast<uintptr_t>(ap) & 15) == 0) {
            *reinterpret_cast<double2*>(ap) = make_double2(o[j][0], o[j][1]);
          } else {
            ap[0] = o[j][0];
            ap[1] = o[j][1];
          }
        }
      }
    }
    __syncthreads();
  }
}

template <bool GS>
static int launch_tc8(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                      const double* w0, cudaStream_t s, const int* cmap) {
  if (p->n != 8 || p->m != 8) return SFK_EUNSUPPORTED;
  using namespace tc8;
  auto kern = hex_laplace_action_tc8<GS>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, THREADS, SMEM, "hex_action_tc8", &sh, true))
    return rc_;
  const Tabs<8, 8> T = make_tabs<8, 8>(p);
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, THREADS, SMEM, s>>>(T, ncells, coords, w0, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_tc8 launch");
}

int launch_hex_action_tc(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s) {
  return launch_tc8<false>(p, ncells, A, coords, w0, s, nullptr);
}

int launch_hex_action_tc_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s) {
  return launch_tc8<true>(p, ncells, y, coords, x, s, cmap);
}

}  // namespace sfk
