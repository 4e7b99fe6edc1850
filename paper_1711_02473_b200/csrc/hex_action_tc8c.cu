// Hex Q_7 Laplace action on the FP64 tensor cores with the collocation-
// derivative schedule — BASELINE C2 at p = 7 (n = m = 8).
//
// The operator and reference mapping of every C2 kernel (forms.py:186-189,
// 235-243; passes.py:672-743).  Schedule of v6 (hex_action6.cu: C = B^-1 D,
// 12 n^4 FMA per cell instead of 16 n^4), stages as batched 8x8x8 GEMMs on
// mma.sync.m8n8k4.f64 (SASS DMMA) as in tc8 (hex_action_tc.cu): 192 DMMA
// per cell instead of tc8's 256.  Fragment forms (lane = 4*gq + kq):
//  * D-form (contraction along x or y; the 8 lines of a tile are the MMA n
//    index): table fragment A[q][k] constant per lane, in[k][line] loaded as
//    64-bit at (k = kq + 4ks, line = gq), outputs D[q = gq][line = 2kq, 2kq+1]
//    stored as one 128-bit word;
//  * D'-form (contraction along z; lines = MMA m index): in[line = gq][k =
//    2kq + ks] is one 128-bit load, the output D[line = gq][q = 2kq, 2kq+1]
//    has exactly that layout, so z stages CHAIN in registers: V = Q B_z feeds
//    gz = V C_z without a store, and G forms t = (tx + ty) + fz C_z^T with
//    the (tx + ty) sum as the accumulator input, then R = t B_z^T.
//   A  x   D-form   u  -> P  = B_x u                 sU -> S1
//   B  y   D-form   P  -> Q  = B_y P                 S1 -> S2
//   C  z   D'-form  Q  -> V  = B_z Q -> gz = C_z V   S2 -> S1 (V), S4 (gz)
//   D  x,y D-form   V  -> gx = C_x V, gy = C_y V     S1 -> S2, S3
//   E  z-lines      geometry + flux in place         S2, S3, S4
//   F  x,y D-form   tx = C_x^T fx, ty = C_y^T fy     in place S2, S3
//   G  z   D'-form  t = tx + ty + fz C_z^T -> R = t B_z^T        -> S1
//   H  y   D-form   S = B_y^T R                      S1 -> S2
//   I  x   D-form   A = B_x^T S                      S2 -> HBM
// Shared layouts are strided + XOR-swizzled per array so that every access
// above is bank-conflict free (tools/tc8c_layout.py searched them under the
// half-/quarter-warp bank model).
#include "async_copy.cuh"
#include "hex_geometry.cuh"

namespace sfk {

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
  // not volatile: a pure function of its operands, so the compiler may
  // interleave independent tiles' MMAs with loads
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct TabsTC8C {
  double B[64];   // B[i*8 + q]
  double C[64];   // C[q'*8 + q]
  double W[8];
  double Bc[16];
};

// One warp per cell: the warp runs all 8 tiles of every stage of its cell
// and two z-lines per lane in stage E, so every exchange is a __syncwarp and
// the CTA never synchronises (the first, CTA-wide version — 4 tiles of mixed
// cells per warp, 9 CTA barriers per batch — measured 2.46 ms, barrier and
// shared-load latency bound).
namespace tc8c {
constexpr int N = 8, NN = 64, N3 = 512;
constexpr int WARPS = 4;
constexpr int CPB = WARPS;               // cells per CTA (one per warp)
constexpr int THREADS = 32 * WARPS;
constexpr int TPW = 8;                   // tiles per warp and stage
constexpr int SLOT = 576;                // doubles per cell and slot (largest layout)
constexpr int UC = 8 * 68;               // u per cell, ix-plane stride 68
constexpr int CSZ = CPB * 24;
// AU: u staged in slot S4 (gz / fz, dead from G to the next C) instead of
// its own buffer — the next batch's u is then fetched after stage G.
constexpr size_t smem_bytes(bool au) {
  return (size_t)(4 * CPB * SLOT + (au ? 0 : CPB * UC) + 2 * CSZ) * sizeof(double);
}

__device__ __forceinline__ int b1(int v) { return ((v >> 1) & 1) << 2; }
// element (a, b, c) = (x, y, z) of one cell's array (tools/tc8c_layout.py)
__device__ __forceinline__ int aP(int a, int b, int c) { return a * 72 + b * 8 + (c ^ b1(b)); }
__device__ __forceinline__ int aQR(int a, int b, int c) { return a * 64 + b * 8 + (c ^ b1(b)); }
__device__ __forceinline__ int aV(int a, int b, int c) { return a * 68 + b * 8 + (c ^ b1(b)); }
__device__ __forceinline__ int aGX(int a, int b, int c) {
  return a * 72 + b * 8 + (c ^ ((((a >> 2) & 1) << 1) | b1(a)));
}
__device__ __forceinline__ int aGY(int a, int b, int c) { return a * 66 + b * 8 + (c ^ b1(b)); }
__device__ __forceinline__ int aGZ(int a, int b, int c) { return a * 66 + b * 8 + c; }
__device__ __forceinline__ int aS(int a, int b, int c) { return a * 68 + b * 8 + c; }
__device__ __forceinline__ int aU(int a, int b, int c) { return a * 68 + b * 8 + c; }
}  // namespace tc8c

// GS: global operator y += sum_c P_c^T A_c P_c x: the cell's dof map
// (int32) is double-buffered in the u staging area (so not with AU), x is
// gathered through it in stage A and y scatter-added in stage I.
// COL: the GLL-collocated (weighted) Laplace action of BASELINE C3 at p = 7
// (hex_colloc.cu's operator: B = I, T.C holds the derivative table D, kappa =
// w1 at the points or nullptr): stages A, B and the B_z halves of C and G drop
// out — C reads u, G's t is the result — and stage E multiplies by kappa.
template <int MINB, bool AU, bool GS = false, bool COL = false>
__global__ void __launch_bounds__(tc8c::THREADS, MINB)
hex_laplace_action_tc8c(const __grid_constant__ TabsTC8C T, int64_t ncells,
                        const double* __restrict__ coords, const double* __restrict__ u,
                        double* __restrict__ A, const int* __restrict__ cmap = nullptr,
                        const double* __restrict__ kappa = nullptr) {
  static_assert(!(GS && AU), "GS keeps the map through stage I: own staging area");
  static_assert(!COL || (!GS && !AU), "COL: E-vector form with its own u staging area");
  using namespace tc8c;
  extern __shared__ __align__(16) double smem[];
  double* S1 = smem;
  double* S2 = S1 + CPB * SLOT;
  double* S3 = S2 + CPB * SLOT;
  double* S4 = S3 + CPB * SLOT;
  static_assert(UC <= SLOT, "u fits a slot");
  double* sU = AU ? S4 : S4 + CPB * SLOT;              // u of cell c at sU + c * (AU ? SLOT : UC)
  double* sCo = S4 + CPB * SLOT + (AU ? 0 : CPB * UC);
  constexpr int US = AU ? SLOT : UC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, gq = lane >> 2;
  const int64_t nbatch = (ncells + CPB - 1) / CPB;

  // table fragments (constant per lane)
  //  D-form fwd A[m=q][k=i] = T[i][q]: *f;  D-form bwd A[m=i][k=q] = T[i][q]: *b
  //  D'-form fwd B[k=i][n=q] = T[i][q] (k = 2kq+ks): z*f; bwd B[k=q][n=i] = T[i][q]: z*b
  double bf[2], bb[2], cf[2], cb[2], zbf[2], zbb[2], zcf[2], zcb[2];
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    bf[ks] = T.B[(4 * ks + kq) * N + gq];
    bb[ks] = T.B[gq * N + 4 * ks + kq];
    cf[ks] = T.C[(4 * ks + kq) * N + gq];
    cb[ks] = T.C[gq * N + 4 * ks + kq];
    zbf[ks] = T.B[(2 * kq + ks) * N + gq];
    zbb[ks] = T.B[gq * N + 2 * kq + ks];
    zcf[ks] = T.C[(2 * kq + ks) * N + gq];
    zcb[ks] = T.C[gq * N + 2 * kq + ks];
  }

  // each warp stages its own cell: u (ix-planes at stride 68) and coords
  auto prefetch = [&](int64_t bt, int buf) {
    const int64_t cg = bt * CPB + warp;
    if (GS && cg < ncells) {
      int* m = reinterpret_cast<int*>(sU + warp * US) + buf * N3;
#pragma unroll
      for (int k = 0; k < N3 / 32; ++k) cp_async4(m + lane + 32 * k, cmap + cg * N3 + lane + 32 * k);
      if (lane < 24) cp_async8(sCo + buf * CSZ + warp * 24 + lane, coords + cg * 24 + lane);
    } else if (cg < ncells) {
      const double* src = u + cg * N3;
      double* du = sU + warp * US;
      if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int r = lane + 32 * k;   // 16-byte chunk of the cell
          cp_async16(du + (r >> 5) * 68 + 2 * (r & 31), src + 2 * r);
        }
      } else {
        for (int e = lane; e < N3; e += 32) cp_async8(du + (e >> 6) * 68 + (e & 63), src + e);
      }
      if (lane < 24) cp_async8(sCo + buf * CSZ + warp * 24 + lane, coords + cg * 24 + lane);
    }
    cp_async_commit();
  };

  int64_t b = blockIdx.x;
  if (b < nbatch) prefetch(b, 0);
  for (int it = 0; b < nbatch; b += gridDim.x, ++it) {
    const int cur = it & 1;
    const int64_t cell0 = b * CPB;
    const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
    cp_async_wait<0>();
    __syncwarp();
    const int c = warp;
    const int* smap = reinterpret_cast<const int*>(sU + warp * US) + cur * N3;   // GS

    // ---- A: x, D-form; tile (c, iy), lines iz: P = B_x u ------------------
    if (!COL) {
      double f[TPW][2], o[TPW][2];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, iy = t & 7;
        const double* in = sU + c * US;
        if (GS) {   // dof (ix, iy, iz) = ix*64 + iy*8 + iz, gathered through the map
          f[j][0] = c < ncb ? __ldg(u + smap[kq * NN + iy * 8 + gq]) : 0.0;
          f[j][1] = c < ncb ? __ldg(u + smap[(4 + kq) * NN + iy * 8 + gq]) : 0.0;
        } else {
          f[j][0] = in[aU(kq, iy, gq)];
          f[j][1] = in[aU(4 + kq, iy, gq)];
        }
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        o[j][0] = o[j][1] = 0.0;
        dmma8(o[j][0], o[j][1], bf[0], f[j][0]);
        dmma8(o[j][0], o[j][1], bf[1], f[j][1]);
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, iy = t & 7;
        *reinterpret_cast<double2*>(S1 + c * SLOT + aP(gq, iy, 2 * kq)) = make_double2(o[j][0], o[j][1]);
      }
    }
    __syncwarp();
    if (!COL && !AU && b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- B: y, D-form; tile (c, qx), lines iz: Q = B_y P -------------------
    if (!COL) {
      double f[TPW][2], o[TPW][2];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, qx = t & 7;
        const double* p = S1 + c * SLOT;
        f[j][0] = p[aP(qx, kq, gq)];
        f[j][1] = p[aP(qx, 4 + kq, gq)];
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        o[j][0] = o[j][1] = 0.0;
        dmma8(o[j][0], o[j][1], bf[0], f[j][0]);
        dmma8(o[j][0], o[j][1], bf[1], f[j][1]);
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, qx = t & 7;
        *reinterpret_cast<double2*>(S2 + c * SLOT + aQR(qx, gq, 2 * kq)) = make_double2(o[j][0], o[j][1]);
      }
    }
    __syncwarp();

    // ---- C: z, D'-form; tile (c, qx), lines qy: V = Q B_z, gz = V C_z -----
    {
      double2 f[TPW];
      double v[TPW][2], g[TPW][2];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, qx = t & 7;
        f[j] = COL ? *reinterpret_cast<const double2*>(sU + c * US + aU(qx, gq, 2 * kq))
                   : *reinterpret_cast<const double2*>(S2 + c * SLOT + aQR(qx, gq, 2 * kq));
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        if (COL) {   // collocated: V = u
          v[j][0] = f[j].x;
          v[j][1] = f[j].y;
        } else {
          v[j][0] = v[j][1] = 0.0;
          dmma8(v[j][0], v[j][1], f[j].x, zbf[0]);
          dmma8(v[j][0], v[j][1], f[j].y, zbf[1]);
        }
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        g[j][0] = g[j][1] = 0.0;
        dmma8(g[j][0], g[j][1], v[j][0], zcf[0]);
        dmma8(g[j][0], g[j][1], v[j][1], zcf[1]);
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, qx = t & 7;
        *reinterpret_cast<double2*>(S1 + c * SLOT + aV(qx, gq, 2 * kq)) = make_double2(v[j][0], v[j][1]);
        *reinterpret_cast<double2*>(S4 + c * SLOT + aGZ(qx, gq, 2 * kq)) = make_double2(g[j][0], g[j][1]);
      }
    }
    __syncwarp();
    if (COL && b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);   // sU was read by C

    // ---- D: gx = C_x V (tile (c, qy), lines qz), gy = C_y V (tile (c, qx)) -
    //      both tile sets' loads first, then their MMAs (2 TPW chains)
    {
      double f[2][TPW][2], o[2][TPW][2];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, tt = t & 7;
        const double* v = S1 + c * SLOT;
        f[0][j][0] = v[aV(kq, tt, gq)];
        f[0][j][1] = v[aV(4 + kq, tt, gq)];
        f[1][j][0] = v[aV(tt, kq, gq)];
        f[1][j][1] = v[aV(tt, 4 + kq, gq)];
      }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          o[s2][j][0] = o[s2][j][1] = 0.0;
          dmma8(o[s2][j][0], o[s2][j][1], cf[0], f[s2][j][0]);
        }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int j = 0; j < TPW; ++j) dmma8(o[s2][j][0], o[s2][j][1], cf[1], f[s2][j][1]);
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, tt = t & 7;
        *reinterpret_cast<double2*>(S2 + c * SLOT + aGX(gq, tt, 2 * kq)) = make_double2(o[0][j][0], o[0][j][1]);
        *reinterpret_cast<double2*>(S3 + c * SLOT + aGY(tt, gq, 2 * kq)) = make_double2(o[1][j][0], o[1][j][1]);
      }
    }
    __syncwarp();

    // ---- E: z-lines (qx, qy) = (r & 7, r >> 3), r = lane and lane + 32:
    //      geometry + flux, two points per step ----------------------------
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      const int qx = r & 7, qy = r >> 3;
      double* gxc = S2 + c * SLOT;
      double* gyc = S3 + c * SLOT;
      double* gzc = S4 + c * SLOT;
      HexLineGeom geo;
      geo.setup(sCo + cur * CSZ + c * 24, T.Bc[qx], T.Bc[N + qx], T.Bc[qy], T.Bc[N + qy]);
      const double wxy = T.W[qx] * T.W[qy];
      const bool wk = COL && kappa != nullptr && c < ncb;
      const double* kp = kappa + (cell0 + (c < ncb ? c : 0)) * N3 + qx * NN + qy * N;
#pragma unroll 1
      for (int q = 0; q < N; q += 2) {
        const double2 kk = wk ? __ldg(reinterpret_cast<const double2*>(kp + q))
                              : make_double2(1.0, 1.0);
        double2* px = reinterpret_cast<double2*>(gxc + aGX(qx, qy, q));
        double2* py = reinterpret_cast<double2*>(gyc + aGY(qx, qy, q));
        double2* pz = reinterpret_cast<double2*>(gzc + aGZ(qx, qy, q));
        double2 gx = *px, gy = *py, gz = *pz;
        {
          double r0[3], r1[3], r2[3];
          const double det = geo.adj(T.Bc[q], T.Bc[N + q], r0, r1, r2);
          double s = (wxy * T.W[q]) * rcp64(fabs(det));
          if (COL) s *= kk.x;
          laplace_flux(r0, r1, r2, s, gx.x, gy.x, gz.x);
        }
        {
          double r0[3], r1[3], r2[3];
          const double det = geo.adj(T.Bc[q + 1], T.Bc[N + q + 1], r0, r1, r2);
          double s = (wxy * T.W[q + 1]) * rcp64(fabs(det));
          if (COL) s *= kk.y;
          laplace_flux(r0, r1, r2, s, gx.y, gy.y, gz.y);
        }
        *px = gx;
        *py = gy;
        *pz = gz;
      }
    }
    __syncwarp();

    // ---- F: tx = C_x^T fx (tile (c, qy)), ty = C_y^T fy (tile (c, qx)), in
    //      place: every warp loads its tiles of both sets, then stores them ---
    {
      double f[2][TPW][2], o[2][TPW][2];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, tt = t & 7;
        const double* gx = S2 + c * SLOT;
        const double* gy = S3 + c * SLOT;
        f[0][j][0] = gx[aGX(kq, tt, gq)];
        f[0][j][1] = gx[aGX(4 + kq, tt, gq)];
        f[1][j][0] = gy[aGY(tt, kq, gq)];
        f[1][j][1] = gy[aGY(tt, 4 + kq, gq)];
      }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          o[s2][j][0] = o[s2][j][1] = 0.0;
          dmma8(o[s2][j][0], o[s2][j][1], cb[0], f[s2][j][0]);
        }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int j = 0; j < TPW; ++j) dmma8(o[s2][j][0], o[s2][j][1], cb[1], f[s2][j][1]);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, tt = t & 7;
        *reinterpret_cast<double2*>(S2 + c * SLOT + aGX(gq, tt, 2 * kq)) = make_double2(o[0][j][0], o[0][j][1]);
        *reinterpret_cast<double2*>(S3 + c * SLOT + aGY(tt, gq, 2 * kq)) = make_double2(o[1][j][0], o[1][j][1]);
      }
    }
    __syncwarp();

    // ---- G: z, D'-form; tile (c, qx), lines qy:
    //      t = (tx + ty) + fz C_z^T, R = t B_z^T ------------------------------
    {
      double2 fz[TPW];
      double tt[TPW][2], rr[TPW][2];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, qx = t & 7;
        const double2 tx = *reinterpret_cast<const double2*>(S2 + c * SLOT + aGX(qx, gq, 2 * kq));
        const double2 ty = *reinterpret_cast<const double2*>(S3 + c * SLOT + aGY(qx, gq, 2 * kq));
        fz[j] = *reinterpret_cast<const double2*>(S4 + c * SLOT + aGZ(qx, gq, 2 * kq));
        tt[j][0] = tx.x + ty.x;
        tt[j][1] = tx.y + ty.y;
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        dmma8(tt[j][0], tt[j][1], fz[j].x, zcb[0]);
        dmma8(tt[j][0], tt[j][1], fz[j].y, zcb[1]);
      }
      if (COL) {
        // collocated: t is the result; lane (gq, kq) of tile qx holds
        // A[qx][gq][2kq, 2kq + 1] — a tile is 64 consecutive doubles
        if (c < ncb) {
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            double* ap = A + (cell0 + c) * N3 + (j & 7) * NN + gq * 8 + 2 * kq;
            if ((reinterpret_cast<uintptr_t>(ap) & 15) == 0) {
              *reinterpret_cast<double2*>(ap) = make_double2(tt[j][0], tt[j][1]);
            } else {
              ap[0] = tt[j][0];
              ap[1] = tt[j][1];
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          rr[j][0] = rr[j][1] = 0.0;
          dmma8(rr[j][0], rr[j][1], tt[j][0], zbb[0]);
          dmma8(rr[j][0], rr[j][1], tt[j][1], zbb[1]);
        }
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          const int t = j, qx = t & 7;
          *reinterpret_cast<double2*>(S1 + c * SLOT + aQR(qx, gq, 2 * kq)) = make_double2(rr[j][0], rr[j][1]);
        }
      }
    }
    __syncwarp();
    if (COL) continue;   // (the prefetch of the next batch was issued after stage C)

    if (AU && b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);   // S4 is free now

    // ---- H: y, D-form bwd; tile (c, qx), lines iz: S = B_y^T R -------------
    {
      double f[TPW][2], o[TPW][2];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, qx = t & 7;
        const double* rp = S1 + c * SLOT;
        f[j][0] = rp[aQR(qx, kq, gq)];
        f[j][1] = rp[aQR(qx, 4 + kq, gq)];
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        o[j][0] = o[j][1] = 0.0;
        dmma8(o[j][0], o[j][1], bb[0], f[j][0]);
        dmma8(o[j][0], o[j][1], bb[1], f[j][1]);
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, qx = t & 7;
        *reinterpret_cast<double2*>(S2 + c * SLOT + aS(qx, gq, 2 * kq)) = make_double2(o[j][0], o[j][1]);
      }
    }
    __syncwarp();

    // ---- I: x, D-form bwd; tile (c, iy), lines iz: A = B_x^T S -------------
    {
      double f[TPW][2], o[TPW][2];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, iy = t & 7;
        const double* sp = S2 + c * SLOT;
        f[j][0] = sp[aS(kq, iy, gq)];
        f[j][1] = sp[aS(4 + kq, iy, gq)];
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        o[j][0] = o[j][1] = 0.0;
        dmma8(o[j][0], o[j][1], bb[0], f[j][0]);
        dmma8(o[j][0], o[j][1], bb[1], f[j][1]);
      }
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int t = j, iy = t & 7;
        if (GS && c < ncb) {
          atomicAdd(A + smap[gq * NN + iy * 8 + 2 * kq], o[j][0]);
          atomicAdd(A + smap[gq * NN + iy * 8 + 2 * kq + 1], o[j][1]);
        } else if (c < ncb) {   // (warp-uniform)
          // D: ix = gq, iz = 2kq + h -> A[cell][ix*64 + iy*8 + iz]
          double* ap = A + (cell0 + c) * N3 + gq * NN + iy * 8 + 2 * kq;
          if ((reinterpret_cast<uintptr_t>(ap) & 15) == 0) {
            *reinterpret_cast<double2*>(ap) = make_double2(o[j][0], o[j][1]);
          } else {
            ap[0] = o[j][0];
            ap[1] = o[j][1];
          }
        }
      }
    }
    // the next batch's stage A writes S1 after this warp's own stage I (same
    // warp: program order + the __syncwarp at the top)
  }
}

int launch_hex_action_tc8c(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, cudaStream_t s) {
  if (p->n != 8 || p->m != 8 || !p->has_ct) return SFK_EUNSUPPORTED;
  using namespace tc8c;
  // default: u staged in S4 and 3 CTAs per SM (1.659 -> 1.633 ms,
  // profiles/r02n_cfg*.json); option v6_cfg = 1 / 2 / 4 selects the others
  const int alt = (int)option(OPT_V6_CFG);
  const bool au = alt == 0 || alt == 1;
  const int minb = (alt == 0 || alt == 2) ? 3 : 2;
  auto kern = minb == 3 ? (au ? hex_laplace_action_tc8c<3, true> : hex_laplace_action_tc8c<3, false>)
                        : (au ? hex_laplace_action_tc8c<2, true> : hex_laplace_action_tc8c<2, false>);
  const size_t smem = smem_bytes(au);
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, THREADS, smem, "hex_action_tc8c", &sh, true))
    return rc_;
  TabsTC8C T;
  for (int i = 0; i < 64; ++i) {
    T.B[i] = p->B[i];
    T.C[i] = p->Ct[i];
  }
  for (int q = 0; q < 8; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[8 + q] = p->Bc[8 + q];
  }
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, THREADS, smem, s>>>(T, ncells, coords, w0, A, nullptr, nullptr);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_tc8c launch");
}

// BASELINE C3 at p = 7 (GLL-collocated weighted Laplace, n = m = 8) on the
// same one-warp-per-cell DMMA kernel (COL): 96 DMMA per cell.  w1 = kappa at
// the points (nullptr: the unweighted collocated action).
int launch_hex_colloc_tc8c(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, const double* w1, cudaStream_t s) {
  if (p->n != 8 || p->m != 8) return SFK_EUNSUPPORTED;
  using namespace tc8c;
  auto kern = hex_laplace_action_tc8c<3, false, false, true>;
  const size_t smem = smem_bytes(false);
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, THREADS, smem, "hex_colloc_tc8c", &sh, true))
    return rc_;
  TabsTC8C T;
  for (int i = 0; i < 64; ++i) {
    T.B[i] = p->B[i];   // (identity at the collocation points; unused)
    T.C[i] = p->D[i];   // D[i*8 + q]: derivative of basis i at point q
  }
  for (int q = 0; q < 8; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[8 + q] = p->Bc[8 + q];
  }
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  if (grid > 0) kern<<<grid, THREADS, smem, s>>>(T, ncells, coords, w0, A, nullptr, w1);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_colloc_tc8c launch");
}

// Global operator (fused gather / scatter) at n = 8: the map needs its own
// staging area, so 2 CTAs per SM (non-AU layout).
int launch_hex_action_tc8c_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                              double* y, const double* coords, cudaStream_t s) {
  if (p->n != 8 || p->m != 8 || !p->has_ct) return SFK_EUNSUPPORTED;
  using namespace tc8c;
  auto kern = hex_laplace_action_tc8c<2, false, true>;
  const size_t smem = smem_bytes(false);
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, THREADS, smem, "hex_action_tc8c_gs", &sh, true))
    return rc_;
  TabsTC8C T;
  for (int i = 0; i < 64; ++i) {
    T.B[i] = p->B[i];
    T.C[i] = p->Ct[i];
  }
  for (int q = 0; q < 8; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[8 + q] = p->Bc[8 + q];
  }
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, THREADS, smem, s>>>(T, ncells, coords, x, y, cmap, nullptr);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_tc8c_gs launch");
}

}  // namespace sfk
