// Hex Q_8 Laplace action on the FP64 tensor cores — BASELINE C2 at p = 8
// (n = m = 9): the collocation-derivative schedule of v6 / tc8c with every
// 9 x 9 line contraction split into an 8 x 8 DMMA core and DFMA edges.
//
// Operator, reference mapping, stages A..I and the one-warp-per-cell form of
// tc8c (hex_action_tc8c.cu; forms.py:186-189, 235-243; passes.py:672-743).
// A 1D contraction out = T in over a tile of 8 lines (9 inputs, 9 outputs):
//   out[0..7] = T[0..7][0..7] in[0..7]   two m8n8k4 DMMA (k = 0..3, 4..7)
//             + T[8][0..7] in[8]         rank-1 edge: 2 DFMA per lane
//   out[8]    = T[0..7][8] in[0..7] + T[8][8] in[8]
//                                        partial dot of the lane's own MMA
//                                        operands, summed over the 4 lanes of
//                                        a row by 2 xor-shuffles
// so 64 of a line's 81 FMAs run on the tensor pipe.  The 81 lines of a stage
// are 10 tiles of 8 plus line 80, run as an 11th tile whose 8 columns all
// read line 80 (one result stored).  D-form (contraction along x or y; the
// 8 lines are the MMA n index) and D'-form (along z; lines = MMA m index, so
// V = Q B_z feeds gz = V C_z in registers, and t = (tx + ty) + fz C_z^T
// feeds R = t B_z^T, as in tc8c).  Stage E (geometry + flux) runs 3 z-lines
// per lane.  Per-cell shared arrays (one warp per cell, __syncwarp only):
//   u, P, S   [x][81]       (dof / line order)
//   Q, V, GX, GY, GZ, R   [(x, y)][10]   (z rows of 10: 16-byte pairs)
#include "async_copy.cuh"
#include "hex_geometry.cuh"

namespace sfk {

__device__ __forceinline__ void dmma9(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double quad_sum(double s) {   // over the 4 lanes of an MMA row
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  return s;
}

struct TabsTC9C {
  double B[81];   // B[i*9 + q]
  double C[81];   // C[q'*9 + q]
  double W[9];
  double Bc[18];
};

// Per-lane constant fragments of one table T[i][q] (lane = 4 gq + kq).
struct Frag9 {
  double df[2], d8q, dk8[2];     // D-form fwd:  out[q][l] = sum_k T[k][q] in[k][l]
  double db[2], b8q, bk8[2];     // D-form bwd:  out[i][l] = sum_q T[i][q] in[q][l]
  double zf[2], zr8[2], zc8[2];  // D'-form fwd: out[l][q] = sum_k in[l][k] T[k][q]
  double zb[2], zbr8[2], zbc8[2];// D'-form bwd: out[l][i] = sum_q in[l][q] T[i][q]
  double t88;
  __device__ __forceinline__ void load(const double* T, int gq, int kq) {
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      df[ks] = T[(kq + 4 * ks) * 9 + gq];
      dk8[ks] = T[(kq + 4 * ks) * 9 + 8];
      db[ks] = T[gq * 9 + kq + 4 * ks];
      bk8[ks] = T[8 * 9 + kq + 4 * ks];
      zf[ks] = T[(2 * kq + ks) * 9 + gq];
      zr8[ks] = T[8 * 9 + 2 * kq + ks];
      zc8[ks] = T[(2 * kq + ks) * 9 + 8];
      zb[ks] = T[gq * 9 + 2 * kq + ks];
      zbr8[ks] = T[(2 * kq + ks) * 9 + 8];
      zbc8[ks] = T[8 * 9 + 2 * kq + ks];
    }
    d8q = T[8 * 9 + gq];
    b8q = T[gq * 9 + 8];
    t88 = T[8 * 9 + 8];
  }
};

// D-form tile: b0 / b1 = in[kq][col gq] / in[kq+4][col gq], e0 / e1 = in[8]
// at cols 2kq / 2kq+1, eg = in[8] at col gq.  Out: d0 / d1 = out[gq][cols
// 2kq, 2kq+1], o8 = out[8][col gq] (every lane of the row).
__device__ __forceinline__ void dtile(const double af[2], double a8q, const double ak8[2],
                                      double a88, double b0, double b1, double e0, double e1,
                                      double eg, double& d0, double& d1, double& o8) {
  d0 = a8q * e0;
  d1 = a8q * e1;
  dmma9(d0, d1, af[0], b0);
  dmma9(d0, d1, af[1], b1);
  o8 = fma(a88, eg, quad_sum(fma(ak8[1], b1, ak8[0] * b0)));
}

// D'-form tile: a0 / a1 = in[row gq][2kq, 2kq+1], a8 = in[row gq][8];
// d0 / d1 / o8 carry the accumulator init in and the result out.
__device__ __forceinline__ void ztile(const double bf[2], const double r8[2], const double c8[2],
                                      double c88, double a0, double a1, double a8, double& d0,
                                      double& d1, double& o8) {
  d0 = fma(a8, r8[0], d0);
  d1 = fma(a8, r8[1], d1);
  dmma9(d0, d1, a0, bf[0]);
  dmma9(d0, d1, a1, bf[1]);
  o8 = fma(c88, a8, o8 + quad_sum(fma(c8[1], a1, c8[0] * a0)));
}

namespace tc9c {
constexpr int NN = 81, N3 = 729;
constexpr int WARPS = 4;                 // cells per CTA (one per warp)
constexpr int THREADS = 32 * WARPS;
constexpr int NT = 11;                   // tiles per stage (10 x 8 lines + line 80)
constexpr int ZS = 10;                   // z-row stride of the [(x, y)][z] arrays
constexpr int SLOT = 810;                // doubles per cell and slot
constexpr int CELL = 4 * SLOT + 48 + 162 + 2;   // slots, coords x2, line-geometry table
constexpr size_t SMEM = (size_t)WARPS * CELL * sizeof(double) + WARPS * sizeof(uint64_t);
__device__ __forceinline__ int line(int t, int j) { return t < 10 ? 8 * t + j : 80; }
}  // namespace tc9c

// D-form stage over the 11 tiles of a cell: IN(k, l) reads, OUT(q, l, v)
// writes; INPLACE: OUT overwrites the array IN reads (a __syncwarp between
// a chunk's loads and its stores; chunks touch disjoint lines).
template <bool INPLACE, class IN, class OUT>
__device__ __forceinline__ void tc9_dstage(const double af[2], double a8q, const double ak8[2],
                                           double a88, int gq, int kq, IN in, OUT out) {
  using namespace tc9c;
#pragma unroll 1
  for (int t0 = 0; t0 < NT; t0 += 4) {
    double b0[4], b1[4], e0[4], e1[4], eg[4], d0[4], d1[4], o8[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = t0 + j < NT ? t0 + j : NT - 1;
      const int lg = line(t, gq);
      b0[j] = in(kq, lg);
      b1[j] = in(kq + 4, lg);
      e0[j] = in(8, line(t, 2 * kq));
      e1[j] = in(8, line(t, 2 * kq + 1));
      eg[j] = in(8, lg);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      dtile(af, a8q, ak8, a88, b0[j], b1[j], e0[j], e1[j], eg[j], d0[j], d1[j], o8[j]);
    if (INPLACE) __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = t0 + j;
      if (t >= NT) break;
      if (t < 10) {
        out(gq, 8 * t + 2 * kq, d0[j]);
        out(gq, 8 * t + 2 * kq + 1, d1[j]);
        if (kq == 0) out(8, 8 * t + gq, o8[j]);
      } else if (kq == 0) {   // tile 10: every column is line 80; column 0 stored
        out(gq, 80, d0[j]);
        if (gq == 0) out(8, 80, o8[j]);
      }
    }
    if (INPLACE) __syncwarp();
  }
}

template <int MINB>
__global__ void __launch_bounds__(tc9c::THREADS, MINB)
hex_laplace_action_tc9c(const __grid_constant__ TabsTC9C T, int64_t ncells,
                        const double* __restrict__ coords, const double* __restrict__ u,
                        double* __restrict__ A) {
  using namespace tc9c;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kq = lane & 3, gq = lane >> 2;
  double* base = smem + warp * CELL;
  double* S1 = base;                     // P, V, R
  double* S2 = S1 + SLOT;                // Q, GX, S
  double* S3 = S2 + SLOT;                // GY
  double* S4 = S3 + SLOT;                // GZ; u from stage G to the next stage A
  double* sCo = S4 + SLOT;               // [2][24]
  double* sLG = sCo + 48;                // [162]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + WARPS * CELL) + warp;
  const int64_t nbatch = (ncells + WARPS - 1) / WARPS;
  const bool cal = (reinterpret_cast<uintptr_t>(coords) & 15) == 0;

  Frag9 FB, FC;
  FB.load(T.B, gq, kq);
  FC.load(T.C, gq, kq);
  const double b88 = FB.t88, c88 = FC.t88;

  auto prefetch = [&](int64_t bt, int buf) {
    const int64_t cg = bt * WARPS + warp;
    if (lane == 0) {
      unsigned bytes = 0;
      if (cg < ncells) {
        fence_proxy_async_smem();
        bytes = bulk_copy_phase(S4, u + cg * N3, N3, bar);
        if (cal) {
          bulk_g2s(sCo + buf * 24, coords + cg * 24, 192u, bar);
          bytes += 192u;
        }
      }
      mbar_arrive_expect_tx(bar, bytes);
    }
    if (!cal && cg < ncells && lane < 24) cp_async8(sCo + buf * 24 + lane, coords + cg * 24 + lane);
    cp_async_commit();
  };

  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  int64_t b = blockIdx.x;
  if (b < nbatch) prefetch(b, 0);
  for (int k = 0; b < nbatch; b += gridDim.x, ++k) {
    const int cur = k & 1;
    const int64_t cell = b * WARPS + warp;
    cp_async_wait<0>();
    mbar_wait(bar, (unsigned)(k & 1));
    __syncwarp();
    const double* su = S4 + dst_shift(u + cell * N3);
    const double* X = sCo + cur * 24;

    // ---- A: x (D-form fwd, B): P[q][l] = sum_k B[k][q] u[k][l], l = (y, z)
    tc9_dstage<false>(FB.df, FB.d8q, FB.dk8, b88, gq, kq,
                      [&](int kk, int l) { return su[kk * NN + l]; },
                      [&](int q, int l, double v) { S1[q * NN + l] = v; });
    for (int e = lane; e < 162; e += 32) sLG[e] = hex_cell_lg(X, T.Bc, 9, e);
    __syncwarp();

    // ---- B: y (D-form fwd, B): lines (x, z): Q[(x, q)][z] ---------------------
    tc9_dstage<false>(FB.df, FB.d8q, FB.dk8, b88, gq, kq,
                      [&](int kk, int l) {
                        const int x = l / 9, z = l - 9 * x;
                        return S1[x * NN + kk * 9 + z];
                      },
                      [&](int q, int l, double v) {
                        const int x = l / 9, z = l - 9 * x;
                        S2[(x * 9 + q) * ZS + z] = v;
                      });
    __syncwarp();

    // ---- C: z (D'-form): rows (x, y): V = Q B_z -> S1, gz = V C_z -> S4 -----
#pragma unroll 1
    for (int t = 0; t < NT; ++t) {
      const int l = line(t, gq);
      const double2 a = *reinterpret_cast<const double2*>(S2 + l * ZS + 2 * kq);
      const double a8 = S2[l * ZS + 8];
      double v0 = 0.0, v1 = 0.0, v8 = 0.0;
      ztile(FB.zf, FB.zr8, FB.zc8, b88, a.x, a.y, a8, v0, v1, v8);
      double g0 = 0.0, g1 = 0.0, g8 = 0.0;
      ztile(FC.zf, FC.zr8, FC.zc8, c88, v0, v1, v8, g0, g1, g8);
      if (t < 10 || gq == 0) {
        *reinterpret_cast<double2*>(S1 + l * ZS + 2 * kq) = make_double2(v0, v1);
        *reinterpret_cast<double2*>(S4 + l * ZS + 2 * kq) = make_double2(g0, g1);
        if (kq == 0) {
          S1[l * ZS + 8] = v8;
          S4[l * ZS + 8] = g8;
        }
      }
    }
    __syncwarp();

    // ---- D: gx = C_x V (lines (y, z)) -> S2; gy = C_y V (lines (x, z)) -> S3
    tc9_dstage<false>(FC.df, FC.d8q, FC.dk8, c88, gq, kq,
                      [&](int kk, int l) {
                        const int y = l / 9, z = l - 9 * y;
                        return S1[(kk * 9 + y) * ZS + z];
                      },
                      [&](int q, int l, double v) {
                        const int y = l / 9, z = l - 9 * y;
                        S2[(q * 9 + y) * ZS + z] = v;
                      });
    tc9_dstage<false>(FC.df, FC.d8q, FC.dk8, c88, gq, kq,
                      [&](int kk, int l) {
                        const int x = l / 9, z = l - 9 * x;
                        return S1[(x * 9 + kk) * ZS + z];
                      },
                      [&](int q, int l, double v) {
                        const int x = l / 9, z = l - 9 * x;
                        S3[(x * 9 + q) * ZS + z] = v;
                      });
    __syncwarp();

    // ---- E: z-lines (x, y) = divmod(l, 9), l = lane + 32 p: geometry + flux
#pragma unroll 1
    for (int l = lane; l < NN; l += 32) {
      const int qx = l / 9, qy = l - 9 * qx;
      double* gxl = S2 + l * ZS;
      double* gyl = S3 + l * ZS;
      double* gzl = S4 + l * ZS;
      HexLineAdj geo;
      geo.setup_lg(sLG, 9, qx, qy, T.Bc[qx], T.Bc[9 + qx]);
      const double wxy = T.W[qx] * T.W[qy];
#pragma unroll 3
      for (int q = 0; q < 9; ++q) {
        double gx = gxl[q], gy = gyl[q], g2 = gzl[q];
        double r0[3], r1[3], r2[3];
        const double det = geo.adj(T.Bc[9 + q], r0, r1, r2);
        const double s = (wxy * T.W[q]) * rcp64(fabs(det));
        laplace_flux(r0, r1, r2, s, gx, gy, g2);
        gxl[q] = gx;
        gyl[q] = gy;
        gzl[q] = g2;
      }
    }
    __syncwarp();

    // ---- F: tx = C_x^T fx (lines (y, z)), ty = C_y^T fy (lines (x, z)) -----
    tc9_dstage<true>(FC.db, FC.b8q, FC.bk8, c88, gq, kq,
                     [&](int kk, int l) {
                       const int y = l / 9, z = l - 9 * y;
                       return S2[(kk * 9 + y) * ZS + z];
                     },
                     [&](int q, int l, double v) {
                       const int y = l / 9, z = l - 9 * y;
                       S2[(q * 9 + y) * ZS + z] = v;
                     });
    tc9_dstage<true>(FC.db, FC.b8q, FC.bk8, c88, gq, kq,
                     [&](int kk, int l) {
                       const int x = l / 9, z = l - 9 * x;
                       return S3[(x * 9 + kk) * ZS + z];
                     },
                     [&](int q, int l, double v) {
                       const int x = l / 9, z = l - 9 * x;
                       S3[(x * 9 + q) * ZS + z] = v;
                     });
    __syncwarp();

    // ---- G: z (D'-form bwd): t = (tx + ty) + fz C_z^T, R = t B_z^T -> S1 -----
#pragma unroll 1
    for (int t = 0; t < NT; ++t) {
      const int l = line(t, gq);
      const double2 tx = *reinterpret_cast<const double2*>(S2 + l * ZS + 2 * kq);
      const double2 ty = *reinterpret_cast<const double2*>(S3 + l * ZS + 2 * kq);
      const double2 fz = *reinterpret_cast<const double2*>(S4 + l * ZS + 2 * kq);
      const double fz8 = S4[l * ZS + 8];
      double t0 = tx.x + ty.x, t1 = tx.y + ty.y, t8 = S2[l * ZS + 8] + S3[l * ZS + 8];
      ztile(FC.zb, FC.zbr8, FC.zbc8, c88, fz.x, fz.y, fz8, t0, t1, t8);
      double r0 = 0.0, r1 = 0.0, r8 = 0.0;
      ztile(FB.zb, FB.zbr8, FB.zbc8, b88, t0, t1, t8, r0, r1, r8);
      if (t < 10 || gq == 0) {
        *reinterpret_cast<double2*>(S1 + l * ZS + 2 * kq) = make_double2(r0, r1);
        if (kq == 0) S1[l * ZS + 8] = r8;
      }
    }
    __syncwarp();
    // S4 (fz) is dead until the next stage C: stage the next batch's u there
    if (b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- H: y (D-form bwd, B): lines (x, iz): S[x][(iy, iz)] -> S2 ---------
    tc9_dstage<false>(FB.db, FB.b8q, FB.bk8, b88, gq, kq,
                      [&](int kk, int l) {
                        const int x = l / 9, z = l - 9 * x;
                        return S1[(x * 9 + kk) * ZS + z];
                      },
                      [&](int q, int l, double v) {
                        const int x = l / 9, z = l - 9 * x;
                        S2[x * NN + q * 9 + z] = v;
                      });
    __syncwarp();

    // ---- I: x (D-form bwd, B): lines (iy, iz) -> A[cell][ix*81 + l] --------
    if (cell < ncells) {
      double* ap = A + cell * N3;
      tc9_dstage<false>(FB.db, FB.b8q, FB.bk8, b88, gq, kq,
                        [&](int kk, int l) { return S2[kk * NN + l]; },
                        [&](int q, int l, double v) { ap[q * NN + l] = v; });
    }
    __syncwarp();
  }
}

int launch_hex_action_tc9c(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, cudaStream_t s) {
  if (p->n != 9 || p->m != 9 || !p->has_ct) return SFK_EUNSUPPORTED;
  using namespace tc9c;
  auto kern = hex_laplace_action_tc9c<2>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, THREADS, SMEM, "hex_action_tc9c", &sh, true))
    return rc_;
  TabsTC9C T;
  for (int i = 0; i < 81; ++i) {
    T.B[i] = p->B[i];
    T.C[i] = p->Ct[i];
  }
  for (int q = 0; q < 9; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[9 + q] = p->Bc[9 + q];
  }
  const int64_t nbatch = (ncells + WARPS - 1) / WARPS;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, THREADS, SMEM, s>>>(T, ncells, coords, w0, A);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_tc9c launch");
}

}  // namespace sfk
