// Hex Q_3 local stiffness matrices on the FP64 tensor cores — BASELINE C5
// at p = 3 (n = m = 4).
//
// Same math and reference mapping as hex_matrix.cu (registry `laplace` on
// `hex`, forms.py:186-189; test index outermost A[i*64 + j], forms.py:402-408),
// same K and Z phases.  The two phases that carry the work are recast as
// small GEMMs with a CONSTANT left operand, so they run as DMMA
// (mma.sync.m8n8k4.f64) with the A fragments held in registers for the whole
// kernel:
//   Y stage  Y_g[qx][(iy,jy),(iz,jz)] = sum_{(l,l') in g, qy}
//              P_g[(iy,jy)][(l,l'),qy] * Z_ll'[qx][qy][(iz,jz)],
//            P_g[(iy,jy)][(l,l'),qy] = T^l_y[iy][qy] T^l'_y[jy][qy]
//            (16 x K_g with K_g = 4 |g| in {4, 8, 8, 16}: one k-step per pair);
//   x stage  A[(ix,jx)][r] = sum_{g,qx} W[(ix,jx)][(g,qx)] * Y_g[qx][r],
//            W[(ix,jx)][(g,qx)] = T^g_x,test[ix][qx] T^g_x,trial[jx][qx]
//            (16 x 16 constant, 256 columns r = (iy,iz,jy,jz) per cell).
// At n = 4 every tile dimension is a multiple of the m8n8k4 shape: no
// padding.  The FMA version of this kernel was shared-memory-issue bound in
// its Y stage (profiles/r01al_C5_p4.md: MIO throttle 25%).
#include "hex_geometry.cuh"

namespace sfk {

struct TabsMat4 {
  double B[16], D[16], W[4], Bc[8];
};

namespace m4 {
constexpr int N = 4, M = 4, N2 = 16, N3 = 64, N4 = 256, M3 = 64;
constexpr int THREADS = 256, WARPS = 8;
constexpr int KS = 6 * M3;              // K (6 unique entries) at every point
constexpr int ZR = 20;                  // Z row stride (16 used; = 4 mod 16: conflict-free B loads)
constexpr int ZS = 9 * M * M * ZR;      // Z[pair][qx*M + qy][ZR]
constexpr int YR = 260;                 // Y row stride (256 used; = 4 mod 16)
constexpr int YS = 4 * M * YR;          // Y[(g*M + qx)][YR]
constexpr size_t SMEM = (size_t)(KS + ZS + YS + 24) * sizeof(double);
}  // namespace m4

__device__ __forceinline__ void dmma4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// pairs (l, l') (index 3l + l') of x-pattern group g = (l == 0) * 2 + (l' == 0)
__device__ __forceinline__ int group_pair(int g, int s) {
  // g = 0: (1,1) (1,2) (2,1) (2,2); g = 1: (1,0) (2,0); g = 2: (0,1) (0,2); g = 3: (0,0)
  return g == 0 ? (s == 0 ? 4 : s == 1 ? 5 : s == 2 ? 7 : 8)
       : g == 1 ? (s == 0 ? 3 : 6) : g == 2 ? (s == 0 ? 1 : 2) : 0;
}
__device__ __forceinline__ int group_size(int g) { return g == 0 ? 4 : g == 3 ? 1 : 2; }

__host__ __device__ constexpr int ksym4(int l, int r) {
  return l == r ? l : (l + r == 1 ? 3 : (l + r == 2 ? 4 : 5));
}

// Persistent CTAs, one cell per iteration; the constant A fragments of the
// three DMMA stages are built once per CTA.
// emap != nullptr: CSR mode — A is the CSR values array and every cell entry
// (i, j) is atomically added at values[emap[cell][i * 64 + j]]
// (sfk_csr_entry_map); the dense offset of the entry indexes the map.
__global__ void __launch_bounds__(m4::THREADS, 3)
hex_laplace_matrix_tc4(const __grid_constant__ TabsMat4 T, int64_t ncells,
                       const double* __restrict__ coords, double* __restrict__ A,
                       const int32_t* __restrict__ emap) {
  using namespace m4;
  extern __shared__ __align__(16) double smem[];
  double* sY = smem;                 // [16][YR]   (16-byte aligned rows)
  double* sZ = sY + YS;              // [9][M*M][ZR]
  double* sK = sZ + ZS;              // [6][M3]  (point index (qx*M + qy)*M + qz)
  double* sC = sK + KS;              // [24]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, kq = lane & 3;

  // --- constant A fragments -------------------------------------------------
  // Y stage: warp = (group g, row tile rt); P_g[(iy,jy)][(pair s, qy = kq)]
  const int yg = warp >> 1, yrt = warp & 1, ynp = group_size(yg);
  double pa[4];
  {
    const int row = yrt * 8 + gq, iy = row / N, jy = row % N;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int pr = group_pair(yg, s < ynp ? s : 0), l = pr / 3, lp = pr % 3;
      pa[s] = (l == 1 ? T.D : T.B)[iy * M + kq] * (lp == 1 ? T.D : T.B)[jy * M + kq];
    }
  }
  // x stage: W[(ix,jx)][(g = s, qx = kq)], row tile = warp & 1
  double wa[4];
  {
    const int row = (warp & 1) * 8 + gq, ix = row / N, jx = row % N;
#pragma unroll
    for (int s = 0; s < 4; ++s)
      wa[s] = ((s & 2) ? T.D : T.B)[ix * M + kq] * ((s & 1) ? T.D : T.B)[jx * M + kq];
  }

  // K at every point of `cell` (threads < M3): reads sC, writes sK
  auto k_phase = [&](int64_t cell) {
    if (tid < M3 && cell < ncells) {
      const int qx = tid / (M * M), qy = (tid / M) % M, qz = tid % M;
      HexLineGeom geo;
      geo.setup(sC, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
      double r0[3], r1[3], r2[3];
      const double det = geo.adj(T.Bc[qz], T.Bc[M + qz], r0, r1, r2);
      const double s = ((T.W[qx] * T.W[qy]) * T.W[qz]) * rcp64(fabs(det));
      const double* rows[3] = {r0, r1, r2};
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int m2 = l; m2 < 3; ++m2) {
          const double* a = rows[l];
          const double* b = rows[m2];
          sK[ksym4(l, m2) * M3 + tid] = s * fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
        }
    }
  };

  // Software pipeline, 3 barriers per cell: the next cell's coords load during
  // this cell's Y stage and its K phase runs beside this cell's x stage (they
  // touch disjoint shared arrays).
  int64_t cell = blockIdx.x;
  if (cell < ncells && tid < 24) sC[tid] = __ldg(coords + cell * 24 + tid);
  __syncthreads();
  k_phase(cell);
  __syncthreads();
  for (; cell < ncells; cell += gridDim.x) {
    const int64_t next = cell + gridDim.x;

    // ---- Z stage (DMMA): Z_pair[(iz,jz)][(qx,qy)] = TT_pair (16 x 4) * K (4 x 16)
    //      tiles (pair, rt, ct): 36 over 8 warps
    for (int t = warp; t < 36; t += WARPS) {
      const int pair = t >> 2, rt = (t >> 1) & 1, ct = t & 1;
      const int l = pair / 3, lp = pair % 3;
      const int zz = rt * 8 + gq, iz = zz / N, jz = zz % N;
      const double a = (l == 2 ? T.D : T.B)[iz * M + kq] * (lp == 2 ? T.D : T.B)[jz * M + kq];
      const double b = sK[ksym4(l, lp) * M3 + (ct * 8 + gq) * M + kq];
      double d0 = 0.0, d1 = 0.0;
      dmma4(d0, d1, a, b);
      // D: row zz = rt*8 + gq, cols qxy = ct*8 + 2kq, +1
      const int qxy = ct * 8 + 2 * kq;
      sZ[(pair * M * M + qxy) * ZR + zz] = d0;
      sZ[(pair * M * M + qxy + 1) * ZR + zz] = d1;
    }
    __syncthreads();

    // ---- Y stage (DMMA); the next cell's coords land meanwhile ----------------
    if (next < ncells && tid >= THREADS - 24) sC[tid - (THREADS - 24)] =
        __ldg(coords + next * 24 + (tid - (THREADS - 24)));
#pragma unroll 1
    for (int qx = 0; qx < M; ++qx) {
#pragma unroll
      for (int ct = 0; ct < 2; ++ct) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          if (s < ynp) {
            const int pr = group_pair(yg, s);
            dmma4(d0, d1, pa[s], sZ[(pr * M * M + qx * M + kq) * ZR + ct * 8 + gq]);
          }
        }
        // D: rows (iy, jy) = rt*8 + gq, cols (iz, jz) = ct*8 + 2kq, +1
        const int oiy = (yrt * 8 + gq) / N, ojy = (yrt * 8 + gq) % N;
        const int col = ct * 8 + 2 * kq, iz = col / N, jz = col % N;
        const int r = ((oiy * N + iz) * N + ojy) * N + jz;
        *reinterpret_cast<double2*>(sY + (yg * M + qx) * YR + r) = make_double2(d0, d1);
      }
    }
    __syncthreads();

    // ---- x stage (DMMA): A[(ix,jx)][r] = W (16 x 16) * Y (16 x 256); then the
    //      next cell's K (disjoint arrays) ------------------------------------
    {
      const int rt = warp & 1;
      double* out = A + cell * (int64_t)(N3 * N3);
#pragma unroll 2
      for (int j = 0; j < 8; ++j) {
        const int ct = (warp >> 1) + 4 * j;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int s = 0; s < 4; ++s) dmma4(d0, d1, wa[s], sY[(s * M + kq) * YR + ct * 8 + gq]);
        const int oix = (rt * 8 + gq) / N, ojx = (rt * 8 + gq) % N;
        const int r = ct * 8 + 2 * kq;
        const int iy = r / (N * N2), iz = (r / N2) % N, jy = (r / N) % N, jz = r % N;
        const int64_t off = (int64_t)(oix * N2 + iy * N + iz) * N3 + ojx * N2 + jy * N + jz;
        if (emap) {
          const int32_t* mp = emap + cell * (int64_t)(N3 * N3) + off;
          atomicAdd(A + __ldg(mp), d0);
          atomicAdd(A + __ldg(mp + 1), d1);
        } else {
          *reinterpret_cast<double2*>(out + off) = make_double2(d0, d1);
        }
      }
    }
    k_phase(next);
    __syncthreads();
  }
}

int launch_hex_matrix_tc4(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          cudaStream_t s, const int32_t* emap) {
  if (p->n != 4 || p->m != 4 || p->collocated) return SFK_EUNSUPPORTED;
  if (!emap && (reinterpret_cast<uintptr_t>(A) & 15) != 0) return SFK_EUNSUPPORTED;   // double2 stores
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)hex_laplace_matrix_tc4, m4::THREADS, m4::SMEM, "hex_matrix_tc4", &sh))
    return rc_;
  TabsMat4 T;
  for (int i = 0; i < 16; ++i) {
    T.B[i] = p->B[i];
    T.D[i] = p->D[i];
  }
  for (int q = 0; q < 4; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[4 + q] = p->Bc[4 + q];
  }
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(ncells < resident ? ncells : resident);
  hex_laplace_matrix_tc4<<<grid, m4::THREADS, m4::SMEM, s>>>(T, ncells, coords, A, emap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_matrix_tc4 launch");
}

}  // namespace sfk

// ===========================================================================
// p = 4 (n = m = 5): the same three DMMA stages with zero padding
// (rows / columns 25 -> 32, K = 5|g| -> multiples of 4; the x stage's K =
// 4 groups x 5 planes = 20 is exact).  Padded A entries are 0; padded B
// entries read zero-initialised shared memory, so no NaN can leak in.
namespace sfk {

namespace m5 {
constexpr int N = 5, M = 5, N2 = 25, N3 = 125, N4 = 625, M3 = 125;
constexpr int THREADS = 512, WARPS = 16;
constexpr int KS = 6 * M3;
constexpr int ZR = 36;                  // Z row stride (32 read, 25 written; = 4 mod 16)
constexpr int ZS = 9 * M * M * ZR;      // Z[pair][qx*M + qy][ZR]
constexpr int YR = 644;                 // Y row stride (632 read, 625 written; = 4 mod 16)
constexpr int YS = 4 * M * YR;          // Y[(g*M + qx)][YR]
constexpr size_t SMEM = (size_t)(YS + ZS + KS + 24) * sizeof(double);
}  // namespace m5

struct TabsMat5 {
  double B[25], D[25], W[5], Bc[10];
};

__global__ void __launch_bounds__(m5::THREADS, 1)
hex_laplace_matrix_tc5(const __grid_constant__ TabsMat5 T, int64_t ncells,
                       const double* __restrict__ coords, double* __restrict__ A,
                       const int32_t* __restrict__ emap) {
  using namespace m5;
  extern __shared__ __align__(16) double smem[];
  double* sY = smem;                 // [20][YR]
  double* sZ = sY + YS;              // [9][M*M][ZR]
  double* sK = sZ + ZS;              // [6][M3]
  double* sC = sK + KS;              // [24]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, kq = lane & 3;

  // padding of Y and Z stays zero: clear everything once
  for (int i = tid; i < YS + ZS; i += THREADS) smem[i] = 0.0;

  auto k_phase = [&](int64_t cell) {
    if (tid < M3 && cell < ncells) {
      const int qx = tid / (M * M), qy = (tid / M) % M, qz = tid % M;
      HexLineGeom geo;
      geo.setup(sC, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
      double r0[3], r1[3], r2[3];
      const double det = geo.adj(T.Bc[qz], T.Bc[M + qz], r0, r1, r2);
      const double s = ((T.W[qx] * T.W[qy]) * T.W[qz]) * rcp64(fabs(det));
      const double* rows[3] = {r0, r1, r2};
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int m2 = l; m2 < 3; ++m2) {
          const double* a = rows[l];
          const double* b = rows[m2];
          sK[ksym4(l, m2) * M3 + tid] = s * fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
        }
    }
  };

  // x-stage A fragments: row tile xrt = warp & 3, W[(ix,jx)][k = (g, qx)] (k = 4s + kq)
  const int xrt = warp & 3;
  double wa[5];
  {
    const int row = xrt * 8 + gq, ix = row / N, jx = row % N;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int k = 4 * s + kq, g = k / M, qx = k % M;
      wa[s] = row < N2 ? ((g & 2) ? T.D : T.B)[ix * M + qx] * ((g & 1) ? T.D : T.B)[jx * M + qx]
                       : 0.0;
    }
  }

  // Z-stage tiles of this warp: (pair = j, rt = (warp >> 2) & 3, ct = warp & 3)
  const int zrt = (warp >> 2) & 3, zct = warp & 3;
  double za[9][2];
  {
    const int zz = zrt * 8 + gq, iz = zz / N, jz = zz % N;
#pragma unroll
    for (int pair = 0; pair < 9; ++pair)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int qz = 4 * s + kq, l = pair / 3, lp = pair % 3;
        za[pair][s] = (zz < N2 && qz < M)
            ? (l == 2 ? T.D : T.B)[iz * M + qz] * (lp == 2 ? T.D : T.B)[jz * M + qz] : 0.0;
      }
  }
  // Y-stage unit of this warp: (g = warp >> 2, rt = warp & 3)
  const int yg = warp >> 2, yrt = warp & 3, ynp = group_size(yg), ykg = 5 * ynp;
  const int ynks = (ykg + 3) / 4;
  double pa[5];
  int prow[5];   // sZ row offset (pair * 25 + qy) of each k-step's B fragment
  {
    const int row = yrt * 8 + gq, iy = row / N, jy = row % N;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int k = 4 * s + kq, sp = k / M, qy = k % M;
      const int pr = group_pair(yg, sp < ynp ? sp : 0);
      double v = 0.0;
      if (row < N2 && k < ykg) {
        const int l = pr / 3, lp = pr % 3;
        v = (l == 1 ? T.D : T.B)[iy * M + qy] * (lp == 1 ? T.D : T.B)[jy * M + qy];
      }
      pa[s] = v;
      prow[s] = pr * M * M + qy;
    }
  }

  int64_t cell = blockIdx.x;
  if (cell < ncells && tid < 24) sC[tid] = __ldg(coords + cell * 24 + tid);
  __syncthreads();
  k_phase(cell);
  __syncthreads();
  for (; cell < ncells; cell += gridDim.x) {
    const int64_t next = cell + gridDim.x;

    // ---- Z stage: Z_pair[(iz,jz)][(qx,qy)] = TT (32 x 8) * K (8 x 32) ----------
    //      this warp: tiles (pair 0..8, zrt, zct), 2 k-steps each (unrolled:
    //      the za fragments stay in registers)
#pragma unroll
    for (int pair = 0; pair < 9; ++pair) {
      const int l = pair / 3, lp = pair % 3;
      const int zz = zrt * 8 + gq, rt = zrt, ct = zct;
      const int qxy = ct * 8 + gq;                       // B column
      const double* kp = sK + ksym4(l, lp) * M3 + qxy * M;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int qz = 4 * s + kq;
        const double b = (qxy < N2 && qz < M) ? kp[qz] : 0.0;
        dmma4(d0, d1, za[pair][s], b);
      }
      (void)rt;
      if (zz < N2) {
        const int c0 = ct * 8 + 2 * kq;                  // D columns c0, c0 + 1 = (qx,qy)
        if (c0 < N2) sZ[(pair * M * M + c0) * ZR + zz] = d0;
        if (c0 + 1 < N2) sZ[(pair * M * M + c0 + 1) * ZR + zz] = d1;
      }
    }
    __syncthreads();

    // ---- Y stage: per (g, qx), Y = P_g (32 x K_g) * Zcat (K_g x 32) ----------
    //      units (g, rt 0..3): 16 over 16 warps; loops qx x ct
    if (next < ncells && tid >= THREADS - 24) sC[tid - (THREADS - 24)] =
        __ldg(coords + next * 24 + (tid - (THREADS - 24)));
    {
      const int g = yg, row = yrt * 8 + gq, iy = row / N, jy = row % N;
#pragma unroll 1
      for (int qx = 0; qx < M; ++qx) {
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) {
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int s = 0; s < 5; ++s) {
            // padded k rows: A is 0 there and prow points at a valid (finite) row
            if (s < ynks) dmma4(d0, d1, pa[s], sZ[(prow[s] + qx * M) * ZR + ct * 8 + gq]);
          }
          if (row < N2) {
            const int c0 = ct * 8 + 2 * kq;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int col = c0 + h;
              if (col < N2) {
                const int iz = col / N, jz = col - iz * N;
                sY[(g * M + qx) * YR + ((iy * N + iz) * N + jy) * N + jz] = h ? d1 : d0;
              }
            }
          }
        }
      }
    }
    __syncthreads();

    // ---- x stage: A[(ix,jx)][r] = W (32 x 20) * Y (20 x 632) ------------------
    {
      double* out = A + cell * (int64_t)(N3 * N3);
      const int row = xrt * 8 + gq, ix = row / N, jx = row % N;
#pragma unroll 2
      for (int ct = warp >> 2; ct < 79; ct += 4) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int s = 0; s < 5; ++s) dmma4(d0, d1, wa[s], sY[(4 * s + kq) * YR + ct * 8 + gq]);
        if (row < N2) {
          // r = (iy*N + iz) * N2 + (jy*N + jz): address = rowpart + (r / 25) * 125 + r % 25
          const int r0 = ct * 8 + 2 * kq;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = r0 + h;
            if (r < N4) {
              const int a = r / N2, b = r - a * N2;
              const int64_t off = (int64_t)(ix * N2 + a) * N3 + jx * N2 + b;
              if (emap) atomicAdd(A + __ldg(emap + cell * (int64_t)(N3 * N3) + off), h ? d1 : d0);
              else out[off] = h ? d1 : d0;
            }
          }
        }
      }
    }
    k_phase(next);
    __syncthreads();
  }
}

int launch_hex_matrix_tc5(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          cudaStream_t s, const int32_t* emap) {
  if (p->n != 5 || p->m != 5 || p->collocated) return SFK_EUNSUPPORTED;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)hex_laplace_matrix_tc5, m5::THREADS, m5::SMEM, "hex_matrix_tc5", &sh))
    return rc_;
  TabsMat5 T;
  for (int i = 0; i < 25; ++i) {
    T.B[i] = p->B[i];
    T.D[i] = p->D[i];
  }
  for (int q = 0; q < 5; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[5 + q] = p->Bc[5 + q];
  }
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(ncells < resident ? ncells : resident);
  hex_laplace_matrix_tc5<<<grid, m5::THREADS, m5::SMEM, s>>>(T, ncells, coords, A, emap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_matrix_tc5 launch");
}

}  // namespace sfk
