// Hex Q_p local stiffness matrices beyond the BASELINE degrees, p = 5..8
// (n = m = 6..9), on the FP64 tensor cores — SURVEY.md §8(f) row 3.
//
// Math and reference mapping as hex_matrix.cu / hex_matrix_tc.cu (registry
// `laplace` on `hex`, forms.py:186-189; test index outermost, A[i*n^3 + j],
// forms.py:402-408): with K_ll'(q) = w_q/|det J| (R R^T)_ll' (R = adj J rows)
//   A[(ix,iy,iz),(jx,jy,jz)] = sum_q sum_ll' K_ll'(q) d^l phi_i(q) d^l' phi_j(q).
// Three contraction stages (z, y, x), as in tc4 / tc5, but the cell is
// processed in CHUNKS of its output so the intermediates fit in shared memory
// at any n (tc5's whole-cell Y is 4 m n^4 doubles: 249 KB at n = 6, 2 MB at
// n = 9).  Chunking by the test z index iz (and blocks of iy) costs no
// recomputation — every intermediate depends on iz (resp. iy) only through
// its own row:
//   for iz:   Z stage  Z_pair[(qx,qy)][jz] = sum_qz K_ll'(qx,qy,qz)
//                                     T^l_z[iz][qz] T^l'_z[jz][qz]      (DFMA)
//     for iy block:
//             Y stage  Y_g[qx][(iy,jy,jz)] = sum_{pair in g, qy}
//                        P_pair[(iy,jy)][qy] Z_pair[(qx,qy)][jz]        (DMMA)
//             x stage  A[(ix,jx)][(iy,jy,jz)] @ iz = sum_{g,qx}
//                        W[(ix,jx)][(g,qx)] Y_g[qx][(iy,jy,jz)]         (DMMA)
// where the 9 (l, l') pairs are grouped by their x pattern g = (l == 0) * 2 +
// (l' == 0) (the x stage needs only 4 tables W_g = T_x,test (x) T_x,trial),
// P_pair = T^l_y (x) T^l'_y and T^d = D when d is the axis, else B.
// Per cell: x stage 4 m n^6, Y 9 m^2 n^4, Z 9 m^3 n^2 MACs (8 n^7 + ... flop
// against the reference's 15 n^7 + ...).
//
// x stage: W (n^2 x 4m) is constant — each warp keeps the A fragments of its
// row tile in registers for the whole kernel, B fragments are one conflict-
// free LDS each, and a row (ix, jx) of an output tile is 8 consecutive
// doubles of A (for fixed (ix, iy, iz, jx) the (jy, jz) entries are
// contiguous): full 32-byte sectors straight from the accumulators.
// Y stage: A fragments from a per-CTA table of P (zero rows pad each group's
// k range to a multiple of 4), B fragments from Z.
// Barriers: 2 per (iz, iy block); Z of the next iz and K of the next cell run
// in the x stage's interval (disjoint arrays).
//
// emap != nullptr: CSR mode (values[emap[cell][i*n^3 + j]] += A_ij, fp64
// atomics; sfk_csr_entry_map) — the (p+1)^6 cell matrices never reach HBM.
#include "hex_geometry.cuh"

namespace sfk {

namespace {

__device__ __forceinline__ void dmma_tcn(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// stride with stride % 16 == 4 (doubles): the four kq rows of a B fragment
// land in distinct bank quarters of a half-warp access
__host__ __device__ constexpr int stride4(int x) { return x + ((4 - x % 16) + 16) % 16; }

__host__ __device__ constexpr int ksym(int l, int r) {
  return l == r ? l : (l + r == 1 ? 3 : (l + r == 2 ? 4 : 5));
}

// pair blocks in x-pattern-group order: g0 = (1,1) (1,2) (2,1) (2,2);
// g1 = (1,0) (2,0); g2 = (0,1) (0,2); g3 = (0,0)
__host__ __device__ constexpr int pair_l(int pb) {
  return pb < 4 ? 1 + pb / 2 : pb < 6 ? 1 + (pb - 4) : 0;
}
__host__ __device__ constexpr int pair_lp(int pb) {
  return pb < 4 ? 1 + pb % 2 : pb < 6 ? 0 : pb < 8 ? 1 + (pb - 6) : 0;
}
__host__ __device__ constexpr int group_pb0(int g) { return g == 0 ? 0 : g == 1 ? 4 : g == 2 ? 6 : 8; }

}  // namespace

template <int N>
struct TabsMatN {
  double B[N * N], D[N * N], W[N], Bc[2 * N];
};

template <int N, int IB, int WX>
struct MatTcnCfg {
  static constexpr int M = N, N2 = N * N, N3 = N2 * N, M2 = M * M, M3 = M2 * M;
  static constexpr int RT = (N2 + 7) / 8;            // x-stage row tiles (ix, jx)
  static constexpr int WARPS = RT * WX, THREADS = 32 * WARPS;
  static constexpr int NB = (N + IB - 1) / IB;       // iy blocks
  static constexpr int XC = IB * N2;                 // x-stage columns of a full block
  static constexpr int CT = (XC + 7) / 8;
  static constexpr int YR = stride4(CT * 8);         // Y[(g, qx)][YR]
  static constexpr int YS = 4 * M * YR;
  static constexpr int ZC = (M * N + 7) / 8 * 8;     // Z columns (qx, jz), padded
  static constexpr int ZR = stride4(ZC);
  static constexpr int ZROWS = 9 * M + 4;            // (pair, qy) + k padding of group 3
  static constexpr int ZS = ZROWS * ZR;
  static constexpr int CTY = ZC / 8;
  static constexpr int KS0 = (4 * M + 3) / 4, KS1 = (2 * M + 3) / 4, KS3 = (M + 3) / 4;
  static constexpr int KSY = KS0 + 2 * KS1 + KS3;    // Y-stage k steps per tile (all groups)
  static constexpr int PR = 4 * KSY;                 // P rows (group-padded k)
  static constexpr int PC = stride4(N2 + 8);         // P columns (iy, jy) + tile overhang
  static constexpr int PS = PR * PC;
  static constexpr int KSZ = 6 * M3;                 // K (6 unique entries) per point
  static constexpr int TS = 2 * N * M;               // B, D tables
  static constexpr size_t SMEM = (size_t)(YS + ZS + PS + KSZ + TS + 24) * sizeof(double);
  static __host__ __device__ constexpr int ks(int g) { return g == 0 ? KS0 : g == 3 ? KS3 : KS1; }
  static __host__ __device__ constexpr int prow0(int g) {
    return g == 0 ? 0 : g == 1 ? 4 * KS0 : g == 2 ? 4 * (KS0 + KS1) : 4 * (KS0 + 2 * KS1);
  }
};

template <int N, int IB, int WX>
__global__ void __launch_bounds__(MatTcnCfg<N, IB, WX>::THREADS, 1)
hex_laplace_matrix_tcn(const __grid_constant__ TabsMatN<N> T, int64_t ncells,
                       const double* __restrict__ coords, double* __restrict__ A,
                       const int32_t* __restrict__ emap) {
  using C = MatTcnCfg<N, IB, WX>;
  constexpr int M = C::M, N2 = C::N2, N3 = C::N3, M2 = C::M2, M3 = C::M3;
  extern __shared__ __align__(16) double smem[];
  double* sY = smem;
  double* sZ = sY + C::YS;
  double* sP = sZ + C::ZS;
  double* sK = sP + C::PS;
  double* sT = sK + C::KSZ;       // sT[0][i][q] = B, sT[1][i][q] = D
  double* sC = sT + C::TS;        // 24 coordinates
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, kq = lane & 3;

  // ---- per-CTA setup: zero the padded arrays, tables, P --------------------
  for (int i = tid; i < C::YS + C::ZS + C::PS; i += C::THREADS) smem[i] = 0.0;
  for (int i = tid; i < N * M; i += C::THREADS) {
    sT[i] = T.B[i];
    sT[N * M + i] = T.D[i];
  }
  __syncthreads();
  // P[(g-padded k)][(iy, jy)]: k = (pair in g, qy); zero beyond the group
  for (int i = tid; i < 9 * M * N2; i += C::THREADS) {
    const int row = i % N2, kk = i / N2;        // kk = pb * M + qy
    const int pb = kk / M, qy = kk % M;
    const int g = pb < 4 ? 0 : pb < 6 ? 1 : pb < 8 ? 2 : 3;
    const int k = kk - group_pb0(g) * M;        // k within the group
    const int l = pair_l(pb), lp = pair_lp(pb), iy = row / N, jy = row % N;
    sP[(C::prow0(g) + k) * C::PC + row] =
        sT[(l == 1) * N * M + iy * M + qy] * sT[(lp == 1) * N * M + jy * M + qy];
  }

  // x-stage A fragments of this warp's row tile: W[(ix,jx)][k = (g, qx)]
  const int xrt = warp % C::RT, xct0 = warp / C::RT;
  double wa[M];
  {
    const int row = xrt * 8 + gq, ix = row / N, jx = row % N;
#pragma unroll
    for (int s = 0; s < M; ++s) {
      const int k = 4 * s + kq, g = k / M, qx = k % M;
      wa[s] = row < N2 ? ((g & 2) ? T.D : T.B)[ix * M + qx] * ((g & 1) ? T.D : T.B)[jx * M + qx]
                       : 0.0;
    }
  }

  auto k_phase = [&](int64_t cell) {
    if (cell >= ncells) return;
    for (int t = tid; t < M3; t += C::THREADS) {
      const int qx = t / M2, qy = (t / M) % M, qz = t % M;
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
          sK[ksym(l, m2) * M3 + t] = s * fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
        }
    }
  };

  // Z stage at test index iz: items (pair block, qy, qx), n outputs (jz) each
  auto z_phase = [&](int iz) {
    for (int t = tid; t < 9 * M2; t += C::THREADS) {
      const int pb = t / M2, qy = (t / M) % M, qx = t % M;
      const int l = pair_l(pb), lp = pair_lp(pb);
      const double* kp = sK + ksym(l, lp) * M3 + (qx * M + qy) * M;
      const double* tl = sT + (l == 2) * N * M + iz * M;
      const double* tr = sT + (lp == 2) * N * M;
      double a[M];
#pragma unroll
      for (int qz = 0; qz < M; ++qz) a[qz] = kp[qz] * tl[qz];
      double* zo = sZ + (pb * M + qy) * C::ZR + qx * N;
#pragma unroll
      for (int jz = 0; jz < N; ++jz) {
        double acc = a[0] * tr[jz * M];
#pragma unroll
        for (int qz = 1; qz < M; ++qz) acc = fma(a[qz], tr[jz * M + qz], acc);
        zo[jz] = acc;
      }
    }
  };

  int64_t cell = blockIdx.x;
  if (cell < ncells && tid < 24) sC[tid] = __ldg(coords + cell * 24 + tid);
  __syncthreads();
  k_phase(cell);
  __syncthreads();
  z_phase(0);
  __syncthreads();

  for (; cell < ncells; cell += gridDim.x) {
    const int64_t next = cell + gridDim.x;
    double* out = A + cell * (int64_t)(N3 * N3);
    const int32_t* mp = emap ? emap + cell * (int64_t)(N3 * N3) : nullptr;
#pragma unroll 1
    for (int iz = 0; iz < N; ++iz) {
#pragma unroll 1
      for (int b = 0; b < C::NB; ++b) {
        const int ib0 = b * IB, nb = (N - ib0) < IB ? (N - ib0) : IB;
        if (iz == 0 && b == 0 && next < ncells && tid < 24)
          sC[tid] = __ldg(coords + next * 24 + tid);   // K(cell) consumed it already

        // ---- Y stage: tiles (rty, cty), all four groups per tile ----------
        {
          const int rty_n = (nb * N + 7) / 8;
          for (int v = warp; v < rty_n * C::CTY; v += C::WARPS) {
            const int rty = v / C::CTY, cty = v % C::CTY;
            const int row = rty * 8 + gq;                      // (iy_l, jy)
            const double* pa = sP + kq * C::PC + ib0 * N + rty * 8 + gq;
            const double* zb = sZ + kq * C::ZR + cty * 8 + gq;
            double d[4][2];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              d[g][0] = 0.0;
              d[g][1] = 0.0;
            }
#pragma unroll
            for (int s = 0; s < C::KS0; ++s) {
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                if (s < C::ks(g)) {
                  const double a = pa[(C::prow0(g) + 4 * s) * C::PC];
                  const double bv = zb[(group_pb0(g) * M + 4 * s) * C::ZR];
                  dmma_tcn(d[g][0], d[g][1], a, bv);
                }
              }
            }
            if (row < nb * N) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int c = cty * 8 + 2 * kq + h;            // (qx, jz)
                if (c < M * N) {
                  const int qx = c / N, jz = c - qx * N;
                  double* yo = sY + qx * C::YR + row * N + jz;
#pragma unroll
                  for (int g = 0; g < 4; ++g) yo[g * M * C::YR] = d[g][h];
                }
              }
            }
          }
        }
        __syncthreads();

        // ---- x stage: A[(ix,jx)][(iy_l, jy, jz)] = W (n^2 x 4m) * Y -------
        {
          const int ncol = nb * N2, ct_n = (ncol + 7) / 8;
          const int row = xrt * 8 + gq, ix = row / N, jx = row % N;
          const bool live = row < N2;
          const int64_t rbase = (int64_t)(((ix * N + ib0) * N + iz) * N3 + jx * N2);
          const double* yb = sY + kq * C::YR + gq;
          constexpr int U = 2;
#pragma unroll 1
          for (int ct = xct0; ct < ct_n; ct += U * WX) {
            double d[U][2];
#pragma unroll
            for (int u = 0; u < U; ++u) d[u][0] = d[u][1] = 0.0;
#pragma unroll
            for (int s = 0; s < M; ++s)
#pragma unroll
              for (int u = 0; u < U; ++u)
                if (u == 0 || ct + u * WX < ct_n)
                  dmma_tcn(d[u][0], d[u][1], wa[s], yb[4 * s * C::YR + (ct + u * WX) * 8]);
            if (live) {
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const int c0 = (ct + u * WX) * 8 + 2 * kq;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const int c = c0 + h;
                  if (c < ncol) {
                    const int iyl = c / N2, rem = c - iyl * N2;
                    const int64_t off = rbase + (int64_t)iyl * (N * N3) + rem;
                    if (mp) atomicAdd(A + __ldg(mp + off), d[u][h]);
                    else __stcs(out + off, d[u][h]);
                  }
                }
              }
            }
          }
        }
        if (b == C::NB - 1) {
          if (iz + 1 < N) z_phase(iz + 1);   // Z read by the last Y stage: synced
          else k_phase(next);                // last Z done; sC(next) loaded at (0, 0)
        }
        __syncthreads();
      }
    }
    if (next < ncells) {
      z_phase(0);
      __syncthreads();
    }
  }
}

template <int N, int IB, int WX>
static int launch_tcn(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                      cudaStream_t s, const int32_t* emap) {
  using C = MatTcnCfg<N, IB, WX>;
  auto kern = hex_laplace_matrix_tcn<N, IB, WX>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_matrix_tcn", &sh))
    return rc_;
  TabsMatN<N> T;
  for (int i = 0; i < N; ++i)
    for (int q = 0; q < N; ++q) {
      T.B[i * N + q] = p->B[i * p->m + q];
      T.D[i * N + q] = p->D[i * p->m + q];
    }
  for (int q = 0; q < N; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[N + q] = p->Bc[p->m + q];
  }
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(ncells < resident ? ncells : resident);
  kern<<<grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, A, emap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_matrix_tcn launch");
}

#ifdef SFK_TCN_ONLY_N
// probe builds (tools/kernel_sweep.py c5h): one instantiation
}  // namespace sfk
extern "C" int SFK_TCN_PROBE_ENTRY(const sfk_plan* p, int64_t ncells, double* A,
                                   const double* coords, const double* w0, void* stream) {
  (void)w0;
  if (p->n != SFK_TCN_ONLY_N || p->m != SFK_TCN_ONLY_N)
    return sfk::fail(SFK_EUNSUPPORTED, "probe build: n = m = %d only", SFK_TCN_ONLY_N);
  return sfk::launch_tcn<SFK_TCN_ONLY_N, SFK_TCNP_IB, SFK_TCNP_WX>(p, ncells, A, coords,
                                                                    (cudaStream_t)stream, nullptr);
}
namespace sfk {
#else
bool hex_matrix_tcn_supported(int n, int m) { return n == m && n >= 6 && n <= 9; }

int launch_hex_matrix_tcn(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          cudaStream_t s, const int32_t* emap) {
  if (p->collocated || p->n != p->m) return SFK_EUNSUPPORTED;
  // (iy block, warps per x-stage row tile) per n: the fastest of all
  // combinations that fit (tools/kernel_sweep.py c5h, profiles/r02cz_c5h_sweep.jsonl:
  // p = 5 / 6 / 7 / 8 3.48 / 4.59 / 3.87 / 6.15 -> 3.24 / 4.34 / 3.72 / 5.46 ms);
  // option c5_hi_cfg = 1, 2 selects earlier alternatives, 5 the r02bb defaults
  const int cfg = (int)option(OPT_C5_HI_CFG);
  switch (p->n) {
    // n = 4: A/B against tc4 (option c5_hi_cfg = 3, 4); n = 5: the default
    // (4.41 ms at 2^16 cells against 5.01 for tc5 and 6.51 for <5, 5, 2>)
    case 4:
      if (cfg == 4) return launch_tcn<4, 4, 2>(p, ncells, A, coords, s, emap);
      return launch_tcn<4, 4, 1>(p, ncells, A, coords, s, emap);
    case 5:
      if (cfg == 4) return launch_tcn<5, 5, 2>(p, ncells, A, coords, s, emap);
      return launch_tcn<5, 5, 1>(p, ncells, A, coords, s, emap);
    case 6:   // 3.48 ms (2^14 cells) vs 3.89 <6,6,2>, 4.62 <6,3,2>
      if (cfg == 1) return launch_tcn<6, 3, 2>(p, ncells, A, coords, s, emap);
      if (cfg == 2) return launch_tcn<6, 6, 2>(p, ncells, A, coords, s, emap);
      if (cfg == 5) return launch_tcn<6, 6, 1>(p, ncells, A, coords, s, emap);
      return launch_tcn<6, 2, 1>(p, ncells, A, coords, s, emap);
    case 7:   // 4.59 ms (2^13 cells) vs 5.54 <7,1,2>, 5.93 <7,7,1>
      if (cfg == 1) return launch_tcn<7, 1, 2>(p, ncells, A, coords, s, emap);
      if (cfg == 2) return launch_tcn<7, 7, 1>(p, ncells, A, coords, s, emap);
      if (cfg == 5) return launch_tcn<7, 4, 2>(p, ncells, A, coords, s, emap);
      return launch_tcn<7, 7, 3>(p, ncells, A, coords, s, emap);
    case 8:   // 3.88 ms (2^12 cells) vs 3.98 <8,2,2>, 4.12 <8,4,1>
      if (cfg == 1) return launch_tcn<8, 2, 2>(p, ncells, A, coords, s, emap);
      if (cfg == 2) return launch_tcn<8, 4, 1>(p, ncells, A, coords, s, emap);
      if (cfg == 5) return launch_tcn<8, 1, 2>(p, ncells, A, coords, s, emap);
      return launch_tcn<8, 4, 2>(p, ncells, A, coords, s, emap);
    case 9:   // 6.17 ms (2^11 cells), <9,1,2> the same (and spills)
      if (cfg == 1) return launch_tcn<9, 1, 2>(p, ncells, A, coords, s, emap);
      if (cfg == 5) return launch_tcn<9, 1, 1>(p, ncells, A, coords, s, emap);
      return launch_tcn<9, 2, 1>(p, ncells, A, coords, s, emap);
    default: return SFK_EUNSUPPORTED;
  }
}

#endif  // SFK_TCN_ONLY_N

}  // namespace sfk
