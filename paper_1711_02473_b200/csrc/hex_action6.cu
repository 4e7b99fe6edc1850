// Hex Q_p Laplace action, line kernel v6 — BASELINE C2 (headline):
// collocation-derivative sum factorisation.
//
// Same operator as v1-v5 (reference forms.py:186-189, 235-243; the spectral
// schedule passes.py:672-743), evaluated with fewer contractions.  With
// Gauss-Legendre points and m = n the 1D interpolation table B (n x n) is
// invertible, so the reference derivative table factors as
//     D = B C,      C = B^-1 D   (m x m, the collocation derivative)
// and the reference gradient at the points,
//     g_x = (D x B x B) u = (C x I x I)(B x B x B) u,
// is three interpolations followed by ONE derivative contraction per
// direction: 3 + 3 line contractions forward instead of 2 + 3 + 3, the same
// backwards (t = C_x^T f_x + C_y^T f_y + C_z^T f_z, then B^T x B^T x B^T).
// 12 n^4 FMA per cell instead of 16 n^4 (-25% of the contraction work).  C is
// solved once per plan on the host in extended precision from the
// reference's own B and D (sfk_api.cu: collocation_derivative), so C is the
// correctly rounded B^-1 D of the reference doubles; cond(B) <= 14 for
// p <= 8 and the results stay within ~2e-15 of the reference's emitted C
// (tests/test_gpu_parity.py, test_fullsize_parity.py).
//
// Pipeline per batch of CPB cells; one thread per line (n^2 lines per cell
// and direction), four shared slots S1..S4 of one n^3 array each:
//   A  x-lines  u (sU)  -> P  = B_x u                     S1
//   B  y-lines  P       -> Q  = B_y P                     S1 -> S2
//   C  z-lines  Q       -> V  = B_z Q (S1), gz = C_z V    (S4)
//   D  x-lines  V       -> gx = C_x V (S2);  y-lines V -> gy = C_y V (S3)
//   E  z-lines  geometry + flux at the line's points: (gx, gy, gz) ->
//               (fx, fy, fz) in place (S2, S3, S4)
//   F  x-lines  tx = C_x^T fx (S2, in place); y-lines ty = C_y^T fy (S3);
//      z-lines  tz = C_z^T fz (S4)
//   G  z-lines  t = tx + ty + tz;  R = B_z^T t         S2, S3, S4 -> S1
//   H  y-lines  R -> B_y^T R                          S1 -> S2
//   I  x-lines  -> A = B_x^T (.)                      S2 -> HBM
// Every array's layout (strides per axis, cell stride) is chosen for the
// two or three line directions that touch it (v6_layout below): the lane
// of a warp that owns line r accesses an address linear (mod 16 banks) in r.
#include "async_copy.cuh"
#include "hex_geometry.cuh"

namespace sfk {

// Tables of v6: row length LD (even, so aligned pairs of consecutive
// entries are one LDCU.128), except n = 8: with 128-bit pairs there the
// compiler hoisted the table set into uniform registers and spilled them
// (168 registers, or spills at the 128 cap); LD = 9 keeps 64-bit loads.
// B[i][q], BT[q][i], C[q'][q], CT[q][q'].
template <int N>
struct TabsV6 {
  static constexpr int LD = N == 8 ? 9 : (N + 1) & ~1;
  alignas(16) double B[N * LD];
  alignas(16) double BT[N * LD];
  alignas(16) double C[N * LD];
  alignas(16) double CT[N * LD];
  double W[N];
  double Bc[2 * N];
};

template <int N>
inline TabsV6<N> make_tabs_v6(const sfk_plan* p) {
  TabsV6<N> t{};
  constexpr int LD = TabsV6<N>::LD;
  for (int i = 0; i < N; ++i)
    for (int q = 0; q < N; ++q) {
      t.B[i * LD + q] = p->B[i * p->m + q];
      t.BT[q * LD + i] = p->B[i * p->m + q];
      t.C[i * LD + q] = p->Ct[i * p->m + q];   // C[q'=i][q]
      t.CT[q * LD + i] = p->Ct[i * p->m + q];
    }
  for (int q = 0; q < N; ++q) {
    t.W[q] = p->wq[q];
    t.Bc[q] = p->Bc[q];
    t.Bc[N + q] = p->Bc[p->m + q];
  }
  return t;
}

// out[o] = sum_i T[i*LD + o] in[i]: NO independent chains of depth NI.
template <int NI, int NO, int LD>
__device__ __forceinline__ void v6_contract(const double* T, const double* in, double* out) {
#pragma unroll
  for (int o = 0; o < NO; ++o) out[o] = T[o] * in[0];
#pragma unroll
  for (int i = 1; i < NI; ++i)
#pragma unroll
    for (int o = 0; o < NO; ++o) out[o] = fma(T[i * LD + o], in[i], out[o]);
}

// Scheduling fence between the independent line tasks of one stage (D, F):
// keeps the compiler from interleaving them, which at n = 8 (every lane
// live, stores unpredicated) raised the kernel to 168 registers.
__device__ __forceinline__ void v6_fence() { __syncwarp(); }

// Strided view of one per-cell array: element (x, y, z) at
// c*cs + x*sx + y*sy + z.
struct V6Arr {
  int sx, sy, cs;
};

__host__ __device__ constexpr int v6_up(int v, int mod, int res) {
  // smallest w >= v with w = res (mod `mod`)
  return v + ((res - v) % mod + mod) % mod;
}

// Layouts (16 banks of 8 bytes per wavefront of 64-bit accesses; LZ odd):
//   x/y array (P): x-line writer lane (y, z) -> y*n + z; y-line reader lane
//     (x, z) -> x*sx + z, linear when sx = n (mod 16).
//   y/z array (Q, Gy, V): [y][x][z], sx = LZ, sy = n*LZ: y-line lane (x, z)
//     -> x*LZ + z (linear for odd n); z-line lane (y, x) -> (y*n + x)*LZ.
//   x/z array (Gx): [x][y][z], sy = LZ, sx = 1 (mod 16): x-line lane (y, z)
//     -> y*LZ + z; z-line lane (y, x) -> x*sx + y*LZ = y*LZ + x (mod 16).
//   V is also read by x-lines (lane (y, z) -> y*n*LZ + z): 2-way there.
template <int N>
struct V6Layout {
  static constexpr int LZ = N | 1;
  static constexpr int NN = N * N;
  static constexpr V6Arr P{v6_up(NN, 16, N % 16), N, v6_up(N * v6_up(NN, 16, N % 16), 16, NN % 16)};
  static constexpr V6Arr YZ{LZ, N * LZ, v6_up(N * N * LZ, 16, (NN * LZ) % 16)};
  static constexpr V6Arr XZ{v6_up(N * LZ, 16, 1), LZ, v6_up(N * v6_up(N * LZ, 16, 1), 16, NN % 16)};
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  static constexpr int SLOT = cmax(cmax(P.cs, YZ.cs), XZ.cs);   // doubles per cell and slot
};

template <int N, int CPB>
struct V6Cfg {
  static constexpr int NN = N * N, N3 = N * N * N;
  static constexpr int THREADS = round_up(CPB * NN, 32);
  static constexpr int SLOT = V6Layout<N>::SLOT;
  static constexpr int S = CPB * SLOT;              // one slot, all cells
  static constexpr int USZ = round_up(CPB * N3 + 1, 2);
  static constexpr int CSZ = CPB * 24;
  static constexpr size_t SMEM = (size_t)(4 * S + USZ + 2 * CSZ + 2) * sizeof(double);
};

template <int N, int CPB, int MINB>
__global__ void __launch_bounds__(V6Cfg<N, CPB>::THREADS, MINB)
hex_laplace_action_v6(const __grid_constant__ TabsV6<N> T, int64_t ncells,
                      const double* __restrict__ coords, const double* __restrict__ u,
                      double* __restrict__ A) {
  using C = V6Cfg<N, CPB>;
  using L = V6Layout<N>;
  constexpr int NN = C::NN, N3 = C::N3, TH = C::THREADS, LD = TabsV6<N>::LD;
  constexpr V6Arr P = L::P, YZ = L::YZ, XZ = L::XZ;
  extern __shared__ __align__(16) double smem[];
  double* S1 = smem;
  double* S2 = S1 + C::S;
  double* S3 = S2 + C::S;
  double* S4 = S3 + C::S;
  double* sU = S4 + C::S;                  // [CPB*N3 (+1 phase shift)]
  double* sCo = sU + C::USZ;               // [2][CPB*24]
  const int tid = threadIdx.x;
  const int64_t nbatch = (ncells + CPB - 1) / CPB;

  // line owned by this thread in every stage: cell c, in-cell index r = a*N + b
  const bool on = tid < CPB * NN;
  const int lt = on ? tid : 0;
  const int c = lt / NN, r = lt - c * NN;
  const int ra = r / N, rb = r - ra * N;   // x-lines: (y, z) = (ra, rb); y-lines: (x, z);
                                           // z-lines: (y, x) = (ra, rb)

  auto prefetch = [&](int64_t b, int buf) {
    const int64_t c0 = b * CPB;
    const int nc = (int)((ncells - c0) < CPB ? (ncells - c0) : CPB);
    async_copy_phase<TH>(sU + dst_shift(u + c0 * N3), u + c0 * N3, nc * N3, tid);
    async_copy<TH>(sCo + buf * C::CSZ, coords + c0 * 24, nc * 24, tid);
    cp_async_commit();
  };

  int64_t b = blockIdx.x;
  if (b < nbatch) prefetch(b, 0);
  for (int k = 0; b < nbatch; b += gridDim.x, ++k) {
    const int cur = k & 1;
    const int64_t cell0 = b * CPB;
    const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
    const bool live = on && c < ncb;
    cp_async_wait<0>();
    __syncthreads();
    const double* su = sU + dst_shift(u + cell0 * N3);

    // ---- A: x-line (y, z): P[x] = sum_i B[i][x] u[i][y][z] -----------------
    {
      double in[N], o[N];
#pragma unroll
      for (int i = 0; i < N; ++i) in[i] = live ? su[c * N3 + i * NN + r] : 0.0;
      v6_contract<N, N, LD>(T.B, in, o);
      double* p = S1 + c * P.cs + ra * P.sy + rb;
      if (on) {
#pragma unroll
        for (int q = 0; q < N; ++q) p[q * P.sx] = o[q];
      }
    }
    __syncthreads();
    if (b + gridDim.x < nbatch) prefetch(b + gridDim.x, cur ^ 1);

    // ---- B: y-line (x, z): Q[y] = B_y P ------------------------------------
    {
      double in[N], o[N];
      const double* p = S1 + c * P.cs + ra * P.sx + rb;
#pragma unroll
      for (int i = 0; i < N; ++i) in[i] = p[i * P.sy];
      v6_contract<N, N, LD>(T.B, in, o);
      double* q = S2 + c * YZ.cs + ra * YZ.sx + rb;
      if (on) {
#pragma unroll
        for (int j = 0; j < N; ++j) q[j * YZ.sy] = o[j];
      }
    }
    __syncthreads();

    // ---- C: z-line (y, x): V = B_z Q (S1), gz = C_z V (S4) -----------------
    {
      double in[N], v[N], gz[N];
      const double* q = S2 + c * YZ.cs + ra * YZ.sy + rb * YZ.sx;
#pragma unroll
      for (int i = 0; i < N; ++i) in[i] = q[i];
      v6_contract<N, N, LD>(T.B, in, v);
      v6_contract<N, N, LD>(T.C, v, gz);
      double* w = S1 + c * YZ.cs + ra * YZ.sy + rb * YZ.sx;
      double* wz = S4 + c * YZ.cs + ra * YZ.sy + rb * YZ.sx;
      if (on) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          w[j] = v[j];
          wz[j] = gz[j];
        }
      }
    }
    __syncthreads();

    // ---- D: x-line (y, z): gx = C_x V -> S2;  y-line (x, z): gy = C_y V -> S3
    {
      double in[N], o[N];
      const double* v = S1 + c * YZ.cs + ra * YZ.sy + rb;           // lane (y, z)
#pragma unroll
      for (int i = 0; i < N; ++i) in[i] = v[i * YZ.sx];
      v6_contract<N, N, LD>(T.C, in, o);
      double* g = S2 + c * XZ.cs + ra * XZ.sy + rb;
      if (on) {
#pragma unroll
        for (int j = 0; j < N; ++j) g[j * XZ.sx] = o[j];
      }
    }
    v6_fence();
    {
      double in[N], o[N];
      const double* v = S1 + c * YZ.cs + ra * YZ.sx + rb;           // lane (x, z)
#pragma unroll
      for (int i = 0; i < N; ++i) in[i] = v[i * YZ.sy];
      v6_contract<N, N, LD>(T.C, in, o);
      double* g = S3 + c * YZ.cs + ra * YZ.sx + rb;
      if (on) {
#pragma unroll
        for (int j = 0; j < N; ++j) g[j * YZ.sy] = o[j];
      }
    }
    __syncthreads();

    // ---- E: z-line (y, x): geometry + flux, in place (S2, S3, S4) ----------
    {
      const int qy = ra, qx = rb;
      double* gxl = S2 + c * XZ.cs + qx * XZ.sx + qy * XZ.sy;
      double* gyl = S3 + c * YZ.cs + qy * YZ.sy + qx * YZ.sx;
      double* gzl = S4 + c * YZ.cs + qy * YZ.sy + qx * YZ.sx;   // gz in, tz out
      const double* sC = sCo + cur * C::CSZ + c * 24;
      HexLineAdj geo;
      geo.setup(sC, T.Bc[qx], T.Bc[N + qx], T.Bc[qy], T.Bc[N + qy]);
      const double wxy = T.W[qx] * T.W[qy];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        double gx = gxl[q], gy = gyl[q], g2 = gzl[q];
        double r0[3], r1[3], r2[3];
        const double det = geo.adj(T.Bc[N + q], r0, r1, r2);
        const double s = (wxy * T.W[q]) * rcp64(fabs(det));
        laplace_flux(r0, r1, r2, s, gx, gy, g2);
        if (on) {
          gxl[q] = gx;
          gyl[q] = gy;
          gzl[q] = g2;
        }
      }
    }
    __syncthreads();

    // ---- F: x-line tx = C_x^T fx (S2 in place); y-line ty = C_y^T fy (S3) ---
    {
      double in[N], o[N];
      double* g = S2 + c * XZ.cs + ra * XZ.sy + rb;
#pragma unroll
      for (int i = 0; i < N; ++i) in[i] = g[i * XZ.sx];
      v6_contract<N, N, LD>(T.CT, in, o);
      if (on) {
#pragma unroll
        for (int j = 0; j < N; ++j) g[j * XZ.sx] = o[j];
      }
    }
    v6_fence();
    {
      double in[N], o[N];
      double* g = S3 + c * YZ.cs + ra * YZ.sx + rb;
#pragma unroll
      for (int i = 0; i < N; ++i) in[i] = g[i * YZ.sy];
      v6_contract<N, N, LD>(T.CT, in, o);
      if (on) {
#pragma unroll
        for (int j = 0; j < N; ++j) g[j * YZ.sy] = o[j];
      }
    }
    v6_fence();
    {
      double in[N], o[N];
      double* g = S4 + c * YZ.cs + ra * YZ.sy + rb * YZ.sx;       // z-line (y, x)
#pragma unroll
      for (int i = 0; i < N; ++i) in[i] = g[i];
      v6_contract<N, N, LD>(T.CT, in, o);
      if (on) {
#pragma unroll
        for (int j = 0; j < N; ++j) g[j] = o[j];
      }
    }
    __syncthreads();

    // ---- G: z-line (y, x): t = tx + ty + tz; R = B_z^T t -> S1 (y/z) -------
    {
      const int qy = ra, qx = rb;
      const double* gxl = S2 + c * XZ.cs + qx * XZ.sx + qy * XZ.sy;
      const double* gyl = S3 + c * YZ.cs + qy * YZ.sy + qx * YZ.sx;
      const double* tzl = S4 + c * YZ.cs + qy * YZ.sy + qx * YZ.sx;
      double* w = S1 + c * YZ.cs + qy * YZ.sy + qx * YZ.sx;
      double t[N], o[N];
#pragma unroll
      for (int q = 0; q < N; ++q) t[q] = (gxl[q] + gyl[q]) + tzl[q];
      v6_contract<N, N, LD>(T.BT, t, o);
      if (on) {
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] = o[i];
      }
    }
    __syncthreads();

    // ---- H: y-line (x, z): B_y^T -> S2 (x/y layout P) ----------------------
    {
      double in[N], o[N];
      const double* q = S1 + c * YZ.cs + ra * YZ.sx + rb;
#pragma unroll
      for (int j = 0; j < N; ++j) in[j] = q[j * YZ.sy];
      v6_contract<N, N, LD>(T.BT, in, o);
      double* p = S2 + c * P.cs + ra * P.sx + rb;
      if (on) {
#pragma unroll
        for (int i = 0; i < N; ++i) p[i * P.sy] = o[i];
      }
    }
    __syncthreads();

    // ---- I: x-line (y, z): A = B_x^T (.) -> HBM ----------------------------
    {
      double in[N], o[N];
      const double* p = S2 + c * P.cs + ra * P.sy + rb;
#pragma unroll
      for (int q = 0; q < N; ++q) in[q] = p[q * P.sx];
      v6_contract<N, N, LD>(T.BT, in, o);
      if (live) {
        double* ap = A + (cell0 + c) * N3 + r;
#pragma unroll
        for (int i = 0; i < N; ++i) ap[i * NN] = o[i];
      }
    }
    // no barrier: the next batch's stage A writes S1 and reads sU, stage I
    // read S2; the barrier at the top of the loop orders sU / coords
  }
}

template <int N, int CPB, int MINB>
static int launch_v6(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* u, cudaStream_t s) {
  using C = V6Cfg<N, CPB>;
  auto kern = hex_laplace_action_v6<N, CPB, MINB>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_action_v6", &sh, true))
    return rc_;
  const TabsV6<N> T = make_tabs_v6<N>(p);
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(nbatch < resident ? nbatch : resident);
  kern<<<grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, u, A);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_v6 launch");
}

// (cells per CTA, min CTAs per SM) per n: the default, then the
// alternatives option v6_cfg = 1..3 selects (A/B runs).
int launch_hex_action_v6(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s) {
  if (p->n != p->m || !p->has_ct) return SFK_EUNSUPPORTED;
  const int alt = (int)option(OPT_V6_CFG);
#define V6_CASE(n_, c0, m0, c1, m1, c2, m2, c3, m3)                         \
  case n_:                                                                   \
    switch (alt) {                                                           \
      case 1: return launch_v6<n_, c1, m1>(p, ncells, A, coords, w0, s);    \
      case 2: return launch_v6<n_, c2, m2>(p, ncells, A, coords, w0, s);    \
      case 3: return launch_v6<n_, c3, m3>(p, ncells, A, coords, w0, s);    \
      default: return launch_v6<n_, c0, m0>(p, ncells, A, coords, w0, s);   \
    }
  switch (p->n) {
    V6_CASE(4, 8, 2, 16, 2, 8, 3, 4, 4)
    V6_CASE(5, 5, 2, 10, 2, 6, 2, 7, 2)
    V6_CASE(6, 7, 2, 8, 2, 5, 3, 3, 3)
    V6_CASE(7, 5, 2, 4, 3, 6, 2, 3, 4)
    V6_CASE(8, 4, 2, 3, 2, 2, 3, 5, 1)
    V6_CASE(9, 3, 2, 2, 3, 4, 1, 2, 2)
    default: return SFK_EUNSUPPORTED;
  }
#undef V6_CASE
}

}  // namespace sfk
