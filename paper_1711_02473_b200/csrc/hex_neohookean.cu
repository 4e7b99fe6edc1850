// Hex Q_p^3 compressible neo-Hookean residual — BASELINE config C4
// (p = 2..6, GL (p+2)^3, mu = 1, lambda = 10).
//
// Reference: not in the reference registry; the
// builder-supplied FormSpec of SURVEY.md §8(a) row a17, lowered by
// forms.lower_form with a vector Q_p test space (elements.py:425-452: dof
// ((ix*n+iy)*n+iz)*3 + comp) and the displacement as coefficient slot 0
// with first derivatives (forms.py:326-350):
//   F = I + grad u,  J = det F,  F^-T = cof(F) / J,
//   P = mu (F - F^-T) + lambda ln(J) F^-T,
//   r[(i, a)] = sum_q w_q |det Jg| sum_k P[a][k] (grad phi_i)_k .
// The same 8 + 8 contraction schedule as the scalar Laplace action is run
// per displacement component (3 x 8 forward, 3 x 8 transposed), with m =
// n + 1 points per axis.
//
// B200 mapping: the scalar line kernel (hex_action2.cu) extended to three
// components; persistent CTAs with cp.async prefetch of the next batch.
// The forward x/y stages run component by component through a shared X buffer into a 9-array Y buffer whose z-lines are stored with a
// stride >= m, so that each z-line thread can overwrite, in place, its own
// 9 lines with (1) the 9 reference-gradient lines, (2) the 9 flux lines and
// (3) the 9 transposed-z lines — no extra shared memory and no barrier
// between those three steps.  Transposed y/x stages then run per component.
#include <cstdlib>

#include "async_copy.cuh"
#include "hex_geometry.cuh"
#include "hex_neohookean_point.cuh"

// Component loops: rolled (one copy of each stage's code) or unrolled x3.
// Rolled, ptxas hoists the stages' table constants out of the loop into vector
// registers and moves them back to uniform registers at every use (R2UR: 15%
// of the executed instructions at p = 4, profiles/r02ce_C4_p4_opmix.txt);
// unrolled, the constants are loaded where they are used.  Same-box A/B
// (profiles/r02cg_c4_*.jsonl): p = 2 0.1603 -> 0.1557, p = 4 0.6758 -> 0.6492
// ms; slower at p = 5, 6 (220-254 registers); p = 3 on the one-shot 6-cell CTAs
// 0.2970 -> 0.2867 ms (profiles/r02ct_c4l_sweep2.jsonl) — so n = 3, 4, 5.
// SFK_NEO_UNROLLA = 0 / 1 (A/B builds) forces rolled / unrolled everywhere.
#ifndef SFK_NEO_UNROLLA
#define SFK_NEO_UNROLLA -1
#endif
__host__ __device__ constexpr int neo_unroll_a(int n) {
  return (SFK_NEO_UNROLLA >= 0 ? SFK_NEO_UNROLLA != 0 : (n >= 3 && n <= 5)) ? 3 : 1;
}
#define NEO_PRAGMA_A _Pragma("unroll (neo_unroll_a(N))")

#ifndef SFK_NEO_YT
#define SFK_NEO_YT 1
#endif

namespace sfk {

#ifdef SFK_C4L_ONLY_N
namespace {   // probe objects differ in macros (SFK_NEO_UNROLLA): keep their instances apart
#endif

constexpr bool NEO_YT = SFK_NEO_YT;

// X-array q-stride and per-cell Y padding from tools/c4_layout.py's bank
// model (x-line writes / y-line reads of X: n = 4..7 modelled wavefronts
// 40 / 40 / 50 / 30 -> 24 / 30 / 34 / 16 with PX 17 / 25 / 37 / 49 ->
// 20 / 37 / 38 / 55; Y cell pad 8 at n = 4, 6: 84 -> 62, 102 -> 90).
__host__ __device__ constexpr int neo_px(int n) {
  return n == 4 ? 20 : n == 5 ? 37 : n == 6 ? 38 : n == 7 ? 55 : (n * n) | 1;
}
__host__ __device__ constexpr int neo_ypad(int n) { return (n == 4 || n == 6) ? 8 : 0; }

template <int N, int M, int CPB>
struct NeoCfg {
  static constexpr int NN = N * N, MN = M * N, MM = M * M;
  static constexpr int THREADS = round_up(CPB * MM, 32);
  static constexpr int PX = neo_px(N);
  static constexpr int LZ = M | 1;             // z-line stride (>= m, odd)
  static constexpr int XA = M * PX;            // one X/R array per cell
  static constexpr int XSZ = 2 * XA;
  static constexpr int YA = MM * LZ;           // one Y array per cell
  static constexpr int YSZ = 9 * YA + neo_ypad(N);
  static constexpr int USZ = round_up(CPB * 3 * N * N * N + 1, 2);   // u of one batch
  static constexpr int CSZ = CPB * 24;
  static constexpr size_t SMEM =
      (size_t)(round_up(CPB * (XSZ + YSZ), 2) + USZ + 2 * CSZ) * sizeof(double);
};

// GS = true: global residual y += sum_c P_c^T r_c(P_c x) (SURVEY.md §8(f)
// item 1): cmap[c][3*node + comp] is the global dof of local dof
// (node, comp); x is gathered into the shared u buffer by per-element
// cp.async through the map, the residual scattered with fp64 atomics.
// WARPS > 0: warp-synchronous mode for small p — each warp owns CPB whole
// cells (every stage has <= 32 lines for them) with its own shared-memory
// slice and prefetch, and the stages sync with __syncwarp instead of CTA
// barriers (the CTA version runs ~13 barriers per batch).
template <int N, int M, int CPB, bool GS = false, int WARPS = 0, int VAR = 0, int MINB = 0>
__global__ void __launch_bounds__(WARPS ? 32 * WARPS : NeoCfg<N, M, CPB>::THREADS, MINB)
hex_neohookean_kernel(const __grid_constant__ Tabs<N, M> T, double mu, double lam,
                      int64_t ncells, const double* __restrict__ coords,
                      const double* __restrict__ u, double* __restrict__ A,
                      const int* __restrict__ cmap = nullptr) {
  using C = NeoCfg<N, M, CPB>;
  constexpr int NN = C::NN, MN = C::MN, MM = C::MM, PX = C::PX, LZ = C::LZ;
  // Y lines qy-major (as hex_action5.cu): the y / y^T stages' accesses
  // (thread (qx, iz), iz fastest) become near-consecutive; the z-line
  // threads keep their odd line stride.  On at n = 6 (p = 5: 1.311 -> 1.243
  // ms; neutral at p = 3, 4, 6, slightly slower at p = 2 —
  // profiles/r01ci_*.jsonl).  SFK_NEO_YT=0 restores qx-major everywhere.
  constexpr bool NYT = NEO_YT && N == 6;
  constexpr int QS = NYT ? M * LZ : LZ;
  constexpr int XA = C::XA, YA = C::YA;
  constexpr int N3 = N * NN;
  constexpr int TH = WARPS ? 32 : C::THREADS;       // threads sharing one cell group
  constexpr int GROUPS = WARPS ? WARPS : 1;         // independent cell groups per CTA
  static_assert(!WARPS || CPB * MM <= 32, "warp-synchronous mode needs CPB*m^2 <= 32");
  extern __shared__ __align__(16) double smem[];
  const int grp = WARPS ? (int)(threadIdx.x >> 5) : 0;
  double* gbase = smem + (size_t)grp * (C::SMEM / sizeof(double));
  double* sX = gbase;
  double* sY = sX + CPB * C::XSZ;
  double* sU = gbase + round_up(CPB * (C::XSZ + C::YSZ), 2);
  double* sCo = sU + C::USZ;
  const int tid = WARPS ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
  auto sync = [] { if (WARPS) __syncwarp(); else __syncthreads(); };
  const int64_t nbatch = (ncells + CPB * GROUPS - 1) / (CPB * GROUPS);
  // persistent CTAs: u (3 components interleaved, as stored) and coords of
  // the next batch stream into shared memory with cp.async while the current
  // batch computes (u once the last x stage consumed it, coords
  // double-buffered because the z stage needs them)
  auto prefetch = [&](int64_t bt, int buf) {
    const int64_t c0 = bt * (CPB * GROUPS) + grp * CPB;
    const int nc = (int)((ncells - c0) < CPB ? (ncells - c0) : CPB);
    if (nc <= 0) {
      cp_async_commit();
      return;
    }
    const double* src = u + c0 * (3 * N3);
    if (GS) {
      const int* mp = cmap + c0 * (3 * N3);
      for (int e = tid; e < nc * 3 * N3; e += TH) cp_async8(sU + e, u + __ldg(mp + e));
    } else {
      async_copy_phase<TH>(sU + dst_shift(src), src, nc * 3 * N3, tid);
    }
    async_copy<TH>(sCo + buf * C::CSZ, coords + c0 * 24, nc * 24, tid);
    cp_async_commit();
  };
  // VAR bit 1: one batch per CTA (grid = batches) instead of the persistent
  // loop (cf. hex_neohookean3.cu ONESHOT)
  constexpr bool OS = (VAR & 2) != 0;
  int64_t batch = blockIdx.x;
  if (batch >= nbatch) return;
  prefetch(batch, 0);
  int it = 0;
  do {
  const int64_t cell0 = batch * (CPB * GROUPS) + grp * CPB;
  const int ncb = (int)((ncells - cell0) < CPB ? ((ncells - cell0) > 0 ? ncells - cell0 : 0)
                                                : CPB);
  cp_async_wait<0>();
  sync();
  const double* sC = sCo + (it & 1) * C::CSZ;
  const double* su = sU + (GS ? 0 : dst_shift(u + cell0 * (3 * N3)));

  // ---------------- forward x / y stages, per component -------------------
NEO_PRAGMA_A
  for (int a = 0; a < 3; ++a) {
    if (tid < CPB * NN) {
      const int c = tid / NN, r = tid - c * NN;
      double uu[N];
      const double* up = su + c * (3 * N3) + 3 * r + a;
#pragma unroll
      for (int i = 0; i < N; ++i) uu[i] = c < ncb ? up[3 * i * NN] : 0.0;
      double* xo = sX + c * C::XSZ + r;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        double b = T.B[q] * uu[0], d = T.D[q] * uu[0];
#pragma unroll
        for (int i = 1; i < N; ++i) {
          b = fma(T.B[i * M + q], uu[i], b);
          d = fma(T.D[i * M + q], uu[i], d);
        }
        xo[q * PX] = b;
        xo[XA + q * PX] = d;
      }
    }
    sync();
    if (!OS && a == 2 && batch + gridDim.x < nbatch) prefetch(batch + gridDim.x, (it & 1) ^ 1);
    if (tid < CPB * MN) {
      const int c = tid / MN, r = tid - c * MN;
      const int qx = r / N, iz = r - qx * N;
      const double* xi = sX + c * C::XSZ + qx * PX + iz;
      double a0[N], a1[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        a0[i] = xi[i * N];
        a1[i] = xi[XA + i * N];
      }
      double* yo = sY + c * C::YSZ + 3 * a * YA + (NYT ? qx * LZ : qx * M * LZ) + iz;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        double bb = T.B[q] * a0[0], bd = T.D[q] * a0[0], db = T.B[q] * a1[0];
#pragma unroll
        for (int i = 1; i < N; ++i) {
          bb = fma(T.B[i * M + q], a0[i], bb);
          bd = fma(T.D[i * M + q], a0[i], bd);
          db = fma(T.B[i * M + q], a1[i], db);
        }
        yo[q * QS] = bb;         // -> d/dz after z stage
        yo[YA + q * QS] = bd;    // -> d/dy
        yo[2 * YA + q * QS] = db;  // -> d/dx
      }
    }
    sync();
  }

  // ---------------- z-lines: gradients, constitutive flux, transposed z ----
  if (tid < CPB * MM) {
    const int c = tid / MM, r = tid - c * MM;
    const int r0 = r / M, r1 = r - r0 * M;
    const int qx = NYT ? r1 : r0, qy = NYT ? r0 : r1;
    double* line = sY + c * C::YSZ + r * LZ;   // component a, slot k: line[(3a+k)*YA + .]
    // (1) reference gradients, in place: slots (0,1,2) <- (d_z, d_y, d_x)
NEO_PRAGMA_A
    for (int a = 0; a < 3; ++a) {
      double bb[N], bd[N], db[N];
      double* l0 = line + 3 * a * YA;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        bb[i] = l0[i];
        bd[i] = l0[YA + i];
        db[i] = l0[2 * YA + i];
      }
#pragma unroll
      for (int q = 0; q < M; ++q) {
        double gz = T.D[q] * bb[0], gy = T.B[q] * bd[0], gx = T.B[q] * db[0];
#pragma unroll
        for (int i = 1; i < N; ++i) {
          gz = fma(T.D[i * M + q], bb[i], gz);
          gy = fma(T.B[i * M + q], bd[i], gy);
          gx = fma(T.B[i * M + q], db[i], gx);
        }
        l0[q] = gz;
        l0[YA + q] = gy;
        l0[2 * YA + q] = gx;
      }
    }
    // (2) pointwise neo-Hookean flux, in place
    HexLineAdj geo;
    geo.setup(sC + c * 24, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
    const double wxy = T.W[qx] * T.W[qy];
    // g[3a + l]: reference derivative l (0 x, 1 y, 2 z) of component a at q
    auto load_point = [&](int q, double g[9]) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int l = 0; l < 3; ++l) g[3 * a + l] = line[(3 * a + 2 - l) * YA + q];
    };
    // flux at point q from its gradients g (overwritten with the 9 fluxes)
    auto point_flux = [&](int q, double g[9]) {
      neo_point_flux(geo, T.Bc[M + q], wxy * T.W[q], mu, lam, g);
    };
    auto store_point = [&](int q, const double g[9]) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int l = 0; l < 3; ++l) line[(3 * a + 2 - l) * YA + q] = g[3 * a + l];   // slot 2 = x
    };
    if (VAR & 1) {
      // two points per iteration: two independent dependency chains
      // (adjugate -> F -> cof -> J -> log -> P -> flux) in flight per thread
#pragma unroll 1
      for (int q = 0; q + 1 < M; q += 2) {
        double g0[9], g1[9];
        load_point(q, g0);
        load_point(q + 1, g1);
        point_flux(q, g0);
        point_flux(q + 1, g1);
        store_point(q, g0);
        store_point(q + 1, g1);
      }
      if (M & 1) {
        double g0[9];
        load_point(M - 1, g0);
        point_flux(M - 1, g0);
        store_point(M - 1, g0);
      }
    } else {
#pragma unroll 1
      for (int q = 0; q < M; ++q) {
        double g0[9];
        load_point(q, g0);
        point_flux(q, g0);
        store_point(q, g0);
      }
    }
    // (3) transposed z, in place: slot 2 <- Bz^T f_x, 1 <- Bz^T f_y, 0 <- Dz^T f_z
NEO_PRAGMA_A
    for (int a = 0; a < 3; ++a) {
      double fz[M], fy[M], fx[M];
      double* l0 = line + 3 * a * YA;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        fz[q] = l0[q];
        fy[q] = l0[YA + q];
        fx[q] = l0[2 * YA + q];
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double sz = T.D[i * M] * fz[0], sy = T.B[i * M] * fy[0], sx = T.B[i * M] * fx[0];
#pragma unroll
        for (int q = 1; q < M; ++q) {
          sz = fma(T.D[i * M + q], fz[q], sz);
          sy = fma(T.B[i * M + q], fy[q], sy);
          sx = fma(T.B[i * M + q], fx[q], sx);
        }
        l0[i] = sz;
        l0[YA + i] = sy;
        l0[2 * YA + i] = sx;
      }
    }
  }
  sync();

  // ---------------- transposed y / x stages, per component ---------------
NEO_PRAGMA_A
  for (int a = 0; a < 3; ++a) {
    if (tid < CPB * MN) {
      const int c = tid / MN, r = tid - c * MN;
      const int qx = r / N, iz = r - qx * N;
      const double* yi = sY + c * C::YSZ + 3 * a * YA + (NYT ? qx * LZ : qx * M * LZ) + iz;
      double pz[M], py[M], px[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        pz[q] = yi[q * QS];
        py[q] = yi[YA + q * QS];
        px[q] = yi[2 * YA + q * QS];
      }
      double* xo = sX + c * C::XSZ + qx * PX + iz;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double r1 = T.B[i * M] * px[0];
        double r2 = fma(T.D[i * M], py[0], T.B[i * M] * pz[0]);
#pragma unroll
        for (int q = 1; q < M; ++q) {
          r1 = fma(T.B[i * M + q], px[q], r1);
          r2 = fma(T.D[i * M + q], py[q], r2);
          r2 = fma(T.B[i * M + q], pz[q], r2);
        }
        xo[i * N] = r1;
        xo[XA + i * N] = r2;
      }
    }
    sync();
    if (tid < CPB * NN) {
      const int c = tid / NN, r = tid - c * NN;
      if (c < ncb) {
        const double* xi = sX + c * C::XSZ + r;
        double p1[M], p2[M];
#pragma unroll
        for (int q = 0; q < M; ++q) {
          p1[q] = xi[q * PX];
          p2[q] = xi[XA + q * PX];
        }
        double* ap = A + (cell0 + c) * (3 * N3) + 3 * r + a;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double v = fma(T.D[i * M], p1[0], T.B[i * M] * p2[0]);
#pragma unroll
          for (int q = 1; q < M; ++q) {
            v = fma(T.D[i * M + q], p1[q], v);
            v = fma(T.B[i * M + q], p2[q], v);
          }
          if (GS) atomicAdd(A + __ldg(cmap + (cell0 + c) * (3 * N3) + 3 * (i * NN + r) + a), v);
          else ap[3 * i * NN] = v;
        }
      }
    }
    sync();
  }
  ++it;
  } while (!OS && (batch += gridDim.x) < nbatch);   // persistent batch loop
}

template <int N, int M, int CPB, bool GS = false, int WARPS = 0, int VAR = 0, int MINB = 0>
static int launch_neo(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                      const double* u, cudaStream_t s, const int* cmap = nullptr) {
  using C = NeoCfg<N, M, CPB>;
  constexpr int THREADS = WARPS ? 32 * WARPS : C::THREADS;
  constexpr size_t SMEM = WARPS ? WARPS * C::SMEM : C::SMEM;
  constexpr int CPBT = WARPS ? WARPS * CPB : CPB;
  auto k = hex_neohookean_kernel<N, M, CPB, GS, WARPS, VAR, MINB>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)k, THREADS, SMEM, "hex_neohookean", &sh, true))
    return rc_;
  const Tabs<N, M> T = make_tabs<N, M>(p);
  const int64_t nbatch = (ncells + CPBT - 1) / CPBT;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)((VAR & 2) || nbatch < resident ? nbatch : resident);
  if (grid > 0)
    k<<<grid, THREADS, SMEM, s>>>(T, p->params[0], p->params[1], ncells, coords, u, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_neohookean_kernel launch");
}

// cells per CTA for m = n + 1 (C4) per degree p (overridable for A/B builds;
// profiles/r01au_c4_cpb.jsonl: p = 2 16 -> 8 cells 0.199 -> 0.164 ms, p = 3
// 8 -> 4, p = 6 2 -> 1; smaller CTAs interleave the barrier-heavy phases)
#ifndef SFK_NEO_WARPS_DEFAULT
#define SFK_NEO_WARPS_DEFAULT 4   // warp-synchronous kernels at p <= 3 (A/B: SFK_NEO_WARPS;
                                  // profiles/r01bb_c4_warps.jsonl: ~3% at p = 2, 3)
#endif
#ifndef SFK_NEO_CPB_P1
#define SFK_NEO_CPB_P1 16
#endif
#ifndef SFK_NEO_CPB_P2
#define SFK_NEO_CPB_P2 8
#endif
#ifndef SFK_NEO_CPB_P3
#define SFK_NEO_CPB_P3 4
#endif
#ifndef SFK_NEO_CPB_P4
#define SFK_NEO_CPB_P4 3
#endif
#ifndef SFK_NEO_CPB_P5
#define SFK_NEO_CPB_P5 3
#endif
#ifndef SFK_NEO_CPB_P6
#define SFK_NEO_CPB_P6 1
#endif

#ifdef SFK_C4L_ONLY_N
// probe builds (tools/kernel_sweep.py c4l): one instantiation of the line kernel
}  // anonymous namespace
}  // namespace sfk
extern "C" int SFK_C4L_PROBE_ENTRY(const sfk_plan* p, int64_t ncells, double* A,
                                   const double* coords, const double* w0, void* stream) {
  if (p->n != SFK_C4L_ONLY_N || p->m != SFK_C4L_ONLY_N + 1)
    return sfk::fail(SFK_EUNSUPPORTED, "probe build: n=%d only", SFK_C4L_ONLY_N);
  return sfk::launch_neo<SFK_C4L_ONLY_N, SFK_C4L_ONLY_N + 1, SFK_C4LP_CPB, false, SFK_C4LP_WARPS,
                         SFK_C4LP_VAR, SFK_C4LP_MINB>(p, ncells, A, coords, w0,
                                                      (cudaStream_t)stream, nullptr);
}
namespace sfk {
#else
template <bool GS>
static int dispatch_neo(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                        const double* w0, cudaStream_t s, const int* cmap) {
  const int n = p->n, m = p->m;
  const int64_t ow = option(OPT_NEO_WARPS);   // 0: built-in, < 0: off
  const int warps = ow == 0 ? SFK_NEO_WARPS_DEFAULT : ow < 0 ? 0 : (int)ow;
  const int var = (int)option(OPT_NEO_CFG);
  // Defaults per degree (m = n + 1), each the fastest of its sweep or A/B run
  // (tools/kernel_sweep.py c4 / c4l; profiles named in brackets):
  //   p = 1     warp-synchronous line kernel, one-shot CTAs
  //   p = 2     the same, two warps per CTA                      [r02cq]
  //   p = 3     CTA-mode line kernel, 6 cells per 160-thread CTA,
  //             one-shot, 3 CTAs per SM, component loops unrolled [r02cq, r02ct]
  //   p = 4     CTA-mode line kernel, 3 cells per CTA, one-shot   [r02cp]
  //   p = 5, 6  component-parallel kernel (hex_neohookean3.cu),
  //             one-shot: 1.257 -> 1.006, 1.759 -> 1.691 ms       [r02cj]
  //             (global operator at p = 6: persistent two-point line
  //             kernel, 1.93 vs 2.17 ms with the atomic scatter)  [r02dj]
  // option neo_cfg: 1 two points per pointwise iteration everywhere, 2 nowhere,
  // 3 the component-parallel kernel wherever it is instantiated, 4 the line
  // kernel everywhere, 5 persistent warp-mode kernels at p <= 3, 6 the one-shot
  // line kernel at p = 4..6.
  if (m == n + 1 && (var == 3 || (var == 0 && (GS ? n == 6 : n >= 6)))) {
    const int rc = GS ? launch_hex_neohookean3_gs(p, ncells, cmap, w0, A, coords, s)
                      : launch_hex_neohookean3(p, ncells, A, coords, w0, s);
    if (rc != SFK_EUNSUPPORTED) return rc;
  }
  if (m == n + 1 && warps > 0 && n <= 4) {
    // warp-synchronous: 3 / 2 / 1 cells per warp at p = 1 / 2 / 3
    if (warps == 8) {
      if (n == 2) return launch_neo<2, 3, 3, GS, 8>(p, ncells, A, coords, w0, s, cmap);
      if (n == 3) return launch_neo<3, 4, 2, GS, 8>(p, ncells, A, coords, w0, s, cmap);
      if (n == 4) return launch_neo<4, 5, 1, GS, 8>(p, ncells, A, coords, w0, s, cmap);
    } else if (var == 5) {   // persistent CTAs (the default until r02cl)
      if (n == 2) return launch_neo<2, 3, 3, GS, 4>(p, ncells, A, coords, w0, s, cmap);
      if (n == 3) return launch_neo<3, 4, 2, GS, 4>(p, ncells, A, coords, w0, s, cmap);
      if (n == 4) return launch_neo<4, 5, 1, GS, 4>(p, ncells, A, coords, w0, s, cmap);
    } else if (var == 1) {
      if (n == 2) return launch_neo<2, 3, 3, GS, 4, 1>(p, ncells, A, coords, w0, s, cmap);
      if (n == 3) return launch_neo<3, 4, 2, GS, 4, 1>(p, ncells, A, coords, w0, s, cmap);
      if (n == 4) return launch_neo<4, 5, 1, GS, 4, 1>(p, ncells, A, coords, w0, s, cmap);
    } else {
      // one-shot CTAs (VAR bit 1): p = 2 0.1566 -> 0.1464, p = 3 0.3738 ->
      // 0.3359 ms (profiles/r02cl_c4_*.jsonl); then the shapes of the c4l sweep
      // (profiles/r02cq_c4l_sweep.jsonl): p = 2 0.1464 -> 0.1392, p = 3 0.3338
      // -> 0.2870 ms
      if (n == 2) return launch_neo<2, 3, 3, GS, 4, 2>(p, ncells, A, coords, w0, s, cmap);
      if (n == 3) return launch_neo<3, 4, 2, GS, 2, 2>(p, ncells, A, coords, w0, s, cmap);
      if (n == 4) return launch_neo<4, 5, 6, GS, 0, 2, 3>(p, ncells, A, coords, w0, s, cmap);
    }
  }
  // the line kernel with one-shot CTAs (VAR bit 1): default at p = 4; option
  // neo_cfg = 6 selects it at p = 5, 6 too (A/B against the component-parallel
  // default there)
  if (m == n + 1 && (var == 6 || (n == 5 && var == 0))) {
    switch (n) {
      case 5: return launch_neo<5, 6, SFK_NEO_CPB_P4, GS, 0, 2>(p, ncells, A, coords, w0, s, cmap);
      case 6: return launch_neo<6, 7, SFK_NEO_CPB_P5, GS, 0, 2>(p, ncells, A, coords, w0, s, cmap);
      case 7: return launch_neo<7, 8, SFK_NEO_CPB_P6, GS, 0, 3>(p, ncells, A, coords, w0, s, cmap);
      default: break;
    }
  }
  // two points per pointwise iteration: p = 6 1.831 -> 1.772 ms, neutral at
  // p = 2..5 (profiles/r02ao_c4_*); option neo_cfg = 2 turns it off at p = 6
  if (m == n + 1 && (var == 1 || (n == 7 && var != 2))) {
    switch (n) {
      case 5: return launch_neo<5, 6, SFK_NEO_CPB_P4, GS, 0, 1>(p, ncells, A, coords, w0, s, cmap);
      case 6: return launch_neo<6, 7, SFK_NEO_CPB_P5, GS, 0, 1>(p, ncells, A, coords, w0, s, cmap);
      case 7: return launch_neo<7, 8, SFK_NEO_CPB_P6, GS, 0, 1>(p, ncells, A, coords, w0, s, cmap);
      default: break;
    }
  }
  if (m == n + 1) {
    switch (n) {
      case 2: return launch_neo<2, 3, SFK_NEO_CPB_P1, GS>(p, ncells, A, coords, w0, s, cmap);
      case 3: return launch_neo<3, 4, SFK_NEO_CPB_P2, GS>(p, ncells, A, coords, w0, s, cmap);
      case 4: return launch_neo<4, 5, SFK_NEO_CPB_P3, GS>(p, ncells, A, coords, w0, s, cmap);
      case 5: return launch_neo<5, 6, SFK_NEO_CPB_P4, GS>(p, ncells, A, coords, w0, s, cmap);
      case 6: return launch_neo<6, 7, SFK_NEO_CPB_P5, GS>(p, ncells, A, coords, w0, s, cmap);
      case 7: return launch_neo<7, 8, SFK_NEO_CPB_P6, GS>(p, ncells, A, coords, w0, s, cmap);
      default: break;
    }
  } else if (m == n) {
    switch (n) {
      case 2: return launch_neo<2, 2, 16, GS>(p, ncells, A, coords, w0, s, cmap);
      case 3: return launch_neo<3, 3, 16, GS>(p, ncells, A, coords, w0, s, cmap);
      case 4: return launch_neo<4, 4, 8, GS>(p, ncells, A, coords, w0, s, cmap);
      default: break;
    }
  }
  return fail(SFK_EUNSUPPORTED,
              "neo-Hookean residual: no kernel for n=%d, m=%d (m==n+1 in 2..7 or m==n in 2..4)",
              n, m);
}

int launch_hex_neohookean(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          const double* w0, cudaStream_t s) {
  return dispatch_neo<false>(p, ncells, A, coords, w0, s, nullptr);
}

int launch_hex_neohookean_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                             double* y, const double* coords, cudaStream_t s) {
  return dispatch_neo<true>(p, ncells, y, coords, x, s, cmap);
}

#endif  // SFK_C4L_ONLY_N

}  // namespace sfk
