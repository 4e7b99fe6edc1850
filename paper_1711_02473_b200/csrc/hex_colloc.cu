// Hex GLL-collocated (weighted) Laplace action — BASELINE config C3
// (p = 4..16, kappa = w1 at the GLL points) and the collocated variant of
// registry `action_laplace` (--variant spectral_gll --quadrature
// collocated-gll).
//
// Reference: `action_form(REGISTRY['weighted_laplace'])` lowered with
// `default_quadrature(..., collocated_gll=True)` (forms.py:192-193, 235-243,
// 291-306).  The element is evaluated at its own nodes, so its value table
// is Delta(i, q) (elements.py:200-220) and delta cancellation
// (passes.py:336-388) leaves, per reference gradient component, ONE 1D
// D-contraction along that component's axis: 3 forward + 3 transposed
// contractions of N^4 each, instead of 8 + 8.
// kappa is a coefficient in the same GLL space: its value at point q is its
// dof q (the Delta property), so it enters pointwise, no contraction.
//
// B200 mapping: one CTA = CPB cells (1 cell for N >= 13: a 17^3 field is
// 38 KB).  Shared memory holds three N^3 arrays per cell with padded
// strides (tools/smem_pads.py):  U (u, later A), GX (d_x u, later f_x),
// GY (d_y u, later f_y), plus K (kappa) for the weighted form.  Phases:
//   1. cp.async u -> U and kappa -> K (kappa lands during phase 2)
//   2. each thread: one x-line (GX = Dx u) and one y-line (GY = Dy u)
//   3. each thread owns a z-line (x, y): d_z u in registers, then per point
//      geometry + kappa + flux, writing f_x, f_y in place and accumulating
//      A_z = Dz^T f_z in registers, stored over its own U line
//   4. x-lines: U += Dx^T f_x;   5. y-lines: U += Dy^T f_y
//   6. coalesced copy U -> A
#include <algorithm>
#include <type_traits>

#include "async_copy.cuh"
#include "hex_geometry.cuh"

namespace sfk {

// Probe builds (tools/c3_sweep.py): -DSFK_C3_ONLY_N=n compiles the dispatch of
// that n alone (no global-operator / warp-mode / DMMA variants) into a small
// library exporting sfk_c3_probe_eval, with SFK_C3P_{PERSIST,KG,SPLITZ,MINB,
// GEOM} (>= 0) overriding the per-n policies below and SFK_C3P_{CPB,SY,SX,CS}
// the launch shape and shared-memory strides.  Product builds leave all of
// them undefined.
#ifndef SFK_C3_ONLY_N
#define SFK_C3_ONLY_N 0
#endif
#ifndef SFK_C3P_PERSIST
#define SFK_C3P_PERSIST -1
#endif
#ifndef SFK_C3P_KG
#define SFK_C3P_KG -1
#endif
#ifndef SFK_C3P_SPLITZ
#define SFK_C3P_SPLITZ -1
#endif
#ifndef SFK_C3P_MINB
#define SFK_C3P_MINB -1
#endif
#ifndef SFK_C3P_GEOM
#define SFK_C3P_GEOM -1
#endif
#ifndef SFK_C3_PROBE_ENTRY
#define SFK_C3_PROBE_ENTRY sfk_c3_probe_eval
#endif
#if SFK_C3_ONLY_N
namespace {   // every variant object of a probe library keeps its own instances
#endif
__host__ __device__ constexpr int c3p(int n, int probe, int dflt) {
  return (SFK_C3_ONLY_N != 0 && n == SFK_C3_ONLY_N && probe >= 0) ? probe : dflt;
}

// Per-n policy (kg, splitz, min CTAs per SM, fuse) — the fastest variant of
// the two sweeps of tools/kernel_sweep.py c3 on the BASELINE batches
// (profiles/r02cb_c3_sweep.jsonl: layout, cells per CTA, persist, kg, splitz,
// min-blocks; profiles/r02ci_c3_sweep2.jsonl: + fuse); what each knob does is
// described where it is used below.
struct C3Policy {
  bool kg, splitz;
  int minb, fuse;
};
__host__ __device__ constexpr C3Policy c3_policy(int n, bool gs = false) {
  // the global-operator form (gather through the dof map, atomic scatter) has
  // its own optimum at four n (tools/kernel_sweep.py c3g,
  // profiles/r02du_c3g_sweep.jsonl: 6-13% over the E-vector form's policy)
  if (gs) {
    switch (n) {
      case 7: case 8: return {false, false, 8, 3};
      case 12: return {true, true, 4, 0};
      case 14: return {false, true, 2, 3};
      default: break;
    }
  }
  switch (n) {
    // n = 5, 6, 8: small CTAs from the wide cells-per-CTA sweep (r02dm_c3_cpb.jsonl)
    case 5: return {false, false, 0, 0};
    case 6: return {false, false, 4, 0};
    case 7: return {true, false, 0, 3};
    case 8: return {true, false, 8, 3};
    case 9: return {false, false, 0, 1};
    case 10: return {false, false, 4, 1};
    case 11: return {false, true, 3, 3};
    case 12: return {true, true, 3, 3};   // third sweep (r02cy_c3_sweep3): with the padded layout
    case 13: return {false, true, 2, 1};
    case 14: return {true, true, 3, 1};
    case 15: return {true, false, 2, 3};
    case 16: return {true, true, 1, 3};
    case 17: return {false, false, 0, 3};
    default: return {false, false, 2, 0};   // n <= 4
  }
}

template <int N>
struct TabsD {
  double D[N * N];
  double W[N];
  double Bc[2 * N];
};

// Persistent CTAs with the next batch's u / kappa / coords prefetched by
// cp.async while the current batch computes.  Round 1 kept it at n = 5 only
// (p = 4 0.1167 -> 0.1127 ms; at n = 6..11 the doubled u / kappa buffers cost
// occupancy, profiles/r01ck_*.jsonl); the round-2 sweep (tools/kernel_sweep.py,
// profiles/r02cb_c3_sweep.jsonl, r02dm_c3_cpb.jsonl) found small one-shot CTAs
// faster there too (0.1127 -> 0.0983 ms), so no n uses it by default.  SFK_COLLOC_PERSIST=n0 (A/B builds) makes every n <= n0 persistent.
#ifdef SFK_COLLOC_PERSIST
__host__ __device__ constexpr bool colloc_persist(int n) { return n <= SFK_COLLOC_PERSIST; }
#else
__host__ __device__ constexpr bool colloc_persist(int n) { return c3p(n, SFK_C3P_PERSIST, false); }
#endif

// KG: kappa read from global memory (through L1/L2) in the pointwise phase
// instead of being staged in shared memory — drops one of the four N^3
// arrays, i.e. more CTAs per SM where shared memory is the limit (round 1:
// n = 16, 139 -> 104 KB per CTA and two CTAs per SM; round 2: see c3_policy).
#ifdef SFK_COLLOC_KG
__host__ __device__ constexpr bool colloc_kg(int n, bool = false) { return n >= SFK_COLLOC_KG; }
#else
__host__ __device__ constexpr bool colloc_kg(int n, bool gs = false) {
  return c3p(n, SFK_C3P_KG, c3_policy(n, gs).kg);
}
#endif

template <int N, int CPB, int SY, int SX, int CS>
struct CollocCfg {
  static constexpr int NN = N * N;
  static constexpr int N3 = N * N * N;
  static constexpr int THREADS = round_up(CPB * NN, 32);
  static constexpr bool persist(int warps) { return warps == 0 && colloc_persist(N); }
  static constexpr size_t smem(bool weighted, int warps = 0, bool gs = false) {
    return persist(warps)
               ? (size_t)((weighted && !colloc_kg(N, gs) ? 6 : 4) * CPB * CS + 2 * CPB * 24) * sizeof(double)
               : (size_t)((weighted && !colloc_kg(N, gs) ? 4 : 3) * CPB * CS + CPB * 24) * sizeof(double);
  }
};

// Register policy (c3_policy.minb): 2 = __launch_bounds__(T, 2) (two CTAs per
// SM, no spills at that cap), 1 = (T, 1), 0 = (T) only — ptxas picks different
// register budgets for the last two (e.g. n = 16: 132 vs 254 registers).
// SPLITZ: phase 3 as three register-light passes over the thread's own lines
// instead of one fused loop (round 1, n = 12..15: p = 11 1.969 -> 1.664 ms,
// p = 13 3.803 -> 3.085, profiles/r01cf_*.jsonl; round 2 adds n = 11 and 16
// and drops 15, see c3_policy).
// SFK_COLLOC_SPLITZ=n0 (A/B builds) splits every n >= n0.
__host__ __device__ constexpr bool colloc_splitz(int n, bool gs = false) {
#ifdef SFK_COLLOC_SPLITZ
  return n >= SFK_COLLOC_SPLITZ;
#else
  return c3p(n, SFK_C3P_SPLITZ, c3_policy(n, gs).splitz);
#endif
}

// FUSE bit 0: phase 2 runs the thread's x-line and y-line together, bit 1:
// phases 4 / 5 compute Dx^T f_x and Dy^T f_y together (the y result waits in
// registers for the barrier) — the two contractions share the table D, so
// each constant (one LDCU per DFMA in the separate form) feeds two DFMAs.
// Same operations in the same order per output: bit-identical.
#ifndef SFK_C3P_FUSE
#define SFK_C3P_FUSE -1
#endif
__host__ __device__ constexpr int colloc_fuse(int n, bool gs = false) {
  return c3p(n, SFK_C3P_FUSE, c3_policy(n, gs).fuse);
}

// UQ: unroll factor of the split z phase's pointwise loop (1 = rolled; 2+:
// that many points' dependency chains in flight per thread, more registers)
#ifndef SFK_C3P_UQ
#define SFK_C3P_UQ -1
#endif
// (sweep: n = 16 4.046 -> 3.799 ms at 2; neutral or slower elsewhere, profiles/r02db_c3_uq.jsonl)
__host__ __device__ constexpr int colloc_uq(int n) { return c3p(n, SFK_C3P_UQ, n == 16 ? 2 : 1); }

__host__ __device__ constexpr int colloc_minb(int n, bool gs = false) {
#ifdef SFK_COLLOC_MINB
  if (SFK_COLLOC_MINB >= 0) return SFK_COLLOC_MINB;   // A/B builds (tools/build_variant.py)
#endif
  if (SFK_C3_ONLY_N != 0 && n == SFK_C3_ONLY_N && SFK_C3P_MINB >= 0) return SFK_C3P_MINB;
  return c3_policy(n, gs).minb;
}

// GS = true: global operator y += sum_c P_c^T A_c P_c x (SURVEY.md §8(f)
// item 1): u = x gathered through cmap[c][i] by per-element cp.async into the
// padded u layout, A = y scatter-added with fp64 atomics at the write-back.
// WARPS > 0: warp-synchronous mode for n <= 5 — each warp owns CPB whole
// cells (CPB * n^2 <= 32 lines) in its own shared-memory slice and the
// phases sync with __syncwarp instead of CTA barriers.
struct C3Arr {
  int sx, sy, cs;
};
// Per-n strides of the GX (x- and z-line accesses) and GY (y- and z-line)
// arrays (tools/c3_layout.py's half-warp bank model of this lane mapping).
// Measured same-box A/B against U's layout for both (profiles/r02aa_c3*):
// n = 6 GY 2.2% faster (kept); n = 7, 9, 11 within +-1% (the bank model's
// 20-30% fewer wavefronts do not show: C3 is not shared-memory bound), kept
// on U's layout.
__host__ __device__ constexpr C3Arr c3_gx(int n, int sx, int sy, int cs) {
  return (void)n, C3Arr{sx, sy, cs};
}
__host__ __device__ constexpr C3Arr c3_gy(int n, int sx, int sy, int cs) {
  return (n == 6 && cs >= 244) ? C3Arr{6, 41, 244} : C3Arr{sx, sy, cs};
}

template <int N, int CPB, int SY, int SX, int CS, bool WEIGHTED, bool GS = false, int WARPS = 0,
          bool C3_CONTIG = true>
__device__ __forceinline__ void colloc_body(const TabsD<N>& T, int64_t ncells,
                                            const double* __restrict__ coords,
                                            const double* __restrict__ u,
                                            const double* __restrict__ kappa,
                                            double* __restrict__ A,
                                            const int* __restrict__ cmap) {
  using C = CollocCfg<N, CPB, SY, SX, CS>;
  constexpr int NN = C::NN, N3 = C::N3;
  // GX / GY get their own strides (x/z- and y/z-accessed arrays, chosen by
  // tools/c3_layout.py's bank model); U keeps (SX, SY, CS)
  constexpr int GXX = c3_gx(N, SX, SY, CS).sx, GXY = c3_gx(N, SX, SY, CS).sy,
                GXC = c3_gx(N, SX, SY, CS).cs;
  constexpr int GYX = c3_gy(N, SX, SY, CS).sx, GYY = c3_gy(N, SX, SY, CS).sy,
                GYC = c3_gy(N, SX, SY, CS).cs;
  static_assert(GXC <= CS && GYC <= CS, "GX / GY must fit the CS-strided buffers");
  constexpr bool SPLITZ = colloc_splitz(N, GS);
  constexpr bool PERSIST = C::persist(WARPS);
  constexpr bool KG = WEIGHTED && colloc_kg(N, GS);
  constexpr bool CONTIG = SY == N && SX == NN && CS == N3 && C3_CONTIG;
  extern __shared__ double smem[];
  constexpr int TH = WARPS ? 32 : C::THREADS;
  static_assert(!WARPS || CPB * NN <= 32, "warp mode needs CPB * n^2 <= 32");
  const int grp = WARPS ? (int)(threadIdx.x >> 5) : 0;
  // one-shot:   [U][GX][GY][coords][K]
  // persistent: [U0][U1][GX][GY][coords0][coords1][K0][K1] (u, coords, kappa
  //             of the next batch stream in while the current one computes)
  double* base = smem + (size_t)grp * (C::smem(WEIGHTED, WARPS, GS) / sizeof(double));
  double* sGX = base + (PERSIST ? 2 : 1) * CPB * CS;
  double* sGY = sGX + CPB * CS;
  double* sC0 = sGY + CPB * CS;
  double* sK0 = sC0 + (PERSIST ? 2 : 1) * CPB * 24;

  const int tid = WARPS ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
  auto sync = [] { if (WARPS) __syncwarp(); else __syncthreads(); };

  // u (group 0) and kappa (group 1) stream into the padded shared layouts
  // with cp.async (one-shot mode: kappa is only needed by the pointwise
  // phase, so its latency hides behind phase 2).
  auto load = [&](int64_t cell0, int ncb, int buf) {
    double* sU = base + buf * (CPB * CS);
    double* sK = sK0 + buf * (CPB * CS);
    double* sC = sC0 + buf * (CPB * 24);
    if (PERSIST) {
      for (int i = tid; i < ncb * 24; i += TH) cp_async8(sC + i, coords + cell0 * 24 + i);
    } else {
      for (int i = tid; i < CPB * 24; i += TH)
        sC[i] = i < ncb * 24 ? __ldg(coords + cell0 * 24 + i) : 0.0;
    }
    // consecutive threads copy consecutive doubles (coalesced global reads);
    // unpadded layouts (CONTIG) are the global order itself: 16-byte copies
    // without the per-element (c, x, y, z) decomposition
    const double* ug = u + cell0 * N3;
    if (CONTIG && !GS) {
      async_copy<TH>(sU, ug, ncb * N3, tid);
    } else {
      for (int i = tid; i < ncb * N3; i += TH) {
        const int c = i / N3, r = i - c * N3;
        const int x = r / NN, yz = r - x * NN, y = yz / N, z = yz - y * N;
        cp_async8(sU + c * CS + x * SX + y * SY + z, GS ? u + __ldg(cmap + cell0 * N3 + i) : ug + i);
      }
    }
    cp_async_commit();
    if (WEIGHTED && !KG) {
      const double* kg = kappa + cell0 * N3;
      if (CONTIG) {
        async_copy<TH>(sK, kg, ncb * N3, tid);
      } else {
        for (int i = tid; i < ncb * N3; i += TH) {
          const int c = i / N3, r = i - c * N3;
          const int x = r / NN, yz = r - x * NN, y = yz / N, z = yz - y * N;
          cp_async8(sK + c * CS + x * SX + y * SY + z, kg + i);
        }
      }
      cp_async_commit();
    }
  };

  auto compute = [&](int64_t cell0, int ncb, int buf) {
    double* sU = base + buf * (CPB * CS);
    const double* sK = sK0 + buf * (CPB * CS);
    const double* sC = sC0 + buf * (CPB * 24);
    const bool act = tid < CPB * NN;
    const int c = tid / NN, r = tid - (tid / NN) * NN;
    const int a = r / N, b = r - (r / N) * N;
    const int cb = c * CS;

    // ---- phase 2: x-line (y=a, z=b) and y-line (x=a, z=b) ---------------
    constexpr int FUSE = colloc_fuse(N, GS);
    if ((FUSE & 1) && act) {
      double ux[N], uy[N];
  #pragma unroll
      for (int i = 0; i < N; ++i) {
        ux[i] = sU[cb + i * SX + a * SY + b];
        uy[i] = sU[cb + a * SX + i * SY + b];
      }
  #pragma unroll
      for (int q = 0; q < N; ++q) {
        double gx = T.D[q] * ux[0], gy = T.D[q] * uy[0];
  #pragma unroll
        for (int i = 1; i < N; ++i) {
          gx = fma(T.D[i * N + q], ux[i], gx);
          gy = fma(T.D[i * N + q], uy[i], gy);
        }
        sGX[c * GXC + q * GXX + a * GXY + b] = gx;
        sGY[c * GYC + a * GYX + q * GYY + b] = gy;
      }
    }
    if (!(FUSE & 1) && act) {
      double ul[N];
  #pragma unroll
      for (int i = 0; i < N; ++i) ul[i] = sU[cb + i * SX + a * SY + b];
  #pragma unroll
      for (int q = 0; q < N; ++q) {
        double g = T.D[q] * ul[0];
  #pragma unroll
        for (int i = 1; i < N; ++i) g = fma(T.D[i * N + q], ul[i], g);
        sGX[c * GXC + q * GXX + a * GXY + b] = g;
      }
  #pragma unroll
      for (int i = 0; i < N; ++i) ul[i] = sU[cb + a * SX + i * SY + b];
  #pragma unroll
      for (int q = 0; q < N; ++q) {
        double g = T.D[q] * ul[0];
  #pragma unroll
        for (int i = 1; i < N; ++i) g = fma(T.D[i * N + q], ul[i], g);
        sGY[c * GYC + a * GYX + q * GYY + b] = g;
      }
    }
    if (WEIGHTED && !PERSIST) cp_async_wait<0>();   // kappa copies of this thread landed
    sync();                     // ... and everybody's are visible

    // ---- phase 3: z-line (x=a, y=b): d_z u, flux, A_z = Dz^T f_z ---------
    // SPLITZ (large n): three register-light passes over the thread's own
    // lines instead of one fused loop (whose d_z input line + A_z accumulators
    // + geometry needed 2n + 24 live doubles: 254 registers at n = 14, one CTA
    // per SM): (a) d_z u written over the U line, (b) pointwise flux in place
    // on the GX / GY / U lines, (c) Dz^T f_z over the U line.  Same operations
    // in the same order per output (bit-identical to the fused loop).
    if (SPLITZ && act) {
      const int base = cb + a * SX + b * SY;
      const int bx = c * GXC + a * GXX + b * GXY, by = c * GYC + a * GYX + b * GYY;
      {
        double ul[N];
  #pragma unroll
        for (int i = 0; i < N; ++i) ul[i] = sU[base + i];
  #pragma unroll
        for (int q = 0; q < N; ++q) {
          double gz = T.D[q] * ul[0];
  #pragma unroll
          for (int i = 1; i < N; ++i) gz = fma(T.D[i * N + q], ul[i], gz);
          sU[base + q] = gz;
        }
      }
      {
        HexLineAdj geo;
        geo.setup(sC + c * 24, T.Bc[a], T.Bc[N + a], T.Bc[b], T.Bc[N + b]);
        const double wxy = T.W[a] * T.W[b];
        const double* kp = KG ? kappa + (cell0 + (c < ncb ? c : 0)) * N3 + a * NN + b * N : sK + base;
  #pragma unroll (colloc_uq(N))
        for (int q = 0; q < N; ++q) {
          double gx = sGX[bx + q], gy = sGY[by + q], gz = sU[base + q];
          double r0[3], r1[3], r2[3];
          const double det = geo.adj(T.Bc[N + q], r0, r1, r2);
          double s = (wxy * T.W[q]) * rcp64(fabs(det));
          if (WEIGHTED) s *= KG ? __ldg(kp + q) : kp[q];
          laplace_flux(r0, r1, r2, s, gx, gy, gz);
          sGX[bx + q] = gx;
          sGY[by + q] = gy;
          sU[base + q] = gz;
        }
      }
      {
        double fz[N];
  #pragma unroll
        for (int q = 0; q < N; ++q) fz[q] = sU[base + q];
  #pragma unroll
        for (int i = 0; i < N; ++i) {
          double az = T.D[i * N] * fz[0];
  #pragma unroll
          for (int q = 1; q < N; ++q) az = fma(T.D[i * N + q], fz[q], az);
          sU[base + i] = az;
        }
      }
    }
    if (!SPLITZ && act) {
      const int base = cb + a * SX + b * SY;
      const int bx = c * GXC + a * GXX + b * GXY, by = c * GYC + a * GYX + b * GYY;
      double ul[N], az[N];
  #pragma unroll
      for (int i = 0; i < N; ++i) {
        ul[i] = sU[base + i];
        az[i] = 0.0;
      }
      // precomputed adjugate polynomials (hex_geometry.cuh) except at n = 15, 16,
      // where their 9 extra registers per thread cost more than they save
      // (same-box A/B, profiles/r01ai_*)
      constexpr bool GEOM = c3p(N, SFK_C3P_GEOM, N == 15 || N == 16);
      using Geo = typename std::conditional<GEOM, HexLineGeom, HexLineAdj>::type;
      Geo geo;
      geo.setup(sC + c * 24, T.Bc[a], T.Bc[N + a], T.Bc[b], T.Bc[N + b]);
      const double wxy = T.W[a] * T.W[b];
      const double* kp = KG ? kappa + (cell0 + (c < ncb ? c : 0)) * N3 + a * NN + b * N : sK + base;
  #pragma unroll
      for (int q = 0; q < N; ++q) {
        double gz = T.D[q] * ul[0];
  #pragma unroll
        for (int i = 1; i < N; ++i) gz = fma(T.D[i * N + q], ul[i], gz);
        double gx = sGX[bx + q], gy = sGY[by + q];
        double r0[3], r1[3], r2[3];
        double det;
        if constexpr (GEOM) det = geo.adj(T.Bc[q], T.Bc[N + q], r0, r1, r2);
        else det = geo.adj(T.Bc[N + q], r0, r1, r2);
        double s = (wxy * T.W[q]) * rcp64(fabs(det));
        if (WEIGHTED) s *= KG ? __ldg(kp + q) : kp[q];
        laplace_flux(r0, r1, r2, s, gx, gy, gz);
        sGX[bx + q] = gx;
        sGY[by + q] = gy;
  #pragma unroll
        for (int i = 0; i < N; ++i) az[i] = fma(T.D[i * N + q], gz, az[i]);
      }
  #pragma unroll
      for (int i = 0; i < N; ++i) sU[base + i] = az[i];
    }
    sync();

    if (FUSE & 2) {
      // ---- phases 4 + 5 fused: both transposed contractions share D -------
      double sy[N];
      if (act) {
        double fx[N], fy[N];
  #pragma unroll
        for (int q = 0; q < N; ++q) {
          fx[q] = sGX[c * GXC + q * GXX + a * GXY + b];
          fy[q] = sGY[c * GYC + a * GYX + q * GYY + b];
        }
  #pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = T.D[i * N] * fx[0];
          double t = T.D[i * N] * fy[0];
  #pragma unroll
          for (int q = 1; q < N; ++q) {
            s = fma(T.D[i * N + q], fx[q], s);
            t = fma(T.D[i * N + q], fy[q], t);
          }
          sU[cb + i * SX + a * SY + b] += s;
          sy[i] = t;
        }
      }
      sync();
      if (act) {
  #pragma unroll
        for (int i = 0; i < N; ++i) sU[cb + a * SX + i * SY + b] += sy[i];
      }
      sync();
    } else {
    // ---- phase 4: x-lines (y=a, z=b): U += Dx^T f_x ----------------------
    if (act) {
      double fl[N];
  #pragma unroll
      for (int q = 0; q < N; ++q) fl[q] = sGX[c * GXC + q * GXX + a * GXY + b];
  #pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = T.D[i * N] * fl[0];
  #pragma unroll
        for (int q = 1; q < N; ++q) s = fma(T.D[i * N + q], fl[q], s);
        sU[cb + i * SX + a * SY + b] += s;
      }
    }
    sync();

    // ---- phase 5: y-lines (x=a, z=b): U += Dy^T f_y ----------------------
    if (act) {
      double fl[N];
  #pragma unroll
      for (int q = 0; q < N; ++q) fl[q] = sGY[c * GYC + a * GYX + q * GYY + b];
  #pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = T.D[i * N] * fl[0];
  #pragma unroll
        for (int q = 1; q < N; ++q) s = fma(T.D[i * N + q], fl[q], s);
        sU[cb + a * SX + i * SY + b] += s;
      }
    }
    sync();

    }

    {
      // coalesced write-back: consecutive threads take consecutive elements of
      // the batch; the (c, x, y, z) decomposition is incremental per thread
      double* ag = A + cell0 * N3;
      if (CONTIG && !GS) {
        const int n = ncb * N3;
        if (((reinterpret_cast<uintptr_t>(ag) | reinterpret_cast<uintptr_t>(sU)) & 15) == 0) {
          for (int i = tid; i < n / 2; i += TH)
            reinterpret_cast<double2*>(ag)[i] = reinterpret_cast<const double2*>(sU)[i];
          if ((n & 1) && tid == 0) ag[n - 1] = sU[n - 1];
        } else {
          for (int i = tid; i < n; i += TH) ag[i] = sU[i];
        }
      } else
      for (int i = tid; i < ncb * N3; i += TH) {
        const int cc = i / N3, rr = i - cc * N3;
        const int x = rr / NN, yz = rr - x * NN, y = yz / N, z = yz - y * N;
        if (GS) atomicAdd(A + __ldg(cmap + cell0 * N3 + i), sU[cc * CS + x * SX + y * SY + z]);
        else ag[i] = sU[cc * CS + x * SX + y * SY + z];
      }
    }
  };

  const int64_t ngroups = (ncells + CPB - 1) / CPB;   // cell batches
  if (PERSIST) {
    int64_t bt = blockIdx.x;
    auto nb_of = [&](int64_t bb) {
      const int64_t rem = ncells - bb * CPB;
      return rem < CPB ? (int)rem : CPB;
    };
    if (bt < ngroups) load(bt * CPB, nb_of(bt), 0);
    for (int k = 0; bt < ngroups; bt += gridDim.x, ++k) {
      const int cur = k & 1;
      cp_async_wait<0>();
      sync();   // this batch landed; the previous batch's write-back is done
      if (bt + gridDim.x < ngroups) load((bt + gridDim.x) * CPB, nb_of(bt + gridDim.x), cur ^ 1);
      compute(bt * CPB, nb_of(bt), cur);
    }
  } else {
    const int64_t cell0 = ((int64_t)blockIdx.x * (WARPS ? WARPS : 1) + grp) * CPB;
    const int64_t rem = ncells - cell0;
    const int ncb = rem < CPB ? (int)rem : CPB;
    load(cell0, ncb, 0);
    if (WEIGHTED && !KG) cp_async_wait<1>();
    else cp_async_wait<0>();
    sync();
    compute(cell0, ncb, 0);
  }
  (void)ngroups;
}

template <int N, int CPB, int SY, int SX, int CS, bool WEIGHTED, int MINB, bool GS, int WARPS,
          int VAR>
__global__ void __launch_bounds__(WARPS ? 32 * WARPS : CollocCfg<N, CPB, SY, SX, CS>::THREADS, MINB)
hex_colloc_action_kernel(const __grid_constant__ TabsD<N> T, int64_t ncells,
                         const double* __restrict__ coords, const double* __restrict__ u,
                         const double* __restrict__ kappa, double* __restrict__ A,
                         const int* __restrict__ cmap) {
  colloc_body<N, CPB, SY, SX, CS, WEIGHTED, GS, WARPS, (VAR & 1) == 0>(T, ncells, coords, u, kappa,
                                                                      A, cmap);
}

template <int N, int CPB, int SY, int SX, int CS, bool WEIGHTED, bool GS, int WARPS, int VAR>
__global__ void __launch_bounds__(WARPS ? 32 * WARPS : CollocCfg<N, CPB, SY, SX, CS>::THREADS)
hex_colloc_action_kernel_free(const __grid_constant__ TabsD<N> T, int64_t ncells,
                              const double* __restrict__ coords, const double* __restrict__ u,
                              const double* __restrict__ kappa, double* __restrict__ A,
                              const int* __restrict__ cmap) {
  colloc_body<N, CPB, SY, SX, CS, WEIGHTED, GS, WARPS, (VAR & 1) == 0>(T, ncells, coords, u, kappa,
                                                                      A, cmap);
}

template <int N, int CPB, int SY, int SX, int CS, bool WEIGHTED, bool GS, int WARPS, int VAR>
static auto colloc_kernel() {
  constexpr int mb = colloc_minb(N, GS);
  if constexpr (mb == 0)
    return hex_colloc_action_kernel_free<N, CPB, SY, SX, CS, WEIGHTED, GS, WARPS, VAR>;
  else return hex_colloc_action_kernel<N, CPB, SY, SX, CS, WEIGHTED, mb, GS, WARPS, VAR>;
}

// VAR bit 0 (option c3_cfg = 1, A/B only): the per-element staging copies
// even where the shared layout is unpadded
template <int N, int CPB, int SY, int SX, int CS, bool GS, int WARPS, int VAR>
static int launch_nv(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* u, const double* kappa, cudaStream_t s, const int* cmap) {
  using C = CollocCfg<N, CPB, SY, SX, CS>;
  constexpr int G = WARPS ? WARPS : 1;                 // cell groups per CTA
  constexpr int THREADS = WARPS ? 32 * WARPS : C::THREADS;
  TabsD<N> T;
  for (int i = 0; i < N * N; ++i) T.D[i] = p->D[i];
  for (int q = 0; q < N; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[N + q] = p->Bc[N + q];
  }
  int64_t grid = (ncells + CPB * G - 1) / (CPB * G);
  // persistent mode: one resident wave of CTAs looping over the batches
  LaunchShape sh;
  if (kappa) {
    auto k = colloc_kernel<N, CPB, SY, SX, CS, true, GS, WARPS, VAR>();
    const size_t sm = G * C::smem(true, WARPS, GS);
    if (const int rc_ = kernel_shape((const void*)k, THREADS, sm, "hex_colloc", &sh)) return rc_;
    if (C::persist(WARPS)) grid = std::min<int64_t>(grid, sh.resident());
    if (grid > 0) k<<<(unsigned)grid, THREADS, sm, s>>>(T, ncells, coords, u, kappa, A, cmap);
  } else {
#if SFK_C3_ONLY_N
    return fail(SFK_EUNSUPPORTED, "probe build: weighted form only");
#else
    auto k = colloc_kernel<N, CPB, SY, SX, CS, false, GS, WARPS, VAR>();
    const size_t sm = G * C::smem(false, WARPS, GS);
    if (const int rc_ = kernel_shape((const void*)k, THREADS, sm, "hex_colloc", &sh)) return rc_;
    if (C::persist(WARPS)) grid = std::min<int64_t>(grid, sh.resident());
    if (grid > 0) k<<<(unsigned)grid, THREADS, sm, s>>>(T, ncells, coords, u, nullptr, A, cmap);
#endif
  }
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_colloc_action_kernel launch");
}

template <int N, int CPB, int SY, int SX, int CS, bool GS = false, int WARPS = 0>
static int launch_n(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                    const double* u, const double* kappa, cudaStream_t s,
                    const int* cmap = nullptr) {
  // unpadded layouts at n = 3, 5, 13 stage with 16-byte copies: p = 4
  // 0.1157 -> 0.1147, p = 12 1.928 -> 1.894 ms; at n = 15, 17 they measured
  // 0.3-0.8% slower and keep the per-element copies (profiles/r02ap_c3_*)
  if constexpr (SY == N && SX == N * N && CS == N * N * N && !GS) {
    if (N >= 15 || option(OPT_C3_CFG) == 1)
      return launch_nv<N, CPB, SY, SX, CS, GS, WARPS, 1>(p, ncells, A, coords, u, kappa, s, cmap);
  }
  return launch_nv<N, CPB, SY, SX, CS, GS, WARPS, 0>(p, ncells, A, coords, u, kappa, s, cmap);
}

#ifndef SFK_COLLOC_WARPS_DEFAULT
#define SFK_COLLOC_WARPS_DEFAULT 0   // warp mode measured slower at p = 4 (profiles/r01bd_c3_warps.jsonl)
#endif

// cells per CTA at n = 10, 12 (overridable for A/B builds)
#ifndef SFK_COLLOC_CPB10
#define SFK_COLLOC_CPB10 1
#endif
#ifndef SFK_COLLOC_CPB12
#define SFK_COLLOC_CPB12 1
#endif

template <bool GS>
static int dispatch_colloc(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, const double* w1, cudaStream_t s,
                           const int* cmap) {
  if (p->n != p->m)
    return fail(SFK_EINVAL, "collocated action needs n_q1d == n_dof1d (got %d, %d)", p->n, p->m);
#if SFK_C3_ONLY_N
  if (p->n != SFK_C3_ONLY_N)
    return fail(SFK_EUNSUPPORTED, "probe build: n=%d only (got %d)", SFK_C3_ONLY_N, p->n);
  return launch_n<SFK_C3_ONLY_N, SFK_C3P_CPB, SFK_C3P_SY, SFK_C3P_SX, SFK_C3P_CS, GS>(
      p, ncells, A, coords, w0, w1, s, cmap);
#else
  // warp-synchronous variants for n <= 5 (option colloc_warps = warps per CTA)
  const int64_t ocw = option(OPT_COLLOC_WARPS);   // 0: built-in, < 0: off
  const int cw = ocw == 0 ? SFK_COLLOC_WARPS_DEFAULT : ocw < 0 ? 0 : (int)ocw;
  if (cw > 0) {
    switch (p->n) {
      case 2: return launch_n<2, 8, 2, 5, 12, GS, 8>(p, ncells, A, coords, w0, w1, s, cmap);
      case 3: return launch_n<3, 3, 3, 9, 27, GS, 8>(p, ncells, A, coords, w0, w1, s, cmap);
      case 4: return launch_n<4, 2, 4, 19, 76, GS, 8>(p, ncells, A, coords, w0, w1, s, cmap);
      case 5: return launch_n<5, 1, 5, 25, 125, GS, 8>(p, ncells, A, coords, w0, w1, s, cmap);
      default: break;
    }
  }
  // (N, cells/CTA, SY, SX, CS): strides from tools/smem_pads.py; the round-2
  // sweep moved n = 6, 9, 10, 11, 14 to the unpadded layout (smaller CTAs,
  // 16-byte staging: more CTAs per SM beat the conflict-free strides) and
  // n = 10, 11 to one cell per CTA (profiles/r02cb_c3_sweep.jsonl); a wider
  // cells-per-CTA sweep at n = 5..9 (r02dm_c3_cpb.jsonl) then moved n = 5, 6, 8
  // to 128- / 128- / 64-thread CTAs (p = 4, 5, 7: 0.1045 / 0.1685 / 0.3686 ->
  // 0.0983 / 0.1577 / 0.3338 ms)
  switch (p->n) {
    case 2: return launch_n<2, 16, 2, 5, 12, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 3: return launch_n<3, 16, 3, 9, 27, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 4: return launch_n<4, 8, 4, 19, 76, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 5: return launch_n<5, 5, 5, 25, 125, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 6: return launch_n<6, 3, 6, 36, 216, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 7: return launch_n<7, GS ? 1 : 5, 7, 52, 369, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 8: return launch_n<8, 1, 9, 72, 576, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 9: return launch_n<9, 3, 9, 81, 729, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 10: return launch_n<10, SFK_COLLOC_CPB10, 10, 100, 1000, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 11: return launch_n<11, 1, 11, 121, 1331, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 12: return launch_n<12, SFK_COLLOC_CPB12, 13, 156, 1872, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 13: return launch_n<13, 1, 13, 169, 2197, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 14: return launch_n<14, 1, 14, 196, 2744, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 15: return launch_n<15, 1, 15, 225, 3375, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 16: return launch_n<16, 1, 17, 272, 4352, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    case 17: return launch_n<17, 1, 17, 289, 4913, GS>(p, ncells, A, coords, w0, w1, s, cmap);
    default:
      return fail(SFK_EUNSUPPORTED, "collocated hex action: n=%d outside [2,17]", p->n);
  }
#endif
}

#if SFK_C3_ONLY_N
}  // anonymous namespace
}  // namespace sfk
// the probe object's only entry point: p is a plan made by the product
// library (a plain host struct), all buffers device pointers as in sfk_eval
#ifndef SFK_C3P_GS
#define SFK_C3P_GS 0
#endif
#if SFK_C3P_GS
// global-operator form: w0 = x (global vector), A = y (accumulated), cmap =
// the cell -> global dof map
extern "C" int SFK_C3_PROBE_ENTRY(const sfk_plan* p, int64_t ncells, double* A,
                                 const double* coords, const double* w0, const double* w1,
                                 const int* cmap, void* stream) {
  return sfk::dispatch_colloc<true>(p, ncells, A, coords, w0, w1, (cudaStream_t)stream, cmap);
}
#else
extern "C" int SFK_C3_PROBE_ENTRY(const sfk_plan* p, int64_t ncells, double* A,
                                 const double* coords, const double* w0, const double* w1,
                                 void* stream) {
  return sfk::dispatch_colloc<false>(p, ncells, A, coords, w0, w1, (cudaStream_t)stream, nullptr);
}
#endif
namespace sfk {
#else
int launch_hex_colloc_action(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                             const double* w0, const double* w1, cudaStream_t s) {
  // option c3_tc = 1: CTA-wide DMMA kernels at n = 8, 12, 16 (hex_colloc_tc.cu,
  // slower); 2: n = 8 on the one-warp-per-cell DMMA kernel (hex_action_tc8c.cu)
  const int rc = launch_hex_colloc_tc(p, ncells, A, coords, w0, w1, s);
  if (rc != SFK_EUNSUPPORTED) return rc;
  if (p->n == 8 && p->m == 8 && option(OPT_C3_TC) == 2)
    return launch_hex_colloc_tc8c(p, ncells, A, coords, w0, w1, s);
  return dispatch_colloc<false>(p, ncells, A, coords, w0, w1, s, nullptr);
}

int launch_hex_colloc_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                         double* y, const double* coords, const double* kappa, cudaStream_t s) {
  return dispatch_colloc<true>(p, ncells, y, coords, x, kappa, s, cmap);
}
#endif

}  // namespace sfk
