// Hex Q_p^3 neo-Hookean residual (BASELINE config C4), component-parallel
// kernel: three thread groups, one per displacement component.
//
// Math, reference mapping and operation order as hex_neohookean.cu (the
// builder FormSpec of SURVEY.md §8(a) row a17; every output is summed in the
// same order, so the two kernels agree bit for bit).  What changes is the
// thread mapping.  hex_neohookean.cu runs the scalar line schedule component
// by component on m^2 threads per cell; its resident warps are capped by the
// 9 m^3 doubles of gradient lines a cell keeps in shared memory (p = 4 / 5 /
// 6: 12 / 10 / 6 warps per SM), and a batch costs 14 CTA barriers.  Here a
// cell gets 3 m^2 threads:
//   * x, y, z contractions (and their transposes): thread (g, line) runs the
//     line of component g — all three components in flight at once, so the
//     x / y stages need one barrier each instead of three;
//   * pointwise stage: thread (g, z-line) takes the points q = g, g + 3, ...
//     of its z-line (all nine gradients of a point are needed together), with
//     its own copy of the line's adjugate polynomials.
// 7 barriers per batch; 16-20 warps per SM at p = 4..6 (96-118 registers in
// the one-shot form, see ONESHOT below).
#include "async_copy.cuh"
#include "hex_geometry.cuh"
#include "hex_neohookean_point.cuh"

namespace sfk {

// probe builds (tools/kernel_sweep.py): -DSFK_C4_ONLY_N=n instantiates that n
// alone with SFK_C4P_{CPB,MINB,PX,LZ,YPAD,NYT,ONESHOT} as given
#ifndef SFK_C4_ONLY_N
#define SFK_C4_ONLY_N 0
#endif
#ifndef SFK_C4P_PQ
#define SFK_C4P_PQ 1
#endif
#ifndef SFK_C4_PROBE_ENTRY
#define SFK_C4_PROBE_ENTRY sfk_c4_probe_eval
#endif
#if SFK_C4_ONLY_N
namespace {
#endif

template <int N, int M, int CPB, int PX_, int LZ_, int YPAD, bool NYT_>
struct Neo3Cfg {
  static constexpr int NN = N * N, MN = M * N, MM = M * M, N3 = N * N * N;
  static constexpr int THREADS = round_up(3 * CPB * MM, 32);
  static constexpr int PX = PX_;               // X-array q stride (>= n^2)
  static constexpr int LZ = LZ_;               // z-line stride (>= m)
  static constexpr bool NYT = NYT_;            // Y lines qy-major
  static constexpr int XA = M * PX;            // one X array (component, table)
  static constexpr int XSZ = 6 * XA;           // 3 components x (B, D)
  static constexpr int YA = MM * LZ;           // one Y array
  static constexpr int YSZ = 9 * YA + YPAD;
  static constexpr int USZ = round_up(CPB * 3 * N3 + 1, 2);
  static constexpr int CSZ = CPB * 24;
  static constexpr size_t SMEM =
      (size_t)(round_up(CPB * (XSZ + YSZ), 2) + USZ + 2 * CSZ) * sizeof(double);
  static_assert(PX >= NN && LZ >= M, "strides");
};

// ONESHOT: one batch per CTA (grid = batches) instead of a persistent loop —
// without the loop ptxas cannot hoist the stages' table constants out of it
// into vector registers (it then moves them back with R2UR at every use and
// the kernel needs 168+ registers at n = 7); the load latency is covered by
// the other resident CTAs.
template <int N, int M, int CPB, int PX_, int LZ_, int YPAD, bool NYT_, int MINB, bool GS,
          bool ONESHOT = false>
__global__ void __launch_bounds__(Neo3Cfg<N, M, CPB, PX_, LZ_, YPAD, NYT_>::THREADS, MINB)
hex_neohookean3_kernel(const __grid_constant__ Tabs<N, M> T, double mu, double lam,
                       int64_t ncells, const double* __restrict__ coords,
                       const double* __restrict__ u, double* __restrict__ A,
                       const int* __restrict__ cmap) {
  using C = Neo3Cfg<N, M, CPB, PX_, LZ_, YPAD, NYT_>;
  constexpr int NN = C::NN, MN = C::MN, MM = C::MM, N3 = C::N3, PX = C::PX, LZ = C::LZ;
  constexpr bool NYT = C::NYT;
  constexpr int QS = NYT ? M * LZ : LZ;
  constexpr int XA = C::XA, YA = C::YA, TH = C::THREADS;
  extern __shared__ __align__(16) double smem[];
  double* sX = smem;
  double* sY = sX + CPB * C::XSZ;
  double* sU = smem + round_up(CPB * (C::XSZ + C::YSZ), 2);
  double* sCo = sU + C::USZ;
  const int tid = (int)threadIdx.x;
  const int64_t nbatch = (ncells + CPB - 1) / CPB;

  auto prefetch = [&](int64_t bt, int buf) {
    const int64_t c0 = bt * CPB;
    const int nc = (int)((ncells - c0) < CPB ? (ncells - c0) : CPB);
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

  int64_t batch = blockIdx.x;
  if (batch >= nbatch) return;
  prefetch(batch, 0);
  int it = 0;
  do {
    const int64_t cell0 = batch * CPB;
    const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
    cp_async_wait<0>();
    __syncthreads();   // this batch's u / coords landed; the previous x^T stage is done with X
    const double* sC = sCo + (it & 1) * C::CSZ;
    const double* su = sU + (GS ? 0 : dst_shift(u + cell0 * (3 * N3)));

    // ---- x: thread (c, g, r = (iy, iz)): B and D along x of component g ----
    if (tid < 3 * CPB * NN) {
      const int c = tid / (3 * NN), cr = tid - c * (3 * NN);
      const int g = cr / NN, r = cr - g * NN;
      double uu[N];
      const double* up = su + c * (3 * N3) + 3 * r + g;
#pragma unroll
      for (int i = 0; i < N; ++i) uu[i] = c < ncb ? up[3 * i * NN] : 0.0;
      double* xo = sX + c * C::XSZ + 2 * g * XA + r;
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
    __syncthreads();
    // sU is free: the next batch's u (and coords, other buffer) stream in
    if (!ONESHOT && batch + gridDim.x < nbatch) prefetch(batch + gridDim.x, (it & 1) ^ 1);

    // ---- y: thread (c, g, qx, iz) ----------------------------------------
    if (tid < 3 * CPB * MN) {
      const int c = tid / (3 * MN), cr = tid - c * (3 * MN);
      const int g = cr / MN, r = cr - g * MN;
      const int qx = r / N, iz = r - qx * N;
      const double* xi = sX + c * C::XSZ + 2 * g * XA + qx * PX + iz;
      double a0[N], a1[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        a0[i] = xi[i * N];
        a1[i] = xi[XA + i * N];
      }
      double* yo = sY + c * C::YSZ + 3 * g * YA + (NYT ? qx * LZ : qx * M * LZ) + iz;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        double bb = T.B[q] * a0[0], bd = T.D[q] * a0[0], db = T.B[q] * a1[0];
#pragma unroll
        for (int i = 1; i < N; ++i) {
          bb = fma(T.B[i * M + q], a0[i], bb);
          bd = fma(T.D[i * M + q], a0[i], bd);
          db = fma(T.B[i * M + q], a1[i], db);
        }
        yo[q * QS] = bb;           // -> d/dz after the z stage
        yo[YA + q * QS] = bd;      // -> d/dy
        yo[2 * YA + q * QS] = db;  // -> d/dx
      }
    }
    __syncthreads();

    // z-line threads (c, g, r): component g's three lines of z-line r
    const bool zact = tid < 3 * CPB * MM;
    const int zc = tid / (3 * MM), zcr = tid - zc * (3 * MM);
    const int zg = zcr / MM, zr = zcr - zg * MM;
    double* line = sY + zc * C::YSZ + zr * LZ;   // slot (3a + k): line[(3a+k)*YA + .]

    // ---- z: reference gradients of component g, in place ------------------
    if (zact) {
      double bb[N], bd[N], db[N];
      double* l0 = line + 3 * zg * YA;
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
    __syncthreads();

    // ---- pointwise flux: points q = g, g + 3, ... of z-line r, in place ----
    if (zact) {
      const int r0 = zr / M, r1 = zr - r0 * M;
      const int qx = NYT ? r1 : r0, qy = NYT ? r0 : r1;
      HexLineAdj geo;
      geo.setup(sC + zc * 24, T.Bc[qx], T.Bc[M + qx], T.Bc[qy], T.Bc[M + qy]);
      const double wxy = T.W[qx] * T.W[qy];
      // (SFK_C4P_PQ > 1, probe builds: that many of the thread's points in flight —
      // measured slower, 128+ registers: profiles/r02ds_c4_pq.jsonl)
      constexpr int PQ = SFK_C4P_PQ;
#pragma unroll (PQ)
      for (int q = zg; q < M; q += 3) {
        double gq[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int l = 0; l < 3; ++l) gq[3 * a + l] = line[(3 * a + 2 - l) * YA + q];
        neo_point_flux(geo, T.Bc[M + q], wxy * T.W[q], mu, lam, gq);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int l = 0; l < 3; ++l) line[(3 * a + 2 - l) * YA + q] = gq[3 * a + l];
      }
    }
    __syncthreads();

    // ---- z^T of component g, in place: slot 2 <- Bz^T f_x, 1 <- Bz^T f_y, 0 <- Dz^T f_z
    if (zact) {
      double fz[M], fy[M], fx[M];
      double* l0 = line + 3 * zg * YA;
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
    __syncthreads();

    // ---- y^T: thread (c, g, qx, iz) ---------------------------------------
    if (tid < 3 * CPB * MN) {
      const int c = tid / (3 * MN), cr = tid - c * (3 * MN);
      const int g = cr / MN, r = cr - g * MN;
      const int qx = r / N, iz = r - qx * N;
      const double* yi = sY + c * C::YSZ + 3 * g * YA + (NYT ? qx * LZ : qx * M * LZ) + iz;
      double pz[M], py[M], px[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        pz[q] = yi[q * QS];
        py[q] = yi[YA + q * QS];
        px[q] = yi[2 * YA + q * QS];
      }
      double* xo = sX + c * C::XSZ + 2 * g * XA + qx * PX + iz;
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
    __syncthreads();

    // ---- x^T: thread (c, g, r = (iy, iz)) -> A ----------------------------
    if (tid < 3 * CPB * NN) {
      const int c = tid / (3 * NN), cr = tid - c * (3 * NN);
      const int g = cr / NN, r = cr - g * NN;
      if (c < ncb) {
        const double* xi = sX + c * C::XSZ + 2 * g * XA + r;
        double p1[M], p2[M];
#pragma unroll
        for (int q = 0; q < M; ++q) {
          p1[q] = xi[q * PX];
          p2[q] = xi[XA + q * PX];
        }
        double* ap = A + (cell0 + c) * (3 * N3) + 3 * r + g;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double v = fma(T.D[i * M], p1[0], T.B[i * M] * p2[0]);
#pragma unroll
          for (int q = 1; q < M; ++q) {
            v = fma(T.D[i * M + q], p1[q], v);
            v = fma(T.B[i * M + q], p2[q], v);
          }
          if (GS) atomicAdd(A + __ldg(cmap + (cell0 + c) * (3 * N3) + 3 * (i * NN + r) + g), v);
          else ap[3 * i * NN] = v;
        }
      }
    }
    ++it;
  } while (!ONESHOT && (batch += gridDim.x) < nbatch);
}

template <int N, int M, int CPB, int PX, int LZ, int YPAD, bool NYT, int MINB, bool GS,
          bool ONESHOT = false>
static int launch_neo3(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                       const double* u, cudaStream_t s, const int* cmap) {
  using C = Neo3Cfg<N, M, CPB, PX, LZ, YPAD, NYT>;
  auto k = hex_neohookean3_kernel<N, M, CPB, PX, LZ, YPAD, NYT, MINB, GS, ONESHOT>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)k, C::THREADS, C::SMEM, "hex_neohookean3", &sh, true))
    return rc_;
  const Tabs<N, M> T = make_tabs<N, M>(p);
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(ONESHOT || nbatch < resident ? nbatch : resident);
  if (grid > 0)
    k<<<grid, C::THREADS, C::SMEM, s>>>(T, p->params[0], p->params[1], ncells, coords, u, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_neohookean3_kernel launch");
}

#if SFK_C4_ONLY_N
}  // anonymous namespace
}  // namespace sfk
extern "C" int SFK_C4_PROBE_ENTRY(const sfk_plan* p, int64_t ncells, double* A,
                                  const double* coords, const double* w0, void* stream) {
  if (p->n != SFK_C4_ONLY_N || p->m != SFK_C4_ONLY_N + 1)
    return sfk::fail(SFK_EUNSUPPORTED, "probe build: n=%d only", SFK_C4_ONLY_N);
  return sfk::launch_neo3<SFK_C4_ONLY_N, SFK_C4_ONLY_N + 1, SFK_C4P_CPB, SFK_C4P_PX, SFK_C4P_LZ,
                          SFK_C4P_YPAD, SFK_C4P_NYT != 0, SFK_C4P_MINB, false,
                          SFK_C4P_ONESHOT != 0>(
      p, ncells, A, coords, w0, (cudaStream_t)stream, nullptr);
}
namespace sfk {
#else

// (cells per CTA, strides, min CTAs per SM, one-shot) per n: the fastest
// variant of tools/kernel_sweep.py c4 (profiles/r02cj_c4_sweep2.jsonl; the
// persistent form: r02cd_c4_sweep.jsonl).  One-shot CTAs win at every n: p = 4
// 0.650 (line kernel) -> 0.616 ms, p = 5 1.257 -> 1.013, p = 6 1.759 -> 1.701;
// the line kernel stays ahead at p = 2, 3 (0.156 / 0.369 vs 0.197 / 0.377).
template <bool GS>
static int dispatch_neo3(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s, const int* cmap) {
  if (p->m != p->n + 1) return SFK_EUNSUPPORTED;
  switch (p->n) {
    case 3: return launch_neo3<3, 4, 2, 9, 5, 0, false, 0, GS, true>(p, ncells, A, coords, w0, s, cmap);
    case 4: return launch_neo3<4, 5, 2, 20, 5, 0, false, 0, GS, true>(p, ncells, A, coords, w0, s, cmap);
    case 5: return launch_neo3<5, 6, 1, 37, 7, 0, true, 5, GS, true>(p, ncells, A, coords, w0, s, cmap);
    case 6: return launch_neo3<6, 7, 1, 38, 7, 0, true, 4, GS, true>(p, ncells, A, coords, w0, s, cmap);
    case 7: return launch_neo3<7, 8, 1, 55, 9, 0, false, 0, GS, true>(p, ncells, A, coords, w0, s, cmap);
    default: return SFK_EUNSUPPORTED;
  }
}

int launch_hex_neohookean3(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, cudaStream_t s) {
  return dispatch_neo3<false>(p, ncells, A, coords, w0, s, nullptr);
}

int launch_hex_neohookean3_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                              double* y, const double* coords, cudaStream_t s) {
  return dispatch_neo3<true>(p, ncells, y, coords, x, s, cmap);
}
#endif

}  // namespace sfk
