// Hex Q_1 Laplace action, one thread per cell — BASELINE C2 at p = 1.
//
// Same math and reference mapping as the other C2 kernels (forms.py:186-189,
// 235-243; passes.py:672-743 schedule; scheduling.py:617-738 emitted
// kernel).  At n = m = 2 a cell is 8 dofs and 8 points: the whole
// sum-factorised pipeline (x, y, z contractions, per-point geometry and
// flux, transposed contractions) fits in one thread's registers, so there
// is no line re-dealing, no shared-memory transposes and no barrier per
// stage.  The CTA stages its cells' coords and u through shared memory with
// 16-byte cp.async (coalesced; per-cell strides padded to 26/10 doubles so
// the per-thread 128-bit reads are bank-conflict free) and each thread
// writes its 8 outputs with four 16-byte vector stores.  128 cells per CTA,
// up to 3 CTAs per SM (166 registers, no spills).
#include "async_copy.cuh"
#include "hex_geometry.cuh"

#ifndef SFK_P1_MINB
#define SFK_P1_MINB 3   // CTAs per SM the register budget allows (A/B builds)
#endif

namespace sfk {

namespace p1 {
constexpr int CS = 26;               // padded coords stride (24 used)
constexpr int US = 10;               // padded u stride (8 used)
constexpr size_t smem(int cpb) { return (size_t)cpb * (CS + US) * sizeof(double); }
}  // namespace p1

// GS = true: global operator y += sum_c P_c^T A_c P_c x (SURVEY.md §8(f)
// item 1): u = x gathered through cmap[c][0..7], A = y scatter-added with
// fp64 atomics.
// PERSIST: a resident grid of CTAs loops over the batches with two staging
// buffers — the next batch's coords / u stream in (cp.async) behind the
// current batch's arithmetic (the one-shot form waits for its loads with
// nothing else to do: 22% long-scoreboard stalls at 12 warps per SM,
// profiles/r02cm_p1.md).  The tables are 2 x 2: nothing for ptxas to hoist.
template <bool GS, int CPB = 128, int MINB = SFK_P1_MINB, bool PERSIST = false>
__global__ void __launch_bounds__(CPB, MINB)
hex_laplace_action_p1(const __grid_constant__ Tabs<2, 2> T, int64_t ncells,
                      const double* __restrict__ coords, const double* __restrict__ u,
                      double* __restrict__ A, const int* __restrict__ cmap = nullptr) {
  using p1::CS;
  using p1::US;
  extern __shared__ __align__(16) double smem[];
  constexpr int BUF = CPB * (CS + US);   // doubles per staging buffer
  const int tid = threadIdx.x;
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  auto stage = [&](int64_t bt, int buf) {
    double* sC = smem + buf * BUF;
    double* sU = sC + CPB * CS;
    const int64_t cell0 = bt * CPB;
    const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
    // 16-byte chunks: coords 12 per cell, u 4 per cell (both 16B-aligned
    // per cell when the bases are; otherwise fall back to 8-byte copies)
    const double* cg = coords + cell0 * 24;
    const double* ug = u + cell0 * 8;
    const bool al = ((reinterpret_cast<uintptr_t>(cg) |
                      (GS ? 0 : reinterpret_cast<uintptr_t>(ug))) & 15) == 0;
    if (al) {
      for (int ch = tid; ch < ncb * 12; ch += CPB) {
        const int c = ch / 12, k = ch - c * 12;
        cp_async16(sC + c * CS + 2 * k, cg + 2 * ch);
      }
      if (!GS)
        for (int ch = tid; ch < ncb * 4; ch += CPB) {
          const int c = ch >> 2, k = ch & 3;
          cp_async16(sU + c * US + 2 * k, ug + 2 * ch);
        }
    } else {
      for (int e = tid; e < ncb * 24; e += CPB) cp_async8(sC + (e / 24) * CS + e % 24, cg + e);
      if (!GS)
        for (int e = tid; e < ncb * 8; e += CPB) cp_async8(sU + (e >> 3) * US + (e & 7), ug + e);
    }
    cp_async_commit();
  };
  int64_t bt = blockIdx.x;
  if (bt >= nbatch) return;
  stage(bt, 0);
  int it = 0;
  do {
  const int cur = PERSIST ? (it & 1) : 0;
  const double* sC = smem + cur * BUF;
  const double* sU = sC + CPB * CS;
  const int64_t cell0 = bt * CPB;
  const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
  cp_async_wait<0>();
  __syncthreads();   // this batch landed; everybody is done reading the other buffer
  if (PERSIST && bt + gridDim.x < nbatch) stage(bt + gridDim.x, cur ^ 1);
  if (tid < ncb) {
  double X[24], uu[8];
  int gm[8];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const double2 v = *reinterpret_cast<const double2*>(sC + tid * CS + 2 * k);
    X[2 * k] = v.x;
    X[2 * k + 1] = v.y;
  }
  if (GS) {
    const int4* mp = reinterpret_cast<const int4*>(cmap + (cell0 + tid) * 8);
    const int4 m0 = __ldg(mp), m1 = __ldg(mp + 1);
    gm[0] = m0.x; gm[1] = m0.y; gm[2] = m0.z; gm[3] = m0.w;
    gm[4] = m1.x; gm[5] = m1.y; gm[6] = m1.z; gm[7] = m1.w;
#pragma unroll
    for (int k = 0; k < 8; ++k) uu[k] = __ldg(u + gm[k]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 v = *reinterpret_cast<const double2*>(sU + tid * US + 2 * k);
      uu[2 * k] = v.x;
      uu[2 * k + 1] = v.y;
    }
  }
  // dof / point index (x, y, z) -> 4x + 2y + z;  tables T.B[i*2+q], T.D[i*2+q]
  // forward: g_x = Dx By Bz u, g_y = Bx Dy Bz u, g_z = Bx By Dz u at 8 points
  double bx[8], dx[8];   // [qx][iy][iz]
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      bx[4 * q + r] = fma(T.B[2 + q], uu[4 + r], T.B[q] * uu[r]);
      dx[4 * q + r] = fma(T.D[2 + q], uu[4 + r], T.D[q] * uu[r]);
    }
  double bb[8], bd[8], db[8];  // [qx][qy][iz]
#pragma unroll
  for (int qx = 0; qx < 2; ++qx)
#pragma unroll
    for (int qy = 0; qy < 2; ++qy)
#pragma unroll
      for (int iz = 0; iz < 2; ++iz) {
        const int o = 4 * qx + 2 * qy + iz, a0 = 4 * qx + iz, a1 = 4 * qx + 2 + iz;
        bb[o] = fma(T.B[2 + qy], bx[a1], T.B[qy] * bx[a0]);
        bd[o] = fma(T.D[2 + qy], bx[a1], T.D[qy] * bx[a0]);
        db[o] = fma(T.B[2 + qy], dx[a1], T.B[qy] * dx[a0]);
      }
  double fx[8], fy[8], fz[8];  // fluxes at the points [qx][qy][qz]
#pragma unroll
  for (int qx = 0; qx < 2; ++qx)
#pragma unroll
    for (int qy = 0; qy < 2; ++qy) {
      HexLineGeom geo;
      geo.setup(X, T.Bc[qx], T.Bc[2 + qx], T.Bc[qy], T.Bc[2 + qy]);
      const double wxy = T.W[qx] * T.W[qy];
      const int l = 4 * qx + 2 * qy;
#pragma unroll
      for (int qz = 0; qz < 2; ++qz) {
        double gz = fma(T.D[2 + qz], bb[l + 1], T.D[qz] * bb[l]);
        double gy = fma(T.B[2 + qz], bd[l + 1], T.B[qz] * bd[l]);
        double gx = fma(T.B[2 + qz], db[l + 1], T.B[qz] * db[l]);
        double r0[3], r1[3], r2[3];
        const double det = geo.adj(T.Bc[qz], T.Bc[2 + qz], r0, r1, r2);
        const double s = (wxy * T.W[qz]) * rcp64(fabs(det));
        laplace_flux(r0, r1, r2, s, gx, gy, gz);
        fx[l + qz] = gx;
        fy[l + qz] = gy;
        fz[l + qz] = gz;
      }
    }
  // transposed z: sx = Bz^T fx, sy = Bz^T fy, sz = Dz^T fz  -> [qx][qy][iz]
  double sx[8], sy[8], sz[8];
#pragma unroll
  for (int l = 0; l < 8; l += 2)
#pragma unroll
    for (int iz = 0; iz < 2; ++iz) {
      sx[l + iz] = fma(T.B[2 * iz + 1], fx[l + 1], T.B[2 * iz] * fx[l]);
      sy[l + iz] = fma(T.B[2 * iz + 1], fy[l + 1], T.B[2 * iz] * fy[l]);
      sz[l + iz] = fma(T.D[2 * iz + 1], fz[l + 1], T.D[2 * iz] * fz[l]);
    }
  // transposed y: r1 = By^T sx, r2 = Dy^T sy + By^T sz  -> [qx][iy][iz]
  double r1[8], r2[8];
#pragma unroll
  for (int qx = 0; qx < 2; ++qx)
#pragma unroll
    for (int iy = 0; iy < 2; ++iy)
#pragma unroll
      for (int iz = 0; iz < 2; ++iz) {
        const int o = 4 * qx + 2 * iy + iz, a0 = 4 * qx + iz, a1 = 4 * qx + 2 + iz;
        r1[o] = fma(T.B[2 * iy + 1], sx[a1], T.B[2 * iy] * sx[a0]);
        r2[o] = fma(T.D[2 * iy + 1], sy[a1], T.D[2 * iy] * sy[a0]);
        r2[o] = fma(T.B[2 * iy + 1], sz[a1], fma(T.B[2 * iy], sz[a0], r2[o]));
      }
  // transposed x: A = Dx^T r1 + Bx^T r2
  double a[8];
#pragma unroll
  for (int ix = 0; ix < 2; ++ix)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double v = T.D[2 * ix] * r1[r];
      v = fma(T.D[2 * ix + 1], r1[4 + r], v);
      v = fma(T.B[2 * ix], r2[r], v);
      v = fma(T.B[2 * ix + 1], r2[4 + r], v);
      a[4 * ix + r] = v;
    }
  if (GS) {
#pragma unroll
    for (int k = 0; k < 8; ++k) atomicAdd(A + gm[k], a[k]);
  } else {
    double* ap = A + (cell0 + tid) * 8;
    if ((reinterpret_cast<uintptr_t>(ap) & 15) == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) reinterpret_cast<double2*>(ap)[k] = make_double2(a[2 * k], a[2 * k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) ap[k] = a[k];
    }
  }
  }   // tid < ncb
  ++it;
  } while (PERSIST && (bt += gridDim.x) < nbatch);
}

template <bool GS, int CPB, int MINB, bool PERSIST = false>
static int launch_p1_cfg(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s, const int* cmap) {
  auto kern = hex_laplace_action_p1<GS, CPB, MINB, PERSIST>;
  const size_t smem = (PERSIST ? 2 : 1) * p1::smem(CPB);
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, CPB, smem, "hex_action_p1", &sh, PERSIST))
    return rc_;
  const Tabs<2, 2> T = make_tabs<2, 2>(p);
  const int64_t nbatch = (ncells + CPB - 1) / CPB;
  const unsigned grid =
      (unsigned)(PERSIST && nbatch > sh.resident() ? sh.resident() : nbatch);
  if (grid > 0) kern<<<grid, CPB, smem, s>>>(T, ncells, coords, w0, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_p1 launch");
}

#ifdef SFK_P1_ONLY
// probe builds (tools/kernel_sweep.py p1): one instantiation
}  // namespace sfk
extern "C" int SFK_P1_PROBE_ENTRY(const sfk_plan* p, int64_t ncells, double* A,
                                  const double* coords, const double* w0, void* stream) {
  if (p->n != 2 || p->m != 2) return sfk::fail(SFK_EUNSUPPORTED, "probe build: n = m = 2 only");
  return sfk::launch_p1_cfg<false, SFK_P1P_CPB, SFK_P1P_MINB, SFK_P1P_PERSIST != 0>(
      p, ncells, A, coords, w0, (cudaStream_t)stream, nullptr);
}
namespace sfk {
#else
// (cells per CTA, min CTAs per SM): option p1_cfg = 1..3 selects the
// alternatives (A/B runs)
template <bool GS>
static int launch_p1(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* w0, cudaStream_t s, const int* cmap) {
  if (p->n != 2 || p->m != 2) return SFK_EUNSUPPORTED;
  switch ((int)option(OPT_P1_CFG)) {
    case 1: return launch_p1_cfg<GS, 64, 6>(p, ncells, A, coords, w0, s, cmap);
    case 2: return launch_p1_cfg<GS, 32, 12>(p, ncells, A, coords, w0, s, cmap);
    case 3: return launch_p1_cfg<GS, 96, 4>(p, ncells, A, coords, w0, s, cmap);
    // persistent, double-buffered staging (A/B): measured slower, 0.0287 vs
    // 0.0246 ms (profiles/r02cy_p1.txt) — the resident grid's 444 CTAs x 168
    // registers leave no room for the extra waves that hide the tail
    case 4: return launch_p1_cfg<GS, 128, SFK_P1_MINB, true>(p, ncells, A, coords, w0, s, cmap);
    case 5: return launch_p1_cfg<GS, 64, 6, true>(p, ncells, A, coords, w0, s, cmap);
    case 6: return launch_p1_cfg<GS, 96, 4, true>(p, ncells, A, coords, w0, s, cmap);
    case 7: return launch_p1_cfg<GS, 32, 12, true>(p, ncells, A, coords, w0, s, cmap);
    default: return launch_p1_cfg<GS, 128, SFK_P1_MINB>(p, ncells, A, coords, w0, s, cmap);
  }
}

int launch_hex_action_p1(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s) {
  return launch_p1<false>(p, ncells, A, coords, w0, s, nullptr);
}

int launch_hex_action_p1_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s) {
  return launch_p1<true>(p, ncells, y, coords, x, s, cmap);
}

#endif  // SFK_P1_ONLY

}  // namespace sfk
