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
constexpr int CPB = 128;             // cells (= threads) per CTA
constexpr int CS = 26;               // padded coords stride (24 used)
constexpr int US = 10;               // padded u stride (8 used)
constexpr size_t SMEM = (size_t)CPB * (CS + US) * sizeof(double);
}  // namespace p1

// GS = true: global operator y += sum_c P_c^T A_c P_c x (SURVEY.md §8(f)
// item 1): u = x gathered through cmap[c][0..7], A = y scatter-added with
// fp64 atomics.
template <bool GS>
__global__ void __launch_bounds__(p1::CPB, SFK_P1_MINB)
hex_laplace_action_p1(const __grid_constant__ Tabs<2, 2> T, int64_t ncells,
                      const double* __restrict__ coords, const double* __restrict__ u,
                      double* __restrict__ A, const int* __restrict__ cmap = nullptr) {
  using namespace p1;
  extern __shared__ __align__(16) double smem[];
  double* sC = smem;
  double* sU = smem + CPB * CS;
  const int tid = threadIdx.x;
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
  {
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
    cp_async_wait<0>();
  }
  __syncthreads();
  if (tid >= ncb) return;

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
    return;
  }
  double* ap = A + (cell0 + tid) * 8;
  if ((reinterpret_cast<uintptr_t>(ap) & 15) == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) reinterpret_cast<double2*>(ap)[k] = make_double2(a[2 * k], a[2 * k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) ap[k] = a[k];
  }
}

template <bool GS>
static int launch_p1(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* w0, cudaStream_t s, const int* cmap) {
  if (p->n != 2 || p->m != 2) return SFK_EUNSUPPORTED;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)hex_laplace_action_p1<GS>, p1::CPB, p1::SMEM,
                                   "hex_action_p1", &sh))
    return rc_;
  const Tabs<2, 2> T = make_tabs<2, 2>(p);
  const unsigned grid = (unsigned)((ncells + p1::CPB - 1) / p1::CPB);
  hex_laplace_action_p1<GS><<<grid, p1::CPB, p1::SMEM, s>>>(T, ncells, coords, w0, A, cmap);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_p1 launch");
}

// ---------------------------------------------------------------------------
// p1c: two threads per cell (lane pair h = 0, 1 owns the points / slab qx = h)
// with the collocation-derivative schedule of v6 (hex_action6.cu):
//   V = (B x B x B) u at the 8 points, g_a = C_a V (C = B^-1 D), flux,
//   t = C_x^T f_x + C_y^T f_y + C_z^T f_z, A = (B^T x B^T x B^T) t.
// Each thread interpolates its own x-slab (the x stage is first, so no data
// is exchanged for it), runs y / z inside the slab, and trades 4 doubles
// with its partner (warp shuffles) three times: V for g_x, f_x for C_x^T
// and the slab result for B_x^T.  Half the geometry per thread (2 of the 4
// z-lines), 96 + 96 contraction FMAs per cell instead of 128 + 128, and
// twice the threads in flight at ~half the registers of the 1-thread kernel.
struct TabsP1C {
  double B[4];    // B[i*2 + q]
  double C[4];    // C[q'*2 + q]  (collocation derivative)
  double W[2];
  double Bc[4];
};

namespace p1c {
constexpr int CPB = 128;                 // cells per CTA
constexpr int THREADS = 2 * CPB;
constexpr int CS = 26, US = 10;          // padded per-cell strides in shared memory
constexpr size_t SMEM = (size_t)CPB * (CS + US) * sizeof(double);
}  // namespace p1c

__device__ __forceinline__ double shx(double v) { return __shfl_xor_sync(0xffffffffu, v, 1); }

__global__ void __launch_bounds__(p1c::THREADS, 2)
hex_laplace_action_p1c(const __grid_constant__ TabsP1C T, int64_t ncells,
                       const double* __restrict__ coords, const double* __restrict__ u,
                       double* __restrict__ A) {
  using namespace p1c;
  extern __shared__ __align__(16) double smem[];
  double* sC = smem;
  double* sU = smem + CPB * CS;
  const int tid = threadIdx.x;
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int ncb = (int)((ncells - cell0) < CPB ? (ncells - cell0) : CPB);
  {
    const double* cg = coords + cell0 * 24;
    const double* ug = u + cell0 * 8;
    const bool al = ((reinterpret_cast<uintptr_t>(cg) | reinterpret_cast<uintptr_t>(ug)) & 15) == 0;
    if (al) {
      for (int ch = tid; ch < ncb * 12; ch += THREADS) {
        const int c = ch / 12, k = ch - c * 12;
        cp_async16(sC + c * CS + 2 * k, cg + 2 * ch);
      }
      for (int ch = tid; ch < ncb * 4; ch += THREADS) {
        const int c = ch >> 2, k = ch & 3;
        cp_async16(sU + c * US + 2 * k, ug + 2 * ch);
      }
    } else {
      for (int e = tid; e < ncb * 24; e += THREADS) cp_async8(sC + (e / 24) * CS + e % 24, cg + e);
      for (int e = tid; e < ncb * 8; e += THREADS) cp_async8(sU + (e >> 3) * US + (e & 7), ug + e);
    }
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();
  const int h = tid & 1, cl = tid >> 1;   // slab qx = h of cell cl
  const bool live = cl < ncb;
  const int cc = live ? cl : 0;           // dead pairs still shuffle (full-warp masks)

  double X[24], uu[8];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const double2 v = *reinterpret_cast<const double2*>(sC + cc * CS + 2 * k);
    X[2 * k] = v.x;
    X[2 * k + 1] = v.y;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double2 v = *reinterpret_cast<const double2*>(sU + cc * US + 2 * k);
    uu[2 * k] = v.x;
    uu[2 * k + 1] = v.y;
  }
  // slab values are indexed [y][z] (2*y + z)
  const double bh0 = T.B[h], bh1 = T.B[2 + h];           // B[i][qx = h]
  double vx[4], vy[4], V[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) vx[r] = fma(bh1, uu[4 + r], bh0 * uu[r]);
#pragma unroll
  for (int qy = 0; qy < 2; ++qy)
#pragma unroll
    for (int iz = 0; iz < 2; ++iz) vy[2 * qy + iz] = fma(T.B[2 + qy], vx[2 + iz], T.B[qy] * vx[iz]);
#pragma unroll
  for (int qy = 0; qy < 2; ++qy)
#pragma unroll
    for (int qz = 0; qz < 2; ++qz)
      V[2 * qy + qz] = fma(T.B[2 + qz], vy[2 * qy + 1], T.B[qz] * vy[2 * qy]);
  double gx[4], gy[4], gz[4];
  {
    // own slab is qx = h, the partner's qx = 1 - h
    const double c0h = T.C[h], c1h = T.C[2 + h];        // C[q'][qx = h]
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double vp = shx(V[k]);
      const double v0 = h ? vp : V[k], v1 = h ? V[k] : vp;
      gx[k] = fma(c1h, v1, c0h * v0);
    }
  }
#pragma unroll
  for (int qy = 0; qy < 2; ++qy)
#pragma unroll
    for (int qz = 0; qz < 2; ++qz) {
      gy[2 * qy + qz] = fma(T.C[2 + qy], V[2 + qz], T.C[qy] * V[qz]);
      gz[2 * qy + qz] = fma(T.C[2 + qz], V[2 * qy + 1], T.C[qz] * V[2 * qy]);
    }
  // geometry + flux at the slab's 4 points (lines qy = 0, 1)
#pragma unroll
  for (int qy = 0; qy < 2; ++qy) {
    HexLineGeom geo;
    geo.setup(X, T.Bc[h], T.Bc[2 + h], T.Bc[qy], T.Bc[2 + qy]);
    const double wxy = T.W[h] * T.W[qy];
#pragma unroll
    for (int qz = 0; qz < 2; ++qz) {
      const int k = 2 * qy + qz;
      double r0[3], r1[3], r2[3];
      const double det = geo.adj(T.Bc[qz], T.Bc[2 + qz], r0, r1, r2);
      const double s = (wxy * T.W[qz]) * rcp64(fabs(det));
      laplace_flux(r0, r1, r2, s, gx[k], gy[k], gz[k]);
    }
  }
  // t = C_x^T f_x + C_y^T f_y + C_z^T f_z on the slab
  double t[4];
  {
    const double ch0 = T.C[2 * h], ch1 = T.C[2 * h + 1];   // C[qx' = h][qx]
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double fp = shx(gx[k]);
      const double f0 = h ? fp : gx[k], f1 = h ? gx[k] : fp;
      t[k] = fma(ch1, f1, ch0 * f0);
    }
  }
#pragma unroll
  for (int qy = 0; qy < 2; ++qy)
#pragma unroll
    for (int qz = 0; qz < 2; ++qz) {
      const int k = 2 * qy + qz;
      t[k] = fma(T.C[2 * qy + 1], gy[2 + qz], fma(T.C[2 * qy], gy[qz], t[k]));
      t[k] = fma(T.C[2 * qz + 1], gz[2 * qy + 1], fma(T.C[2 * qz], gz[2 * qy], t[k]));
    }
  // B_z^T, B_y^T on the slab, then B_x^T across the pair
  double sz[4], ry[4];
#pragma unroll
  for (int qy = 0; qy < 2; ++qy)
#pragma unroll
    for (int iz = 0; iz < 2; ++iz) sz[2 * qy + iz] = fma(T.B[2 * iz + 1], t[2 * qy + 1], T.B[2 * iz] * t[2 * qy]);
#pragma unroll
  for (int iy = 0; iy < 2; ++iy)
#pragma unroll
    for (int iz = 0; iz < 2; ++iz) ry[2 * iy + iz] = fma(T.B[2 * iy + 1], sz[2 + iz], T.B[2 * iy] * sz[iz]);
  double a[4];
  {
    const double bx0 = T.B[2 * h], bx1 = T.B[2 * h + 1];   // B[ix = h][qx]
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double rp = shx(ry[k]);
      const double r0v = h ? rp : ry[k], r1v = h ? ry[k] : rp;
      a[k] = fma(bx1, r1v, bx0 * r0v);
    }
  }
  if (!live) return;
  // A[cell][4*ix + 2*iy + iz], ix = h
  double* ap = A + (cell0 + cl) * 8 + 4 * h;
  if ((reinterpret_cast<uintptr_t>(ap) & 15) == 0) {
    reinterpret_cast<double2*>(ap)[0] = make_double2(a[0], a[1]);
    reinterpret_cast<double2*>(ap)[1] = make_double2(a[2], a[3]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) ap[k] = a[k];
  }
}

int launch_hex_action_p1c(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          const double* w0, cudaStream_t s) {
  if (p->n != 2 || p->m != 2 || !p->has_ct) return SFK_EUNSUPPORTED;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)hex_laplace_action_p1c, p1c::THREADS, p1c::SMEM,
                                   "hex_action_p1c", &sh))
    return rc_;
  TabsP1C T;
  for (int k = 0; k < 4; ++k) {
    T.B[k] = p->B[k];
    T.C[k] = p->Ct[k];
    T.Bc[k] = p->Bc[k];
  }
  T.W[0] = p->wq[0];
  T.W[1] = p->wq[1];
  const unsigned grid = (unsigned)((ncells + p1c::CPB - 1) / p1c::CPB);
  hex_laplace_action_p1c<<<grid, p1c::THREADS, p1c::SMEM, s>>>(T, ncells, coords, w0, A);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_laplace_action_p1c launch");
}

int launch_hex_action_p1(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s) {
  return launch_p1<false>(p, ncells, A, coords, w0, s, nullptr);
}

int launch_hex_action_p1_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s) {
  return launch_p1<true>(p, ncells, y, coords, x, s, cmap);
}

}  // namespace sfk
