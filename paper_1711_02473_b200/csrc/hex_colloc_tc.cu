// Hex GLL-collocated (weighted) Laplace action on the FP64 tensor cores —
// BASELINE config C3 at n = 8, 12, 16 (p = 7, 11, 15).
//
// Same math and reference mapping as hex_colloc.cu (action_form of
// weighted_laplace, collocated GLL: one D-contraction per gradient component
// and per transposed component, forms.py:192-193, passes.py:336-388).  Every
// contraction is a GEMM with the constant table D on one side, run as DMMA
// (mma.sync.m8n8k4.f64) with D's fragments in registers for the whole
// kernel:
//   GX[qx][(y,z)]  = sum_i D[i][qx] U[i][(y,z)]       (D^T as A)
//   GY[x][qy][z]   = sum_i D[i][qy] U[x][i][z]        (D^T as A, per x)
//   GZ[(x,y)][qz]  = sum_i U[(x,y)][i] D[i][qz]       (D as B)
//   pointwise flux per z-line (geometry, kappa) in place
//   U[i][(y,z)]    = sum_q D[i][q] FX[q][(y,z)]       (D as A)
//   U[x][i][z]    += sum_q D[i][q] FY[x][q][z]        (D as A, C = U)
//   U[(x,y)][i]   += sum_q FZ[(x,y)][q] D[i][q]       (D^T as B, C = U)
// D^T-as-A and D-as-B fragments are the same per-lane values (and so are
// D-as-A and D^T-as-B), so two register sets serve all six.  Shared arrays
// U, GX, GY, GZ share one padded (x, y, z) layout with row strides = 4 mod 16,
// which makes every fragment load conflict-free; kappa is read from HBM in
// the pointwise pass (each value once).  n = 12 pads the 12-wide dimensions
// to 16 with zero fragments and zero-initialised padding.
#include <cstdlib>

#include "async_copy.cuh"
#include "hex_geometry.cuh"

namespace sfk {

template <int N_>
struct CollocTcCfg {
  static constexpr int N = N_, NP = (N_ + 7) / 8 * 8, NN = N_ * N_, N3 = N_ * N_ * N_;
  static constexpr int KST = N_ / 4;              // k-steps over an N-long index
  static constexpr int RT = NP / 8;               // 8-wide tiles over an N-long index
  static constexpr int SY = (NP % 16 == 8) ? NP + 4 : NP + 4;   // = 4 or 12 mod 16
  static constexpr int SX0 = N_ * SY;
  static constexpr int SX = SX0 + ((4 - SX0 % 16) + 16) % 16;   // = 4 mod 16
  static constexpr int AS = N_ * SX;              // one array
  static constexpr int WARPS = 8, THREADS = 256;
  static constexpr size_t SMEM = (size_t)(4 * AS + 24) * sizeof(double);
  static_assert(N_ % 4 == 0, "n must be a multiple of 4");
};

template <int N>
struct TabsD2 {
  double D[N * N];
  double W[N];
  double Bc[2 * N];
};

__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int N, bool WEIGHTED>
__global__ void __launch_bounds__(CollocTcCfg<N>::THREADS, 1)
hex_colloc_tc_kernel(const __grid_constant__ TabsD2<N> T, int64_t ncells,
                     const double* __restrict__ coords, const double* __restrict__ u,
                     const double* __restrict__ kappa, double* __restrict__ A) {
  using C = CollocTcCfg<N>;
  constexpr int NP = C::NP, NN = C::NN, N3 = C::N3, KST = C::KST, RT = C::RT;
  constexpr int SY = C::SY, SX = C::SX, AS = C::AS, WARPS = C::WARPS, TH = C::THREADS;
  extern __shared__ __align__(16) double smem[];
  double* sU = smem;
  double* sGX = sU + AS;
  double* sGY = sGX + AS;
  double* sGZ = sGY + AS;
  double* sC = sGZ + AS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, kq = lane & 3;

  for (int i = tid; i < 4 * AS; i += TH) smem[i] = 0.0;   // padding stays 0
  // fragments: dt[rt][ks] = D[ks*4+kq][rt*8+gq] (D^T as A  ==  D as B),
  //            dd[rt][ks] = D[rt*8+gq][ks*4+kq] (D as A   ==  D^T as B)
  double dt[RT][KST], dd[RT][KST];
#pragma unroll
  for (int rt = 0; rt < RT; ++rt)
#pragma unroll
    for (int ks = 0; ks < KST; ++ks) {
      const int r = rt * 8 + gq, k = ks * 4 + kq;
      dt[rt][ks] = r < N ? T.D[k * N + r] : 0.0;
      dd[rt][ks] = r < N ? T.D[r * N + k] : 0.0;
    }
  __syncthreads();

  for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
    // ---- u -> U (padded layout), coords ------------------------------------
    {
      const double* ug = u + cell * N3;
      for (int i = tid; i < N3; i += TH) {
        const int x = i / NN, yz = i - x * NN, y = yz / N, z = yz - y * N;
        cp_async8(sU + x * SX + y * SY + z, ug + i);
      }
      if (tid < 24) sC[tid] = __ldg(coords + cell * 24 + tid);
      cp_async_commit();
      cp_async_wait<0>();
    }
    __syncthreads();

    // ---- forward: GX, GY, GZ (independent; one barrier) -----------------------
    // GX[qx][(y,z)]: tiles (rt over qx, ct over (y,z))
    for (int t = warp; t < RT * (NN / 8); t += WARPS) {
      const int rt = t % RT, ct = t / RT;
      double d0 = 0.0, d1 = 0.0;
      const int n = ct * 8 + gq, y = n / N, z = n - y * N;
#pragma unroll
      for (int ks = 0; ks < KST; ++ks)
        dmma_c(d0, d1, dt[rt][ks], sU[(ks * 4 + kq) * SX + y * SY + z]);
      const int qx = rt * 8 + gq;
      if (qx < N) {
        const int n0 = ct * 8 + 2 * kq, y0 = n0 / N, z0 = n0 - y0 * N;
        sGX[qx * SX + y0 * SY + z0] = d0;
        const int n1 = n0 + 1, y1 = n1 / N, z1 = n1 - y1 * N;
        sGX[qx * SX + y1 * SY + z1] = d1;
      }
    }
    // GY[x][qy][z]: tiles (x, rt over qy, ct over z)
    for (int t = warp; t < N * RT * RT; t += WARPS) {
      const int x = t / (RT * RT), rt = (t / RT) % RT, ct = t % RT;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KST; ++ks)
        dmma_c(d0, d1, dt[rt][ks], sU[x * SX + (ks * 4 + kq) * SY + ct * 8 + gq]);
      const int qy = rt * 8 + gq, z0 = ct * 8 + 2 * kq;
      if (qy < N) {
        if (z0 < N) sGY[x * SX + qy * SY + z0] = d0;
        if (z0 + 1 < N) sGY[x * SX + qy * SY + z0 + 1] = d1;
      }
    }
    // GZ[(x,y)][qz]: A = U rows (x,y), B = D; tiles (rows over (x,y), ct over qz)
    for (int t = warp; t < (NN / 8) * RT; t += WARPS) {
      const int rr = t / RT, ct = t % RT;
      const int row = rr * 8 + gq, x = row / N, y = row - x * N;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KST; ++ks)
        dmma_c(d0, d1, sU[x * SX + y * SY + ks * 4 + kq], dt[ct][ks]);
      const int r0 = rr * 8 + gq, x0 = r0 / N, y0 = r0 - x0 * N, q0 = ct * 8 + 2 * kq;
      if (q0 < N) sGZ[x0 * SX + y0 * SY + q0] = d0;
      if (q0 + 1 < N) sGZ[x0 * SX + y0 * SY + q0 + 1] = d1;
    }
    __syncthreads();

    // ---- pointwise: z-line (x, y) per thread: geometry, kappa, flux ----------
    for (int l = tid; l < NN; l += TH) {
      const int x = l / N, y = l - x * N;
      const int base = x * SX + y * SY;
      HexLineAdj geo;
      geo.setup(sC, T.Bc[x], T.Bc[N + x], T.Bc[y], T.Bc[N + y]);
      const double wxy = T.W[x] * T.W[y];
      const double* kp = kappa + cell * N3 + l * N;
#pragma unroll 2
      for (int q = 0; q < N; ++q) {
        double gx = sGX[base + q], gy = sGY[base + q], gz = sGZ[base + q];
        double r0[3], r1[3], r2[3];
        const double det = geo.adj(T.Bc[N + q], r0, r1, r2);
        double s = (wxy * T.W[q]) * rcp64(fabs(det));
        if (WEIGHTED) s *= __ldg(kp + q);
        laplace_flux(r0, r1, r2, s, gx, gy, gz);
        sGX[base + q] = gx;
        sGY[base + q] = gy;
        sGZ[base + q] = gz;
      }
    }
    __syncthreads();

    // ---- transposed x: U[i][(y,z)] = D FX (D as A) -----------------------------
    for (int t = warp; t < RT * (NN / 8); t += WARPS) {
      const int rt = t % RT, ct = t / RT;
      double d0 = 0.0, d1 = 0.0;
      const int n = ct * 8 + gq, y = n / N, z = n - y * N;
#pragma unroll
      for (int ks = 0; ks < KST; ++ks)
        dmma_c(d0, d1, dd[rt][ks], sGX[(ks * 4 + kq) * SX + y * SY + z]);
      const int i = rt * 8 + gq;
      if (i < N) {
        const int n0 = ct * 8 + 2 * kq, y0 = n0 / N, z0 = n0 - y0 * N;
        sU[i * SX + y0 * SY + z0] = d0;
        const int n1 = n0 + 1, y1 = n1 / N, z1 = n1 - y1 * N;
        sU[i * SX + y1 * SY + z1] = d1;
      }
    }
    __syncthreads();
    // ---- transposed y: U[x][i][z] += D FY[x] (C = U) ----------------------------
    for (int t = warp; t < N * RT * RT; t += WARPS) {
      const int x = t / (RT * RT), rt = (t / RT) % RT, ct = t % RT;
      const int i = rt * 8 + gq, z0 = ct * 8 + 2 * kq;
      double* up = sU + x * SX + i * SY + z0;
      double d0 = (i < N && z0 < N) ? up[0] : 0.0, d1 = (i < N && z0 + 1 < N) ? up[1] : 0.0;
#pragma unroll
      for (int ks = 0; ks < KST; ++ks)
        dmma_c(d0, d1, dd[rt][ks], sGY[x * SX + (ks * 4 + kq) * SY + ct * 8 + gq]);
      if (i < N) {
        if (z0 < N) up[0] = d0;
        if (z0 + 1 < N) up[1] = d1;
      }
    }
    __syncthreads();
    // ---- transposed z: U[(x,y)][i] += FZ[(x,y)] D^T (C = U, D^T as B) -----------
    for (int t = warp; t < (NN / 8) * RT; t += WARPS) {
      const int rr = t / RT, ct = t % RT;
      const int row = rr * 8 + gq, x = row / N, y = row - x * N;
      const int i0 = ct * 8 + 2 * kq;
      double* up = sU + x * SX + y * SY + i0;
      double d0 = i0 < N ? up[0] : 0.0, d1 = i0 + 1 < N ? up[1] : 0.0;
#pragma unroll
      for (int ks = 0; ks < KST; ++ks)
        dmma_c(d0, d1, sGZ[x * SX + y * SY + ks * 4 + kq], dd[ct][ks]);
      if (i0 < N) up[0] = d0;
      if (i0 + 1 < N) up[1] = d1;
    }
    __syncthreads();

    // ---- U -> A (coalesced) ----------------------------------------------------
    {
      double* ag = A + cell * N3;
      for (int i = tid; i < N3; i += TH) {
        const int x = i / NN, yz = i - x * NN, y = yz / N, z = yz - y * N;
        ag[i] = sU[x * SX + y * SY + z];
      }
    }
    __syncthreads();   // U is rewritten by the next cell's load
  }
}

template <int N>
static int launch_colloc_tc(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                            const double* u, const double* kappa, cudaStream_t s) {
  using C = CollocTcCfg<N>;
  TabsD2<N> T;
  for (int i = 0; i < N * N; ++i) T.D[i] = p->D[i];
  for (int q = 0; q < N; ++q) {
    T.W[q] = p->wq[q];
    T.Bc[q] = p->Bc[q];
    T.Bc[N + q] = p->Bc[N + q];
  }
  auto kern = kappa ? hex_colloc_tc_kernel<N, true> : hex_colloc_tc_kernel<N, false>;
  LaunchShape sh;
  if (const int rc_ = kernel_shape((const void*)kern, C::THREADS, C::SMEM, "hex_colloc_tc", &sh))
    return rc_;
  const int64_t resident = sh.resident();
  const unsigned grid = (unsigned)(ncells < resident ? ncells : resident);
  kern<<<grid, C::THREADS, C::SMEM, s>>>(T, ncells, coords, u, kappa, A);
  note_launch();
  return cuda_status(cudaGetLastError(), "hex_colloc_tc launch");
}

// DMMA path for n = 8, 12, 16 — OPT-IN (option c3_tc = 1).  Measured slower than
// the line kernel (p = 7: 1.25 vs 0.385 ms, p = 15: 5.51 vs 4.89 ms,
// profiles/r01bn_c3_dmma.jsonl): one cell at a time per CTA with an exposed
// per-cell u load and 1 CTA/SM by registers; kept correct (parity-tested)
// as the starting point for a prefetching, multi-cell version.
int launch_hex_colloc_tc(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, const double* w1, cudaStream_t s) {
  const bool off = option(OPT_C3_TC) != 1;
  if (off || p->n != p->m) return SFK_EUNSUPPORTED;
  switch (p->n) {
    case 8: return launch_colloc_tc<8>(p, ncells, A, coords, w0, w1, s);
    case 12: return launch_colloc_tc<12>(p, ncells, A, coords, w0, w1, s);
    case 16: return launch_colloc_tc<16>(p, ncells, A, coords, w0, w1, s);
    default: return SFK_EUNSUPPORTED;
  }
}

}  // namespace sfk
