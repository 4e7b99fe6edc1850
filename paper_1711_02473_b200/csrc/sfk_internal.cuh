// Internal declarations shared by the sfk CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sfk.h"
#include "sfk_options.h"

#define SFK_MAXN 17   // dofs per axis (p <= 16)
#define SFK_MAXM 18   // quadrature points per axis

// The plan behind the opaque sfk_plan* handle.  Tables are HOST copies: they
// are passed by value (as __grid_constant__ kernel parameters, i.e. constant
// bank 0) to every launch, so a plan owns no device memory and is usable on
// any device / stream.
struct sfk_plan {
  int kind, dim, degree, n, m, collocated, nparams;
  double B[SFK_MAXN * SFK_MAXM];   // B[i*m + q]
  double D[SFK_MAXN * SFK_MAXM];   // D[i*m + q]
  double wq[SFK_MAXM];
  double xq[SFK_MAXM];
  double Bc[2 * SFK_MAXM];         // P1 values  Bc[v*m + q]
  double Dc[2 * SFK_MAXM];         // P1 derivatives (-1, +1)
  double params[8];
  // collocation derivative C = B^-1 D (n == m only, has_ct): C[q'*m + q],
  // solved at plan creation in extended precision (sfk_api.cu)
  double Ct[SFK_MAXM * SFK_MAXM];
  int has_ct;
  int64_t coords_size, w0_size, w1_size, a_size;
};

namespace sfk {

// Thread-local error text + status helpers (sfk_api.cu).
int fail(int status, const char* fmt, ...);
int cuda_status(cudaError_t err, const char* what);
void note_launch(int64_t k = 1);

// Tables in the form kernels consume them (kernel parameter => constant
// bank).  On sm_100a DFMA takes no constant-bank operand: an entry with a
// compile-time index reaches it through a uniform register (LDCU, then
// DFMA R, R, UR, R) — one extra instruction per use unless the entry feeds
// several DFMAs, and a reason to keep such kernels free of loops ptxas could
// hoist the loads out of.
template <int N, int M>
struct Tabs {
  double B[N * M];
  double D[N * M];
  double W[M];
  double Bc[2 * M];
  double X[M];
};

template <int N, int M>
inline Tabs<N, M> make_tabs(const sfk_plan* p) {
  Tabs<N, M> t;
  for (int i = 0; i < N; ++i)
    for (int q = 0; q < M; ++q) {
      t.B[i * M + q] = p->B[i * p->m + q];
      t.D[i * M + q] = p->D[i * p->m + q];
    }
  for (int q = 0; q < M; ++q) {
    t.W[q] = p->wq[q];
    t.X[q] = p->xq[q];
    t.Bc[q] = p->Bc[q];
    t.Bc[M + q] = p->Bc[p->m + q];
  }
  return t;
}

// Tables plus (B, D) pairs interleaved, for the line kernels (v2, v4, v5):
// they use B[i][q] and D[i][q] together, so one 128-bit constant load
// (LDCU.128) feeds both.  A separate type so the other kernels keep the
// compact parameter block (the tc8 kernel measured 10% slower with the
// pairs in its parameters: profiles/r01bw_*.jsonl).
template <int N, int M>
struct TabsBD {
  alignas(16) double BD[2 * N * M];
  double B[N * M];
  double D[N * M];
  double W[M];
  double Bc[2 * M];
  double X[M];
};

template <int N, int M>
inline TabsBD<N, M> make_tabs_bd(const sfk_plan* p) {
  const Tabs<N, M> t = make_tabs<N, M>(p);
  TabsBD<N, M> o;
  for (int k = 0; k < N * M; ++k) {
    o.B[k] = t.B[k];
    o.D[k] = t.D[k];
    o.BD[2 * k] = t.B[k];
    o.BD[2 * k + 1] = t.D[k];
  }
  for (int q = 0; q < M; ++q) {
    o.W[q] = t.W[q];
    o.X[q] = t.X[q];
    o.Bc[q] = t.Bc[q];
    o.Bc[M + q] = t.Bc[M + q];
  }
  return o;
}

// Family launchers (one translation unit each).
int launch_hex_action(const sfk_plan* p, int64_t ncells, double* A,
                      const double* coords, const double* w0,
                      const double* w1, cudaStream_t s);
int launch_hex_action_v2(const sfk_plan* p, int64_t ncells, double* A,
                         const double* coords, const double* w0, cudaStream_t s);
int launch_hex_action_v3(const sfk_plan* p, int64_t ncells, double* A,
                         const double* coords, const double* w0, cudaStream_t s);
int launch_hex_action_tc(const sfk_plan* p, int64_t ncells, double* A,
                         const double* coords, const double* w0, cudaStream_t s);
int launch_hex_action_p1(const sfk_plan* p, int64_t ncells, double* A,
                         const double* coords, const double* w0, cudaStream_t s);
int launch_hex_action_p1_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s);
int launch_hex_action_v2_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s);
int launch_hex_action_tc_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s);
int launch_hex_neohookean_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                             double* y, const double* coords, cudaStream_t s);
// C3 at n = 8 on the one-warp-per-cell DMMA kernel (hex_action_tc8c.cu, COL mode)
int launch_hex_colloc_tc8c(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, const double* w1, cudaStream_t s);
// component-parallel C4 kernel (hex_neohookean3.cu); SFK_EUNSUPPORTED where not instantiated
int launch_hex_neohookean3(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, cudaStream_t s);
int launch_hex_neohookean3_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                              double* y, const double* coords, cudaStream_t s);
int launch_hex_colloc_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                         double* y, const double* coords, const double* kappa, cudaStream_t s);
int launch_hex_action_v5_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s);
int launch_hex_action_cell_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                              double* y, const double* coords, cudaStream_t s);
int launch_hex_action_cell(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, cudaStream_t s);
int launch_hex_action_v5(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s);
int launch_hex_action_v6_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s);
int launch_hex_action_tc8c_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                              double* y, const double* coords, cudaStream_t s);
int launch_hex_action_tc8c(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                           const double* w0, cudaStream_t s);
int launch_hex_action_v6(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s);
int launch_hex_action_v4(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, cudaStream_t s);
int launch_hex_action_v4_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                            double* y, const double* coords, cudaStream_t s);
int launch_hex_colloc_tc(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         const double* w0, const double* w1, cudaStream_t s);
int launch_hex_action_gs(const sfk_plan* p, int64_t ncells, const int* cmap, const double* x,
                         double* y, const double* coords, cudaStream_t s);
int launch_hex_colloc_action(const sfk_plan* p, int64_t ncells, double* A,
                             const double* coords, const double* w0,
                             const double* w1, cudaStream_t s);
int launch_quad_action(const sfk_plan* p0, const sfk_plan* p1, int64_t ncells,
                       double* A0, double* A1, const double* coords,
                       const double* w0, cudaStream_t s);
int launch_hex_matrix_p1(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                         cudaStream_t s);
int launch_hex_matrix_tc4(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          cudaStream_t s, const int32_t* emap = nullptr);
int launch_hex_matrix_tc5(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          cudaStream_t s, const int32_t* emap = nullptr);
int launch_hex_matrix_tcn(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          cudaStream_t s, const int32_t* emap = nullptr);
bool hex_matrix_tcn_supported(int n, int m);
int launch_hex_matrix(const sfk_plan* p, int64_t ncells, double* A,
                      const double* coords, cudaStream_t s);
int launch_hex_matrix_csr(const sfk_plan* p, int64_t ncells, const int32_t* dofs,
                          const double* coords, const int64_t* row_ptr, const int32_t* col_idx,
                          const int32_t* emap, double* values, cudaStream_t s);
int launch_hex_neohookean(const sfk_plan* p, int64_t ncells, double* A,
                          const double* coords, const double* w0,
                          cudaStream_t s);
int launch_hex_mass(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                    const double* w0, cudaStream_t s);
bool hex_mass_supported(int n, int m);
int launch_sum_squares(const double* x, int64_t n, double* out, cudaStream_t s);
int run_fp64_peak(double seconds, double* dfma, double* dmma);

}  // namespace sfk

// Table entry accessors of the line kernels: TB(k) = B[k], TD(k) = D[k]
// (k = i*M + q), read from the interleaved pairs unless SFK_TAB_PAIRS=0.
#ifndef SFK_TAB_PAIRS
#define SFK_TAB_PAIRS 1
#endif
#if SFK_TAB_PAIRS
#define TB(k) T.BD[2 * (k)]
#define TD(k) T.BD[2 * (k) + 1]
#else
#define TB(k) T.B[k]
#define TD(k) T.D[k]
#endif
// Per-instantiation choice (a kernel defines `constexpr bool PAIRS`).
#define TBP(k) (PAIRS ? T.BD[2 * (k)] : T.B[k])
#define TDP(k) (PAIRS ? T.BD[2 * (k) + 1] : T.D[k])

// ---------------------------------------------------------------------------
// device helpers

namespace sfk {

// 1/x to full double precision: MUFU.RCP64H seed + two Newton steps.
__device__ __forceinline__ double rcp64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  return y;
}

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

}  // namespace sfk
