// C-ABI entry points of libsfk.so (declared in include/sfk.h).
//
// This is the drop-in boundary: the reference hands a per-cell C function to
// the caller's cell loop (scheduling.py:617-738); these entry
// points ARE that loop, batched on the device.  Validation and error
// reporting mirror the reference's: a missing argument is UnboundVariable,
// a mis-sized one ShapeMismatch (interpreter.py:23-28, 291-299) — on the C
// side both surface as SFK_EINVAL with the argument name in sfk_last_error,
// and the Python layer raises the reference exception types before calling.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>

#include "sfk_internal.cuh"

namespace sfk {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int cuda_status(cudaError_t err, const char* what) {
  if (err == cudaSuccess) return SFK_OK;
  return fail(err == cudaErrorMemoryAllocation ? SFK_ENOMEM : SFK_ECUDA,
              "%s: %s (%s)", what, cudaGetErrorName(err), cudaGetErrorString(err));
}

void note_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// Hex Laplace action (BASELINE C2) kernel generation per degree.  The
// default ("auto") is the fastest measured generation for each n = p+1
// (profiles/r01*_*.json A/B runs); option c2_kernel (sfk_set_option) forces one
// (tuning / A-B runs; a generation that has no instance for n falls back).
//   v1: line kernel, thread per line, non-persistent       (hex_action.cu)
//   v2: persistent, cp.async prefetch, in-place z passes    (hex_action2.cu)
//   v3: v2 + input-streaming contractions, searched pads    (hex_action3.cu)
//   tc: FP64 tensor-core (DMMA) stages, n = 8               (hex_action_tc.cu)
//   cell: one thread per cell, everything in registers, n = 2 (hex_action_p1.cu)
//   v4: v3 with whole cells per warp, no CTA barriers, n = 3..5 (hex_action4.cu)
static int c2_variant() { return (int)option(OPT_C2_KERNEL); }

static int c2_auto(int n) {
  switch (n) {
    case 2: return 5;
    case 3: return 8;   // thread-per-cell over v4: 0.1245 -> 0.1115 ms (profiles/r01cq_*.jsonl)
    case 4: return 10;  // v6 warp-synchronous over v4: 0.2088 -> 0.2034 ms (profiles/r02h_cfg3.json)
    // v6 (collocation derivative, 12 n^4 instead of 16 n^4 FMA) over v3 / v5:
    // p = 4 0.503 -> 0.441, p = 5 0.925 -> 0.813, p = 6 1.448 -> 1.247,
    // p = 8 3.341 -> 2.791 ms (profiles/r02c_v6.json vs r02c_clean.json)
    case 5: return 10;
    case 6: return 10;
    case 7: return 10;
    case 8: return 11;  // tc8c (collocation on DMMA, warp per cell) over tc8: 2.086 -> 1.660 ms (profiles/r02m_*)
    case 9: return 10;
    default: return 1;
  }
}

static int launch_c2(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                     const double* w0, cudaStream_t s) {
  int v = c2_variant();
  if (v == 0) v = c2_auto(p->n);
  int rc = SFK_EUNSUPPORTED;
  if (v == 11) {
    rc = launch_hex_action_tc8c(p, ncells, A, coords, w0, s);
    if (rc == SFK_EUNSUPPORTED) v = c2_auto(p->n);
  }
  if (v == 10) {
    rc = launch_hex_action_v6(p, ncells, A, coords, w0, s);
    if (rc == SFK_EUNSUPPORTED) v = c2_auto(p->n);
  }
  if (v == 8) {
    rc = launch_hex_action_cell(p, ncells, A, coords, w0, s);
    if (rc == SFK_EUNSUPPORTED) v = 3;
  }
  if (v == 7) {
    rc = launch_hex_action_v5(p, ncells, A, coords, w0, s);
    if (rc == SFK_EUNSUPPORTED) v = 2;
  }
  if (v == 6) {
    rc = launch_hex_action_v4(p, ncells, A, coords, w0, s);
    if (rc == SFK_EUNSUPPORTED) v = 3;
  }
  if (v == 5) rc = launch_hex_action_p1(p, ncells, A, coords, w0, s);
  if (v == 4) rc = launch_hex_action_tc(p, ncells, A, coords, w0, s);
  if (v >= 4 && rc == SFK_EUNSUPPORTED) v = 3;
  if (rc == SFK_EUNSUPPORTED && v >= 3) rc = launch_hex_action_v3(p, ncells, A, coords, w0, s);
  if (rc == SFK_EUNSUPPORTED && v >= 2) rc = launch_hex_action_v2(p, ncells, A, coords, w0, s);
  if (rc == SFK_EUNSUPPORTED) rc = launch_hex_action(p, ncells, A, coords, w0, nullptr, s);
  return rc;
}

static int dispatch(const sfk_plan* p, int64_t ncells, double* A,
                    const double* coords, const double* w0, const double* w1,
                    cudaStream_t s) {
  switch (p->kind) {
    case SFK_KIND_ACTION_LAPLACE:
      if (p->dim == 3) {
        if (p->collocated) return launch_hex_colloc_action(p, ncells, A, coords, w0, nullptr, s);
        return launch_c2(p, ncells, A, coords, w0, s);
      }
      return launch_quad_action(p, nullptr, ncells, A, nullptr, coords, w0, s);
    case SFK_KIND_ACTION_WEIGHTED_LAPLACE:
      return launch_hex_colloc_action(p, ncells, A, coords, w0, w1, s);
    case SFK_KIND_ACTION_MASS:
      if (p->dim == 2) return launch_quad_action(p, nullptr, ncells, A, nullptr, coords, w0, s);
      return launch_hex_mass(p, ncells, A, coords, w0, s);
    case SFK_KIND_LAPLACE_MATRIX:
      if (p->dim == 3) return launch_hex_matrix(p, ncells, A, coords, s);
      return fail(SFK_EUNSUPPORTED, "laplace matrix: only the hex kernel is instantiated");
    case SFK_KIND_NEOHOOKEAN_RESIDUAL:
      return launch_hex_neohookean(p, ncells, A, coords, w0, s);
    default:
      return fail(SFK_EUNSUPPORTED, "unknown kernel kind %d", p->kind);
  }
}


// Per-device staging for sfk_eval_host: streams and device buffers are
// created once and reused (the r01 version allocated them per call, which
// cost milliseconds on small batches).  Calls on one device serialise on the
// context mutex.
#ifndef SFK_HOST_STREAMS
#define SFK_HOST_STREAMS 8   // 8 > 4 > 2 streams for e2e (profiles/r01bf_e2e_streams.jsonl)
#endif
struct HostCtx {
  static constexpr int NS = SFK_HOST_STREAMS;
  std::mutex mu;
  bool init = false;
  cudaStream_t stream[NS] = {};
  cudaEvent_t done[NS] = {};   // scratch events (mesh upload fences)
  double* buf[NS] = {};
  size_t cap = 0;
  int reserve(size_t bytes) {
    if (!init) {
      for (int i = 0; i < NS; ++i) {
        int rc = cuda_status(cudaStreamCreateWithFlags(&stream[i], cudaStreamNonBlocking),
                             "cudaStreamCreate(eval_host)");
        if (rc == SFK_OK)
          rc = cuda_status(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming),
                           "cudaEventCreate(eval_host)");
        if (rc != SFK_OK) return rc;
      }
      init = true;
    }
    if (bytes <= cap) return SFK_OK;
    // growing: earlier (possibly asynchronous) calls may still use the buffers
    for (int i = 0; i < NS; ++i) {
      int rc = cuda_status(cudaStreamSynchronize(stream[i]), "cudaStreamSynchronize(eval_host)");
      if (rc != SFK_OK) return rc;
    }
    for (int i = 0; i < NS; ++i) {
      if (buf[i]) cudaFree(buf[i]);
      buf[i] = nullptr;
    }
    cap = 0;
    for (int i = 0; i < NS; ++i) {
      int rc = cuda_status(cudaMalloc(&buf[i], bytes), "cudaMalloc(eval_host staging)");
      if (rc != SFK_OK) return rc;
    }
    cap = bytes;
    return SFK_OK;
  }
};

static HostCtx* host_ctx(int dev) {
  static HostCtx ctx[64];
  return (dev >= 0 && dev < 64) ? &ctx[dev] : nullptr;
}

// The instance table of dispatch(): true when (kind, cell dim, n, m,
// collocated) reaches a kernel.  sfk_plan_create rejects every other
// combination, so an unsupported request fails when the plan is built (the
// reference raises at compile time, cli.py:155-208), never at eval.
// Collocation derivative C = B^-1 D for square tables (n == m): D = B C
// with B[i][q] (basis i, point q).  Gaussian elimination with partial
// pivoting in long double plus one refinement step, then rounded to double,
// so C is (almost always) the correctly rounded product of the reference's
// own tables.  Returns false when B is singular.
static bool collocation_derivative(int n, const double* B, const double* D, double* C) {
  typedef long double R;
  R a[SFK_MAXN][SFK_MAXN], x[SFK_MAXN][SFK_MAXN], rhs[SFK_MAXN][SFK_MAXN];
  int piv[SFK_MAXN];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) a[i][j] = B[i * n + j];
  for (int i = 0; i < n; ++i) piv[i] = i;
  // LU of B (rows i), B = P^T L U
  for (int k = 0; k < n; ++k) {
    int best = k;
    for (int i = k + 1; i < n; ++i)
      if (fabsl(a[i][k]) > fabsl(a[best][k])) best = i;
    if (a[best][k] == 0) return false;
    if (best != k) {
      for (int j = 0; j < n; ++j) {
        R t = a[k][j]; a[k][j] = a[best][j]; a[best][j] = t;
      }
      int t = piv[k]; piv[k] = piv[best]; piv[best] = t;
    }
    for (int i = k + 1; i < n; ++i) {
      a[i][k] /= a[k][k];
      for (int j = k + 1; j < n; ++j) a[i][j] -= a[i][k] * a[k][j];
    }
  }
  auto solve = [&](R (*b)[SFK_MAXN], R (*out)[SFK_MAXN]) {
    for (int col = 0; col < n; ++col) {
      R y[SFK_MAXN];
      for (int i = 0; i < n; ++i) {
        R s = b[piv[i]][col];
        for (int j = 0; j < i; ++j) s -= a[i][j] * y[j];
        y[i] = s;
      }
      for (int i = n - 1; i >= 0; --i) {
        R s = y[i];
        for (int j = i + 1; j < n; ++j) s -= a[i][j] * out[j][col];
        out[i][col] = s / a[i][i];
      }
    }
  };
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) rhs[i][j] = D[i * n + j];
  solve(rhs, x);
  for (int it = 0; it < 2; ++it) {   // refinement: r = D - B x
    R res[SFK_MAXN][SFK_MAXN], dx[SFK_MAXN][SFK_MAXN];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        R s = D[i * n + j];
        for (int k = 0; k < n; ++k) s -= (R)B[i * n + k] * x[k][j];
        res[i][j] = s;
      }
    solve(res, dx);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) x[i][j] += dx[i][j];
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) C[i * n + j] = (double)x[i][j];
  return true;
}

static bool kernel_available(int kind, int dim, int n, int m, int colloc) {
  const bool hex_line = (n == m && n >= 2 && n <= 10) || (m == n + 1 && n >= 2 && n <= 8);
  const bool quad = dim == 2 && !colloc && n == m && n >= 2 && n <= 17;
  const bool colloc_hex = dim == 3 && colloc && n == m && n >= 2 && n <= 17;
  switch (kind) {
    case SFK_KIND_ACTION_LAPLACE:
      return dim == 3 ? (colloc ? colloc_hex : hex_line) : quad;
    case SFK_KIND_ACTION_WEIGHTED_LAPLACE:
      return colloc_hex;
    case SFK_KIND_ACTION_MASS:
      return dim == 3 ? hex_mass_supported(n, m) : quad;
    case SFK_KIND_LAPLACE_MATRIX:
      return dim == 3 && !colloc && n == m && n >= 2 && n <= 9;
    case SFK_KIND_NEOHOOKEAN_RESIDUAL:
      return dim == 3 && !colloc &&
             ((m == n + 1 && n >= 2 && n <= 7) || (m == n && n >= 2 && n <= 4));
    default:
      return false;
  }
}

static int validate(const sfk_plan* p, int64_t ncells, const double* A,
                    const double* coords, const double* w0, const double* w1) {
  if (!p) return fail(SFK_EINVAL, "plan is NULL");
  if (ncells < 0) return fail(SFK_EINVAL, "ncells < 0");
  if (ncells == 0) return SFK_OK;
  if (!A) return fail(SFK_EINVAL, "A is NULL");
  if (!coords) return fail(SFK_EINVAL, "coords is NULL");
  if (p->w0_size > 0 && !w0) return fail(SFK_EINVAL, "w0 is NULL");
  if (p->w1_size > 0 && !w1) return fail(SFK_EINVAL, "w1 is NULL");
  return SFK_OK;
}

}  // namespace sfk

using namespace sfk;

extern "C" {

int sfk_abi_version(void) { return SFK_ABI_VERSION; }

int sfk_plan_create(int kind, int cell_dim, int degree, int n, int m, int collocated,
                    const double* B, const double* D, const double* wq, const double* xq,
                    const double* Bc, const double* Dc, const double* params, int nparams,
                    sfk_plan** out) {
  if (!out) return fail(SFK_EINVAL, "out is NULL");
  *out = nullptr;
  if (kind < SFK_KIND_ACTION_LAPLACE || kind > SFK_KIND_NEOHOOKEAN_RESIDUAL)
    return fail(SFK_EINVAL, "unknown kind %d", kind);
  if (cell_dim != 2 && cell_dim != 3) return fail(SFK_EINVAL, "cell_dim must be 2 or 3");
  if (n < 2 || n > SFK_MAXN) return fail(SFK_EUNSUPPORTED, "n_dof1d=%d outside [2,%d]", n, SFK_MAXN);
  if (m < 1 || m > SFK_MAXM) return fail(SFK_EUNSUPPORTED, "n_q1d=%d outside [1,%d]", m, SFK_MAXM);
  if (!B || !D || !wq || !xq || !Bc || !Dc) return fail(SFK_EINVAL, "NULL table pointer");
  if (nparams < 0 || nparams > 8 || (nparams > 0 && !params))
    return fail(SFK_EINVAL, "bad params (nparams=%d)", nparams);
  if (!kernel_available(kind, cell_dim, n, m, collocated ? 1 : 0))
    return fail(SFK_EUNSUPPORTED,
                "no kernel for kind %d on a %s with %d dofs/axis, %d points/axis%s", kind,
                cell_dim == 3 ? "hex" : "quad", n, m, collocated ? " (collocated)" : "");
  sfk_plan* p = new (std::nothrow) sfk_plan();
  if (!p) return fail(SFK_ENOMEM, "plan allocation failed");
  p->kind = kind;
  p->dim = cell_dim;
  p->degree = degree;
  p->n = n;
  p->m = m;
  p->collocated = collocated ? 1 : 0;
  p->nparams = nparams;
  memcpy(p->B, B, sizeof(double) * n * m);
  memcpy(p->D, D, sizeof(double) * n * m);
  memcpy(p->wq, wq, sizeof(double) * m);
  memcpy(p->xq, xq, sizeof(double) * m);
  memcpy(p->Bc, Bc, sizeof(double) * 2 * m);
  memcpy(p->Dc, Dc, sizeof(double) * 2 * m);
  if (nparams) memcpy(p->params, params, sizeof(double) * nparams);
  p->has_ct = (n == m && n <= SFK_MAXN) ? collocation_derivative(n, B, D, p->Ct) : 0;
  const int64_t nd = cell_dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
  p->coords_size = cell_dim == 3 ? 24 : 8;
  p->w0_size = 0;
  p->w1_size = 0;
  switch (kind) {
    case SFK_KIND_ACTION_LAPLACE:
    case SFK_KIND_ACTION_MASS:
      p->w0_size = nd;
      p->a_size = nd;
      break;
    case SFK_KIND_ACTION_WEIGHTED_LAPLACE:
      p->w0_size = nd;
      p->w1_size = nd;
      p->a_size = nd;
      break;
    case SFK_KIND_LAPLACE_MATRIX:
      p->a_size = nd * nd;
      break;
    case SFK_KIND_NEOHOOKEAN_RESIDUAL:
      p->w0_size = 3 * nd;
      p->a_size = 3 * nd;
      if (nparams < 2) {
        delete p;
        return fail(SFK_EINVAL, "neo-Hookean plan needs params {mu, lambda}");
      }
      break;
  }
  *out = p;
  return SFK_OK;
}

int sfk_kernel_available(int kind, int cell_dim, int n_dof1d, int n_q1d, int collocated) {
  return kernel_available(kind, cell_dim, n_dof1d, n_q1d, collocated ? 1 : 0) ? 1 : 0;
}

int sfk_plan_destroy(sfk_plan* plan) {
  delete plan;
  return SFK_OK;
}

int sfk_plan_sizes(const sfk_plan* p, int64_t* cs, int64_t* w0s, int64_t* w1s, int64_t* as) {
  if (!p) return fail(SFK_EINVAL, "plan is NULL");
  if (cs) *cs = p->coords_size;
  if (w0s) *w0s = p->w0_size;
  if (w1s) *w1s = p->w1_size;
  if (as) *as = p->a_size;
  return SFK_OK;
}

int sfk_eval(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
             const double* w0, const double* w1, void* stream) {
  int st = validate(p, ncells, A, coords, w0, w1);
  if (st != SFK_OK || ncells == 0) return st;
  return dispatch(p, ncells, A, coords, w0, w1, (cudaStream_t)stream);
}

int sfk_eval_pair(const sfk_plan* p0, const sfk_plan* p1, int64_t ncells, double* A0,
                  double* A1, const double* coords, const double* w0, void* stream) {
  int st = validate(p0, ncells, A0, coords, w0, nullptr);
  if (st == SFK_OK) st = validate(p1, ncells, A1, coords, w0, nullptr);
  if (st != SFK_OK || ncells == 0) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const bool fusable = p0->dim == 2 && p1->dim == 2 && p0->n == p1->n && p0->m == p1->m &&
                       !p0->collocated && !p1->collocated &&
                       (p0->kind == SFK_KIND_ACTION_MASS || p0->kind == SFK_KIND_ACTION_LAPLACE) &&
                       (p1->kind == SFK_KIND_ACTION_MASS || p1->kind == SFK_KIND_ACTION_LAPLACE) &&
                       memcmp(p0->wq, p1->wq, sizeof(double) * p0->m) == 0 &&
                       memcmp(p0->B, p1->B, sizeof(double) * p0->n * p0->m) == 0;
  if (fusable) return launch_quad_action(p0, p1, ncells, A0, A1, coords, w0, s);
  st = dispatch(p0, ncells, A0, coords, w0, nullptr, s);
  if (st != SFK_OK) return st;
  return dispatch(p1, ncells, A1, coords, w0, nullptr, s);
}

struct sfk_mesh_impl;
static int eval_host_impl(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                          const double* w0, const double* w1, int64_t chunk, bool wait,
                          const double* dcoords = nullptr, cudaEvent_t ready = nullptr) {
  // dcoords: device-resident coordinates (sfk_mesh), no coords H2D; `ready`
  // orders every staging stream after the mesh upload
  int st = validate(p, ncells, A, dcoords ? dcoords : coords, w0, w1);
  if (st != SFK_OK || ncells == 0) return st;
  const int64_t per_cell = (dcoords ? 0 : p->coords_size) + p->w0_size + p->w1_size + p->a_size;
  if (chunk <= 0) {
    // ~128 MiB of traffic per chunk: H2D of chunk k+1, the kernel of chunk k
    // and the D2H of chunk k-1 overlap (separate copy engines per direction;
    // tools/pcie_probe.py: 55 GB/s H2D, 57 GB/s D2H, 100 GB/s concurrent).
    // e2e GDoF/s by chunk size 16 / 32 / 64 / 128 / 256 MiB: 4.34 / 4.74 /
    // 4.94 / 5.09 / 4.79 (profiles/r01df_*.jsonl)
    const long long mb = option(OPT_HOST_CHUNK_MB) > 0 ? option(OPT_HOST_CHUNK_MB) : 128ll;
    chunk = (int64_t)((mb << 20) / (8 * per_cell));
    if (chunk < 1024) chunk = 1024;
  }
  if (chunk > ncells) chunk = ncells;
  int dev = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc != SFK_OK) return rc;
  HostCtx* ctx = host_ctx(dev);
  if (!ctx) return fail(SFK_EINVAL, "device %d out of range for sfk_eval_host", dev);
  std::lock_guard<std::mutex> lock(ctx->mu);
  const size_t bytes = (size_t)chunk * per_cell * sizeof(double);
  rc = ctx->reserve(bytes);
  if (rc != SFK_OK) return rc;
  int64_t k = 0;
  for (int64_t c0 = 0; c0 < ncells && rc == SFK_OK; c0 += chunk, ++k) {
    const int64_t nc = (ncells - c0) < chunk ? (ncells - c0) : chunk;
    const int i = (int)(k % HostCtx::NS);
    cudaStream_t s = ctx->stream[i];
    double* dc = ctx->buf[i];
    double* dw0 = dc + (dcoords ? 0 : chunk * p->coords_size);
    double* dw1 = dw0 + chunk * p->w0_size;
    double* dA = dw1 + chunk * p->w1_size;
    if (dcoords) {
      dc = const_cast<double*>(dcoords) + c0 * p->coords_size;
      if (ready && k < HostCtx::NS)
        rc = cuda_status(cudaStreamWaitEvent(s, ready, 0), "cudaStreamWaitEvent(mesh)");
    } else {
      rc = cuda_status(cudaMemcpyAsync(dc, coords + c0 * p->coords_size,
                                       nc * p->coords_size * sizeof(double),
                                       cudaMemcpyHostToDevice, s), "H2D coords");
    }
    if (rc == SFK_OK && p->w0_size)
      rc = cuda_status(cudaMemcpyAsync(dw0, w0 + c0 * p->w0_size, nc * p->w0_size * sizeof(double),
                                       cudaMemcpyHostToDevice, s), "H2D w0");
    if (rc == SFK_OK && p->w1_size)
      rc = cuda_status(cudaMemcpyAsync(dw1, w1 + c0 * p->w1_size, nc * p->w1_size * sizeof(double),
                                       cudaMemcpyHostToDevice, s), "H2D w1");
    if (rc == SFK_OK)
      rc = dispatch(p, nc, dA, dc, p->w0_size ? dw0 : nullptr, p->w1_size ? dw1 : nullptr, s);
    if (rc == SFK_OK)
      rc = cuda_status(cudaMemcpyAsync(A + c0 * p->a_size, dA, nc * p->a_size * sizeof(double),
                                       cudaMemcpyDeviceToHost, s), "D2H A");
  }
  if (!wait && rc == SFK_OK) return SFK_OK;
  for (int i = 0; i < HostCtx::NS; ++i) {
    cudaError_t e = cudaStreamSynchronize(ctx->stream[i]);
    if (rc == SFK_OK) rc = cuda_status(e, "cudaStreamSynchronize(eval_host)");
  }
  return rc;
}

int sfk_eval_host(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                  const double* w0, const double* w1, int64_t chunk) {
  return eval_host_impl(p, ncells, A, coords, w0, w1, chunk, true);
}

int sfk_eval_host_async(const sfk_plan* p, int64_t ncells, double* A, const double* coords,
                        const double* w0, const double* w1, int64_t chunk) {
  return eval_host_impl(p, ncells, A, coords, w0, w1, chunk, false);
}

int sfk_host_wait(void) {
  int dev = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc != SFK_OK) return rc;
  HostCtx* ctx = host_ctx(dev);
  if (!ctx) return fail(SFK_EINVAL, "device %d out of range", dev);
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (!ctx->init) return SFK_OK;
  for (int i = 0; i < HostCtx::NS; ++i) {
    cudaError_t e = cudaStreamSynchronize(ctx->stream[i]);
    if (rc == SFK_OK) rc = cuda_status(e, "cudaStreamSynchronize(host_wait)");
  }
  return rc;
}

// ---- device-resident meshes ------------------------------------------------
struct sfk_mesh {
  int dev = 0;
  int64_t ncells = 0;
  int coords_size = 0;
  double* d = nullptr;
  cudaEvent_t ready = nullptr;
};

int sfk_mesh_create(int64_t ncells, int coords_size, sfk_mesh** out) {
  if (!out) return fail(SFK_EINVAL, "out is NULL");
  *out = nullptr;
  if (ncells < 0) return fail(SFK_EINVAL, "ncells < 0");
  if (coords_size != 24 && coords_size != 8)
    return fail(SFK_EINVAL, "coords_size must be 24 (hex) or 8 (quad), got %d", coords_size);
  sfk_mesh* m = new (std::nothrow) sfk_mesh();
  if (!m) return fail(SFK_ENOMEM, "mesh allocation failed");
  int rc = cuda_status(cudaGetDevice(&m->dev), "cudaGetDevice");
  if (rc == SFK_OK && ncells > 0)
    rc = cuda_status(cudaMalloc(&m->d, (size_t)ncells * coords_size * sizeof(double)),
                     "cudaMalloc(mesh)");
  if (rc == SFK_OK)
    rc = cuda_status(cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming),
                     "cudaEventCreate(mesh)");
  if (rc != SFK_OK) {
    if (m->d) cudaFree(m->d);
    delete m;
    return rc;
  }
  m->ncells = ncells;
  m->coords_size = coords_size;
  *out = m;
  return SFK_OK;
}

int sfk_mesh_destroy(sfk_mesh* m) {
  if (!m) return SFK_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(m->dev);
  cudaEventSynchronize(m->ready);
  if (m->d) cudaFree(m->d);
  cudaEventDestroy(m->ready);
  cudaSetDevice(cur);
  delete m;
  return SFK_OK;
}

const double* sfk_mesh_coords(const sfk_mesh* m) { return m ? m->d : nullptr; }

int sfk_mesh_upload(sfk_mesh* m, const double* coords) {
  if (!m) return fail(SFK_EINVAL, "mesh is NULL");
  if (m->ncells == 0) return SFK_OK;
  if (!coords) return fail(SFK_EINVAL, "coords is NULL");
  int dev = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc != SFK_OK) return rc;
  if (dev != m->dev) return fail(SFK_EINVAL, "mesh lives on device %d, current is %d", m->dev, dev);
  HostCtx* ctx = host_ctx(dev);
  std::lock_guard<std::mutex> lock(ctx->mu);
  rc = ctx->reserve(0);   // streams exist
  if (rc != SFK_OK) return rc;
  cudaStream_t s = ctx->stream[0];
  // earlier evaluations on the other staging streams may still read the
  // mesh: order the overwrite after them
  for (int i = 1; i < HostCtx::NS && rc == SFK_OK; ++i) {
    cudaEvent_t e = ctx->done[i];
    rc = cuda_status(cudaEventRecord(e, ctx->stream[i]), "cudaEventRecord(mesh fence)");
    if (rc == SFK_OK) rc = cuda_status(cudaStreamWaitEvent(s, e, 0), "cudaStreamWaitEvent(mesh fence)");
  }
  if (rc != SFK_OK) return rc;
  rc = cuda_status(cudaMemcpyAsync(m->d, coords, (size_t)m->ncells * m->coords_size * sizeof(double),
                                   cudaMemcpyHostToDevice, s), "H2D mesh");
  if (rc == SFK_OK) rc = cuda_status(cudaEventRecord(m->ready, s), "cudaEventRecord(mesh)");
  return rc;
}

int sfk_eval_host_mesh(const sfk_plan* p, const sfk_mesh* m, int64_t first_cell, int64_t ncells,
                       double* A, const double* w0, const double* w1, int64_t chunk_cells,
                       int wait) {
  if (!m) return fail(SFK_EINVAL, "mesh is NULL");
  if (!p) return fail(SFK_EINVAL, "plan is NULL");
  if (p->coords_size != m->coords_size)
    return fail(SFK_EINVAL, "plan takes %lld coordinates per cell, the mesh holds %d",
                (long long)p->coords_size, m->coords_size);
  if (first_cell < 0 || ncells < 0 || first_cell + ncells > m->ncells)
    return fail(SFK_EINVAL, "cells [%lld, %lld) outside the mesh (%lld cells)",
                (long long)first_cell, (long long)(first_cell + ncells), (long long)m->ncells);
  int dev = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc != SFK_OK) return rc;
  if (dev != m->dev) return fail(SFK_EINVAL, "mesh lives on device %d, current is %d", m->dev, dev);
  if (ncells == 0) return SFK_OK;
  return eval_host_impl(p, ncells, A, nullptr, w0, w1, chunk_cells, wait != 0,
                        m->d + first_cell * m->coords_size, m->ready);
}

int sfk_eval_gather_scatter(const sfk_plan* p, int64_t ncells, const int32_t* cell_dofs,
                            const double* x, double* y, const double* coords, void* stream) {
  if (!p) return fail(SFK_EINVAL, "plan is NULL");
  if (ncells < 0) return fail(SFK_EINVAL, "ncells < 0");
  if (ncells == 0) return SFK_OK;
  if (!cell_dofs || !x || !y || !coords) return fail(SFK_EINVAL, "NULL pointer argument");
  if (p->kind != SFK_KIND_ACTION_LAPLACE || p->dim != 3 || p->collocated || p->n != p->m)
    return fail(SFK_EUNSUPPORTED,
                "gather/scatter operator: hex action_laplace with m == n only");
  return launch_hex_action_gs(p, ncells, cell_dofs, x, y, coords, (cudaStream_t)stream);
}

int sfk_eval_global(const sfk_plan* p, int64_t ncells, const int32_t* cell_dofs,
                    const double* x, double* y, const double* coords, const double* w1,
                    void* stream) {
  if (!p) return fail(SFK_EINVAL, "plan is NULL");
  if (ncells < 0) return fail(SFK_EINVAL, "ncells < 0");
  if (ncells == 0) return SFK_OK;
  if (!cell_dofs || !x || !y || !coords) return fail(SFK_EINVAL, "NULL pointer argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (p->dim != 3) return fail(SFK_EUNSUPPORTED, "global operator: hex plans only");
  switch (p->kind) {
    case SFK_KIND_ACTION_LAPLACE:
      if (w1) return fail(SFK_EINVAL, "action_laplace takes no w1");
      if (p->collocated) return launch_hex_colloc_gs(p, ncells, cell_dofs, x, y, coords, nullptr, s);
      if (p->n != p->m)
        return fail(SFK_EUNSUPPORTED, "global operator: action_laplace with m == n only");
      return launch_hex_action_gs(p, ncells, cell_dofs, x, y, coords, s);
    case SFK_KIND_ACTION_WEIGHTED_LAPLACE:
      if (!w1) return fail(SFK_EINVAL, "w1 (kappa per cell) is NULL");
      return launch_hex_colloc_gs(p, ncells, cell_dofs, x, y, coords, w1, s);
    case SFK_KIND_NEOHOOKEAN_RESIDUAL:
      if (w1) return fail(SFK_EINVAL, "neohookean_residual takes no w1");
      return launch_hex_neohookean_gs(p, ncells, cell_dofs, x, y, coords, s);
    default:
      return fail(SFK_EUNSUPPORTED, "global operator: kind %d has no fused gather/scatter",
                  p->kind);
  }
}

int sfk_assemble_csr(const sfk_plan* p, int64_t ncells, const int32_t* cell_dofs,
                     const double* coords, const int64_t* row_ptr, const int32_t* col_idx,
                     const int32_t* entry_map, double* values, void* stream) {
  if (!p) return fail(SFK_EINVAL, "plan is NULL");
  if (ncells < 0) return fail(SFK_EINVAL, "ncells < 0");
  if (ncells == 0) return SFK_OK;
  if (!cell_dofs || !coords || !row_ptr || !col_idx || !values)
    return fail(SFK_EINVAL, "NULL pointer argument");
  if (p->kind != SFK_KIND_LAPLACE_MATRIX || p->dim != 3)
    return fail(SFK_EUNSUPPORTED, "CSR assembly: hex laplace (matrix) plans only");
  return launch_hex_matrix_csr(p, ncells, cell_dofs, coords, row_ptr, col_idx, entry_map, values,
                               (cudaStream_t)stream);
}

int sfk_sum_squares(const double* x, int64_t n, double* out, void* stream) {
  if (n < 0) return fail(SFK_EINVAL, "n < 0");
  if (!out) return fail(SFK_EINVAL, "out is NULL");
  if (n == 0) return SFK_OK;
  if (!x) return fail(SFK_EINVAL, "x is NULL");
  return launch_sum_squares(x, n, out, (cudaStream_t)stream);
}

int64_t sfk_launch_count(void) { return g_launches.load(); }

int sfk_last_error(char* buf, int64_t size) {
  if (!buf || size <= 0) return SFK_EINVAL;
  snprintf(buf, (size_t)size, "%s", g_err);
  return SFK_OK;
}

int sfk_device_info(int device, int* sm_count, int* sm_clock_khz, int* mem_clock_khz,
                    int* mem_bus_bits, char* name, int name_size) {
  cudaDeviceProp prop;
  int rc = cuda_status(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (rc != SFK_OK) return rc;
  if (sm_count) *sm_count = prop.multiProcessorCount;
  int v = 0;
  if (sm_clock_khz) {
    cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, device);
    *sm_clock_khz = v;
  }
  if (mem_clock_khz) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMemoryClockRate, device);
    *mem_clock_khz = v;
  }
  if (mem_bus_bits) {
    cudaDeviceGetAttribute(&v, cudaDevAttrGlobalMemoryBusWidth, device);
    *mem_bus_bits = v;
  }
  if (name && name_size > 0) snprintf(name, (size_t)name_size, "%s", prop.name);
  return SFK_OK;
}

int sfk_fp64_peak(double seconds, double* dfma, double* dmma) {
  return run_fp64_peak(seconds, dfma, dmma);
}

}  // extern "C"
