/*
 * sfk.h — C ABI of the B200 (sm_100a) sum-factorised cell-kernel library
 * (libsfk.so, built from paper_1711_02473_b200/csrc).
 *
 * What it replaces.  The reference `sumfact` emits one C99 function per
 * kernel,
 *
 *     void NAME(double *restrict A, const double *restrict coords,
 *               const double *restrict w0 [, const double *restrict w1]);
 *
 * (reference pkg/src/sumfact/scheduling.py:731-735) and leaves the loop over
 * cells to the caller.  `sfk_eval` is that loop, for a whole
 * batch of cells, on the GPU: same argument order (A first, then coords,
 * w0, w1), same per-cell layouts, same overwrite
 * semantics (the emitted kernel zero-fills A first, scheduling.py:372).
 * `sfk_plan_create` replaces the static const tables T0..Tk the emitted C
 * embeds (scheduling.py:724-728): the caller passes the reference-bit-exact
 * 1D tables produced on the host by `compile_kernel` (cli.py:211-217).
 *
 * Conventions.
 *   - Every function returns 0 (SFK_OK) or a non-zero sfk_status; the text of
 *     the last error on the calling thread is available from sfk_last_error.
 *   - Batched arrays are C-contiguous row-major [ncells][size] fp64.
 *   - sfk_eval* take DEVICE pointers, enqueue on `stream` (a cudaStream_t,
 *     NULL = legacy default stream) and return without synchronising.  They
 *     do not allocate.  A must not alias the inputs; it is overwritten.
 *   - sfk_eval_host takes HOST pointers and is synchronous: it is the
 *     drop-in for the caller's `for c in cells: NAME(A+c*nA, coords+c*nc,
 *     w0+c*nw)` loop, with host<->device copies pipelined against compute.
 *   - Plans are immutable after creation and may be used concurrently from
 *     several threads/streams (the emitted kernels are reentrant).
 */
#ifndef SFK_H
#define SFK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFK_ABI_VERSION 1

typedef struct sfk_plan sfk_plan;

typedef enum sfk_status {
  SFK_OK = 0,
  SFK_EINVAL = 1,        /* bad argument (null pointer, negative count, ...)  */
  SFK_EUNSUPPORTED = 2,  /* no kernel instantiated for this kind/degree/points */
  SFK_ECUDA = 3,         /* CUDA runtime error                                 */
  SFK_ENOMEM = 4         /* host or device allocation failed                   */
} sfk_status;

typedef enum sfk_kind {
  /* hex or quad Laplace action b = K u (registry `action_laplace`,
   * reference forms.py:186-189, 235-243, 261-263); GL(m) or collocated GLL */
  SFK_KIND_ACTION_LAPLACE = 1,
  /* hex weighted Laplace action b = K_kappa u, kappa = w1 at GLL points
   * (action_form(REGISTRY['weighted_laplace']), forms.py:192-193)        */
  SFK_KIND_ACTION_WEIGHTED_LAPLACE = 2,
  /* mass action b = M u (registry `action_mass`, forms.py:173)            */
  SFK_KIND_ACTION_MASS = 3,
  /* local stiffness matrix, test-major A[i*N+j] (registry `laplace`)      */
  SFK_KIND_LAPLACE_MATRIX = 4,
  /* vector Q_p^3 neo-Hookean residual (builder FormSpec);
   * params = {mu, lambda}                                                 */
  SFK_KIND_NEOHOOKEAN_RESIDUAL = 5
} sfk_kind;

/* ABI version of the loaded library (== SFK_ABI_VERSION). */
int sfk_abi_version(void);

/*
 * Create a plan.  Host pointers, copied into the plan:
 *   B, D    [n_dof1d * n_q1d]  1D basis / derivative tables, basis-major
 *           (T[n_q1d*i + q], as the emitted C indexes its tables)
 *   wq      [n_q1d]            1D quadrature weights on [0,1]
 *   xq      [n_q1d]            1D quadrature points on [0,1]
 *   Bc, Dc  [2 * n_q1d]        P1 coordinate-element tables at the points
 *   params  [nparams]          form parameters (neo-Hookean: mu, lambda)
 * cell_dim: 2 (quad) or 3 (hex).  collocated: 1 when B is the identity
 * (GLL element evaluated at its own nodes, reference elements.py:200-220).
 * Replaces: the static const tables of the emitted kernel
 * (reference scheduling.py:724-728); built by compile_kernel (cli.py:211).
 */
int sfk_plan_create(int kind, int cell_dim, int degree, int n_dof1d,
                    int n_q1d, int collocated, const double *B,
                    const double *D, const double *wq, const double *xq,
                    const double *Bc, const double *Dc, const double *params,
                    int nparams, sfk_plan **out);

int sfk_plan_destroy(sfk_plan *plan);

/* 1 when a kernel is instantiated for this (kind, cell_dim, n_dof1d, n_q1d,
 * collocated), else 0.  Host-only, no CUDA call.  sfk_plan_create fails with
 * SFK_EUNSUPPORTED for every combination this rejects, and compile_kernel
 * raises Unsupported for them (the reference raises at compile time,
 * cli.py:155-208). */
int sfk_kernel_available(int kind, int cell_dim, int n_dof1d, int n_q1d,
                         int collocated);

/* Per-cell sizes of the plan's arguments, in doubles (for validation). */
int sfk_plan_sizes(const sfk_plan *plan, int64_t *coords_size,
                   int64_t *w0_size, int64_t *w1_size, int64_t *a_size);

/*
 * Batched evaluation on the device (replaces the caller's C cell loop around
 * the emitted `NAME(A, coords, w0[, w1])`, scheduling.py:731-735).
 *   A      [ncells][a_size]       output, overwritten
 *   coords [ncells][2^d * d]      vertex coordinates, v = 4a+2b+c, comp inner
 *   w0     [ncells][w0_size]      coefficient 0 (trial dofs for actions)
 *   w1     [ncells][w1_size]      coefficient 1 (kappa) or NULL
 */
int sfk_eval(const sfk_plan *plan, int64_t ncells, double *A,
             const double *coords, const double *w0, const double *w1,
             void *stream);

/*
 * Fused evaluation of two plans sharing (coords, w0) in one launch
 * (BASELINE config C1: quad Q3 action_mass + action_laplace).  Falls back to
 * two launches when the pair has no fused kernel.
 */
int sfk_eval_pair(const sfk_plan *plan0, const sfk_plan *plan1,
                  int64_t ncells, double *A0, double *A1,
                  const double *coords, const double *w0, void *stream);

/*
 * Host-buffer evaluation: synchronous, chunked, copies pipelined with
 * compute on internal streams.  Same layouts as sfk_eval.  chunk_cells <= 0
 * picks a default.  Pinned (page-locked) host buffers give full PCIe
 * bandwidth; pageable buffers work but copy slower.
 */
int sfk_eval_host(const sfk_plan *plan, int64_t ncells, double *A,
                  const double *coords, const double *w0, const double *w1,
                  int64_t chunk_cells);

/*
 * The same, enqueued only: returns once every copy and kernel of the batch is
 * queued on the library's per-device staging streams, so consecutive calls
 * (e.g. one per degree) overlap their copy pipelines.  The host buffers must
 * stay valid and untouched until sfk_host_wait() returns; results are in A
 * only then.
 */
int sfk_eval_host_async(const sfk_plan *plan, int64_t ncells, double *A,
                        const double *coords, const double *w0,
                        const double *w1, int64_t chunk_cells);
/* Wait for every sfk_eval_host_async call on the current device. */
int sfk_host_wait(void);

/*
 * Device-resident meshes.  The reference's caller loop passes the same
 * coordinates to every kernel it runs on a mesh (scheduling.py:731-735 takes
 * `coords` per call); with several operators, degrees or iterations over one
 * mesh the host path would re-send them on every call.  A mesh holds them on
 * the current device: upload once (sfk_mesh_upload: asynchronous, on the
 * host path's first staging stream; every later sfk_eval_host_mesh call on
 * the device is ordered after it), then evaluate with host w0 / w1 / A only.
 *   coords_size: 24 (hex) or 8 (quad) doubles per cell.
 */
typedef struct sfk_mesh sfk_mesh;
int sfk_mesh_create(int64_t ncells, int coords_size, sfk_mesh **out);
int sfk_mesh_upload(sfk_mesh *mesh, const double *coords_host);
/* device pointer of the mesh coordinates ([ncells][coords_size]) for sfk_eval */
const double *sfk_mesh_coords(const sfk_mesh *mesh);
int sfk_mesh_destroy(sfk_mesh *mesh);
/* cells [first_cell, first_cell + ncells) of the mesh; A, w0, w1 are HOST
 * arrays for those cells.  wait = 0: asynchronous like sfk_eval_host_async
 * (complete after sfk_host_wait); wait != 0: synchronous like sfk_eval_host. */
int sfk_eval_host_mesh(const sfk_plan *plan, const sfk_mesh *mesh, int64_t first_cell,
                       int64_t ncells, double *A, const double *w0, const double *w1,
                       int64_t chunk_cells, int wait);

/*
 * Global (assembled) operator application, matrix-free:
 *     y += sum_c P_c^T A_c P_c x
 * P_c gathers the cell's local dofs from the global vector x through
 * cell_dofs[c][i] (global index of local dof i of cell c, reference local
 * order (ix*n+iy)*n+iz); A_c is the plan's cell kernel; the scatter-add into
 * y is fused (fp64 atomics, so the summation order of shared dofs is not
 * fixed).  DEVICE pointers, stream-ordered; y is accumulated into (zero it
 * first for y = K x).  Supported: hex action_laplace, GL (m == n).
 * Replaces: the caller's assembly loop around the emitted kernel — the
 * "global gather/scatter" next step of SURVEY.md §8(f) (the reference
 * scopes global assembly out).
 */
int sfk_eval_gather_scatter(const sfk_plan *plan, int64_t ncells,
                            const int32_t *cell_dofs, const double *x,
                            double *y, const double *coords, void *stream);

/*
 * The same for every action kernel with a fused gather/scatter mode:
 *     y += sum_c P_c^T K_c(P_c x)
 * hex action_laplace (GL or collocated GLL), action_weighted_laplace (w1 =
 * kappa per cell, [ncells][n^3], NOT gathered) and the neo-Hookean residual
 * (cell_dofs[c][3*node + comp], the reference's vector dof order; y is the
 * assembled nonlinear residual r(x)).  Same conventions as
 * sfk_eval_gather_scatter, which is this call with w1 = NULL.
 */
int sfk_eval_global(const sfk_plan *plan, int64_t ncells,
                    const int32_t *cell_dofs, const double *x, double *y,
                    const double *coords, const double *w1, void *stream);

/*
 * Assembled sparse matrices (local-matrix assembly +
 * sparse insertion; the paper's "global assembly" step, PAPER.md:166-167,
 * scoped out by the reference).
 *
 * sfk_csr_create: the CSR sparsity pattern of sum_c P_c^T A_c P_c for the
 * cell -> dof map cell_dofs[ncells][ndofs_per_cell] (DEVICE, int32 global
 * dof numbers < ndofs): rows 0..ndofs-1, row_ptr int64, col_idx int32
 * sorted ascending within each row.  Built on the device (radix sort +
 * unique of the (row, col) pairs), synchronous on `stream`; the pattern
 * owns its device arrays (sfk_csr_info exposes them, sfk_csr_destroy frees
 * them).  Requires ndofs^2 < 2^64.
 */
typedef struct sfk_csr sfk_csr;
int sfk_csr_create(int64_t ncells, int ndofs_per_cell, const int32_t *cell_dofs,
                   int64_t ndofs, void *stream, sfk_csr **out);
int sfk_csr_info(const sfk_csr *pattern, int64_t *nrows, int64_t *nnz,
                 int64_t **row_ptr, int32_t **col_idx);
/* Entry map of a pattern: map[c][i][j] (DEVICE, int32, caller-allocated,
 * ncells * ndofs_per_cell^2) = position of the cell entry (i, j) in
 * col_idx/values.  Computed once per pattern (binary search per entry);
 * passed to sfk_assemble_csr it turns every insertion into one load and one
 * atomic.  Requires nnz < 2^31. */
int sfk_csr_entry_map(const sfk_csr *pattern, int64_t ncells, int ndofs_per_cell,
                      const int32_t *cell_dofs, int32_t *map, void *stream);
int sfk_csr_destroy(sfk_csr *pattern);

/*
 * values[nnz] += sum_c P_c^T A_c P_c for DENSE per-cell matrices
 * cell_matrices[ncells][nd][nd] (test index outer — the reference's return
 * layout, forms.py:402-408) produced by ANY kernel: a hand-written family or
 * a generated LoopProgram (every registry matrix form, any cell / degree /
 * vector layout).  Positions from entry_map (sfk_csr_entry_map) when
 * non-NULL, else a binary search per entry in row_ptr / col_idx.  DEVICE
 * pointers, stream-ordered, fp64 atomics.  Replaces: the caller's insertion
 * loop around any emitted matrix kernel.
 */
int sfk_csr_insert(int64_t ncells, int ndofs_per_cell, const double *cell_matrices,
                   const int32_t *cell_dofs, const int64_t *row_ptr, const int32_t *col_idx,
                   const int32_t *entry_map, double *values, void *stream);

/*
 * values[nnz] += the assembled hex Laplace stiffness matrix: the C5 kernel
 * (plan kind SFK_KIND_LAPLACE_MATRIX, p <= 4) computes each cell matrix in
 * shared memory/registers and scatter-adds it straight into the CSR values
 * (fp64 atomics) — the (p+1)^6 local matrix never reaches HBM.  Positions
 * come from entry_map (sfk_csr_entry_map) when it is non-NULL, else from a
 * binary search of the column in its row.  DEVICE pointers, stream-ordered;
 * zero `values` first.  Replaces: the caller's insertion loop around the
 * emitted `laplace` kernel.
 */
int sfk_assemble_csr(const sfk_plan *plan, int64_t ncells,
                     const int32_t *cell_dofs, const double *coords,
                     const int64_t *row_ptr, const int32_t *col_idx,
                     const int32_t *entry_map, double *values, void *stream);

/*
 * Functionals/checksums of a device array x[0..n):
 *   out[0] = sum x_i^2,  out[1] = sum x_i        (overwritten)
 * `out` is a DEVICE buffer of at least SFK_SUM_WORKSPACE doubles (the tail is
 * scratch for per-CTA partials, so the call does not allocate).  The
 * summation order depends only on n, so the result is bitwise reproducible.
 * Used for the Frobenius checksum all-reduced over ranks (BASELINE C5).
 */
#define SFK_SUM_WORKSPACE 1024
int sfk_sum_squares(const double *x, int64_t n, double *out, void *stream);

/* ------------------------------------------------------------------------
 * LoopProgram path: any kernel the reference can
 * compile, given as its loss-free JSON serialization
 *     sumfact.scheduling.serialize_program(program)   (scheduling.py:465-532)
 * of the LoopProgram returned by cli.compile_kernel (cli.py:211-217) or
 * scheduling.schedule (scheduling.py:341).  libsfk generates a batched
 * sm_100a kernel from the statement list (one CTA-wide phase per loop nest,
 * buffers in shared memory, cells across threads) and compiles it with
 * NVRTC.  Replaces: emit_c + the host C compiler + the caller's per-cell
 * loop (scheduling.py:617-738).  Without SFK_PROGRAM_FMA every
 * target element is summed in the reference's loop order with separately
 * rounded multiplies and adds, i.e. bit-identical to the reference's C
 * compiled with -ffp-contract=off (IEEE division and sqrt on both sides).
 * ---------------------------------------------------------------------- */
typedef struct sfk_program sfk_program;

#define SFK_PROGRAM_FMA 1     /* allow FMA contraction (not bit-exact)       */
#define SFK_PROGRAM_NO_JIT 2  /* parse + generate only (inspect the source)  */

/* json: the serialize_program text (len < 0: NUL-terminated).  Parses,
 * generates and JIT-compiles (NVRTC, no GPU needed); the module is loaded on
 * a device at its first sfk_program_eval there.  Malformed programs ->
 * SFK_EINVAL (the reference's UnloweredNode / parse errors); NVRTC missing
 * -> SFK_EUNSUPPORTED. */
int sfk_program_create(const char *json, int64_t len, int flags,
                       sfk_program **out);
int sfk_program_destroy(sfk_program *program);

/* program.return_buffer[1] and the sizes of program.arguments, in order. */
int sfk_program_sizes(const sfk_program *program, int64_t *return_size,
                      int *nargs, int64_t *arg_sizes, int max_args);

/* Launch geometry: out[0..10] = cells per CTA, threads, slots per cell,
 * dynamic smem bytes, global-scratch flag, phases, serial phases, barriers,
 * cubin bytes, warp mode (1: each warp owns whole cells, barriers are
 * __syncwarp), phases fused into the previous phase's loop. */
int sfk_program_config(const sfk_program *program, int64_t *out, int n);

/* what = 0: generated CUDA source, 1: kernel entry name, 2: program name. */
int sfk_program_text(const sfk_program *program, int what, char *buf,
                     int64_t size, int64_t *length);

/* A[ncells][return_size] = NAME(coords, w0, ...) per cell.  DEVICE pointers
 * (args[k] is [ncells][arg_sizes[k]], in program.arguments order), enqueued
 * on `stream`; A is overwritten (the emitted kernel zero-fills it). */
int sfk_program_eval(const sfk_program *program, int64_t ncells, double *A,
                     const double *const *args, int nargs, void *stream);

/* Number of sfk kernels launched by this process so far (all threads). */
int64_t sfk_launch_count(void);

/* Copy the calling thread's last error message (NUL-terminated). */
int sfk_last_error(char *buf, int64_t size);

/* Device facts for the roofline logs. */
int sfk_device_info(int device, int *sm_count, int *sm_clock_khz,
                    int *mem_clock_khz, int *mem_bus_bits, char *name,
                    int name_size);

/*
 * FP64 peak micro-benchmark on the current device: DFMA chains and
 * DMMA (mma.sync m8n8k4 f64).  Runs about `seconds` in total.
 */
int sfk_fp64_peak(double seconds, double *tflops_dfma, double *tflops_dmma);

/*
 * Tuning options (A/B runs of kernel variants; no reference counterpart —
 * the reference has no runtime).  `name` is one of the lower-case option
 * names of csrc/sfk_options.h ("c2_kernel", "c2_g", "host_chunk_mb", ...);
 * 0 restores the built-in, measured-best choice.  Process-wide and
 * thread-safe.  The library reads no environment variables for dispatch:
 * these calls are the only way to change a kernel choice.
 */
int sfk_set_option(const char *name, int64_t value);
int sfk_get_option(const char *name, int64_t *value);

#ifdef __cplusplus
}
#endif

#endif /* SFK_H */
