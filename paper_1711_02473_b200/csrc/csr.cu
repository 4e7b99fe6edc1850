// CSR sparsity pattern of an assembled operator from a cell -> dof map
// ("local-matrix assembly plus sparse insertion";
// the reference scopes global assembly out).
//
// Symbolic phase on the device: every (row, col) = (dof[c][i], dof[c][j])
// pair becomes a 64-bit key row*ndofs + col; CUB radix-sorts the keys (only
// the bits ndofs^2 needs), removes duplicates, and row_ptr[r] is the lower
// bound of r*ndofs in the unique keys.  col_idx within a row is therefore
// sorted ascending, which the numeric phase (hex_matrix.cu, CSR epilogue)
// binary-searches.  The pattern owns its device arrays (sfk_csr_destroy).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "sfk_internal.cuh"

struct sfk_csr {
  int64_t nrows = 0, nnz = 0;
  int64_t* row_ptr = nullptr;  // [nrows + 1]
  int32_t* col_idx = nullptr;  // [nnz]
  int device = 0;
};

namespace sfk {

__global__ void csr_keys_kernel(int64_t ncells, int ndpc, const int32_t* __restrict__ dofs,
                                int64_t ndofs, uint64_t* __restrict__ keys) {
  const int64_t per = (int64_t)ndpc * ndpc;
  const int64_t total = ncells * per;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = k / per;
    const int r = (int)(k - c * per);
    const int i = r / ndpc, j = r - i * ndpc;
    const int64_t row = __ldg(dofs + c * ndpc + i), col = __ldg(dofs + c * ndpc + j);
    keys[k] = (uint64_t)(row * ndofs + col);
  }
}

__global__ void csr_rows_kernel(const uint64_t* __restrict__ keys, int64_t nnz, int64_t ndofs,
                                int64_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t k = t0; k < nnz; k += stride) col_idx[k] = (int32_t)(keys[k] % (uint64_t)ndofs);
  for (int64_t r = t0; r <= ndofs; r += stride) {
    const uint64_t target = (uint64_t)r * (uint64_t)ndofs;
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    row_ptr[r] = lo;
  }
}

// map[c][i][j] = position of (dof[c][i], dof[c][j]) in the CSR arrays
// (binary search within the row; done once per pattern).
__global__ void csr_map_kernel(int64_t ncells, int ndpc, const int32_t* __restrict__ dofs,
                               const int64_t* __restrict__ row_ptr,
                               const int32_t* __restrict__ col_idx, int32_t* __restrict__ map) {
  const int64_t per = (int64_t)ndpc * ndpc;
  const int64_t total = ncells * per;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = k / per;
    const int r = (int)(k - c * per);
    const int i = r / ndpc, j = r - i * ndpc;
    const int32_t row = __ldg(dofs + c * ndpc + i), col = __ldg(dofs + c * ndpc + j);
    int64_t lo = __ldg(row_ptr + row), hi = __ldg(row_ptr + row + 1);
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(col_idx + mid) < col) lo = mid + 1; else hi = mid;
    }
    map[k] = (int32_t)lo;
  }
}

// values[pos(c, i, j)] += Ac[c][i][j] for dense per-cell matrices (test
// index outer, as every reference kernel returns them): the insertion half of
// sfk_assemble_csr for matrices produced by any kernel (hand-written or a
// generated LoopProgram).  pos from the entry map, else a binary search of
// the column within its row.
__global__ void csr_insert_kernel(int64_t ncells, int ndpc, const double* __restrict__ Ac,
                                  const int32_t* __restrict__ dofs,
                                  const int64_t* __restrict__ row_ptr,
                                  const int32_t* __restrict__ col_idx,
                                  const int32_t* __restrict__ map, double* __restrict__ values) {
  const int64_t per = (int64_t)ndpc * ndpc;
  const int64_t total = ncells * per;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t pos;
    if (map) {
      pos = __ldg(map + k);
    } else {
      const int64_t c = k / per;
      const int r = (int)(k - c * per);
      const int i = r / ndpc, j = r - i * ndpc;
      const int32_t row = __ldg(dofs + c * ndpc + i), col = __ldg(dofs + c * ndpc + j);
      int64_t lo = __ldg(row_ptr + row), hi = __ldg(row_ptr + row + 1);
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(col_idx + mid) < col) lo = mid + 1; else hi = mid;
      }
      pos = lo;
    }
    atomicAdd(values + pos, __ldg(Ac + k));
  }
}

}  // namespace sfk

using namespace sfk;

extern "C" {

int sfk_csr_create(int64_t ncells, int ndofs_per_cell, const int32_t* cell_dofs, int64_t ndofs,
                   void* stream, sfk_csr** out) {
  if (!out) return fail(SFK_EINVAL, "sfk_csr_create: out is NULL");
  *out = nullptr;
  if (ncells < 0 || ndofs_per_cell <= 0 || ndofs <= 0 || ndofs > INT32_MAX)
    return fail(SFK_EINVAL, "sfk_csr_create: bad sizes");
  if (ncells > 0 && !cell_dofs) return fail(SFK_EINVAL, "sfk_csr_create: cell_dofs is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  auto* P = new (std::nothrow) sfk_csr;
  if (!P) return fail(SFK_ENOMEM, "sfk_csr_create: out of memory");
  P->nrows = ndofs;
  cudaGetDevice(&P->device);
  const int64_t nkeys = ncells * (int64_t)ndofs_per_cell * ndofs_per_cell;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  int64_t* dnum = nullptr;
  void* tmp = nullptr;
  int rc = SFK_OK;
  auto cleanup = [&]() {
    cudaFreeAsync(k0, s);
    cudaFreeAsync(k1, s);
    cudaFreeAsync(dnum, s);
    cudaFreeAsync(tmp, s);
  };
  do {
    if ((rc = cuda_status(cudaMalloc(&P->row_ptr, (ndofs + 1) * sizeof(int64_t)), "csr row_ptr")))
      break;
    if (nkeys == 0) {
      rc = cuda_status(cudaMemsetAsync(P->row_ptr, 0, (ndofs + 1) * sizeof(int64_t), s), "memset");
      break;
    }
    if ((rc = cuda_status(cudaMallocAsync(&k0, nkeys * 8, s), "csr keys"))) break;
    if ((rc = cuda_status(cudaMallocAsync(&k1, nkeys * 8, s), "csr keys"))) break;
    if ((rc = cuda_status(cudaMallocAsync(&dnum, 8, s), "csr count"))) break;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((nkeys + threads - 1) / threads, 148 * 32);
    csr_keys_kernel<<<(unsigned)blocks, threads, 0, s>>>(ncells, ndofs_per_cell, cell_dofs, ndofs, k0);
    note_launch();
    int end_bit = 1;
    while (end_bit < 64 && ((uint64_t)1 << end_bit) < (uint64_t)ndofs * (uint64_t)ndofs) ++end_bit;
    size_t b_sort = 0, b_uniq = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b_sort, k0, k1, nkeys, 0, end_bit, s);
    cub::DeviceSelect::Unique(nullptr, b_uniq, k1, k0, dnum, nkeys, s);
    if ((rc = cuda_status(cudaMallocAsync(&tmp, std::max(b_sort, b_uniq), s), "csr cub temp"))) break;
    if ((rc = cuda_status(cub::DeviceRadixSort::SortKeys(tmp, b_sort, k0, k1, nkeys, 0, end_bit, s),
                          "cub sort")))
      break;
    if ((rc = cuda_status(cub::DeviceSelect::Unique(tmp, b_uniq, k1, k0, dnum, nkeys, s), "cub unique")))
      break;
    note_launch(2);
    if ((rc = cuda_status(cudaMemcpyAsync(&P->nnz, dnum, 8, cudaMemcpyDeviceToHost, s), "nnz")))
      break;
    if ((rc = cuda_status(cudaStreamSynchronize(s), "csr sync"))) break;
    if ((rc = cuda_status(cudaMalloc(&P->col_idx, std::max<int64_t>(1, P->nnz) * sizeof(int32_t)),
                          "csr col_idx")))
      break;
    const int64_t work = std::max(P->nnz, ndofs + 1);
    const int64_t b2 = std::min<int64_t>((work + threads - 1) / threads, 148 * 32);
    csr_rows_kernel<<<(unsigned)b2, threads, 0, s>>>(k0, P->nnz, ndofs, P->row_ptr, P->col_idx);
    note_launch();
    rc = cuda_status(cudaGetLastError(), "csr_rows_kernel");
  } while (false);
  cleanup();
  if (rc == SFK_OK) rc = cuda_status(cudaStreamSynchronize(s), "csr sync");
  if (rc != SFK_OK) {
    cudaFree(P->row_ptr);
    cudaFree(P->col_idx);
    delete P;
    return rc;
  }
  *out = P;
  return SFK_OK;
}

int sfk_csr_entry_map(const sfk_csr* P, int64_t ncells, int ndofs_per_cell,
                      const int32_t* cell_dofs, int32_t* map, void* stream) {
  if (!P) return fail(SFK_EINVAL, "sfk_csr_entry_map: NULL pattern");
  if (ncells < 0 || ndofs_per_cell <= 0) return fail(SFK_EINVAL, "sfk_csr_entry_map: bad sizes");
  if (ncells == 0) return SFK_OK;
  if (!cell_dofs || !map) return fail(SFK_EINVAL, "sfk_csr_entry_map: NULL pointer argument");
  if (P->nnz >= INT32_MAX)
    return fail(SFK_EUNSUPPORTED, "sfk_csr_entry_map: nnz >= 2^31 does not fit int32 positions");
  const int64_t total = ncells * (int64_t)ndofs_per_cell * ndofs_per_cell;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 32);
  csr_map_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      ncells, ndofs_per_cell, cell_dofs, P->row_ptr, P->col_idx, map);
  note_launch();
  return cuda_status(cudaGetLastError(), "csr_map_kernel");
}

int sfk_csr_insert(int64_t ncells, int ndofs_per_cell, const double* cell_matrices,
                   const int32_t* cell_dofs, const int64_t* row_ptr, const int32_t* col_idx,
                   const int32_t* entry_map, double* values, void* stream) {
  if (ncells < 0 || ndofs_per_cell <= 0) return fail(SFK_EINVAL, "sfk_csr_insert: bad sizes");
  if (ncells == 0) return SFK_OK;
  if (!cell_matrices || !values || (!entry_map && (!cell_dofs || !row_ptr || !col_idx)))
    return fail(SFK_EINVAL, "sfk_csr_insert: NULL pointer argument");
  const int64_t total = ncells * (int64_t)ndofs_per_cell * ndofs_per_cell;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 32);
  csr_insert_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      ncells, ndofs_per_cell, cell_matrices, cell_dofs, row_ptr, col_idx, entry_map, values);
  note_launch();
  return cuda_status(cudaGetLastError(), "csr_insert_kernel");
}

int sfk_csr_info(const sfk_csr* P, int64_t* nrows, int64_t* nnz, int64_t** row_ptr,
                 int32_t** col_idx) {
  if (!P) return fail(SFK_EINVAL, "sfk_csr_info: NULL pattern");
  if (nrows) *nrows = P->nrows;
  if (nnz) *nnz = P->nnz;
  if (row_ptr) *row_ptr = P->row_ptr;
  if (col_idx) *col_idx = P->col_idx;
  return SFK_OK;
}

int sfk_csr_destroy(sfk_csr* P) {
  if (!P) return SFK_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(P->device);
  cudaFree(P->row_ptr);
  cudaFree(P->col_idx);
  cudaSetDevice(cur);
  delete P;
  return SFK_OK;
}

}  // extern "C"
