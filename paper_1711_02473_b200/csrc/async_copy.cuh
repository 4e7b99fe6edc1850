// cp.async (LDGSTS) helpers: global -> shared copies that complete
// asynchronously, so the next cell batch streams in while the current one
// computes.
#pragma once

#include <stdint.h>

namespace sfk {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K));
}

// Copy `n` doubles global -> shared (both arrays 8B aligned; 16B chunks when
// the source allows it).  Called by every thread of the CTA.
template <int THREADS>
__device__ __forceinline__ void async_copy(double* dst, const double* src, int n, int tid) {
  const bool al16 = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (al16) {
    const int n2 = n >> 1;
    for (int i = tid; i < n2; i += THREADS) cp_async16(dst + 2 * i, src + 2 * i);
    if ((n & 1) && tid == 0) cp_async8(dst + n - 1, src + n - 1);
  } else {
    for (int i = tid; i < n; i += THREADS) cp_async8(dst + i, src + i);
  }
}

}  // namespace sfk
