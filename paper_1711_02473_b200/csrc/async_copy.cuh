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
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K));
}

// Copy `n` doubles global -> shared (both arrays 8B aligned; 16B chunks when
// the source allows it).  Called by every thread of the CTA.  Callers that
// can choose the destination should use dst_shift() to give dst the same
// 16-byte phase as src, so the 16-byte path is always taken.
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

// 0 or 1: the shift (in doubles) that gives a shared buffer the 16-byte
// phase of the global source address.
__device__ __forceinline__ int dst_shift(const void* src) {
  return (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
}

template <int THREADS>
__device__ __forceinline__ void async_copy_phase(double* dst, const double* src, int n, int tid) {
  // dst and src share the 16-byte phase: one leading 8-byte copy if needed
  if (n <= 0) return;   // (n = 0 with lead = 1 would copy src[-1])
  const int lead = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
  if (lead && tid == 0 && n > 0) cp_async8(dst, src);
  const int m = n - lead;
  const int n2 = m >> 1;
  for (int i = tid; i < n2; i += THREADS) cp_async16(dst + lead + 2 * i, src + lead + 2 * i);
  if ((m & 1) && tid == 0) cp_async8(dst + n - 1, src + n - 1);
}

}  // namespace sfk
