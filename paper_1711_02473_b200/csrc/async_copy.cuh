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

// ---------------------------------------------------------------------------
// Bulk (TMA-engine) copies global -> shared completing on an mbarrier
// (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP): one thread moves a
// whole contiguous block; consumers wait on the barrier's phase parity.

namespace sfk {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// order this thread's earlier generic-proxy shared accesses before the async
// proxy's writes of a following bulk copy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// bytes: multiple of 16; dst, src 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

// Stage n doubles starting at src into dst + phase(src) (element 0 at
// dst + ((src >> 3) & 1), as async_copy_phase): the 16-byte aligned body as
// ONE bulk copy on `bar`, the at most two odd end elements as 8-byte
// cp.async (committed: the consumer also waits cp.async groups).  Called by
// ONE thread.  Returns the bytes the barrier must expect.
__device__ __forceinline__ unsigned bulk_copy_phase(double* dst, const double* src, int n,
                                                    uint64_t* bar) {
  if (n <= 0) return 0;
  const int lead = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
  double* d0 = dst + lead;                       // element 0
  if (lead) cp_async8(d0, src);
  const int m = n - lead, body = m & ~1;
  if (m & 1) cp_async8(d0 + n - 1, src + n - 1);
  cp_async_commit();
  if (body > 0) bulk_g2s(d0 + lead, src + lead, (unsigned)body * 8u, bar);
  return (unsigned)body * 8u;
}

}  // namespace sfk
