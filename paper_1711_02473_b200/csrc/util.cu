// Reductions for checksums/functionals and the FP64 peak micro-benchmark.
#include <chrono>

#include "sfk_internal.cuh"

namespace sfk {

constexpr int kSumBlocks = 508;   // (SFK_SUM_WORKSPACE - 2) / 2 partial pairs
constexpr int kSumThreads = 256;

// Fixed grid, fixed per-thread stride order, fixed tree => result depends on
// n only (bitwise reproducible run to run).
__global__ void __launch_bounds__(kSumThreads)
sum_partials_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  double s2 = 0.0, s1 = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kSumThreads;
  for (int64_t i = (int64_t)blockIdx.x * kSumThreads + threadIdx.x; i < n; i += stride) {
    const double v = __ldg(x + i);
    s2 = fma(v, v, s2);
    s1 += v;
  }
  __shared__ double r2[kSumThreads], r1[kSumThreads];
  r2[threadIdx.x] = s2;
  r1[threadIdx.x] = s1;
  __syncthreads();
  for (int w = kSumThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      r2[threadIdx.x] += r2[threadIdx.x + w];
      r1[threadIdx.x] += r1[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = r2[0];
    part[2 * blockIdx.x + 1] = r1[0];
  }
}

__global__ void sum_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double r2[512], r1[512];
  const int t = threadIdx.x;
  r2[t] = t < nb ? part[2 * t] : 0.0;
  r1[t] = t < nb ? part[2 * t + 1] : 0.0;
  __syncthreads();
  for (int w = 256; w > 0; w >>= 1) {
    if (t < w) {
      r2[t] += r2[t + w];
      r1[t] += r1[t + w];
    }
    __syncthreads();
  }
  if (t == 0) {
    out[0] = r2[0];
    out[1] = r1[0];
  }
}

int launch_sum_squares(const double* x, int64_t n, double* out, cudaStream_t s) {
  int64_t nb64 = (n + kSumThreads - 1) / kSumThreads;
  const int nb = nb64 < kSumBlocks ? (int)nb64 : kSumBlocks;
  sum_partials_kernel<<<nb, kSumThreads, 0, s>>>(x, n, out + 2);
  int rc = cuda_status(cudaGetLastError(), "sum_partials_kernel launch");
  if (rc != SFK_OK) return rc;
  sum_final_kernel<<<1, 512, 0, s>>>(out + 2, nb, out);
  note_launch(2);
  return cuda_status(cudaGetLastError(), "sum_final_kernel launch");
}

// ---------------------------------------------------------------------------
// FP64 peak: independent DFMA chains / DMMA m8n8k4 accumulators per thread.

template <int CH>
__global__ void peak_dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 123.456) out[0] = s;
}

template <int CH>
__global__ void peak_dmma_kernel(double* out, int iters, double a0, double b0) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    c[i][0] = threadIdx.x;
    c[i][1] = i;
  }
  const double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}

int run_fp64_peak(double seconds, double* dfma, double* dmma) {
  int dev = 0, sms = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  rc = cuda_status(cudaMalloc(&d, 8), "cudaMalloc");
  if (rc) return rc;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double budget = seconds > 0 ? seconds / 2 : 0.25;
  double best_f = 0, best_m = 0;
  int it_f = 2000, it_m = 500;
  for (int pass = 0; pass < 2; ++pass) {
    // pass 0 calibrates the iteration count, pass 1 runs for ~budget
    const int tpb = 512;
    const int bf = sms * 4, bm = sms * 2;
    float ms = 0;
    cudaEventRecord(e0);
    peak_dfma_kernel<8><<<bf, tpb>>>(d, it_f, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best_f = fmax(best_f, 2.0 * 8 * it_f * (double)bf * tpb / (ms * 1e-3) / 1e12);
    if (pass == 0 && ms > 0) it_f = (int)fmin(2e8, it_f * (budget * 1e3 / ms));
    cudaEventRecord(e0);
    peak_dmma_kernel<4><<<bm, tpb>>>(d, it_m, 1.0, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best_m = fmax(best_m, 2.0 * 256 * 4 * it_m * (double)bm * (tpb / 32) / (ms * 1e-3) / 1e12);
    if (pass == 0 && ms > 0) it_m = (int)fmin(2e8, it_m * (budget * 1e3 / ms));
  }
  note_launch(4);
  rc = cuda_status(cudaGetLastError(), "fp64 peak kernels");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (dfma) *dfma = best_f;
  if (dmma) *dmma = best_m;
  return rc;
}

}  // namespace sfk
