// DFMA dependent-chain latency and per-warp ILP needed to saturate the FP64
// pipe: one CTA of W warps on one SM, each warp running K independent chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double* out, long long* cyc, int iters, double a, double b) {
  double x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = threadIdx.x * 1e-3 + k;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < K; ++k) x[k] = fma(x[k], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
void run(int warps, double* out, long long* cyc) {
  const int iters = 2000;
  chains<K><<<1, warps * 32>>>(out, cyc, iters, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  chains<K><<<1, warps * 32>>>(out, cyc, iters, 0.999999, 1e-7);
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double n_inst = (double)iters * 16 * K * warps;   // warp-level DFMA
  printf("K=%d warps=%2d  cycles/DFMA-per-warp-chain=%.2f  warp-DFMA per SM-cycle=%.3f\n", K, warps,
         (double)c / (iters * 16), n_inst / c);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1024);
  for (int w : {1, 4, 8, 16, 32}) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<4>(w, out, cyc);
    run<8>(w, out, cyc);
  }
  return 0;
}
