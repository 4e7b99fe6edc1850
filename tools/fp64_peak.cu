// FP64 peak microbenchmarks for B200 (sm_100a): DFMA chains and DMMA (mma.sync m8n8k4 f64).
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
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
__global__ void dmma_kernel(double* out, int iters, double a0, double b0) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int rep = 0; rep < 3; ++rep) {
    for (int tpb : {256, 512}) {
      int blocks = sms * (2048 / tpb);
      dfma_kernel<8><<<blocks, tpb>>>(d, 100, 1.0000001, 1e-7);
      cudaEventRecord(e0);
      dfma_kernel<8><<<blocks, tpb>>>(d, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * (double)blocks * tpb;
      printf("DFMA tpb=%d blocks=%d: %.3f ms  %.2f TFLOP/s\n", tpb, blocks, ms, fl / ms / 1e9);
    }
    for (int tpb : {128, 256, 512}) {
      int blocks = sms * (1024 / tpb);
      dmma_kernel<4><<<blocks, tpb>>>(d, 100, 1.0, 1.0);
      cudaEventRecord(e0);
      dmma_kernel<4><<<blocks, tpb>>>(d, iters / 4, 1.0, 1.0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 256 * 4 * (iters / 4) * (double)blocks * (tpb / 32);
      printf("DMMA tpb=%d blocks=%d: %.3f ms  %.2f TFLOP/s\n", tpb, blocks, ms, fl / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s sms=%d clock=%d kHz\n", p.name, sms, p.clockRate);
  return 0;
}
