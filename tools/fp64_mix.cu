// Do DMMA (FP64 tensor) and DFMA (FP64 pipe) overlap on B200?  Run each alone
// and both concurrently (warp-specialised and interleaved in one warp).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// mode 0: DFMA only, 1: DMMA only, 2: warp-specialised (even warps DFMA, odd DMMA),
// 3: interleaved in every warp
__global__ void mix(double* out, int itf, int itm, int mode) {
  const int w = threadIdx.x / 32;
  double f[8], c[4][2];
  for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) { c[i][0] = i; c[i][1] = threadIdx.x; }
  const double a = 1.0000001, b = 1e-7, x = 1.0 + threadIdx.x * 1e-9, y = 1.0;
  bool do_f = mode == 0 || mode == 3 || (mode == 2 && (w & 1) == 0);
  bool do_m = mode == 1 || mode == 3 || (mode == 2 && (w & 1) == 1);
  if (mode == 3) {
    for (int it = 0; it < itm; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(c[i][0], c[i][1], x, y);
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fma(f[i], a, b);
    }
  } else {
    if (do_f)
      for (int it = 0; it < itf; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fma(f[i], a, b);
    if (do_m)
      for (int it = 0; it < itm; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma(c[i][0], c[i][1], x, y);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += f[i];
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int tpb = 512, blocks = sms * 2;
  // per-warp work: DFMA: itf*8*32 FMA ; DMMA: itm*4*256 FMA
  const int itf = 40000, itm = 10000;   // 10.24M vs 10.24M FMA per warp
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 4; ++mode) {
      mix<<<blocks, tpb>>>(d, 100, 25, mode);
      cudaEventRecord(e0);
      mix<<<blocks, tpb>>>(d, itf, itm, mode);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warps = (double)blocks * tpb / 32;
      double fl_f = 2.0 * itf * 8 * 32, fl_m = 2.0 * itm * 4 * 256;
      double tot = 0;
      if (mode == 0) tot = warps * fl_f;
      if (mode == 1) tot = warps * fl_m;
      if (mode == 2) tot = warps / 2 * (fl_f + fl_m);
      if (mode == 3) tot = warps * (2.0 * itm * 4 * 8 * 32 + fl_m);
      printf("mode %d: %.3f ms  %.2f TFLOP/s total\n", mode, ms, tot / ms / 1e9);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
