// Stand-ins for the sfk_api.cu helpers a probe library (tools/c3_sweep.py)
// needs: error text to stderr, no launch counter.
#include <cstdarg>
#include <cstdio>

#include "sfk_internal.cuh"

namespace sfk {

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfprintf(stderr, fmt, ap);
  va_end(ap);
  fputc('\n', stderr);
  return status;
}

int cuda_status(cudaError_t err, const char* what) {
  if (err == cudaSuccess) return 0;
  return fail(SFK_ECUDA, "%s: %s", what, cudaGetErrorString(err));
}

void note_launch(int64_t) {}

}  // namespace sfk
