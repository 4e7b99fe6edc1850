// sfk_set_option / sfk_get_option and the per-device launch-shape cache.
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include <cuda_runtime.h>

#include "../../include/sfk.h"
#include "sfk_options.h"

namespace sfk {

int fail(int status, const char* fmt, ...);
int cuda_status(cudaError_t err, const char* what);

static const char* const kNames[OPT_COUNT] = {
    "c2_kernel",     "c2_g",        "v5_cpb6",   "c2_r",         "c2_roll",
    "c2g_small",     "c2g_kernel",  "cell_th",   "cell_minb",    "colloc_warps",
    "c3_tc",         "c5_p1",       "c5_p3",     "c5_p4",        "csr_dmma",
    "c5_p1_minb",    "neo_warps",   "host_chunk_mb", "lp_smem_kb", "lp_max_threads",
    "lp_warp",       "lp_minb",     "lp_fuse",   "v6_cfg",       "neo_cfg",
    "c3_cfg",        "c5_hi_cfg",   "p1_cfg",
};

static std::atomic<int64_t> g_opt[OPT_COUNT];

int64_t option(Option o) { return g_opt[o].load(std::memory_order_relaxed); }

const char* option_name(int o) { return (o >= 0 && o < OPT_COUNT) ? kNames[o] : nullptr; }

static int find(const char* name) {
  if (!name) return -1;
  for (int i = 0; i < OPT_COUNT; ++i)
    if (std::strcmp(name, kNames[i]) == 0) return i;
  return -1;
}

using ShapeKey = std::tuple<const void*, int, int, size_t>;

int kernel_shape(const void* func, int threads, size_t smem, const char* name,
                 LaunchShape* out, bool max_carveout) {
  static std::mutex mu;
  static std::map<ShapeKey, LaunchShape> cache;
  int dev = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc != SFK_OK) return rc;
  const ShapeKey key{func, dev, threads, smem};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return SFK_OK;
  }
  LaunchShape sh;
  rc = cuda_status(cudaDeviceGetAttribute(&sh.sms, cudaDevAttrMultiProcessorCount, dev),
                   "cudaDeviceGetAttribute(SM count)");
  if (rc != SFK_OK) return rc;
  if (smem > 48 * 1024) {
    rc = cuda_status(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem), name);
    if (rc != SFK_OK) return rc;
  }
  if (max_carveout) {
    cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaGetLastError();   // the carveout is a hint; never leave it as an error
  }
  rc = cuda_status(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sh.per_sm, func, threads, smem),
                   "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if (rc != SFK_OK) return rc;
  if (sh.per_sm < 1 || sh.sms < 1)
    return fail(SFK_ECUDA, "%s: kernel does not fit on an SM (threads %d, smem %zu)", name,
                threads, smem);
  cache.emplace(key, sh);
  *out = sh;
  return SFK_OK;
}

}  // namespace sfk

extern "C" {

int sfk_set_option(const char* name, int64_t value) {
  const int i = sfk::find(name);
  if (i < 0) return sfk::fail(SFK_EINVAL, "unknown option '%s'", name ? name : "(null)");
  sfk::g_opt[i].store(value, std::memory_order_relaxed);
  return SFK_OK;
}

int sfk_get_option(const char* name, int64_t* value) {
  const int i = sfk::find(name);
  if (i < 0) return sfk::fail(SFK_EINVAL, "unknown option '%s'", name ? name : "(null)");
  if (!value) return sfk::fail(SFK_EINVAL, "value is NULL");
  *value = sfk::g_opt[i].load(std::memory_order_relaxed);
  return SFK_OK;
}

}  // extern "C"
