// C ABI for LoopProgram kernels (include/sfk.h, "LoopProgram path"):
// JSON -> generated CUDA (lp_codegen.cpp) -> NVRTC cubin for sm_100a ->
// module per device -> persistent batched launch.
//
// NVRTC is loaded with dlopen (libnvrtc.so.12; SFK_NVRTC overrides the
// path) and the driver entry points come from the static cudart
// (cudaGetDriverEntryPoint), so libsfk.so keeps no link-time dependency on
// either and still loads on a machine without a GPU (the CPU test tier
// exercises parse + generate + NVRTC compile there).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "lp_program.h"
#include "sfk_internal.cuh"

struct sfk_program {
  sfk::lp::Program prog;
  sfk::lp::Generated gen;
  std::vector<char> cubin;
  int flags = 0;
  std::mutex mu;
  struct PerDevice {
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
    int blocks = 0;  // persistent grid size
  };
  // fixed storage: pointers handed out by module_for stay valid while other
  // threads load the module on further devices
  static constexpr int kMaxDevices = 64;
  PerDevice dev[kMaxDevices];
};

namespace {

// ---- NVRTC (dlopen) -------------------------------------------------------
struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetErrorString) err = nullptr;
  std::string why;
  bool ok = false;
};

Nvrtc& nvrtc() {
  static Nvrtc N;
  static std::once_flag once;
  std::call_once(once, [] {
    std::vector<std::string> cands;
    if (const char* e = std::getenv("SFK_NVRTC")) cands.push_back(e);
    cands.push_back("libnvrtc.so.12");
    cands.push_back("/usr/local/cuda/lib64/libnvrtc.so.12");
    cands.push_back("libnvrtc.so");
    void* h = nullptr;
    for (const auto& c : cands)
      if ((h = dlopen(c.c_str(), RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) {
      N.why = std::string("cannot dlopen libnvrtc.so.12: ") + dlerror();
      return;
    }
#define SFK_SYM(field, name)                                      \
  N.field = reinterpret_cast<decltype(N.field)>(dlsym(h, name)); \
  if (!N.field) { N.why = "libnvrtc lacks " name; return; }
    SFK_SYM(create, "nvrtcCreateProgram")
    SFK_SYM(compile, "nvrtcCompileProgram")
    SFK_SYM(log_size, "nvrtcGetProgramLogSize")
    SFK_SYM(log, "nvrtcGetProgramLog")
    SFK_SYM(cubin_size, "nvrtcGetCUBINSize")
    SFK_SYM(cubin, "nvrtcGetCUBIN")
    SFK_SYM(destroy, "nvrtcDestroyProgram")
    SFK_SYM(err, "nvrtcGetErrorString")
#undef SFK_SYM
    N.ok = true;
  });
  return N;
}

// ---- driver entry points via cudart ---------------------------------------
struct Driver {
  decltype(&cuModuleLoadData) load = nullptr;
  decltype(&cuModuleGetFunction) get = nullptr;
  decltype(&cuModuleUnload) unload = nullptr;
  decltype(&cuFuncSetAttribute) set_attr = nullptr;
  decltype(&cuLaunchKernel) launch = nullptr;
  decltype(&cuOccupancyMaxActiveBlocksPerMultiprocessor) occ = nullptr;
  decltype(&cuGetErrorString) err = nullptr;
  bool ok = false;
  std::string why;
};

Driver& driver() {
  static Driver D;
  static std::once_flag once;
  std::call_once(once, [] {
    auto sym = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    bool ok = sym("cuModuleLoadData", (void**)&D.load) &&
              sym("cuModuleGetFunction", (void**)&D.get) &&
              sym("cuModuleUnload", (void**)&D.unload) &&
              sym("cuFuncSetAttribute", (void**)&D.set_attr) &&
              sym("cuLaunchKernel", (void**)&D.launch) &&
              sym("cuOccupancyMaxActiveBlocksPerMultiprocessor", (void**)&D.occ) &&
              sym("cuGetErrorString", (void**)&D.err);
    D.ok = ok;
    if (!ok) D.why = "CUDA driver entry points unavailable (no GPU driver?)";
  });
  return D;
}

int cu_status(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return SFK_OK;
  const char* s = "unknown";
  if (driver().err) driver().err(r, &s);
  return sfk::fail(SFK_ECUDA, "%s: %s", what, s);
}

const int64_t kSmemLimit = 227 * 1024;  // opt-in dynamic smem per CTA on sm_100

int compile(sfk_program* P) {
  Nvrtc& N = nvrtc();
  if (!N.ok) return sfk::fail(SFK_EUNSUPPORTED, "LoopProgram JIT: %s", N.why.c_str());
  nvrtcProgram prog;
  nvrtcResult r = N.create(&prog, P->gen.source.c_str(), "sfk_lp.cu", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return sfk::fail(SFK_ECUDA, "nvrtcCreateProgram: %s", N.err(r));
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device",
                                   "--extra-device-vectorization"};
  opts.push_back((P->flags & SFK_PROGRAM_FMA) ? "--fmad=true" : "--fmad=false");
  r = N.compile(prog, (int)opts.size(), opts.data());
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    N.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) N.log(prog, &log[0]);
    N.destroy(&prog);
    return sfk::fail(SFK_ECUDA, "NVRTC compile of LoopProgram '%s' failed: %.400s",
                     P->prog.name.c_str(), log.c_str());
  }
  size_t n = 0;
  N.cubin_size(prog, &n);
  P->cubin.resize(n);
  N.cubin(prog, P->cubin.data());
  N.destroy(&prog);
  return SFK_OK;
}

int module_for(sfk_program* P, int dev, sfk_program::PerDevice** out) {
  if (dev < 0 || dev >= sfk_program::kMaxDevices)
    return sfk::fail(SFK_EINVAL, "device %d out of range", dev);
  std::lock_guard<std::mutex> lk(P->mu);
  sfk_program::PerDevice& d = P->dev[dev];
  if (!d.fn) {
    if (P->cubin.empty()) return sfk::fail(SFK_EUNSUPPORTED, "program was created without JIT");
    Driver& D = driver();
    if (!D.ok) return sfk::fail(SFK_ECUDA, "%s", D.why.c_str());
    int rc = sfk::cuda_status(cudaSetDevice(dev), "cudaSetDevice");
    if (rc) return rc;
    rc = sfk::cuda_status(cudaFree(nullptr), "context init");
    if (rc) return rc;
    if ((rc = cu_status(D.load(&d.mod, P->cubin.data()), "cuModuleLoadData"))) return rc;
    if ((rc = cu_status(D.get(&d.fn, d.mod, P->gen.entry.c_str()), "cuModuleGetFunction"))) return rc;
    const auto& C = P->gen.cfg;
    if ((rc = cu_status(D.set_attr(d.fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                   (int)C.smem_bytes),
                        "cuFuncSetAttribute")))
      return rc;
    int per_sm = 0;
    if ((rc = cu_status(D.occ(&per_sm, d.fn, C.threads, (size_t)C.smem_bytes), "occupancy"))) return rc;
    if (per_sm < 1) return sfk::fail(SFK_EUNSUPPORTED, "LoopProgram kernel does not fit an SM");
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (C.global_scratch) per_sm = std::min(per_sm, 2);
    d.blocks = sms * per_sm;
  }
  *out = &d;
  return SFK_OK;
}

}  // namespace

extern "C" {

int sfk_program_create(const char* json_text, int64_t len, int flags, sfk_program** out) {
  if (!json_text || !out) return sfk::fail(SFK_EINVAL, "sfk_program_create: null argument");
  *out = nullptr;
  auto* P = new (std::nothrow) sfk_program;
  if (!P) return sfk::fail(SFK_ENOMEM, "sfk_program_create: out of memory");
  P->flags = flags;
  try {
    const size_t n = len >= 0 ? (size_t)len : std::strlen(json_text);
    P->prog = sfk::lp::parse_program(json_text, n);
    if (P->prog.args.size() > 8) throw std::runtime_error("more than 8 arguments");
    P->gen = sfk::lp::generate(P->prog, kSmemLimit, (flags & SFK_PROGRAM_FMA) != 0);
  } catch (const std::exception& e) {
    delete P;
    return sfk::fail(SFK_EINVAL, "LoopProgram: %s", e.what());
  }
  if (!(flags & SFK_PROGRAM_NO_JIT)) {
    const int rc = compile(P);
    if (rc) {
      delete P;
      return rc;
    }
  }
  *out = P;
  return SFK_OK;
}

int sfk_program_destroy(sfk_program* P) {
  if (!P) return SFK_OK;
  if (driver().ok)
    for (auto& d : P->dev)
      if (d.mod) driver().unload(d.mod);
  delete P;
  return SFK_OK;
}

int sfk_program_sizes(const sfk_program* P, int64_t* return_size, int* nargs, int64_t* arg_sizes,
                      int max_args) {
  if (!P) return sfk::fail(SFK_EINVAL, "sfk_program_sizes: null program");
  if (return_size) *return_size = P->prog.ret_size;
  if (nargs) *nargs = (int)P->prog.args.size();
  if (arg_sizes)
    for (int k = 0; k < (int)P->prog.args.size() && k < max_args; ++k)
      arg_sizes[k] = P->prog.args[k].second;
  return SFK_OK;
}

int sfk_program_config(const sfk_program* P, int64_t* out, int n) {
  if (!P || !out) return sfk::fail(SFK_EINVAL, "sfk_program_config: null argument");
  const auto& C = P->gen.cfg;
  const int64_t v[] = {C.cells_per_block, C.threads, C.slots, C.smem_bytes, C.global_scratch,
                       C.phases, C.serial_phases, C.barriers, (int64_t)P->cubin.size(),
                       C.warp_mode, C.fused_phases};
  for (int k = 0; k < n && k < (int)(sizeof v / sizeof v[0]); ++k) out[k] = v[k];
  return SFK_OK;
}

int sfk_program_text(const sfk_program* P, int what, char* buf, int64_t size, int64_t* length) {
  if (!P) return sfk::fail(SFK_EINVAL, "sfk_program_text: null program");
  const std::string& s = what == 0 ? P->gen.source : what == 1 ? P->gen.entry : P->prog.name;
  if (length) *length = (int64_t)s.size();
  if (buf && size > 0) {
    const size_t n = std::min<size_t>(s.size(), (size_t)size - 1);
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return SFK_OK;
}

int sfk_program_eval(const sfk_program* Pc, int64_t ncells, double* A, const double* const* args,
                     int nargs, void* stream) {
  auto* P = const_cast<sfk_program*>(Pc);
  if (!P) return sfk::fail(SFK_EINVAL, "sfk_program_eval: null program");
  if (ncells < 0) return sfk::fail(SFK_EINVAL, "sfk_program_eval: negative ncells");
  if (nargs != (int)P->prog.args.size())
    return sfk::fail(SFK_EINVAL, "sfk_program_eval: program takes %d arguments, got %d",
                     (int)P->prog.args.size(), nargs);
  if (ncells == 0) return SFK_OK;
  if (!A) return sfk::fail(SFK_EINVAL, "sfk_program_eval: null A");
  for (int k = 0; k < nargs; ++k)
    if (!args || !args[k])
      return sfk::fail(SFK_EINVAL, "sfk_program_eval: null argument '%s'",
                       P->prog.args[k].first.c_str());
  int dev = 0;
  int rc = sfk::cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  sfk_program::PerDevice* d = nullptr;
  if ((rc = module_for(P, dev, &d))) return rc;
  const auto& C = P->gen.cfg;
  const int64_t nchunks = (ncells + C.cells_per_block - 1) / C.cells_per_block;
  const int blocks = (int)std::min<int64_t>(nchunks, d->blocks);
  cudaStream_t s = (cudaStream_t)stream;
  double* arena = nullptr;
  if (C.global_scratch) {
    rc = sfk::cuda_status(
        cudaMallocAsync((void**)&arena, (size_t)blocks * C.arena_doubles_per_block * 8, s),
        "cudaMallocAsync(arena)");
    if (rc) return rc;
  }
  void* params[12];
  int np = 0;
  params[np++] = &A;
  const double* a[8];
  for (int k = 0; k < nargs; ++k) {
    a[k] = args[k];
    params[np++] = &a[k];
  }
  long long nc = ncells;
  params[np++] = &nc;
  params[np++] = &arena;
  rc = cu_status(driver().launch(d->fn, blocks, 1, 1, C.threads, 1, 1, (unsigned)C.smem_bytes,
                                 (CUstream)s, params, nullptr),
                 "cuLaunchKernel(LoopProgram)");
  sfk::note_launch();
  if (arena) cudaFreeAsync(arena, s);
  return rc;
}

}  // extern "C"
