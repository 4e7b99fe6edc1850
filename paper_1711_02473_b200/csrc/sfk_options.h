// Tuning options and per-device launch shapes (host side, shared by the CUDA
// translation units and the LoopProgram generator).
//
// Options replace the round-1 environment switches: the library reads no
// environment variables for dispatch.  Every option defaults to 0 = the
// built-in (measured-best) choice; callers doing A/B runs set one explicitly
// through sfk_set_option(name, value).  Values are process-wide atomics, so
// reading them from concurrent sfk_eval calls is race-free.
#pragma once

#include <stddef.h>
#include <stdint.h>

namespace sfk {

enum Option : int {
  OPT_C2_KERNEL,     // C2 generation: 1 v1, 2 v2, 3 v3, 4 tc, 5 cell(p1), 6 v4, 7 v5, 8 cellv, 10 v6, 11 tc8c
  OPT_C2_G,          // v5 output group size
  OPT_V5_CPB6,       // v5 cells per CTA at n = 6 (8 = the pair-free 288-thread variant)
  OPT_C2_R,          // v2 lines per thread
  OPT_C2_ROLL,       // v2 pointwise loop rolling
  OPT_C2G_SMALL,     // 3: global operator at p = 2, 3 through v3
  OPT_C2G_KERNEL,    // global operator: 0 v6 / tc8c, 1 round-1 selection, 2 / 3 forced v2 / v3
  OPT_CELL_TH,       // cellv threads per CTA
  OPT_CELL_MINB,     // cellv min CTAs per SM
  OPT_COLLOC_WARPS,  // C3 warp-synchronous variant: warps per CTA, -1 = off
  OPT_C3_TC,         // 1: C3 CTA-wide DMMA variants (n = 8, 12, 16), 2: n = 8 on the one-warp-per-cell DMMA kernel
  OPT_C5_P1,         // 1: C5 p = 1 through the CTA-phase kernel
  OPT_C5_P3,         // 1: C5 p = 3 through the FMA phase kernel
  OPT_C5_P4,         // 1: C5 p = 4 through the FMA phase kernel, 2: through tc5
  OPT_CSR_DMMA,      // 1: CSR epilogue on the DMMA matrix kernels
  OPT_C5_P1_MINB,    // 3: C5 p = 1 kernel with min 3 CTAs per SM
  OPT_NEO_WARPS,     // C4 warp-synchronous variant: warps per CTA, -1 = off
  OPT_HOST_CHUNK_MB, // sfk_eval_host staging chunk (MiB)
  OPT_LP_SMEM_KB,    // LoopProgram: shared-memory budget per CTA (KiB)
  OPT_LP_MAX_THREADS,
  OPT_LP_WARP,       // LoopProgram warp mode: -1 = off
  OPT_LP_MINB,
  OPT_LP_FUSE,       // LoopProgram loop fusion: -1 = off
  OPT_V6_CFG,        // v6 launch-shape / schedule alternatives per n (1..9: A/B history; 10, 11, 12: the persistent and earlier one-shot defaults)
  OPT_NEO_CFG,       // C4 variant: 1 two points per pointwise iteration at every p, 2 at none, 3 component-parallel kernel everywhere, 4 line kernel everywhere, 5 persistent warp-mode line kernel (p <= 3), 6 one-shot line kernel at p = 4..6
  OPT_C3_CFG,        // C3 variant: 1 per-element staging copies everywhere
  OPT_C5_HI_CFG,
  OPT_P1_CFG,        // C2 p = 1 kernel: (cells per CTA, min CTAs per SM) alternative 1..3     // C5 p = 5..8 DMMA kernel: (iy block, warps per row tile) alternative 1, 2
  OPT_COUNT
};

int64_t option(Option o);
const char* option_name(int o);

// Resident-grid shape of one kernel on the CURRENT device: the >48 KB
// dynamic shared-memory opt-in and carveout are applied for that device, and
// the occupancy result is cached per (kernel, device, threads, smem) under a
// mutex and only published after every setup step succeeded.
struct LaunchShape {
  int sms = 0;
  int per_sm = 0;
  long long resident() const { return (long long)sms * per_sm; }
};
// max_carveout: also prefer the largest shared-memory carveout (a hint).
int kernel_shape(const void* func, int threads, size_t smem, const char* name,
                 LaunchShape* out, bool max_carveout = false);

}  // namespace sfk
