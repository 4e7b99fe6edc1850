// Shared-memory layout of the v2 / v5 line kernels (hex_action2.cu,
// hex_action5.cu): per cell an X/R pair [2][M][PX] and a Y/S triple
// [3][M*M][LZ], one u buffer for the batch and double-buffered coords.
#pragma once

#include "sfk_internal.cuh"

namespace sfk {

// YPAD: extra doubles per cell after the Y/S triple (cell-stride tuning,
// tools/smem_pads_yt.py).
template <int N, int M, int CPB, int R, int YPAD = 0>
struct HexAction2Cfg {
  static constexpr int NN = N * N, MN = M * N, MM = M * M, N3 = N * N * N;
  static constexpr int LINES = (MM > NN ? MM : NN) * CPB;   // max lines of a stage
  static constexpr int THREADS = round_up((LINES + R - 1) / R, 32);
  static constexpr int PX = (N >= 4) ? NN + (((N - NN) % 16) + 16) % 16 : NN;
  static constexpr int LZ = (M > N ? M : N) | 1;   // z-line stride, >= m (in-place z)
  static constexpr int XA = M * PX;                // one X/R array per cell
  static constexpr int XSZ = 2 * XA;
  static constexpr int YA = MM * LZ;               // one Y/S array per cell
  static constexpr int YSZ = 3 * YA + YPAD;
  static constexpr int USZ = round_up(CPB * N3 + 1, 2); // u buffer (16B multiple)
  static constexpr int CSZ = CPB * 24;
  static constexpr size_t SMEM =
      (size_t)(round_up(CPB * XSZ + CPB * YSZ, 2) + USZ + 2 * CSZ) * sizeof(double);
};

}  // namespace sfk
