// Shared pieces of the collocation-derivative C2 kernels (hex_action6.cu,
// hex_action7.cu): the table block passed by value and the register line
// contraction.
#pragma once

#include "sfk_internal.cuh"

namespace sfk {

// Tables of v6: row length LD (even, so aligned pairs of consecutive
// entries are one LDCU.128), except n = 8: with 128-bit pairs there the
// compiler hoisted the table set into uniform registers and spilled them
// (168 registers, or spills at the 128 cap); LD = 9 keeps 64-bit loads.
// B[i][q], BT[q][i], C[q'][q], CT[q][q'].
template <int N>
struct TabsV6 {
  static constexpr int LD = N == 8 ? 9 : (N + 1) & ~1;
  alignas(16) double B[N * LD];
  alignas(16) double BT[N * LD];
  alignas(16) double C[N * LD];
  alignas(16) double CT[N * LD];
  double W[N];
  double Bc[2 * N];
};

template <int N>
inline TabsV6<N> make_tabs_v6(const sfk_plan* p) {
  TabsV6<N> t{};
  constexpr int LD = TabsV6<N>::LD;
  for (int i = 0; i < N; ++i)
    for (int q = 0; q < N; ++q) {
      t.B[i * LD + q] = p->B[i * p->m + q];
      t.BT[q * LD + i] = p->B[i * p->m + q];
      t.C[i * LD + q] = p->Ct[i * p->m + q];   // C[q'=i][q]
      t.CT[q * LD + i] = p->Ct[i * p->m + q];
    }
  for (int q = 0; q < N; ++q) {
    t.W[q] = p->wq[q];
    t.Bc[q] = p->Bc[q];
    t.Bc[N + q] = p->Bc[p->m + q];
  }
  return t;
}

// out[o] = sum_i T[i*LD + o] in[i]: NO independent chains of depth NI.
template <int NI, int NO, int LD>
__device__ __forceinline__ void v6_contract(const double* T, const double* in, double* out) {
#pragma unroll
  for (int o = 0; o < NO; ++o) out[o] = T[o] * in[0];
#pragma unroll
  for (int i = 1; i < NI; ++i)
#pragma unroll
    for (int o = 0; o < NO; ++o) out[o] = fma(T[i * LD + o], in[i], out[o]);
}

}  // namespace sfk
