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
// Even-odd form of a centro-(anti)symmetric N x N table (T[N-1-i][N-1-o] =
// s T[i][o]): with e_i = in_i + in_{N-1-i}, o_i = in_i - in_{N-1-i} (i < H)
// and m = in_H (odd N),
//   out[o] = E_o + O_o,  out[N-1-o] = s (E_o - O_o)     (o < H)
//   E_o = sum_i Pe[i][o] e_i + M[o] m,  O_o = sum_i Po[i][o] o_i,
// and out[H] = sum_i Pe[i][H] e_i + M[H] m (s = +1) or sum_i Po[i][H] o_i
// (s = -1): n = 5 / 6 take 21 / 30 FP64 ops per line instead of 25 / 36.
template <int N>
struct EOTab {
  static constexpr int H = N / 2, HO = (N + 1) / 2;
  double Pe[H * HO];   // [i][o]
  double Po[H * HO];
  double M[HO];
};

template <int N>
struct TabsV6 {
  static constexpr int LD = N == 8 ? 9 : (N + 1) & ~1;
  alignas(16) double B[N * LD];
  alignas(16) double BT[N * LD];
  alignas(16) double C[N * LD];
  alignas(16) double CT[N * LD];
  double W[N];
  double Bc[2 * N];
  EOTab<N> eB, eBT, eC, eCT;   // even-odd forms (filled by make_tabs_v6; used by EO kernels)
};

// Even-odd coefficients of table T (T[i*ld + o]) after symmetrisation with
// sign s.  Only used where the reference's tables are centro-symmetric to a
// few ulp (n <= 6: the symmetrised results stay within 4e-14 of the
// reference's emitted C).
template <int N>
inline void make_eo(const double* T, int ld, int s, EOTab<N>* e) {
  constexpr int H = EOTab<N>::H, HO = EOTab<N>::HO;
  double Ts[N][N];
  for (int i = 0; i < N; ++i)
    for (int o = 0; o < N; ++o) Ts[i][o] = 0.5 * (T[i * ld + o] + s * T[(N - 1 - i) * ld + (N - 1 - o)]);
  for (int i = 0; i < H; ++i)
    for (int o = 0; o < HO; ++o) {
      e->Pe[i * HO + o] = 0.5 * (Ts[i][o] + Ts[N - 1 - i][o]);
      e->Po[i * HO + o] = 0.5 * (Ts[i][o] - Ts[N - 1 - i][o]);
    }
  for (int o = 0; o < HO; ++o) e->M[o] = (N & 1) ? Ts[H][o] : 0.0;
}

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
  make_eo<N>(t.B, LD, 1, &t.eB);
  make_eo<N>(t.BT, LD, 1, &t.eBT);
  make_eo<N>(t.C, LD, -1, &t.eC);
  make_eo<N>(t.CT, LD, -1, &t.eCT);
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

// Two lines through the same table in one pass: every table entry (one LDCU
// per use on sm_100a, DFMA takes no constant-bank operand) feeds two DFMAs.
// Per output the operations and their order are those of v6_contract.
template <int NI, int NO, int LD>
__device__ __forceinline__ void v6_contract2(const double* T, const double* in1, const double* in2,
                                             double* out1, double* out2) {
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    out1[o] = T[o] * in1[0];
    out2[o] = T[o] * in2[0];
  }
#pragma unroll
  for (int i = 1; i < NI; ++i)
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      out1[o] = fma(T[i * LD + o], in1[i], out1[o]);
      out2[o] = fma(T[i * LD + o], in2[i], out2[o]);
    }
}

// out[o] = sum_i T[i][o] in[i] in even-odd form (EOTab), S = +1 / -1.
template <int N, int S>
__device__ __forceinline__ void v6_contract_eo(const EOTab<N>& E, const double* in, double* out) {
  constexpr int H = EOTab<N>::H, HO = EOTab<N>::HO;
  double e[H], o[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    e[i] = in[i] + in[N - 1 - i];
    o[i] = in[i] - in[N - 1 - i];
  }
#pragma unroll
  for (int q = 0; q < H; ++q) {
    double Ev = (N & 1) ? E.M[q] * in[H] : E.Pe[q] * e[0];
    double Ov = E.Po[q] * o[0];
#pragma unroll
    for (int i = (N & 1) ? 0 : 1; i < H; ++i) Ev = fma(E.Pe[i * HO + q], e[i], Ev);
#pragma unroll
    for (int i = 1; i < H; ++i) Ov = fma(E.Po[i * HO + q], o[i], Ov);
    out[q] = Ev + Ov;
    out[N - 1 - q] = S > 0 ? Ev - Ov : Ov - Ev;
  }
  if (N & 1) {
    double v = S > 0 ? E.M[H] * in[H] : E.Po[H] * o[0];
#pragma unroll
    for (int i = S > 0 ? 0 : 1; i < H; ++i)
      v = S > 0 ? fma(E.Pe[i * HO + H], e[i], v) : fma(E.Po[i * HO + H], o[i], v);
    out[H] = v;
  }
}

}  // namespace sfk
