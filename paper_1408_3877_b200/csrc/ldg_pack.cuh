// Packed FP32 block layout of the mixed-precision smoother (ldg_smooth.cu),
// shared with the block-Jacobi setup that writes P^-1 in it (ldg_apply.cu).
#pragma once

// -DLDG_UNR_P4=n: column groups of a packed block in flight per step at p = 4 (tuning builds)
#ifndef LDG_UNR_P4
#define LDG_UNR_P4 1
#endif

namespace ldgb {

// Packing of the stored N x N blocks into float4 quads.
//  flat (p <= 1): the block column-major, padded to a multiple of 4 values;
//    streamed fully unrolled.
//  chunked (p >= 2): each block on its own, columns grouped CC at a time
//    (CC*N a multiple of 4, N padded with zero columns to NCOL), QC quads per
//    group.  The stream is a rolled loop over column groups whose body has a
//    compile-time (row, column) map: a bounded number of loads in flight per
//    thread (a fully unrolled 57-quad block made ptxas hoist every load, 255
//    registers and spills) and only the group's CC vector values live.
template <int P>
struct SmCfg {
  static constexpr int N = (P + 1) * (P + 2) / 2;
  static constexpr int NN = N * N;
  static constexpr int NF = (N + 3) / 4 * 4;
  static constexpr bool kFlat = P <= 1;
  static constexpr int CC = (N % 2 == 0) ? 2 : 4;
  static constexpr int NCOL = (N + CC - 1) / CC * CC;
  static constexpr int QC = kFlat ? 1 : CC * N / 4;       // quads per column group
  static constexpr int NCH = NCOL / CC;                   // column groups per block
  static constexpr int QS = NCH * QC;                     // quads per block (chunked)
  static constexpr int QP = kFlat ? (NN + 3) / 4 : QS;    // quads of one packed block (E^m_kk or P^-1)
  static constexpr int Q = (3 * P + 2) / 2;               // edge rule of the matrix-free off-diagonal E
  static constexpr int EDGE = (12 * Q * N + Q + 3) / 4 * 4;  // FP32 edge tables (pe, pth, we), padded
  static constexpr int UNR = kFlat ? 1 : (P == 4 ? LDG_UNR_P4 : (16 / QC > 0 ? 16 / QC : 1));  // groups unrolled per step
};

// (quad, component) of value (i, j) of a packed block: flat = column-major
// j*N + i; chunked = group j / CC, position (j % CC)*N + i within the group
template <int P>
__host__ __device__ inline int sm_packed_slot(int i, int j) {
  using C = SmCfg<P>;
  if (C::kFlat) return j * C::N + i;
  return (j / C::CC) * C::QC * 4 + (j % C::CC) * C::N + i;
}

// float index of P^-1[i][j] of element k in the packed layout
template <int P>
__device__ __forceinline__ long sm_packed_p_index(int i, int j, long Kp, long k) {
  const int v = sm_packed_slot<P>(i, j);
  return (static_cast<long>(v >> 2) * Kp + k) * 4 + (v & 3);
}

}  // namespace ldgb
