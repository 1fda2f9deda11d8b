// Off-diagonal blocks of E^m = -G^m + R^m + R_D^m, evaluated matrix-free.
//
// The block of E^m coupling element k to its neighbour kp across k's edge n
// (kp's edge np) is pure R^m (assembly.hpp:214-252, the kp-side half of the
// edge average).  With d_h sampled at the Qe Gauss points of an edge rule
// exact for degree 3p (the rank-Q form of k_assemble, ldg_assemble.cu):
//
//   E^m_{k,kp} = co_m  U_n diag(w_q d_kp(theta(x_q)))  V_{n,np}^T,
//   co_m = |E_n| nu^m_n / 2,   U_n[i][q] = phi_i(x_q),   V[j][q] = phi_j(theta(x_q)),
//
// so sum_m E^m_{k,kp} t^m_kp = U_n (wd (.) V^T (co_1 t^1 + co_2 t^2)_kp): 3 N Qe
// FMAs per edge from D_kp and t_kp, instead of streaming 2 N^2 stored values.
// Only the diagonal blocks E^m_kk are stored (ldg_device.cuh).
#pragma once

namespace ldgb {

// z[q] = w_q (d_kp . V[:, q]) (u . V[:, q]),  u = co_1 t^1_kp + co_2 t^2_kp;
// pth = V^t of the edge pair ([q][j]), we = rule weights; d(j), u(j) load the
// j-th value (column-outer order: 2 Q accumulators live, no N-vectors)
template <int N, int Q, typename S, typename FD, typename FU>
__device__ __forceinline__ void offdiag_z(const S* __restrict__ pth, const S* __restrict__ we, FD d, FU u, S* z) {
  S dv[Q], uv[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) dv[q] = uv[q] = S(0);
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const S dj = d(j), uj = u(j);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const S p = pth[q * N + j];
      dv[q] = fma(dj, p, dv[q]);
      uv[q] = fma(uj, p, uv[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) z[q] = we[q] * dv[q] * uv[q];
}

// acc[i] += scale * sum_q U[i][q] z[q]   (pe_n = U^t of edge n, [q][i])
template <int N, int Q, typename S>
__device__ __forceinline__ void offdiag_rows(const S* __restrict__ pe_n, const S* z, S scale, S* acc) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    S s = S(0);
#pragma unroll
    for (int q = 0; q < Q; ++q) s = fma(pe_n[q * N + i], z[q], s);
    acc[i] = fma(scale, s, acc[i]);
  }
}

// row i only
template <int N, int Q, typename S>
__device__ __forceinline__ S offdiag_row(const S* __restrict__ pe_n, const S* z, int i) {
  S s = S(0);
#pragma unroll
  for (int q = 0; q < Q; ++q) s = fma(pe_n[q * N + i], z[q], s);
  return s;
}

}  // namespace ldgb
