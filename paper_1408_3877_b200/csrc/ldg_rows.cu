// Row-parallel variants of the operator kernels (the ones the solver runs).
//
// One CTA owns a tile of 32 consecutive elements; warp i of the CTA computes
// output row i of the N x N block rows of those 32 elements (lane = element).
// Compared with one thread per element this gives N times the threads, a
// dependency chain of a few load rounds per thread instead of ~N*8, and it
// keeps every access coalesced: for fixed (block, i, j) a warp reads 32
// consecutive elements of one plane, and the vector gathers of a tile are
// shared through L1 by its N warps.  Coarse multigrid levels (a few hundred
// elements) were pure latency with a thread per element (80-90 us per
// launch); this layout makes them a few microseconds.
//
// Reference tables are read through the read-only cache (all lanes of a warp
// read the same table entry: one broadcast transaction), stored transposed,
// T^t[j][i] at j*NP + i (ldg_tables.cpp).
#include <cmath>

#include "ldg_internal.hpp"
#include "ldg_offdiag.cuh"

namespace ldgb {

namespace {

constexpr int kTile = 32;

template <int P>
struct Cfg {
  static constexpr int N = (P + 1) * (P + 2) / 2;
  static constexpr int NP = (N % 2) ? N + 1 : N;
  static constexpr int Q = (3 * P + 2) / 2;  // edge rule of the off-diagonal E blocks
};

inline unsigned tiles_of(int K) { return static_cast<unsigned>((K + kTile - 1) / kTile); }

#define LDG_DISPATCH_P(p, CALL) \
  switch (p) {                  \
    case 0: { CALL(0); break; } \
    case 1: { CALL(1); break; } \
    case 2: { CALL(2); break; } \
    case 3: { CALL(3); break; } \
    default: { CALL(4); break; } \
  }

struct RowCtx {
  int k;      // element
  int i;      // output row
  bool live;  // k < K
};

__device__ __forceinline__ RowCtx row_ctx(int K) {
  RowCtx c;
  c.k = blockIdx.x * kTile + (threadIdx.x & (kTile - 1));
  c.i = threadIdx.x / kTile;
  c.live = c.k < K;
  return c;
}

// (T x[.][col])_i with T^t stored at tab (read-only path, broadcast)
template <int N, int NP>
__device__ __forceinline__ double row_dot(const double* __restrict__ tab, int i, const double* __restrict__ x,
                                          long Kp, int col) {
  double tv[N], xv[N];  // loads first, then the chain (see ldg_small.cu trow)
#pragma unroll
  for (int j = 0; j < N; ++j) {
    tv[j] = __ldg(tab + j * NP + i);
    xv[j] = x[j * Kp + col];
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) s = fma(tv[j], xv[j], s);
  return s;
}

// t^m_i = inv2a [sigma (mhat^-1 vz^m)_i + tau (mhat^-1 B^m x)_i]  (stage 1)
// with the mhat^-1-premultiplied tables: one pass, no cross-row exchange.
template <int P>
__global__ void __launch_bounds__(kTile * Cfg<P>::N) k_stage1_rows(DevMesh m, DevTables T,
                                                                   const double* __restrict__ vz, double sigma,
                                                                   const double* __restrict__ x, double tau,
                                                                   double* __restrict__ tout) {
  constexpr int N = Cfg<P>::N, NP = Cfg<P>::NP, NNP = N * NP;
  pdl_wait();
  pdl_trigger();
  const RowCtx c = row_ctx(m.K);
  if (!c.live) return;
  const int k = c.k, i = c.i;
  const long Kp = m.Kp;
  const double* g = m.geom;
  const double* tb = T.base;
  double u1 = 0.0, u2 = 0.0;
  if (x) {
    // diagonal block: -H^m_k + sum_n c^m_n s_diag_n, x_k shared by the 5 tables
    double dH1 = 0.0, dH2 = 0.0, dS0 = 0.0, dS1 = 0.0, dS2 = 0.0;
    const double* mH = tb + T.tmH;
    const double* mS = tb + T.tmSd;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const double xj = x[j * Kp + k];
      const int o = j * NP + i;
      dH1 = fma(__ldg(mH + o), xj, dH1);
      dH2 = fma(__ldg(mH + NNP + o), xj, dH2);
      dS0 = fma(__ldg(mS + o), xj, dS0);
      dS1 = fma(__ldg(mS + NNP + o), xj, dS1);
      dS2 = fma(__ldg(mS + 2 * NNP + o), xj, dS2);
    }
    const double b11 = g[kB11 * Kp + k], b12 = g[kB12 * Kp + k], b21 = g[kB21 * Kp + k], b22 = g[kB22 * Kp + k];
    u1 = -b22 * dH1 + b21 * dH2;
    u2 = b12 * dH1 - b11 * dH2;
    const double dS[3] = {dS0, dS1, dS2};
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      const int kind = m.kind[n * Kp + k];
      const double len = g[(kLen0 + n) * Kp + k];
      const double f = kind == kInterior ? 0.5 * len : (kind == kNeumann ? len : 0.0);
      u1 = fma(f * g[(kNux0 + n) * Kp + k], dS[n], u1);
      u2 = fma(f * g[(kNuy0 + n) * Kp + k], dS[n], u2);
      const int kp = m.nbr[n * Kp + k];
      if (kp >= 0) {  // off-diagonal: nu^m |E| / 2 s_off(n, n+) x_{k+}
        const double d = row_dot<N, NP>(tb + T.tmSo + (n * 3 + m.nbrn[n * Kp + k]) * NNP, i, x, Kp, kp);
        u1 = fma(0.5 * len * g[(kNux0 + n) * Kp + k], d, u1);
        u2 = fma(0.5 * len * g[(kNuy0 + n) * Kp + k], d, u2);
      }
    }
    u1 *= tau;
    u2 *= tau;
  }
  if (vz) {
    u1 = fma(sigma, row_dot<N, NP>(tb + T.tMinv, i, vz, Kp, k), u1);
    u2 = fma(sigma, row_dot<N, NP>(tb + T.tMinv, i, vz + N * Kp, Kp, k), u2);
  }
  const double inv2a = 1.0 / (2.0 * g[kArea * Kp + k]);
  tout[i * Kp + k] = inv2a * u1;
  tout[(N + i) * Kp + k] = inv2a * u2;
}

// y_i = alpha (M x_k)_i + beta ((S + S_D) x)_i - gamma sum_m sum_s (E^m[s] tz^m_col)_i + delta w_i
// (diagonal E blocks stored, off-diagonal ones matrix-free: ldg_offdiag.cuh)
template <int P, typename TE>
__global__ void __launch_bounds__(kTile * Cfg<P>::N) k_stage2_rows(DevMesh m, DevTables T, const TE* __restrict__ E,
                                                                   const double* __restrict__ D,
                                                                   const double* __restrict__ x, double alpha,
                                                                   double beta, const double* __restrict__ tz,
                                                                   double gamma, const double* __restrict__ w,
                                                                   double delta, double* __restrict__ y) {
  constexpr int N = Cfg<P>::N, NN = N * N, NP = Cfg<P>::NP, NNP = N * NP, Q = Cfg<P>::Q;
  pdl_wait();
  pdl_trigger();
  const RowCtx c = row_ctx(m.K);
  if (!c.live) return;
  const int k = c.k, i = c.i;
  const long Kp = m.Kp;
  const double* tb = T.base;
  const double* g = m.geom;
  int nbr[3];
#pragma unroll
  for (int n = 0; n < 3; ++n) nbr[n] = m.nbr[n * Kp + k];
  double acc = 0.0;
  if (tz) {
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const TE* blk = E + (static_cast<long>(cc) * NN + i * N) * Kp + k;
      const double* tc = tz + static_cast<long>(cc) * N * Kp + k;
      double part = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) part = fma(static_cast<double>(__ldcs(blk + j * Kp)), tc[j * Kp], part);
      acc += part;
    }
#pragma unroll 1
    for (int n = 0; n < 3; ++n) {
      const int kp = m.nbr[n * Kp + k];
      if (kp < 0) continue;
      const double hl = 0.5 * g[(kLen0 + n) * Kp + k];
      const double co1 = hl * g[(kNux0 + n) * Kp + k], co2 = hl * g[(kNuy0 + n) * Kp + k];
      double z[Q];
      offdiag_z<N, Q, double>(
          tb + T.pth + (n * 3 + m.nbrn[n * Kp + k]) * Q * N, tb + T.we, [&](int j) { return D[j * Kp + kp]; },
          [&](int j) { return fma(co1, tz[j * Kp + kp], co2 * tz[(N + j) * Kp + kp]); }, z);
      acc += offdiag_row<N, Q, double>(tb + T.pe + n * Q * N, z, i);
    }
    acc *= -gamma;
  }
  if (x) {
    if (alpha != 0.0) acc = fma(alpha * 2.0 * m.geom[kArea * Kp + k], row_dot<N, NP>(tb + T.tM, i, x, Kp, k), acc);
    if (beta != 0.0) {
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        const int kind = m.kind[n * Kp + k];
        if (kind == kInterior || kind == kDirichlet)
          acc = fma(beta, row_dot<N, NP>(tb + T.tSd + n * NNP, i, x, Kp, k), acc);
        if (nbr[n] >= 0)
          acc = fma(-beta, row_dot<N, NP>(tb + T.tSo + (n * 3 + m.nbrn[n * Kp + k]) * NNP, i, x, Kp, nbr[n]), acc);
      }
    }
  }
  if (w) acc = fma(delta, w[i * Kp + k], acc);
  y[i * Kp + k] = acc;
}

// y_i = beta y_i + omega (P_k^-1 x_k)_i
template <int P, typename TP>
__global__ void __launch_bounds__(kTile * Cfg<P>::N) k_bjac_rows(int K, long Kp, const TP* __restrict__ Pinv,
                                                                 const double* __restrict__ x, double omega,
                                                                 double beta, double* __restrict__ y) {
  constexpr int N = Cfg<P>::N;
  pdl_wait();
  pdl_trigger();
  const RowCtx c = row_ctx(K);
  if (!c.live) return;
  const int k = c.k, i = c.i;
  const TP* blk = Pinv + static_cast<long>(i) * N * Kp + k;
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) s = fma(static_cast<double>(__ldcs(blk + j * Kp)), x[j * Kp + k], s);
  y[i * Kp + k] = (beta == 0.0 ? 0.0 : beta * y[i * Kp + k]) + omega * s;
}

}  // namespace

void rows_stage1(Handle& h, const double* vz, double sigma, const double* x, double tau, double* tout) {
#define CALL(P)                                                                                         \
  launch_pdl(k_stage1_rows<P>, tiles_of(h.K), kTile * Cfg<P>::N, 0, h.stream, h.mesh(), h.dtab, vz, sigma, x, \
             tau, tout)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

template <typename TE>
void rows_stage2(Handle& h, const TE* E, const double* x, double alpha, double beta, const double* tz, double gamma,
                 const double* w, double delta, double* y) {
#define CALL(P)                                                                                           \
  launch_pdl(k_stage2_rows<P, TE>, tiles_of(h.K), kTile * Cfg<P>::N, 0, h.stream, h.mesh(), h.dtab, E, h.D.ptr, \
             x, alpha, beta, tz, gamma, w, delta, y)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}
template void rows_stage2<double>(Handle&, const double*, const double*, double, double, const double*, double,
                                  const double*, double, double*);
template void rows_stage2<float>(Handle&, const float*, const double*, double, double, const double*, double,
                                 const double*, double, double*);

template <typename TP>
void rows_bjac(Handle& h, const TP* Pinv, const double* x, double omega, double beta, double* y) {
#define CALL(P) \
  launch_pdl(k_bjac_rows<P, TP>, tiles_of(h.K), kTile * Cfg<P>::N, 0, h.stream, h.K, h.Kp, Pinv, x, omega, beta, y)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}
template void rows_bjac<double>(Handle&, const double*, const double*, double, double, double*);
template void rows_bjac<float>(Handle&, const float*, const double*, double, double, double*);

}  // namespace ldgb
