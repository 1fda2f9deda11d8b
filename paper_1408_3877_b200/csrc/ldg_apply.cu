// K6 — block-SpMV of the LDG operator, with the static blocks applied
// matrix-free.
//
// Of the blocks of W + dt A (system.hpp:120-135, 162-167) only E^m =
// -G^m + R^m + R_D^m (the C rows' Z columns) depend on d(t); they are
// assembled every step (ldg_assemble.cu) and streamed from HBM here.  The
// static ones — M = 2|T| mhat, B^m = -H^m + Q^m + Q_N^m (Z rows' C column) and
// eta (S + S_D) (C row's C column) — are linear combinations of at most 14
// reference matrices (hhat, s_diag, s_offdiag, mhat; assembly.hpp:76-208)
// with per-element scalars (B_k, |T_k|, nu_kn, |E_kn|, edge kinds), so they
// are rebuilt on the fly from shared memory instead of being read: 8 of the
// 20 N x N blocks per element remain in HBM traffic.
// The reference tables are stored transposed and padded (row j of T^t is 16
// bytes aligned), so one 128-bit shared load feeds two FP64 FMAs and every
// lane of a warp reads the same address (broadcast).
#include <cmath>
#include <cstdlib>

#include "ldg_internal.hpp"
#include "ldg_offdiag.cuh"

// min resident CTAs per SM of the thread-per-element kernels: at p = 4 the
// register-heavy kernels are latency-bound at 1 CTA; 4 CTAs (<= 128 registers)
// measured 7-15% faster there (2, 6, 7 CTAs: +24 / +48 / +38 % Schur apply).
// At p = 3, 7 CTAs (one wave of the 256^2 level): Schur apply 145 -> 110 us,
// full apply 153 -> 115 us.  With the rank-form kernels p = 1, 2 want one wave
// too (7 CTAs: 150 / 91 registers otherwise, 2.3 / 1.4 waves; Schur apply
// 55.4 -> 51.1 us and full apply 62 -> 52 us at p = 2).  (-DLDG_MINB_STAGE=n
// overrides all, -DLDG_MINB_STAGE_P<p>=n one degree.)
#ifdef LDG_MINB_STAGE
#define LDG_MINB_STAGE_P(P) LDG_MINB_STAGE
#else
#ifndef LDG_MINB_STAGE_P3
#define LDG_MINB_STAGE_P3 7
#endif
#ifndef LDG_MINB_STAGE_P4
#define LDG_MINB_STAGE_P4 4
#endif
#ifndef LDG_MINB_STAGE_P2
#define LDG_MINB_STAGE_P2 7
#endif
#ifndef LDG_MINB_STAGE_P1
#define LDG_MINB_STAGE_P1 7
#endif
#define LDG_MINB_STAGE_P(P) \
  ((P) == 4 ? LDG_MINB_STAGE_P4 : ((P) == 3 ? LDG_MINB_STAGE_P3 : ((P) == 2 ? LDG_MINB_STAGE_P2 : ((P) == 1 ? LDG_MINB_STAGE_P1 : 1))))
#endif
// stage 2 alone at p = 4 (tuning builds): 5 / 6 / 7 CTAs measured Schur apply
// 274 / 298 / 308 us against 238 us at 4
#ifdef LDG_MINB_STAGE2_P4
#define LDG_MINB_S2STAGE_P(P) ((P) == 4 ? LDG_MINB_STAGE2_P4 : LDG_MINB_STAGE_P(P))
#else
#define LDG_MINB_S2STAGE_P(P) LDG_MINB_STAGE_P(P)
#endif

namespace ldgb {

namespace {

template <int P>
struct Cfg {
  static constexpr int N = (P + 1) * (P + 2) / 2;
  static constexpr int NP = (N % 2) ? N + 1 : N;
  static constexpr int TAB = 16 * N * NP;  // tH(2) + tSd(3) + tSo(9) + tM + tMinv
  static constexpr int Q = (3 * P + 2) / 2;  // edge rule of the off-diagonal E blocks
  static constexpr int EDGE = (12 * Q * N + Q + 1) / 2 * 2;  // pe(3) + pth(9) + we, padded to even
};

inline unsigned grid_of(long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

#define LDG_DISPATCH_P(p, CALL) \
  switch (p) {                  \
    case 0: { CALL(0); break; } \
    case 1: { CALL(1); break; } \
    case 2: { CALL(2); break; } \
    case 3: { CALL(3); break; } \
    default: { CALL(4); break; } \
  }

// shared-memory image of the static tables: [tH 2 | tSd 3 | tSo 9 | tM | tMinv]
template <int P>
struct STab {
  static constexpr int N = Cfg<P>::N, NP = Cfg<P>::NP, NNP = N * NP;
  const double* s;
  __device__ const double* H(int m) const { return s + m * NNP; }
  __device__ const double* Sd(int n) const { return s + (2 + n) * NNP; }
  __device__ const double* So(int nm, int np) const { return s + (5 + nm * 3 + np) * NNP; }
  __device__ const double* M() const { return s + 14 * NNP; }
  __device__ const double* Minv() const { return s + 15 * NNP; }
};

// The five table blocks are contiguous in the device table buffer in this
// order (ldg_tables.cpp), so staging is one vectorised copy.  With EDGE the
// edge tables of the matrix-free off-diagonal E blocks follow them
// (pe [3][Q][N] | pth [9][Q][N] | we [Q]).
template <int P, bool EDGE = false>
__device__ __forceinline__ STab<P> stage_tables(double* sm, const DevTables& T) {
  constexpr int n = Cfg<P>::TAB, N = Cfg<P>::N, Q = Cfg<P>::Q;
  const double2* src = reinterpret_cast<const double2*>(T.base + T.tH);
  double2* dst = reinterpret_cast<double2*>(sm);
  for (int i = threadIdx.x; i < n / 2; i += blockDim.x) dst[i] = src[i];
  if constexpr (EDGE) {
    double* e = sm + n;
    for (int i = threadIdx.x; i < 3 * Q * N; i += blockDim.x) e[i] = T.base[T.pe + i];
    for (int i = threadIdx.x; i < 9 * Q * N; i += blockDim.x) e[3 * Q * N + i] = T.base[T.pth + i];
    for (int i = threadIdx.x; i < Q; i += blockDim.x) e[12 * Q * N + i] = T.base[T.we + i];
  }
  __syncthreads();
  return STab<P>{sm};
}


// w = T x with x in registers (T^t in shared memory, rows of NP doubles)
template <int N, int NP>
__device__ __forceinline__ void tab_mv(const double* sT, const double* x, double* w) {
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const double xj = x[j];
    const double2* row = reinterpret_cast<const double2*>(sT + j * NP);
#pragma unroll
    for (int q = 0; q < N / 2; ++q) {
      const double2 t = row[q];
      w[2 * q] = fma(t.x, xj, w[2 * q]);
      w[2 * q + 1] = fma(t.y, xj, w[2 * q + 1]);
    }
    if (N & 1) w[N - 1] = fma(sT[j * NP + N - 1], xj, w[N - 1]);
  }
}

// w = T x[.][col] with x streamed from memory (L1-resident after first use):
// for N > 6 the column loop stays rolled so at most N accumulators and one
// table row are live (p = 3, 4 would spill with x and T fully unrolled).
template <int N, int NP>
__device__ __forceinline__ void tab_mv_g(const double* sT, const double* __restrict__ x, long Kp, int col,
                                         double* w) {
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] = 0.0;
#pragma unroll(N <= 6 ? N : 1)
  for (int j = 0; j < N; ++j) {
    const double xj = x[j * Kp + col];
    const double2* row = reinterpret_cast<const double2*>(sT + j * NP);
#pragma unroll
    for (int q = 0; q < N / 2; ++q) {
      const double2 t = row[q];
      w[2 * q] = fma(t.x, xj, w[2 * q]);
      w[2 * q + 1] = fma(t.y, xj, w[2 * q + 1]);
    }
    if (N & 1) w[N - 1] = fma(sT[j * NP + N - 1], xj, w[N - 1]);
  }
}

// out[i][k] = scale * (T u)_i for u in registers: rows of T (columns of the
// stored transpose) one at a time, results stored directly.
template <int N, int NP>
__device__ __forceinline__ void tab_mv_store(const double* sT, const double* u, double scale,
                                             double* __restrict__ out, long Kp, int k) {
#pragma unroll(N <= 6 ? N : 1)
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(sT[j * NP + i], u[j], s);
    out[i * Kp + k] = scale * s;
  }
}

template <int N>
__device__ __forceinline__ void load_vec(const double* __restrict__ x, long Kp, int col, double* xv) {
#pragma unroll
  for (int j = 0; j < N; ++j) xv[j] = x[j * Kp + col];
}

// acc[i] += sum_j blk[(i*N+j)][k] * x[j][col]: a stored block streamed one
// column at a time (N coalesced loads in flight, N live accumulators)
template <int N, typename TB>
__device__ __forceinline__ void block_mv_gather(const TB* __restrict__ blk, long Kp, int k,
                                                const double* __restrict__ x, int col, double* acc) {
  const long NKp = static_cast<long>(N) * Kp;
  if constexpr (N <= 6) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const double xj = x[j * Kp + col];
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = fma(static_cast<double>(blk[i * NKp + j * Kp + k]), xj, acc[i]);
    }
  } else {
    // U block columns per round: U*N streaming loads in flight per thread
    // (one round per column left the warps latency-bound at ~60% of HBM;
    // U = 5 for FP32 blocks measured slower: 126 registers, lower occupancy)
    constexpr int U = (N % 3 == 0) ? 3 : 2;
    const TB* bj = blk + k;
#pragma unroll 1
    for (int j = 0; j < N; j += U, bj += U * Kp) {
      double xj[U];
      TB v[U][N];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        xj[u] = x[(j + u) * Kp + col];
#pragma unroll
        for (int i = 0; i < N; ++i) v[u][i] = __ldcs(bj + u * Kp + i * NKp);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = fma(static_cast<double>(v[u][i]), xj[u], acc[i]);
    }
  }
}

struct EdgeData {
  int kind[3], nbr[3], nbrn[3];
  double len[3], nux[3], nuy[3];
};

__device__ __forceinline__ EdgeData load_edges(const DevMesh& m, int k) {
  EdgeData e;
  const long Kp = m.Kp;
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    e.kind[n] = m.kind[n * Kp + k];
    e.nbr[n] = m.nbr[n * Kp + k];
    e.nbrn[n] = m.nbrn[n * Kp + k];
    e.len[n] = m.geom[(kLen0 + n) * Kp + k];
    e.nux[n] = m.geom[(kNux0 + n) * Kp + k];
    e.nuy[n] = m.geom[(kNuy0 + n) * Kp + k];
  }
  return e;
}

// sum_m E^m_{k,kp} t^m_kp over the interior edges of k, added to acc
// (ldg_offdiag.cuh); edge tables staged after the STab block
template <int P>
__device__ __forceinline__ void offdiag_all(const double* sm_edge, const double* __restrict__ D,
                                            const double* __restrict__ t, long Kp, const EdgeData& e,
                                            double* acc) {
  constexpr int N = Cfg<P>::N, Q = Cfg<P>::Q;
  const double* pe = sm_edge;
  const double* pth = sm_edge + 3 * Q * N;
  const double* we = sm_edge + 12 * Q * N;
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kp = e.nbr[n];
    if (kp < 0) continue;
    const double co1 = 0.5 * e.len[n] * e.nux[n], co2 = 0.5 * e.len[n] * e.nuy[n];
    double z[Q];
    offdiag_z<N, Q, double>(
        pth + (n * 3 + e.nbrn[n]) * Q * N, we, [&](int j) { return D[j * Kp + kp]; },
        [&](int j) { return fma(co1, t[j * Kp + kp], co2 * t[(N + j) * Kp + kp]); }, z);
    offdiag_rows<N, Q, double>(pe + n * Q * N, z, 1.0, acc);
  }
}

// u^m += sum_s B^m[s] x_col(s), B^m = -H^m + Q^m + Q_N^m rebuilt from tables
// (assembly.hpp:92-109, 174-208): diagonal -H^m_k + sum_n c^m_n s_diag_n with
// c = nu^m |E|/2 (interior), nu^m |E| (Neumann); off-diagonal nu^m|E|/2 s_off.
template <int P>
__device__ __forceinline__ void apply_B(const STab<P>& tb, const DevMesh& m, const EdgeData& e, int k, double b11,
                                        double b12, double b21, double b22, const double* __restrict__ x,
                                        double* u1, double* u2) {
  constexpr int N = Cfg<P>::N, NP = Cfg<P>::NP;
  const long Kp = m.Kp;
  double w[N];
  tab_mv_g<N, NP>(tb.H(0), x, Kp, k, w);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    u1[i] = fma(-b22, w[i], u1[i]);
    u2[i] = fma(b12, w[i], u2[i]);
  }
  tab_mv_g<N, NP>(tb.H(1), x, Kp, k, w);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    u1[i] = fma(b21, w[i], u1[i]);
    u2[i] = fma(-b11, w[i], u2[i]);
  }
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const double c = e.kind[n] == kInterior ? 0.5 * e.len[n] : (e.kind[n] == kNeumann ? e.len[n] : 0.0);
    if (c == 0.0) continue;
    tab_mv_g<N, NP>(tb.Sd(n), x, Kp, k, w);
    const double c1 = c * e.nux[n], c2 = c * e.nuy[n];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      u1[i] = fma(c1, w[i], u1[i]);
      u2[i] = fma(c2, w[i], u2[i]);
    }
  }
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    if (e.nbr[n] < 0) continue;
    tab_mv_g<N, NP>(tb.So(n, e.nbrn[n]), x, Kp, e.nbr[n], w);
    const double c1 = 0.5 * e.len[n] * e.nux[n], c2 = 0.5 * e.len[n] * e.nuy[n];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      u1[i] = fma(c1, w[i], u1[i]);
      u2[i] = fma(c2, w[i], u2[i]);
    }
  }
}

// acc += beta (S + S_D) x  (assembly.hpp:142-168: + s_diag on interior and
// Dirichlet edges, - s_offdiag to the neighbour; the edge length cancels)
template <int P>
__device__ __forceinline__ void apply_S(const STab<P>& tb, const DevMesh& m, const EdgeData& e, int k,
                                        const double* __restrict__ x, double beta, double* acc) {
  constexpr int N = Cfg<P>::N, NP = Cfg<P>::NP;
  const long Kp = m.Kp;
  double w[N];
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    if (e.kind[n] != kInterior && e.kind[n] != kDirichlet) continue;
    tab_mv_g<N, NP>(tb.Sd(n), x, Kp, k, w);
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = fma(beta, w[i], acc[i]);
  }
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    if (e.nbr[n] < 0) continue;
    tab_mv_g<N, NP>(tb.So(n, e.nbrn[n]), x, Kp, e.nbr[n], w);
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = fma(-beta, w[i], acc[i]);
  }
}

// stage 1: tout^m = M_k^-1 (sigma vz^m + tau sum_s B^m[s] x_col(s))
template <int P>
__global__ void __launch_bounds__(128, LDG_MINB_STAGE_P(P)) k_stage1(DevMesh m, DevTables T, const double* __restrict__ vz, double sigma,
                                                const double* __restrict__ x, double tau, double* __restrict__ tout,
                                                int k0, int k1) {
  constexpr int N = Cfg<P>::N, NP = Cfg<P>::NP;
  extern __shared__ __align__(16) double sm[];
  const STab<P> tb = stage_tables<P>(sm, T);
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  const long Kp = m.Kp;
  const double* g = m.geom;
  double u1[N], u2[N];
#pragma unroll
  for (int i = 0; i < N; ++i) u1[i] = u2[i] = 0.0;
  if (x) {
    const EdgeData e = load_edges(m, k);
    apply_B<P>(tb, m, e, k, g[kB11 * Kp + k], g[kB12 * Kp + k], g[kB21 * Kp + k], g[kB22 * Kp + k], x, u1, u2);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      u1[i] *= tau;
      u2[i] *= tau;
    }
  }
  if (vz) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      u1[i] = fma(sigma, vz[i * Kp + k], u1[i]);
      u2[i] = fma(sigma, vz[(N + i) * Kp + k], u2[i]);
    }
  }
  const double inv2a = 1.0 / (2.0 * g[kArea * Kp + k]);
  tab_mv_store<N, NP>(tb.Minv(), u1, inv2a, tout, Kp, k);
  tab_mv_store<N, NP>(tb.Minv(), u2, inv2a, tout + N * Kp, Kp, k);
}

// stage 1 of the Krylov operator, tout^m = tau M_k^-1 B^m x (no vz term):
// the same products against the m_hat^-1-premultiplied tables (tmH | tmSd |
// tmSo, the STab offsets of tH | tSd | tSo), so the result is a scale by
// 1/(2|T_k|) instead of a trailing M^-1 product (225 scalar table loads and
// FMAs per component at p = 4)
template <int P>
__global__ void __launch_bounds__(128, LDG_MINB_STAGE_P(P)) k_stage1m(DevMesh m, DevTables T,
                                                                      const double* __restrict__ x, double tau,
                                                                      double* __restrict__ tout, int k0, int k1) {
  constexpr int N = Cfg<P>::N, NNP = N * Cfg<P>::NP;
  extern __shared__ __align__(16) double sm[];
  {
    const double2* src = reinterpret_cast<const double2*>(T.base + T.tmH);
    double2* dst = reinterpret_cast<double2*>(sm);
    for (int i = threadIdx.x; i < 14 * NNP / 2; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
  }
  const STab<P> tb{sm};
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  const long Kp = m.Kp;
  const double* g = m.geom;
  double u1[N], u2[N];
#pragma unroll
  for (int i = 0; i < N; ++i) u1[i] = u2[i] = 0.0;
  const EdgeData e = load_edges(m, k);
  apply_B<P>(tb, m, e, k, g[kB11 * Kp + k], g[kB12 * Kp + k], g[kB21 * Kp + k], g[kB22 * Kp + k], x, u1, u2);
  const double sc = tau / (2.0 * g[kArea * Kp + k]);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    tout[i * Kp + k] = sc * u1[i];
    tout[(N + i) * Kp + k] = sc * u2[i];
  }
}

// ---- rank-Qe edge form (TableLayout rkR..rkW, when DevTables::rank_ok) ------
// Every edge operator is a Qe-point quadrature sum (s_diag_n = pe_n^t W pe_n,
// s_offdiag_{n,np} = pe_n^t W pth_{n,np}, the off-diagonal E blocks with the
// sampled d, ldg_offdiag.cuh), so an edge costs the projections of the
// vectors onto its points, a pointwise combination and ONE product back
// instead of an N x N table product per term; the derivative tables are
// degree-lower-triangular and their zero chunks are skipped.  Same integrals
// as the tables (exact rule), different rounding (<= 1e-15 relative).
template <int P>
struct RkCfg {
  static constexpr int N = Cfg<P>::N, NP = Cfg<P>::NP, Q = Cfg<P>::Q, QP = (Q + 1) / 2 * 2;
  static constexpr int kR = 0, kRm = 3 * Q * NP, kT = 6 * Q * NP, kV = kT + 3 * N * QP, kW = kV + 9 * N * QP;
  static constexpr int kCount = kW + QP;
};

// copies two launch-invariant table blocks (even counts, 16-byte aligned) into shared memory
__device__ __forceinline__ void stage_d2(double* sm, const double* a, int na, const double* b, int nb) {
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  double2* d2 = reinterpret_cast<double2*>(sm);
  for (int i = threadIdx.x; i < na / 2; i += blockDim.x) d2[i] = a2[i];
  for (int i = threadIdx.x; i < nb / 2; i += blockDim.x) d2[na / 2 + i] = b2[i];
  __syncthreads();
}

// z[0..QP) += row[.] v
template <int QP>
__device__ __forceinline__ void rk_acc(const double* row, double v, double* z) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
  for (int c = 0; c < QP / 2; ++c) {
    const double2 t = r2[c];
    z[2 * c] = fma(t.x, v, z[2 * c]);
    z[2 * c + 1] = fma(t.y, v, z[2 * c + 1]);
  }
}

// out[0..N) += sum_q R[q][.] z[q]
template <int N, int NP, int Q>
__device__ __forceinline__ void rk_out(const double* R, const double* z, double* out) {
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double2* r2 = reinterpret_cast<const double2*>(R + q * NP);
#pragma unroll
    for (int c = 0; c < N / 2; ++c) {
      const double2 t = r2[c];
      out[2 * c] = fma(t.x, z[q], out[2 * c]);
      out[2 * c + 1] = fma(t.y, z[q], out[2 * c + 1]);
    }
    if (N & 1) out[N - 1] = fma(R[q * NP + N - 1], z[q], out[N - 1]);
  }
}

__host__ __device__ constexpr int hier_first_row(int j) {
  int d = 0;
  while ((d + 1) * (d + 2) / 2 <= j) ++d;  // degree of phi_j
  return (d + 1) * (d + 2) / 2;            // first basis function of degree d + 1
}

// u^m = B^m x in rank form (B^m = -H^m + Q^m + Q_N^m): the H part from the two
// derivative tables at sH (tH, or tmH with m_hat^-1 applied), the edge parts
// through rows rR of the output table (rkR, or rkRm with m_hat^-1 applied)
template <int P>
__device__ __forceinline__ void apply_B_rank(const double* sH, const double* rk, int rR, const DevMesh& m, int k,
                                             const double* __restrict__ x, double* u1, double* u2) {
  using RC = RkCfg<P>;
  constexpr int N = Cfg<P>::N, NP = Cfg<P>::NP, NNP = N * NP, Q = RC::Q, QP = RC::QP;
  const long Kp = m.Kp;
  const double* g = m.geom;
  {
    double w1[N], w2[N];
#pragma unroll
    for (int i = 0; i < N; ++i) w1[i] = w2[i] = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const double xj = x[j * Kp + k];
      const int first = hier_first_row(j);
      const double2* r1 = reinterpret_cast<const double2*>(sH + j * NP);
      const double2* r2 = reinterpret_cast<const double2*>(sH + NNP + j * NP);
#pragma unroll
      for (int c = 0; c < N / 2; ++c) {
        if (2 * c + 1 < first) continue;
        const double2 a = r1[c], b = r2[c];
        w1[2 * c] = fma(a.x, xj, w1[2 * c]);
        w1[2 * c + 1] = fma(a.y, xj, w1[2 * c + 1]);
        w2[2 * c] = fma(b.x, xj, w2[2 * c]);
        w2[2 * c + 1] = fma(b.y, xj, w2[2 * c + 1]);
      }
      if ((N & 1) && N - 1 >= first) {
        w1[N - 1] = fma(sH[j * NP + N - 1], xj, w1[N - 1]);
        w2[N - 1] = fma(sH[NNP + j * NP + N - 1], xj, w2[N - 1]);
      }
    }
    const double b11 = g[kB11 * Kp + k], b12 = g[kB12 * Kp + k], b21 = g[kB21 * Kp + k], b22 = g[kB22 * Kp + k];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      u1[i] = fma(b21, w2[i], -b22 * w1[i]);
      u2[i] = fma(-b11, w2[i], b12 * w1[i]);
    }
  }
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kind = m.kind[n * Kp + k];
    const int kp = m.nbr[n * Kp + k];
    const double len = g[(kLen0 + n) * Kp + k];
    const double co = kind == kInterior ? 0.5 * len : (kind == kNeumann ? len : 0.0);
    if (co == 0.0 && kp < 0) continue;
    double z[QP];
#pragma unroll
    for (int q = 0; q < QP; ++q) z[q] = 0.0;
    if (co != 0.0) {
      const double* tT = rk + RC::kT + n * N * QP;
#pragma unroll
      for (int j = 0; j < N; ++j) rk_acc<QP>(tT + j * QP, co * x[j * Kp + k], z);
    }
    if (kp >= 0) {
      const double hl = 0.5 * len;
      const double* tV = rk + RC::kV + (n * 3 + m.nbrn[n * Kp + k]) * N * QP;
#pragma unroll
      for (int j = 0; j < N; ++j) rk_acc<QP>(tV + j * QP, hl * x[j * Kp + kp], z);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) z[q] *= rk[RC::kW + q];
    double sv[N];
#pragma unroll
    for (int i = 0; i < N; ++i) sv[i] = 0.0;
    rk_out<N, NP, Q>(rk + rR + n * Q * NP, z, sv);
    const double nux = g[(kNux0 + n) * Kp + k], nuy = g[(kNuy0 + n) * Kp + k];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      u1[i] = fma(nux, sv[i], u1[i]);
      u2[i] = fma(nuy, sv[i], u2[i]);
    }
  }
}

// stage 1 of the Krylov operator in rank form: tout^m = tau M_k^-1 B^m x
template <int P>
__global__ void __launch_bounds__(128, LDG_MINB_STAGE_P(P)) k_stage1r(DevMesh m, DevTables T,
                                                                      const double* __restrict__ x, double tau,
                                                                      double* __restrict__ tout, int k0, int k1) {
  using RC = RkCfg<P>;
  constexpr int N = Cfg<P>::N, NNP = N * Cfg<P>::NP;
  extern __shared__ __align__(16) double sm[];
  stage_d2(sm, T.base + T.tmH, 2 * NNP, T.base + T.rkR, RC::kCount);
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  const long Kp = m.Kp;
  double u1[N], u2[N];
  apply_B_rank<P>(sm, sm + 2 * NNP, RC::kRm, m, k, x, u1, u2);
  const double sc = tau / (2.0 * m.geom[kArea * Kp + k]);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    tout[i * Kp + k] = sc * u1[i];
    tout[(N + i) * Kp + k] = sc * u2[i];
  }
}

// Everything crossing the edges of element k in the C row, rank form:
//   acc += ce sum_{kp} E_{k,kp} t_kp  +  beta ((S + S_D) x)_k
// t = (t^1, t^2) at stride N Kp (null: no E term), x null / beta 0: no S term
template <int P>
__device__ __forceinline__ void edges_rank(const double* rk, const DevMesh& m, int k, const double* __restrict__ D,
                                           const double* __restrict__ t, double ce, const double* __restrict__ x,
                                           double beta, double* acc) {
  using RC = RkCfg<P>;
  constexpr int N = Cfg<P>::N, NP = Cfg<P>::NP, Q = RC::Q, QP = RC::QP;
  const long Kp = m.Kp;
  const double* g = m.geom;
  const bool sx = x != nullptr && beta != 0.0;
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kind = m.kind[n * Kp + k];
    const int kp = m.nbr[n * Kp + k];
    const bool pen = sx && (kind == kInterior || kind == kDirichlet);
    if (!pen && kp < 0) continue;
    double z[QP];
#pragma unroll
    for (int q = 0; q < QP; ++q) z[q] = 0.0;
    if (pen) {
      const double* tT = rk + RC::kT + n * N * QP;
#pragma unroll
      for (int j = 0; j < N; ++j) rk_acc<QP>(tT + j * QP, beta * x[j * Kp + k], z);
    }
    if (kp >= 0) {
      const double* tV = rk + RC::kV + (n * 3 + m.nbrn[n * Kp + k]) * N * QP;
      if (t) {
        const double hl = 0.5 * g[(kLen0 + n) * Kp + k];
        const double co1 = hl * g[(kNux0 + n) * Kp + k], co2 = hl * g[(kNuy0 + n) * Kp + k];
        double dv[QP], uv[QP];
#pragma unroll
        for (int q = 0; q < QP; ++q) dv[q] = uv[q] = 0.0;
#pragma unroll(N <= 6 ? N : 3)
        for (int j = 0; j < N; ++j) {
          const double dj = D[j * Kp + kp];
          const double uj = fma(co1, t[j * Kp + kp], co2 * t[(N + j) * Kp + kp]);
          const double xj = sx ? -beta * x[j * Kp + kp] : 0.0;
          const double2* r2 = reinterpret_cast<const double2*>(tV + j * QP);
#pragma unroll
          for (int c = 0; c < QP / 2; ++c) {
            const double2 tt = r2[c];
            dv[2 * c] = fma(tt.x, dj, dv[2 * c]);
            dv[2 * c + 1] = fma(tt.y, dj, dv[2 * c + 1]);
            uv[2 * c] = fma(tt.x, uj, uv[2 * c]);
            uv[2 * c + 1] = fma(tt.y, uj, uv[2 * c + 1]);
            z[2 * c] = fma(tt.x, xj, z[2 * c]);
            z[2 * c + 1] = fma(tt.y, xj, z[2 * c + 1]);
          }
        }
#pragma unroll
        for (int q = 0; q < QP; ++q) z[q] = fma(ce * dv[q], uv[q], z[q]);
      } else if (sx) {
#pragma unroll
        for (int j = 0; j < N; ++j) rk_acc<QP>(tV + j * QP, -beta * x[j * Kp + kp], z);
      }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) z[q] *= rk[RC::kW + q];
    rk_out<N, NP, Q>(rk + RC::kR + n * Q * NP, z, acc);
  }
}

// stage 2: y = alpha M_k x_k + beta (S + S_D) x - gamma sum_m sum_s E^m[s] tz^m_col + delta w
// (the Krylov operator, FP64): stored diagonal blocks streamed, off-diagonal
// blocks matrix-free from D.
template <int P, bool RK>
__global__ void __launch_bounds__(128, LDG_MINB_S2STAGE_P(P)) k_stage2(DevMesh m, DevTables T, const double* __restrict__ E,
                                                const double* __restrict__ D, const double* __restrict__ x,
                                                double alpha, double beta, const double* __restrict__ tz,
                                                double gamma, const double* __restrict__ w, double delta,
                                                double* __restrict__ y, int k0, int k1) {
  constexpr int N = Cfg<P>::N, NN = N * N, NP = Cfg<P>::NP;
  extern __shared__ __align__(16) double sm[];
  if constexpr (RK) {  // tM | rank-Qe edge block
    stage_d2(sm, T.base + T.tM, N * NP, T.base + T.rkR, RkCfg<P>::kCount);
    const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= k1) return;
    const long Kp = m.Kp;
    double acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = 0.0;
    if (tz) {
#pragma unroll 1
      for (int c = 0; c < 2; ++c)
        block_mv_gather<N>(E + static_cast<long>(c) * NN * Kp, Kp, k, tz + static_cast<long>(c) * N * Kp, k, acc);
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] *= -gamma;
    }
    edges_rank<P>(sm + N * NP, m, k, D, tz, -gamma, x, beta, acc);
    if (x && alpha != 0.0) {
      double v[N];
      tab_mv_g<N, NP>(sm, x, Kp, k, v);
      const double sa = alpha * 2.0 * m.geom[kArea * Kp + k];
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = fma(sa, v[i], acc[i]);
    }
    if (w) {
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = fma(delta, w[i * Kp + k], acc[i]);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) y[i * Kp + k] = acc[i];
    return;
  }
  const STab<P> tb = stage_tables<P, true>(sm, T);
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  const long Kp = m.Kp;
  double acc[N];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = 0.0;
  const EdgeData e = load_edges(m, k);
  if (tz) {
#pragma unroll 1
    for (int c = 0; c < 2; ++c)
      block_mv_gather<N>(E + static_cast<long>(c) * NN * Kp, Kp, k, tz + static_cast<long>(c) * N * Kp, k, acc);
    offdiag_all<P>(sm + Cfg<P>::TAB, D, tz, Kp, e, acc);
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] *= -gamma;
  }
  if (x) {
    if (alpha != 0.0) {
      double v[N];
      tab_mv_g<N, NP>(tb.M(), x, Kp, k, v);
      const double sa = alpha * 2.0 * m.geom[kArea * Kp + k];
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = fma(sa, v[i], acc[i]);
    }
    if (beta != 0.0) apply_S<P>(tb, m, e, k, x, beta, acc);
  }
  if (w) {
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = fma(delta, w[i * Kp + k], acc[i]);
  }
#pragma unroll
  for (int i = 0; i < N; ++i) y[i * Kp + k] = acc[i];
}

// full (W + dt A) Y, Y = [Z1; Z2; C] (system.hpp:161-167):
//   out_Zm = dt (M z^m_k + B^m c)
//   out_C  = wm M c_k + dt (sum_m E^m z^m + eta (S + S_D) c)
template <int P, bool RK>
__global__ void __launch_bounds__(128, LDG_MINB_STAGE_P(P)) k_full(DevMesh m, DevTables T, const double* __restrict__ E,
                                              const double* __restrict__ D, const double* __restrict__ Yin,
                                              double wm, double dt, double eta, double* __restrict__ out) {
  constexpr int N = Cfg<P>::N, NN = N * N, NP = Cfg<P>::NP;
  extern __shared__ __align__(16) double sm[];
  if constexpr (RK) {  // tH 2 | tM | rank-Qe edge block
    {
      const double2* a2 = reinterpret_cast<const double2*>(T.base + T.tH);
      const double2* b2 = reinterpret_cast<const double2*>(T.base + T.tM);
      const double2* c2 = reinterpret_cast<const double2*>(T.base + T.rkR);
      double2* d2 = reinterpret_cast<double2*>(sm);
      for (int i = threadIdx.x; i < N * NP; i += blockDim.x) d2[i] = a2[i];
      for (int i = threadIdx.x; i < N * NP / 2; i += blockDim.x) d2[N * NP + i] = b2[i];
      for (int i = threadIdx.x; i < RkCfg<P>::kCount / 2; i += blockDim.x) d2[3 * N * NP / 2 + i] = c2[i];
      __syncthreads();
    }
    const double* sM = sm + 2 * N * NP;
    const double* rk = sm + 3 * N * NP;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m.K) return;
    const long Kp = m.Kp;
    const double two_a = 2.0 * m.geom[kArea * Kp + k];
    const double* C = Yin + 2L * N * Kp;
    double w[N];
    {
      double u1[N], u2[N];
      apply_B_rank<P>(sm, rk, RkCfg<P>::kR, m, k, C, u1, u2);
      tab_mv_g<N, NP>(sM, Yin, Kp, k, w);
#pragma unroll
      for (int i = 0; i < N; ++i) out[i * Kp + k] = dt * fma(two_a, w[i], u1[i]);
      tab_mv_g<N, NP>(sM, Yin + static_cast<long>(N) * Kp, Kp, k, w);
#pragma unroll
      for (int i = 0; i < N; ++i) out[(N + i) * Kp + k] = dt * fma(two_a, w[i], u2[i]);
    }
    double acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = 0.0;
#pragma unroll 1
    for (int c = 0; c < 2; ++c)
      block_mv_gather<N>(E + static_cast<long>(c) * NN * Kp, Kp, k, Yin + static_cast<long>(c) * N * Kp, k, acc);
    edges_rank<P>(rk, m, k, D, Yin, 1.0, C, eta, acc);
    tab_mv_g<N, NP>(sM, C, Kp, k, w);
#pragma unroll
    for (int i = 0; i < N; ++i) out[(2 * N + i) * Kp + k] = fma(wm * two_a, w[i], dt * acc[i]);
    return;
  }
  const STab<P> tb = stage_tables<P, true>(sm, T);
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m.K) return;
  const long Kp = m.Kp;
  const double* g = m.geom;
  const double two_a = 2.0 * g[kArea * Kp + k];
  const double* C = Yin + 2L * N * Kp;
  const EdgeData e = load_edges(m, k);
  double w[N];
  {
    double u1[N], u2[N];
#pragma unroll
    for (int i = 0; i < N; ++i) u1[i] = u2[i] = 0.0;
    apply_B<P>(tb, m, e, k, g[kB11 * Kp + k], g[kB12 * Kp + k], g[kB21 * Kp + k], g[kB22 * Kp + k], C, u1, u2);
    tab_mv_g<N, NP>(tb.M(), Yin, Kp, k, w);
#pragma unroll
    for (int i = 0; i < N; ++i) out[i * Kp + k] = dt * fma(two_a, w[i], u1[i]);
    tab_mv_g<N, NP>(tb.M(), Yin + static_cast<long>(N) * Kp, Kp, k, w);
#pragma unroll
    for (int i = 0; i < N; ++i) out[(N + i) * Kp + k] = dt * fma(two_a, w[i], u2[i]);
  }
  double acc[N];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = 0.0;
#pragma unroll 1
  for (int c = 0; c < 2; ++c)
    block_mv_gather<N>(E + static_cast<long>(c) * NN * Kp, Kp, k, Yin + static_cast<long>(c) * N * Kp, k, acc);
  offdiag_all<P>(sm + Cfg<P>::TAB, D, Yin, Kp, e, acc);
  apply_S<P>(tb, m, e, k, C, eta, acc);
  tab_mv_g<N, NP>(tb.M(), C, Kp, k, w);
#pragma unroll
  for (int i = 0; i < N; ++i) out[(2 * N + i) * Kp + k] = fma(wm * two_a, w[i], dt * acc[i]);
}

// y = beta y + omega P^-1 x  (beta = 0: plain block-Jacobi application)
template <int P, typename TP>
__global__ void __launch_bounds__(128) k_bjac_axpy(int K, long Kp, const TP* __restrict__ Pinv,
                                                   const double* __restrict__ x, double omega, double beta,
                                                   double* __restrict__ y) {
  constexpr int N = Cfg<P>::N;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double acc[N];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = 0.0;
  block_mv_gather<N>(Pinv, Kp, k, x, k, acc);
#pragma unroll
  for (int i = 0; i < N; ++i) y[i * Kp + k] = (beta == 0.0 ? 0.0 : beta * y[i * Kp + k]) + omega * acc[i];
}

template <int P>
size_t tab_smem() {
  return sizeof(double) * Cfg<P>::TAB;
}
template <int P>
size_t tab_edge_smem() {
  return sizeof(double) * (Cfg<P>::TAB + Cfg<P>::EDGE);
}

template <typename Kern>
void set_smem(Kern kern, size_t bytes) {
  if (bytes > 48 * 1024)
    LDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

__global__ void k_to_f32(long n, const double* __restrict__ src, float* __restrict__ dst) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<float>(src[i]);
}

// Kernel shape per launch: thread-per-element (this file) keeps each vector
// value in a register for all N rows and issues the fewest load
// instructions, which wins once a level fills the GPU; the row-parallel
// kernels (ldg_rows.cu) win on small levels, where a thread's serial load
// chain is the latency (measured at p = 4: fine level 246 vs 354 us, coarse
// levels 35 vs 90 us; with the packed FP16/FP32 smoother, matrix-free
// off-diagonal blocks and loads issued ahead of the FMA chains, the 8192- and
// 2048-element levels sweep in 27 / 26 us on thread-per-element kernels vs
// 57 / 54 us otherwise at p = 4, hence the default of 2048).
// LDG_ROWS_BELOW overrides the switch.
// LDG_RANK_FORM=0: the table kernels even when the tensors allow the rank form (A/B, tests)
bool rank_form() {
  static const bool on = [] {
    const char* s = std::getenv("LDG_RANK_FORM");
    return s ? std::atoi(s) != 0 : true;
  }();
  return on;
}

bool use_rows(const Handle& h) {
  static const long below = [] {
    const char* s = std::getenv("LDG_ROWS_BELOW");
    return s ? std::atol(s) : 2048L;
  }();
  return h.K < below;
}

}  // namespace

void launch_stage1(Handle& h, const double* vz, double sigma, const double* x, double tau, double* tout, int k0,
                   int k1) {
  if (k1 < 0) k1 = h.K;
  if (k1 <= k0) return;
  if (use_rows(h)) {
    if (k0 != 0 || k1 != h.K) throw Error(LDG_EINVAL, "element range on the row kernels");
    return rows_stage1(h, vz, sigma, x, tau, tout);
  }
  const unsigned grid = grid_of(k1 - k0, 128);
  // the Krylov operator's stage 1 (x only): premultiplied tables, no trailing M^-1 product
#define CALL(P)                                                                                               \
  do {                                                                                                        \
    if (!vz && x && h.dtab.rank_ok && rank_form()) {                                                          \
      const size_t smr = sizeof(double) * (2 * Cfg<P>::N * Cfg<P>::NP + RkCfg<P>::kCount);                    \
      set_smem(k_stage1r<P>, smr);                                                                            \
      k_stage1r<P><<<grid, 128, smr, h.stream>>>(h.mesh(), h.dtab, x, tau, tout, k0, k1);                     \
    } else if (!vz && x) {                                                                                    \
      const size_t sm14 = sizeof(double) * 14 * Cfg<P>::N * Cfg<P>::NP;                                       \
      set_smem(k_stage1m<P>, sm14);                                                                           \
      k_stage1m<P><<<grid, 128, sm14, h.stream>>>(h.mesh(), h.dtab, x, tau, tout, k0, k1);                    \
    } else {                                                                                                  \
      set_smem(k_stage1<P>, tab_smem<P>());                                                                   \
      k_stage1<P><<<grid, 128, tab_smem<P>(), h.stream>>>(h.mesh(), h.dtab, vz, sigma, x, tau, tout, k0, k1); \
    }                                                                                                         \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_stage2(Handle& h, const double* x, double alpha_m, double beta_s, const double* tz, double gamma_e,
                   const double* w, double delta, double* y, int k0, int k1) {
  if (k1 < 0) k1 = h.K;
  if (k1 <= k0) return;
  if (use_rows(h)) {
    if (k0 != 0 || k1 != h.K) throw Error(LDG_EINVAL, "element range on the row kernels");
    return rows_stage2<double>(h, h.E.ptr, x, alpha_m, beta_s, tz, gamma_e, w, delta, y);
  }
  const unsigned grid = grid_of(k1 - k0, 128);
#define CALL(P)                                                                                               \
  do {                                                                                                        \
    if (h.dtab.rank_ok && rank_form()) {                                                                      \
      const size_t smr = sizeof(double) * (Cfg<P>::N * Cfg<P>::NP + RkCfg<P>::kCount);                        \
      set_smem(k_stage2<P, true>, smr);                                                                       \
      k_stage2<P, true><<<grid, 128, smr, h.stream>>>(h.mesh(), h.dtab, h.E.ptr, h.D.ptr, x, alpha_m, beta_s, \
                                                      tz, gamma_e, w, delta, y, k0, k1);                      \
    } else {                                                                                                  \
      set_smem(k_stage2<P, false>, tab_edge_smem<P>());                                                       \
      k_stage2<P, false><<<grid, 128, tab_edge_smem<P>(), h.stream>>>(h.mesh(), h.dtab, h.E.ptr, h.D.ptr, x,  \
                                                                      alpha_m, beta_s, tz, gamma_e, w, delta, \
                                                                      y, k0, k1);                             \
    }                                                                                                         \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_full_apply(Handle& h, const double* Y, double wm, double dt, double* out) {
  const unsigned grid = grid_of(h.K, 128);
#define CALL(P)                                                                                                 \
  do {                                                                                                          \
    if (h.dtab.rank_ok && rank_form()) {                                                                        \
      const size_t smr = sizeof(double) * (3 * Cfg<P>::N * Cfg<P>::NP + RkCfg<P>::kCount);                      \
      set_smem(k_full<P, true>, smr);                                                                           \
      k_full<P, true><<<grid, 128, smr, h.stream>>>(h.mesh(), h.dtab, h.E.ptr, h.D.ptr, Y, wm, dt, h.prob.eta,  \
                                                    out);                                                       \
    } else {                                                                                                    \
      set_smem(k_full<P, false>, tab_edge_smem<P>());                                                           \
      k_full<P, false><<<grid, 128, tab_edge_smem<P>(), h.stream>>>(h.mesh(), h.dtab, h.E.ptr, h.D.ptr, Y, wm,  \
                                                                    dt, h.prob.eta, out);                       \
    }                                                                                                           \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_bjac_setup(Handle& h, double wm, double dt) { launch_bjac(h, wm, dt, 0); }

// FP32 inverses from the FP64 E of the level (row-kernel smoother copies)

void launch_bjac_setup_f32_from64(Handle& h, double wm, double dt) { launch_bjac(h, wm, dt, 1); }

bool level_uses_rows(const Handle& h) { return use_rows(h); }

// Levels below LDG_SMALL_BELOW elements (default 4096) run the multigrid
// smoother on the lane-split kernels of ldg_small.cu (latency-bound sizes);
// measured at p = 4 on an 8192-element level they were 3x slower than the
// row kernels, whose streams stay coalesced.
bool level_is_small(const Handle& h) {
  static const long below = [] {
    const char* s = std::getenv("LDG_SMALL_BELOW");
    return s ? std::atol(s) : 4096L;
  }();
  return h.K < below;
}

void launch_bjac_apply(Handle& h, const double* x, double* y) { launch_bjac_axpy(h, x, 1.0, 0.0, y); }

template <typename TP>
void bjac_axpy_impl(Handle& h, const TP* Pinv, const double* x, double omega, double beta, double* y) {
  if (use_rows(h)) return rows_bjac<TP>(h, Pinv, x, omega, beta, y);
  const unsigned grid = grid_of(h.K, 128);
#define CALL(P) k_bjac_axpy<P, TP><<<grid, 128, 0, h.stream>>>(h.K, h.Kp, Pinv, x, omega, beta, y)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_bjac_axpy(Handle& h, const double* x, double omega, double beta, double* y) {
  bjac_axpy_impl<double>(h, h.Pinv.ptr, x, omega, beta, y);
}

void launch_bjac_axpy_f32(Handle& h, const double* x, double omega, double beta, double* y) {
  bjac_axpy_impl<float>(h, h.Pinv32.ptr, x, omega, beta, y);
}

void launch_to_f32(Handle& h, long n, const double* src, float* dst) {
  k_to_f32<<<1184, 256, 0, h.stream>>>(n, src, dst);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

}  // namespace ldgb
