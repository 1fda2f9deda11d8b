// Mixed-precision multigrid smoother kernels (the preconditioner's hot path).
//
// The V-cycle spends most of each implicit-Euler step in three operations per
// smoothing sweep on the large levels: t^m = M^-1 B^m x (stage 1), the
// residual r = b - S_c x (stage 2) and the damped block-Jacobi update
// x += omega P^-1 r.  Here they run in FP32 arithmetic on FP32 operator
// copies; vectors stay FP64 and the outer Krylov operator is untouched, so
// only the preconditioner's contraction depends on the rounding.
//
//  * The stored blocks (E^m_kk, P_k^-1) are FP16, scaled per element, packed
//    four values to a 64-bit quad in the (column group, column, row) order of
//    ldg_pack.cuh and streamed one quad plane at a time: a warp moves 256
//    contiguous bytes per load instruction.
//  * Stage 2 and the block-Jacobi update are one kernel: the residual of the
//    element never leaves registers (ping-pong x_in -> x_out, since stage 2
//    reads the neighbours' x).
//  * Every edge term is applied in rank-Qe form from small shared-memory
//    tables (RankCfg below); from p = 3 on stage 1 hands its projections to
//    stage 2 as edge traces, and chained sweeps reuse the traces stage 2
//    leaves of its output.
//
// Reference operators restated (as in ldg_apply.cu): B^m = -H^m + Q^m + Q_N^m
// (assembly.hpp:92-109, 174-208), S + S_D (assembly.hpp:142-168), M = 2|T| mhat.
#include <cuda_fp16.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <type_traits>

#include "ldg_internal.hpp"
#include "ldg_pack.cuh"
#include "ldg_offdiag.cuh"

// min resident CTAs per SM of the thread-per-element kernels, per degree
// p = 0..4 (stage 1 | stage 2).  The level-0 grids are 1024 CTAs of 128
// (256^2 FK): 7-8 CTAs/SM (<= 72 / 64 registers) run them in ONE wave, and
// anything that takes stage 2 above one wave loses (round 2, p = 4, with the
// trace-form kernel: two column groups in flight at 5 / 6 CTAs 86 / 100 us
// per sweep against 76 at 7; 8 CTAs 84).  Stage 1 at p = 4 stays at 4 CTAs
// (128 registers; 5 / 6 / 7 CTAs: sweep 81.7 / 85.2 / 77.4 us against 76.8,
// chained or not), at p = 3 7 CTAs beat 8 (41.8 vs 45.1 us per sweep).  8 at
// p <= 1 measured slower; 7 at p = 1 is needed all the same: left alone the
// compiler takes 80 registers, 6 CTAs/SM hold 888 of the level's 1024 CTAs
// and the rest runs as a second wave (p = 1 sweep 14.3 -> 9.6 us, 10-step
// C2 bench 30.7 -> 29.9 ms: every degree >= 2 smooths a p = 1 level of 256^2).
// -DLDG_MINB_S1=abcde / -DLDG_MINB_S1C=abcde (chained sweeps) /
// -DLDG_MINB_S2=abcde (one digit per p = 0..4) override (tuning builds).
#ifndef LDG_MINB_S1
#define LDG_MINB_S1 17874
#endif
#ifndef LDG_MINB_S2
#define LDG_MINB_S2 17777
#endif

namespace ldgb {

namespace {

constexpr int minb_digit(int code, int p) { return p == 4 ? code % 10 : minb_digit(code / 10, p + 1); }
constexpr int kMinbS1[5] = {minb_digit(LDG_MINB_S1, 0), minb_digit(LDG_MINB_S1, 1), minb_digit(LDG_MINB_S1, 2),
                            minb_digit(LDG_MINB_S1, 3), minb_digit(LDG_MINB_S1, 4)};
// stage 1 on chained sweeps (no projections of x: fewer registers)
#ifndef LDG_MINB_S1C
#define LDG_MINB_S1C 17874
#endif
constexpr int kMinbS1c[5] = {minb_digit(LDG_MINB_S1C, 0), minb_digit(LDG_MINB_S1C, 1), minb_digit(LDG_MINB_S1C, 2),
                             minb_digit(LDG_MINB_S1C, 3), minb_digit(LDG_MINB_S1C, 4)};
constexpr int kMinbS2[5] = {minb_digit(LDG_MINB_S2, 0), minb_digit(LDG_MINB_S2, 1), minb_digit(LDG_MINB_S2, 2),
                            minb_digit(LDG_MINB_S2, 3), minb_digit(LDG_MINB_S2, 4)};
static_assert(kMinbS1[0] == LDG_MINB_S1 / 10000 && kMinbS2[4] == LDG_MINB_S2 % 10, "min-blocks digits");

template <int P>
using Cfg = SmCfg<P>;

inline unsigned grid_of(long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

#define LDG_DISPATCH_P(p, CALL) \
  switch (p) {                  \
    case 0: { CALL(0); break; } \
    case 1: { CALL(1); break; } \
    case 2: { CALL(2); break; } \
    case 3: { CALL(3); break; } \
    default: { CALL(4); break; } \
  }

__device__ __forceinline__ long Kp_of(const DevMesh& m) { return m.Kp; }

__device__ __forceinline__ float comp(const float4& v, int r) {
  return r == 0 ? v.x : (r == 1 ? v.y : (r == 2 ? v.z : v.w));
}

// copies `count` floats of the FP32 tables into shared memory
__device__ __forceinline__ const float* stage_f(float* sm, const float* src, int count) {
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(sm);
  for (int i = threadIdx.x; i < count / 4; i += blockDim.x) d4[i] = s4[i];
  __syncthreads();
  return sm;
}

// w = T x, T^t rows of NF floats in shared memory.  Paired FP32 FMAs
// (FFMA2, sm_100): one 128-bit broadcast load feeds two of them, half the
// FMA instructions of the scalar form (these kernels are issue-bound).
template <int N, int NF>
__device__ __forceinline__ void ftab_mv(const float* sT, const float* x, float* w) {
  float2 acc[NF / 2];
#pragma unroll
  for (int q = 0; q < NF / 2; ++q) acc[q] = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float4* row = reinterpret_cast<const float4*>(sT + j * NF);
    const float2 xj = make_float2(x[j], x[j]);
#pragma unroll
    for (int q = 0; q < NF / 4; ++q) {
      const float4 t = row[q];
      acc[2 * q] = __ffma2_rn(make_float2(t.x, t.y), xj, acc[2 * q]);
      if (4 * q + 2 < N) acc[2 * q + 1] = __ffma2_rn(make_float2(t.z, t.w), xj, acc[2 * q + 1]);
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] = (i & 1) ? acc[i / 2].y : acc[i / 2].x;
}

template <int N>
__device__ __forceinline__ void load_f(const double* __restrict__ x, long Kp, int col, float* v) {
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = static_cast<float>(x[j * Kp + col]);
}

// ---- rank-Qe edge terms --------------------------------------------------
// Every edge matrix of the smoother is a quadrature sum over the Qe points
// of the edge rule (FTables: s_diag_n = peR_n^t diag(we) peR_n, s_offdiag =
// peR_n^t diag(we) pthT_{n,np}^t, and the off-diagonal E blocks with the
// sampled d, ldg_offdiag.cuh), so one edge costs its projections onto the
// points (N Qe each), a pointwise combination, and ONE product back
// (Qe N) instead of an N x N table product per term: per edge at p = 4,
// stage 2 runs 525 FMAs where the table form ran 765, stage 1 315 for 510,
// and the staged tables shrink from 13-14 N x NF blocks to 7 KB.
// Edge traces between stage 1 and stage 2 from this degree on (measured at
// 256^2, level-0 sweep: p = 4 88.3 -> 76.2 us; p = 3 42.8 either way; p <= 2
// and the small levels lose 2 us per sweep to the longer stage 1)
#ifndef LDG_TRACE_MINP
#define LDG_TRACE_MINP 3
#endif
constexpr int kTraceMinP = LDG_TRACE_MINP;

template <int P>
struct RankCfg {
  static constexpr int N = Cfg<P>::N, NF = Cfg<P>::NF, Q = Cfg<P>::Q, QF = (Q + 3) / 4 * 4;
  static constexpr int kPeT = 3 * Q * NF, kPthT = kPeT + 3 * N * QF, kWe = kPthT + 9 * N * QF;
  static constexpr int kFloats = kWe + QF;  // [peR | peT | pthT | weR]
};

// z (QF values as pairs) += T[j][.] v: row j of a [N][QF] projection table
template <int QF>
__device__ __forceinline__ void rank_acc(const float* rowj, float v, float2* z) {
  const float2 vv = make_float2(v, v);
  const float4* r4 = reinterpret_cast<const float4*>(rowj);
#pragma unroll
  for (int c = 0; c < QF / 4; ++c) {
    const float4 t = r4[c];
    z[2 * c] = __ffma2_rn(make_float2(t.x, t.y), vv, z[2 * c]);
    z[2 * c + 1] = __ffma2_rn(make_float2(t.z, t.w), vv, z[2 * c + 1]);
  }
}

// The same for column j of a derivative table h_hat(., ., m): the modal basis
// is hierarchical by degree (N = 1, 3, 6, 10, 15 functions up to degree
// 0..4) and d phi_i has a lower degree than phi_i, so H[i][j] = int d_m phi_i
// phi_j vanishes unless deg phi_i > deg phi_j: the 4-row chunks below the
// first row of degree deg(j) + 1 are skipped (29 of 60 chunks remain at p = 4).
__host__ __device__ constexpr int hier_first_row(int j) {
  int d = 0;
  while ((d + 1) * (d + 2) / 2 <= j) ++d;  // degree of phi_j
  return (d + 1) * (d + 2) / 2;            // first basis function of degree d + 1
}
template <int NF>
__device__ __forceinline__ void hier_acc(const float* rowj, float v, float2* z, int j) {
  const float2 vv = make_float2(v, v);
  const float4* r4 = reinterpret_cast<const float4*>(rowj);
  const int first = hier_first_row(j);
#pragma unroll
  for (int c = 0; c < NF / 4; ++c) {
    if (4 * c + 3 < first) continue;
    const float4 t = r4[c];
    z[2 * c] = __ffma2_rn(make_float2(t.x, t.y), vv, z[2 * c]);
    z[2 * c + 1] = __ffma2_rn(make_float2(t.z, t.w), vv, z[2 * c + 1]);
  }
}

// out (NF values as pairs) += sum_q R[q][.] z[q]: the rows of peR_n
template <int Q, int NF>
__device__ __forceinline__ void rank_out(const float* R, const float2* z, float2* out) {
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const float zq = (q & 1) ? z[q / 2].y : z[q / 2].x;
    const float2 vv = make_float2(zq, zq);
    const float4* r4 = reinterpret_cast<const float4*>(R + q * NF);
#pragma unroll
    for (int c = 0; c < NF / 4; ++c) {
      const float4 t = r4[c];
      out[2 * c] = __ffma2_rn(make_float2(t.x, t.y), vv, out[2 * c]);
      out[2 * c + 1] = __ffma2_rn(make_float2(t.z, t.w), vv, out[2 * c + 1]);
    }
  }
}

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return make_float2(a.x * b.x, a.y * b.y); }

// copies two launch-invariant table blocks into shared memory (one barrier)
__device__ __forceinline__ void stage_f2(float* sm, const float* a, int na, const float* b, int nb) {
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* d4 = reinterpret_cast<float4*>(sm);
  for (int i = threadIdx.x; i < na / 4; i += blockDim.x) d4[i] = a4[i];
  for (int i = threadIdx.x; i < nb / 4; i += blockDim.x) d4[na / 4 + i] = b4[i];
  __syncthreads();
}

// tout^m = M_k^-1 B^m x (both m), FP32 arithmetic, FP64 in/out.  The element
// part -H^m from the two m_hat^-1-premultiplied tables, the edge parts
// Q^m + Q_N^m in rank-Qe form (m_hat = I to rounding in FP32).
//
// With `tr` (single-rank levels) the element also leaves its edge traces for
// stage 2, [n][q][Kp] at the Qe points of its own edges: x (already
// projected here) and -(c1 t^1 + c2 t^2), c = nu |E| / 2 — what the
// neighbour across edge n needs of this element, with the neighbour's sign
// of the normal.  Stage 2 then reads Qe values per edge and quantity instead
// of gathering the neighbour's N-vectors and projecting them again.
// CH ("chained"): x is the output of the preceding stage-2 launch, which
// left its x traces already (k_s2f epilogue): no projection of x at all here,
// the neighbours' contribution is Qe trace values per edge.
// tr = x traces [3][Q][Kp] (read if CH, written otherwise) | u traces [3][Q][Kp] at tr + utr_off.
template <int P, typename TT, bool CH>
__global__ void __launch_bounds__(128, CH ? kMinbS1c[P] : kMinbS1[P]) k_s1f(DevMesh m, DevTables T,
                                             const double* __restrict__ x, TT* __restrict__ tout,
                                             float* __restrict__ tr, long utr_off, int k0, int k1) {
  using RC = RankCfg<P>;
  constexpr int N = Cfg<P>::N, NF = Cfg<P>::NF, TAB = N * NF, Q = RC::Q, QF = RC::QF;
  extern __shared__ __align__(16) float smf[];
  const long Kp = m.Kp;
  const double* g = m.geom;
  const int kt = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  const int k = kt < k1 ? kt : k1 - 1;
  // the element's mesh data is launch-invariant: in flight across the table
  // staging and the dependency wait
  int kind[3], nb[3], nbn[3];
  float c1[3], c2[3];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    kind[n] = m.kind[n * Kp + k];
    nb[n] = m.nbr[n * Kp + k];
    nbn[n] = m.nbrn[n * Kp + k];
    const double hl = 0.5 * g[(kLen0 + n) * Kp + k];
    c1[n] = static_cast<float>(hl * g[(kNux0 + n) * Kp + k]);
    c2[n] = static_cast<float>(hl * g[(kNuy0 + n) * Kp + k]);
  }
  const float b11 = static_cast<float>(g[kB11 * Kp + k]), b12 = static_cast<float>(g[kB12 * Kp + k]);
  const float b21 = static_cast<float>(g[kB21 * Kp + k]), b22 = static_cast<float>(g[kB22 * Kp + k]);
  const float inv2a = static_cast<float>(1.0 / (2.0 * g[kArea * Kp + k]));
  stage_f2(smf, T.fbase + T.fmH, 2 * TAB, T.fbase + T.fR, RC::kFloats);
  const float* tb = smf;
  const float* s_R = smf + 2 * TAB;
  pdl_wait();
  pdl_trigger();
  if (kt >= k1) return;
  float2 u1[NF / 2], u2[NF / 2];
  {
    float2 w1[NF / 2], w2[NF / 2];
    float2 zo[3][QF / 2];  // own projections onto the three edges' points
#pragma unroll
    for (int c = 0; c < NF / 2; ++c) w1[c] = w2[c] = f2(0.f);
#pragma unroll
    for (int n = 0; n < 3; ++n)
#pragma unroll
      for (int c = 0; c < QF / 2; ++c) zo[n][c] = f2(0.f);
    // one pass over the element's x: both H products and (with traces) the three projections
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const float xj = static_cast<float>(x[j * Kp + k]);
      hier_acc<NF>(tb + j * NF, xj, w1, j);
      hier_acc<NF>(tb + TAB + j * NF, xj, w2, j);
      if (!CH && tr) {
#pragma unroll
        for (int n = 0; n < 3; ++n) rank_acc<QF>(s_R + RC::kPeT + (n * N + j) * QF, xj, zo[n]);
      }
    }
    if (!CH && tr) {
#pragma unroll
      for (int n = 0; n < 3; ++n)
#pragma unroll
        for (int q = 0; q < Q; ++q) tr[(n * Q + q) * Kp + k] = (q & 1) ? zo[n][q / 2].y : zo[n][q / 2].x;
    }
#pragma unroll
    for (int c = 0; c < NF / 2; ++c) {
      u1[c] = __ffma2_rn(f2(b21), w2[c], mul2(f2(-b22), w1[c]));
      u2[c] = __ffma2_rn(f2(-b11), w2[c], mul2(f2(b12), w1[c]));
    }
  }
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    // own side: nu |E| / 2 on interior edges, nu |E| on Neumann edges, none on Dirichlet edges
    const float fo = kind[n] == kInterior ? 1.f : (kind[n] == kNeumann ? 2.f : 0.f);
    if (fo == 0.f && nb[n] < 0) continue;
    float2 z[QF / 2];
#pragma unroll
    for (int c = 0; c < QF / 2; ++c) z[c] = f2(0.f);
    if (fo != 0.f) {
      if (tr) {  // the element's own x trace, just written
        float zq[QF];
#pragma unroll
        for (int q = 0; q < QF; ++q) zq[q] = q < Q ? fo * tr[(n * Q + q) * Kp + k] : 0.f;
#pragma unroll
        for (int c = 0; c < QF / 2; ++c) z[c] = make_float2(zq[2 * c], zq[2 * c + 1]);
      } else {
        const float* pT = s_R + RC::kPeT + n * N * QF;
#pragma unroll
        for (int j = 0; j < N; ++j) rank_acc<QF>(pT + j * QF, fo * static_cast<float>(x[j * Kp + k]), z);
      }
    }
    if (nb[n] >= 0) {
      const int kp = nb[n];
      if constexpr (CH) {  // the neighbour's x trace at the matching points (its edge runs the other way)
        const float* xt = tr + static_cast<long>(nbn[n]) * Q * Kp + kp;
        float zq[QF];
#pragma unroll
        for (int q = 0; q < QF; ++q) zq[q] = q < Q ? xt[(Q - 1 - q) * Kp] : 0.f;
#pragma unroll
        for (int c = 0; c < QF / 2; ++c) {
          z[c].x += zq[2 * c];
          z[c].y += zq[2 * c + 1];
        }
      } else {
        const float* tT = s_R + RC::kPthT + (n * 3 + nbn[n]) * N * QF;
#pragma unroll
        for (int j = 0; j < N; ++j) rank_acc<QF>(tT + j * QF, static_cast<float>(x[j * Kp + kp]), z);
      }
    }
    const float4* we4 = reinterpret_cast<const float4*>(s_R + RC::kWe);
#pragma unroll
    for (int c = 0; c < QF / 4; ++c) {
      const float4 w = we4[c];
      z[2 * c] = mul2(z[2 * c], make_float2(w.x, w.y));
      z[2 * c + 1] = mul2(z[2 * c + 1], make_float2(w.z, w.w));
    }
    float2 sv[NF / 2];
#pragma unroll
    for (int c = 0; c < NF / 2; ++c) sv[c] = f2(0.f);
    rank_out<Q, NF>(s_R + n * Q * NF, z, sv);
#pragma unroll
    for (int c = 0; c < NF / 2; ++c) {
      u1[c] = __ffma2_rn(f2(c1[n]), sv[c], u1[c]);
      u2[c] = __ffma2_rn(f2(c2[n]), sv[c], u2[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < NF / 2; ++c) {
    u1[c] = mul2(u1[c], f2(inv2a));
    u2[c] = mul2(u2[c], f2(inv2a));
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    tout[i * Kp + k] = static_cast<TT>((i & 1) ? u1[i / 2].y : u1[i / 2].x);
    tout[(N + i) * Kp + k] = static_cast<TT>((i & 1) ? u2[i / 2].y : u2[i / 2].x);
  }
  if (tr) {
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      float2 zu[QF / 2];
#pragma unroll
      for (int c = 0; c < QF / 2; ++c) zu[c] = f2(0.f);
      const float* pT = s_R + RC::kPeT + n * N * QF;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const float t1 = (j & 1) ? u1[j / 2].y : u1[j / 2].x, t2 = (j & 1) ? u2[j / 2].y : u2[j / 2].x;
        rank_acc<QF>(pT + j * QF, -fmaf(c1[n], t1, c2[n] * t2), zu);
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) tr[utr_off + (n * Q + q) * Kp + k] = (q & 1) ? zu[q / 2].y : zu[q / 2].x;
    }
  }
}

// d_h at the edge points of every element (per step and level): dtr[n][q][k] = sum_j peR_n[q][j] D[j][k]
template <int P>
__global__ void __launch_bounds__(128) k_dtrace(long Kp, int Kg, const float* __restrict__ peR,
                                                const double* __restrict__ D, float* __restrict__ dtr) {
  constexpr int N = Cfg<P>::N, NF = Cfg<P>::NF, Q = RankCfg<P>::Q;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= Kg) return;
  float dv[N];
  load_f<N>(D, Kp, k, dv);
#pragma unroll 1
  for (int nq = 0; nq < 3 * Q; ++nq) {
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fmaf(__ldg(peR + nq * NF + j), dv[j], s);
    dtr[nq * Kp + k] = s;
  }
}

// A quad of the packed stream: float4 (FP32 copy) or four FP16 values in a
// uint2 (E scaled per element into [-1, 1], written by k_bjac_warp, ldg_bjac.cu)
__device__ __forceinline__ float4 ld_quad(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ float4 ld_quad(const uint2* p) {
  const uint2 u = __ldcs(p);
  const float2 fa = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 fb = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  return make_float4(fa.x, fa.y, fb.x, fb.y);
}

// acc[i] += sum_j blk[i][j] v[j] over one column group: quad q of the group
// holds values u = 4q..4q+3, u = jj*N + i, column j0 + jj
template <int N, int QC, typename TQ>
__device__ __forceinline__ void group_mv(const TQ* __restrict__ g, long Kp, const float* v, float* acc) {
  float4 e[QC];
#pragma unroll
  for (int q = 0; q < QC; ++q) e[q] = ld_quad(g + q * Kp);
#pragma unroll
  for (int q = 0; q < QC; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int u = 4 * q + r;
      acc[u % N] = fmaf(comp(e[q], r), v[u / N], acc[u % N]);
    }
}

// acc += blk v for one packed N x N block (E^m_kk or P_k^-1, ldg_pack.cuh
// layout), v from `load(j)` (FP32 value of column j)
template <int P, typename TQ, typename F>
__device__ __forceinline__ void packed_apply(const TQ* __restrict__ blk, long Kp, F load, float* acc) {
  using C = Cfg<P>;
  constexpr int N = C::N, NN = C::NN;
  if constexpr (C::kFlat) {
    float r[N];
#pragma unroll
    for (int j = 0; j < N; ++j) r[j] = load(j);
#pragma unroll
    for (int q = 0; q < C::QP; ++q) {
      const float4 e = ld_quad(blk + q * Kp);
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int v = 4 * q + rr;
        if (v < NN) acc[v % N] = fmaf(comp(e, rr), r[v / N], acc[v % N]);
      }
    }
  } else {
#pragma unroll(C::UNR)
    for (int ch = 0; ch < C::NCH; ++ch) {
      float v[C::CC];
#pragma unroll
      for (int jj = 0; jj < C::CC; ++jj) {
        const int j = ch * C::CC + jj;
        v[jj] = (C::NCOL == N || j < N) ? load(j) : 0.f;
      }
      group_mv<N, C::QC, TQ>(blk + static_cast<long>(ch) * C::QC * Kp, Kp, v, acc);
    }
  }
}

// d = P^-1 r (FP32 packed, or FP16 packed times the element's scale)
template <int P, typename TQ, typename F>
__device__ __forceinline__ void pinv_apply(const TQ* __restrict__ Pk, long Kp, F load, float* d) {
#pragma unroll
  for (int i = 0; i < Cfg<P>::N; ++i) d[i] = 0.f;
  packed_apply<P, TQ>(Pk, Kp, load, d);
}

// r = b - [wm M x + dt (eta S x - sum_m E^m t^m)] on the element, then
//   MODE 0: out = r
//   MODE 1: out = x + omega P^-1 r        (one damped block-Jacobi sweep)
template <int P, int MODE, typename TQ, typename TP, typename TT>
__global__ void __launch_bounds__(128, kMinbS2[P]) k_s2f(DevMesh m, DevTables T, const TQ* __restrict__ Eq,
                                             const float* __restrict__ Escale, const double* __restrict__ D,
                                             const double* __restrict__ x,
                                             const TT* __restrict__ tz, const double* __restrict__ b, double wm,
                                             double dteta, double dt, const TP* __restrict__ Pq,
                                             const float* __restrict__ Pscale, float omega, double* out,
                                             double cheb_beta, int prev_zero, int k0, int k1,
                                             const float* __restrict__ tr, const float* __restrict__ utr,
                                             const float* __restrict__ dtr, float* __restrict__ xtr_out) {
  using C = Cfg<P>;
  using RC = RankCfg<P>;
  constexpr int N = C::N, NF = C::NF, Q = RC::Q, QF = RC::QF;
  extern __shared__ __align__(16) float smf[];
  const float* s_R = stage_f(smf, T.fbase + T.fR, RC::kFloats);  // peR | peT | pthT | weR
  __shared__ float s_r[MODE == 1 && !C::kFlat ? N : 1][128];  // the residual, for the grouped P^-1 stream
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  pdl_trigger();
  if (k >= k1) return;
  const long Kp = m.Kp;
  const double* g = m.geom;
  float acc[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) acc[i] = 0.f;
  const float fdt = static_cast<float>(dt), fdteta = static_cast<float>(dteta);
  // diagonal blocks E^m_kk t^m_k (packed stream), scaled copy
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    const TT* tc = tz + static_cast<long>(c) * N * Kp + k;
    packed_apply<P, TQ>(Eq + static_cast<long>(c) * C::QP * Kp + k, Kp,
                        [&](int j) { return static_cast<float>(tc[j * Kp]); }, acc);
  }
  {
    const float es = (Escale ? Escale[k] : 1.0f) * fdt;
    const float sm = static_cast<float>(-wm * 2.0 * g[kArea * Kp + k]);  // mass term, m_hat = I in FP32
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = fmaf(sm, static_cast<float>(x[i * Kp + k]), es * acc[i]);
  }
  // Everything that crosses edge n, in rank-Qe form with one product back:
  //   + dt   E^m_{k,kp} t^m_kp  (matrix-free from D, ldg_offdiag.cuh)   interior
  //   - dt eta s_diag_n x_k                                            interior, Dirichlet
  //   + dt eta s_offdiag_{n,np} x_kp                                   interior
  if constexpr (std::is_same<TT, float>::value && P >= kTraceMinP) {
    // single-rank levels: the traces stage 1 left at the edge points (the
    // neighbour's point q' = Qe - 1 - q: its edge runs the other way)
#pragma unroll 1
    for (int n = 0; n < 3; ++n) {
      const int kind = m.kind[n * Kp + k];
      const int kp = m.nbr[n * Kp + k];
      const bool pen = kind == kInterior || kind == kDirichlet;
      if (!pen && kp < 0) continue;
      float z[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) z[q] = pen ? -fdteta * tr[(n * Q + q) * Kp + k] : 0.f;
      if (kp >= 0) {
        const long at = static_cast<long>(m.nbrn[n * Kp + k]) * Q * Kp + kp;
        const float* xt = tr + at;
        const float* ut = utr + at;
        const float* dt_ = dtr + at;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const long o = static_cast<long>(Q - 1 - q) * Kp;
          z[q] = fmaf(fdteta, xt[o], fmaf(fdt * dt_[o], ut[o], z[q]));
        }
      }
      const float* we = s_R + RC::kWe;
#pragma unroll
      for (int q = 0; q < Q; ++q) z[q] *= we[q];
      float2* out2 = reinterpret_cast<float2*>(acc);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float2 vv = f2(z[q]);
        const float4* r4 = reinterpret_cast<const float4*>(s_R + (n * Q + q) * NF);
#pragma unroll
        for (int c = 0; c < NF / 4; ++c) {
          const float4 t = r4[c];
          out2[2 * c] = __ffma2_rn(make_float2(t.x, t.y), vv, out2[2 * c]);
          out2[2 * c + 1] = __ffma2_rn(make_float2(t.z, t.w), vv, out2[2 * c + 1]);
        }
      }
    }
  } else {
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kind = m.kind[n * Kp + k];
    const int kp = m.nbr[n * Kp + k];
    const bool pen = kind == kInterior || kind == kDirichlet;
    if (!pen && kp < 0) continue;
    float2 z[QF / 2];
#pragma unroll
    for (int c = 0; c < QF / 2; ++c) z[c] = f2(0.f);
    if (pen) {
      const float* pT = s_R + RC::kPeT + n * N * QF;
#pragma unroll
      for (int j = 0; j < N; ++j) rank_acc<QF>(pT + j * QF, static_cast<float>(x[j * Kp + k]), z);
#pragma unroll
      for (int c = 0; c < QF / 2; ++c) z[c] = mul2(z[c], f2(-fdteta));
    }
    if (kp >= 0) {
      const double hl = 0.5 * g[(kLen0 + n) * Kp + k];
      const float co1 = static_cast<float>(hl * g[(kNux0 + n) * Kp + k]);
      const float co2 = static_cast<float>(hl * g[(kNuy0 + n) * Kp + k]);
      const float* tT = s_R + RC::kPthT + (n * 3 + m.nbrn[n * Kp + k]) * N * QF;
      float2 dv[QF / 2], uv[QF / 2], xn[QF / 2];
#pragma unroll
      for (int c = 0; c < QF / 2; ++c) dv[c] = uv[c] = xn[c] = f2(0.f);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const float dj = static_cast<float>(D[j * Kp + kp]);
        const float uj =
            fmaf(co1, static_cast<float>(tz[j * Kp + kp]), co2 * static_cast<float>(tz[(N + j) * Kp + kp]));
        const float xj = static_cast<float>(x[j * Kp + kp]);
        const float4* r4 = reinterpret_cast<const float4*>(tT + j * QF);
#pragma unroll
        for (int c = 0; c < QF / 4; ++c) {
          const float4 t = r4[c];
          const float2 ta = make_float2(t.x, t.y), tb2 = make_float2(t.z, t.w);
          dv[2 * c] = __ffma2_rn(ta, f2(dj), dv[2 * c]);
          dv[2 * c + 1] = __ffma2_rn(tb2, f2(dj), dv[2 * c + 1]);
          uv[2 * c] = __ffma2_rn(ta, f2(uj), uv[2 * c]);
          uv[2 * c + 1] = __ffma2_rn(tb2, f2(uj), uv[2 * c + 1]);
          xn[2 * c] = __ffma2_rn(ta, f2(xj), xn[2 * c]);
          xn[2 * c + 1] = __ffma2_rn(tb2, f2(xj), xn[2 * c + 1]);
        }
      }
#pragma unroll
      for (int c = 0; c < QF / 2; ++c)
        z[c] = __ffma2_rn(f2(fdteta), xn[c], __ffma2_rn(mul2(f2(fdt), dv[c]), uv[c], z[c]));
    }
    const float4* we4 = reinterpret_cast<const float4*>(s_R + RC::kWe);
#pragma unroll
    for (int c = 0; c < QF / 4; ++c) {
      const float4 w = we4[c];
      z[2 * c] = mul2(z[2 * c], make_float2(w.x, w.y));
      z[2 * c + 1] = mul2(z[2 * c + 1], make_float2(w.z, w.w));
    }
    rank_out<Q, NF>(s_R + n * Q * NF, z, reinterpret_cast<float2*>(acc));
  }
  }
  if constexpr (MODE == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i * Kp + k] = b[i * Kp + k] + static_cast<double>(acc[i]);
  } else {
    float d[N];
    if constexpr (C::kFlat) {
      pinv_apply<P, TP>(Pq + k, Kp,
                        [&](int j) { return static_cast<float>(b[j * Kp + k] + static_cast<double>(acc[j])); }, d);
    } else {
      const int tid = threadIdx.x;
#pragma unroll
      for (int i = 0; i < N; ++i) s_r[i][tid] = static_cast<float>(b[i * Kp + k] + static_cast<double>(acc[i]));
      pinv_apply<P, TP>(Pq + k, Kp, [&](int j) { return s_r[j][tid]; }, d);
    }
    const float om = Pscale ? omega * Pscale[k] : omega;
    if (cheb_beta == 0.0) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double xn = fma(static_cast<double>(om), static_cast<double>(d[i]), x[i * Kp + k]);
        out[i * Kp + k] = xn;
        d[i] = static_cast<float>(xn);
      }
    } else {  // Chebyshev step: out (holding x_{k-1}, or 0) <- x + a P^-1 r + beta (x - x_{k-1})
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double xi = x[i * Kp + k], xp = prev_zero ? 0.0 : out[i * Kp + k];
        const double xn = fma(static_cast<double>(om), static_cast<double>(d[i]), fma(cheb_beta, xi - xp, xi));
        out[i * Kp + k] = xn;
        d[i] = static_cast<float>(xn);
      }
    }
    if constexpr (std::is_same<TT, float>::value && P >= kTraceMinP) {
      // the new x at the edge points, for the next sweep's stage 1 and stage 2 (the other
      // trace buffer: neighbours still read this sweep's)
      if (xtr_out) {
#pragma unroll 1
        for (int n = 0; n < 3; ++n) {
          float2 z[QF / 2];
#pragma unroll
          for (int c = 0; c < QF / 2; ++c) z[c] = f2(0.f);
          const float* pT = s_R + RC::kPeT + n * N * QF;
#pragma unroll
          for (int j = 0; j < N; ++j) rank_acc<QF>(pT + j * QF, d[j], z);
#pragma unroll
          for (int q = 0; q < Q; ++q) xtr_out[(n * Q + q) * Kp + k] = (q & 1) ? z[q / 2].y : z[q / 2].x;
        }
      }
    }
  }
}

// out = omega P^-1 b  (the first sweep from x = 0)
template <int P, typename TP>
__global__ void __launch_bounds__(128) k_bjf(int K, long Kp, const TP* __restrict__ Pq,
                                             const float* __restrict__ Pscale, const double* __restrict__ b,
                                             float omega, double* __restrict__ out) {
  constexpr int N = Cfg<P>::N;
  pdl_wait();
  pdl_trigger();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  float d[N];
  pinv_apply<P, TP>(Pq + k, Kp, [&](int j) { return static_cast<float>(b[j * Kp + k]); }, d);
  const float om = Pscale ? omega * Pscale[k] : omega;
#pragma unroll
  for (int i = 0; i < N; ++i) out[i * Kp + k] = static_cast<double>(om * d[i]);
}

template <int P>
size_t s1_smem() {
  return sizeof(float) * (2 * Cfg<P>::N * Cfg<P>::NF + RankCfg<P>::kFloats);
}
template <int P>
size_t s2_smem() {
  return sizeof(float) * RankCfg<P>::kFloats;
}

}  // namespace

int smooth_trace_min_p() { return kTraceMinP; }

long packed_p_quads(int p) {
  switch (p) {
    case 0: return Cfg<0>::QP;
    case 1: return Cfg<1>::QP;
    case 2: return Cfg<2>::QP;
    case 3: return Cfg<3>::QP;
    default: return Cfg<4>::QP;
  }
}

// Buffers of the FP16 copy of the level's diagonal E blocks for the big-level
// smoother, scaled per element into [-1, 1] (half the bytes of FP32 in the
// HBM-bound stage 2; FP32 copies measured slower in round 1 at equal iterations)
void smooth_pack_alloc(Handle& h) {
  if (h.Eh.ptr) return;
  h.Eh.alloc(2L * packed_p_quads(h.p) * h.Kp, &h.bytes);
  h.Escale.alloc(h.Kp, &h.bytes);
}

// d_h at the edge points for the trace-form smoother (per step; the FP16 copy of E
// itself, Eh / Escale, is written by the block-Jacobi setup from its staged blocks,
// ldg_bjac.cu)
void smooth_dtraces(Handle& h) {
#define CALL(P)                                                                                          \
  do {                                                                                                   \
    if (h.dtr32.ptr && P >= kTraceMinP) {                                                                \
      k_dtrace<P><<<grid_of(h.Kg, 128), 128, 0, h.stream>>>(h.Kp, h.Kg, h.dtab.fbase + h.dtab.fR, h.D.ptr, \
                                                            h.dtr32.ptr);                                \
      ++h.launches;                                                                                      \
    }                                                                                                    \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
}

// Trace buffers of a single-rank level (tr32): x traces A | u traces | x traces B,
// 3 Q planes each.  h.xtr_cur selects the x-trace buffer that belongs to the
// vector stage 1 is given; a MODE 1 stage 2 writes the other one and flips.
void smooth_stage1(Handle& h, const double* x, int k0, int k1, bool chained) {
  if (k1 < 0) k1 = h.K;
  if (k1 <= k0) return;
  const unsigned grid = grid_of(k1 - k0, 128);
#define CALL(P)                                                                                               \
  do {                                                                                                        \
    if (h.tz32.ptr) {                                                                                         \
      const long planes = 3L * RankCfg<P>::Q * h.Kp;                                                          \
      float* xt = (P >= kTraceMinP && h.tr32.ptr) ? h.tr32.ptr + (h.xtr_cur ? 2 * planes : 0) : nullptr;      \
      const long uoff = h.xtr_cur ? -planes : planes;                                                         \
      if (chained && xt)                                                                                      \
        launch_pdl(k_s1f<P, float, true>, grid, 128, s1_smem<P>(), h.stream, h.mesh(), h.dtab, x, h.tz32.ptr, \
                   xt, uoff, k0, k1);                                                                         \
      else                                                                                                    \
        launch_pdl(k_s1f<P, float, false>, grid, 128, s1_smem<P>(), h.stream, h.mesh(), h.dtab, x,            \
                   h.tz32.ptr, xt, uoff, k0, k1);                                                             \
    } else {                                                                                                  \
      launch_pdl(k_s1f<P, double, false>, grid, 128, s1_smem<P>(), h.stream, h.mesh(), h.dtab, x, h.tz.ptr,   \
                 static_cast<float*>(nullptr), 0L, k0, k1);                                                   \
    }                                                                                                         \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void smooth_stage2(Handle& h, int mode, const double* x, const double* b, double wm, double dt, double omega,
                   double* out, double cheb_beta, int prev_zero, int k0, int k1) {
  const double dteta = dt * h.prob.eta;
  const float om = static_cast<float>(omega);
  if (k1 < 0) k1 = h.K;
  if (k1 <= k0) return;
  const unsigned grid = grid_of(k1 - k0, 128);
  bool traced = false;
#define LAUNCH(P, M, TT, TZ)                                                                                      \
  do {                                                                                                            \
    const long planes = 3L * RankCfg<P>::Q * h.Kp;                                                                \
    const bool trp = P >= kTraceMinP && h.tr32.ptr && static_cast<const void*>(TZ) == h.tz32.ptr;                 \
    const float* xt = trp ? h.tr32.ptr + (h.xtr_cur ? 2 * planes : 0) : nullptr;                                  \
    float* xo = (trp && M == 1) ? h.tr32.ptr + (h.xtr_cur ? 0 : 2 * planes) : nullptr;                            \
    launch_pdl(k_s2f<P, M, uint2, uint2, TT>, grid, 128, s2_smem<P>(), h.stream, h.mesh(), h.dtab, h.Eh.ptr,      \
               h.Escale.ptr, h.D.ptr, x, TZ, b, wm, dteta, dt, h.Ph.ptr, h.Pscale.ptr, om, out, cheb_beta,        \
               prev_zero, k0, k1, xt, trp ? h.tr32.ptr + planes : nullptr, h.dtr32.ptr, xo);                      \
    traced = xo != nullptr;                                                                                       \
  } while (0)
#define CALL(P)                                           \
  do {                                                    \
    if (mode == 0 && h.tz32.ptr)                          \
      LAUNCH(P, 0, float, h.tz32.ptr);                    \
    else if (mode == 0)                                   \
      LAUNCH(P, 0, double, h.tz.ptr);                     \
    else if (h.tz32.ptr)                                  \
      LAUNCH(P, 1, float, h.tz32.ptr);                    \
    else                                                  \
      LAUNCH(P, 1, double, h.tz.ptr);                     \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
#undef LAUNCH
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
  if (traced) h.xtr_cur ^= 1;  // the x traces of `out` are in the other buffer
}

void smooth_zero(Handle& h, const double* b, double omega, double* out) {
#define CALL(P)                                                                                              \
  launch_pdl(k_bjf<P, uint2>, grid_of(h.K, 128), 128, 0, h.stream, h.K, h.Kp, h.Ph.ptr, h.Pscale.ptr, b,         \
             static_cast<float>(omega), out)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

}  // namespace ldgb
