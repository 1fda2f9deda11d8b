// Mixed-precision multigrid smoother kernels (the preconditioner's hot path).
//
// The V-cycle spends most of each implicit-Euler step in three operations per
// smoothing sweep on the large levels: t^m = M^-1 B^m x (stage 1), the
// residual r = b - S_c x (stage 2) and the damped block-Jacobi update
// x += omega P^-1 r.  Here they run in FP32 arithmetic on FP32 operator
// copies; vectors stay FP64 and the outer Krylov operator is untouched, so
// only the preconditioner's contraction depends on the rounding.
//
//  * Stored blocks are packed per element and streamed as float4: Eq[c][q][k]
//    holds values 4q..4q+3 of component c's four blocks in (slot, column, row)
//    order, so a warp moves 512 contiguous bytes per load instruction and the
//    quarter as many load instructions as the FP32 scalar layout issues.
//    P^-1 is packed the same way (column-major, NN rounded up to 4).
//  * Stage 2 and the block-Jacobi update are one kernel: the residual of the
//    element never leaves registers (ping-pong x_in -> x_out, since stage 2
//    reads the neighbours' x).
//  * The reference tables live in shared memory as FP32 rows of NF = N
//    rounded to 4 (one 128-bit broadcast load per 4 entries).
//
// Reference operators restated (as in ldg_apply.cu): B^m = -H^m + Q^m + Q_N^m
// (assembly.hpp:92-109, 174-208), S + S_D (assembly.hpp:142-168), M = 2|T| mhat.
#include <cuda_fp16.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "ldg_internal.hpp"
#include "ldg_pack.cuh"
#include "ldg_offdiag.cuh"

// min resident CTAs per SM of the thread-per-element kernels, per degree
// p = 0..4 (stage 1 | stage 2).  The level-0 grids are 1024 CTAs of 128
// (256^2 FK): 7-8 CTAs/SM (<= 73 / 64 registers, a few spilled bytes) run
// them in one wave: V-cycle -13% at p = 2 and -14% at p = 3 (stage 2 at 7,
// stage 1 at 8: 0.515 / 0.764 ms against 0.600 / 0.883 ms with 1 CTA).  At
// p = 4 stage 2 at 7 CTAs (72 registers, 48 bytes spilled) runs the level in
// one wave: V-cycle 1557 -> 1435 us, step 38.4 -> 36.2 ms (5 and 6 CTAs,
// 96 / 80 registers without spills, stay at two waves and were 1-2 % slower
// than 4; 8 CTAs spill more: +6 %).  Stage 1 at p = 4 stays at 4 CTAs: 6, 7,
// 8 CTAs (also with one neighbour at a time, LDG_S1_SEQ_P) measured
// +3 / +7 / +16 % V-cycle.  8 at p <= 1 measured slower.
// -DLDG_MINB_S1=abcde / -DLDG_MINB_S2=abcde (one digit per p = 0..4)
// override (tuning builds).
#ifndef LDG_MINB_S1
#define LDG_MINB_S1 11884
#endif
#ifndef LDG_MINB_S2
#define LDG_MINB_S2 11777
#endif

namespace ldgb {

namespace {

constexpr int minb_digit(int code, int p) { return p == 4 ? code % 10 : minb_digit(code / 10, p + 1); }
constexpr int kMinbS1[5] = {minb_digit(LDG_MINB_S1, 0), minb_digit(LDG_MINB_S1, 1), minb_digit(LDG_MINB_S1, 2),
                            minb_digit(LDG_MINB_S1, 3), minb_digit(LDG_MINB_S1, 4)};
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

// tout^m = M_k^-1 B^m x (both m), FP32 arithmetic, FP64 in/out
template <int P, typename TT>
__global__ void __launch_bounds__(128, kMinbS1[P]) k_s1f(DevMesh m, DevTables T, const double* __restrict__ x,
                                             TT* __restrict__ tout, int k0, int k1) {
  constexpr int N = Cfg<P>::N, NF = Cfg<P>::NF, TAB = N * NF;
  extern __shared__ __align__(16) float smf[];
  const float* tb = stage_f(smf, T.fbase + T.fmH, 14 * TAB);  // tmH 2 | tmSd 3 | tmSo 9
  pdl_wait();
  pdl_trigger();
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  const long Kp = m.Kp;
  const double* g = m.geom;
  float xv[N], w[N], u1[N], u2[N];
  load_f<N>(x, Kp, k, xv);
  const float b11 = static_cast<float>(g[kB11 * Kp + k]), b12 = static_cast<float>(g[kB12 * Kp + k]);
  const float b21 = static_cast<float>(g[kB21 * Kp + k]), b22 = static_cast<float>(g[kB22 * Kp + k]);
  ftab_mv<N, NF>(tb, xv, w);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    u1[i] = -b22 * w[i];
    u2[i] = b12 * w[i];
  }
  ftab_mv<N, NF>(tb + TAB, xv, w);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    u1[i] = fmaf(b21, w[i], u1[i]);
    u2[i] = fmaf(-b11, w[i], u2[i]);
  }
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kind = m.kind[n * Kp + k];
    const double len = g[(kLen0 + n) * Kp + k];
    const double f = kind == kInterior ? 0.5 * len : (kind == kNeumann ? len : 0.0);
    if (f == 0.0) continue;
    ftab_mv<N, NF>(tb + (2 + n) * TAB, xv, w);
    const float c1 = static_cast<float>(f * g[(kNux0 + n) * Kp + k]);
    const float c2 = static_cast<float>(f * g[(kNuy0 + n) * Kp + k]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      u1[i] = fmaf(c1, w[i], u1[i]);
      u2[i] = fmaf(c2, w[i], u2[i]);
    }
  }
  // the neighbours' x: every load issued before the products (one latency
  // round instead of one per neighbour; one neighbour at a time at 6-8 CTAs
  // per SM measured 3-16 % slower at p = 4)
  int nb[3], nbn[3];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    nb[n] = m.nbr[n * Kp + k];
    nbn[n] = m.nbrn[n * Kp + k];
  }
  float xn[3][N];
#pragma unroll
  for (int n = 0; n < 3; ++n)
#pragma unroll
    for (int j = 0; j < N; ++j) xn[n][j] = nb[n] >= 0 ? static_cast<float>(x[j * Kp + nb[n]]) : 0.f;
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    if (nb[n] < 0) continue;
    ftab_mv<N, NF>(tb + (5 + n * 3 + nbn[n]) * TAB, xn[n], w);
    const double hl = 0.5 * g[(kLen0 + n) * Kp + k];
    const float c1 = static_cast<float>(hl * g[(kNux0 + n) * Kp + k]);
    const float c2 = static_cast<float>(hl * g[(kNuy0 + n) * Kp + k]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      u1[i] = fmaf(c1, w[i], u1[i]);
      u2[i] = fmaf(c2, w[i], u2[i]);
    }
  }
  const float inv2a = static_cast<float>(1.0 / (2.0 * g[kArea * Kp + k]));
#pragma unroll
  for (int i = 0; i < N; ++i) {
    tout[i * Kp + k] = static_cast<TT>(inv2a * u1[i]);
    tout[(N + i) * Kp + k] = static_cast<TT>(inv2a * u2[i]);
  }
}

// A quad of the packed stream: float4 (FP32 copy) or four FP16 values in a
// uint2 (E scaled per element into [-1, 1], ldg_smooth.cu k_pack_e)
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
                                             double cheb_beta, int prev_zero, int k0, int k1) {
  using C = Cfg<P>;
  constexpr int N = C::N, NF = C::NF, TAB = N * NF;
  constexpr int Q = C::Q;
  extern __shared__ __align__(16) float smf[];
  // tM | tSd 3 | tSo 9 | pe 3 | pth 9 | we (contiguous in the FP32 table buffer)
  const float* tb = stage_f(smf, T.fbase + T.fM, 13 * TAB + C::EDGE);
  const float* s_pe = tb + 13 * TAB;
  const float* s_pth = s_pe + 3 * Q * N;
  const float* s_we = s_pth + 9 * Q * N;
  __shared__ float s_r[MODE == 1 && !C::kFlat ? N : 1][128];  // the residual, for the grouped P^-1 stream
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  pdl_trigger();
  if (k >= k1) return;
  const long Kp = m.Kp;
  const double* g = m.geom;
  float acc[N];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = 0.f;
  // diagonal blocks E^m_kk t^m_k (packed stream), scaled copy
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    const TT* tc = tz + static_cast<long>(c) * N * Kp + k;
    packed_apply<P, TQ>(Eq + static_cast<long>(c) * C::QP * Kp + k, Kp,
                        [&](int j) { return static_cast<float>(tc[j * Kp]); }, acc);
  }
  if (Escale) {
    const float es = Escale[k];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] *= es;
  }
  // off-diagonal blocks, matrix-free from D (ldg_offdiag.cuh)
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kp = m.nbr[n * Kp + k];
    if (kp < 0) continue;
    const double hl = 0.5 * g[(kLen0 + n) * Kp + k];
    const float co1 = static_cast<float>(hl * g[(kNux0 + n) * Kp + k]);
    const float co2 = static_cast<float>(hl * g[(kNuy0 + n) * Kp + k]);
    float z[Q];
    offdiag_z<N, Q, float>(
        s_pth + (n * 3 + m.nbrn[n * Kp + k]) * Q * N, s_we, [&](int j) { return static_cast<float>(D[j * Kp + kp]); },
        [&](int j) {
          return fmaf(co1, static_cast<float>(tz[j * Kp + kp]), co2 * static_cast<float>(tz[(N + j) * Kp + kp]));
        },
        z);
    offdiag_rows<N, Q, float>(s_pe + n * Q * N, z, 1.0f, acc);
  }
  const float fdt = static_cast<float>(dt), fdteta = static_cast<float>(dteta);
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] *= fdt;
  {
    float xv[N], w[N];
    load_f<N>(x, Kp, k, xv);
    ftab_mv<N, NF>(tb, xv, w);
    const float sm = static_cast<float>(-wm * 2.0 * g[kArea * Kp + k]);
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = fmaf(sm, w[i], acc[i]);
#pragma unroll 1
    for (int n = 0; n < 3; ++n) {
      const int kind = m.kind[n * Kp + k];
      if (kind != kInterior && kind != kDirichlet) continue;
      ftab_mv<N, NF>(tb + (1 + n) * TAB, xv, w);
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = fmaf(-fdteta, w[i], acc[i]);
    }
  }
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kp = m.nbr[n * Kp + k];
    if (kp < 0) continue;
    float xn[N], w[N];
    load_f<N>(x, Kp, kp, xn);
    ftab_mv<N, NF>(tb + (4 + n * 3 + m.nbrn[n * Kp + k]) * TAB, xn, w);
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = fmaf(fdteta, w[i], acc[i]);
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
      for (int i = 0; i < N; ++i)
        out[i * Kp + k] = fma(static_cast<double>(om), static_cast<double>(d[i]), x[i * Kp + k]);
    } else {  // Chebyshev step: out (holding x_{k-1}, or 0) <- x + a P^-1 r + beta (x - x_{k-1})
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double xi = x[i * Kp + k], xp = prev_zero ? 0.0 : out[i * Kp + k];
        out[i * Kp + k] = fma(static_cast<double>(om), static_cast<double>(d[i]), fma(cheb_beta, xi - xp, xi));
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

// FP16 packed copy of the diagonal blocks E[(c*NN + i*N + j)][k] (FP64),
// one thread per element: pass 1 the element's scale max |E| over its two
// blocks, pass 2 the quads of ldg_pack.cuh (slot v -> (i, j), zero padding)
// as 8-byte stores, each pass a coalesced sweep over the 2 N^2 planes.
// (Was two kernels, a per-element max and one thread per FP16 value with
// 2-byte scattered stores: 68 + 264 us at p = 4, 256^2.)
template <int P>
__global__ void __launch_bounds__(128) k_pack_eh(long Kp, const double* __restrict__ E, float* __restrict__ scale,
                                                 uint2* __restrict__ Eq) {
  using C = Cfg<P>;
  constexpr int N = C::N, NN = C::NN;
  const long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (k >= Kp) return;
  double mx = 0.0;
#pragma unroll 8
  for (int v = 0; v < 2 * NN; ++v) mx = fmax(mx, fabs(E[v * Kp + k]));
  const float sc = mx > 0.0 ? static_cast<float>(mx) : 1.0f;
  scale[k] = sc;
  const float inv = 1.0f / sc;
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
#pragma unroll 4
    for (int q = 0; q < C::QP; ++q) {
      __half hv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int v = 4 * q + r;
        int i, j;
        bool ok;
        if constexpr (C::kFlat) {
          j = v / N;
          i = v % N;
          ok = v < NN;
        } else {
          const int g = v / (C::QC * 4), w = v % (C::QC * 4);
          j = g * C::CC + w / N;
          i = w % N;
          ok = j < N;
        }
        const float val = ok ? static_cast<float>(E[(static_cast<long>(c) * NN + i * N + j) * Kp + k]) : 0.0f;
        hv[r] = __float2half_rn(val * inv);
      }
      uint2 u;
      u.x = static_cast<unsigned>(__half_as_ushort(hv[0])) | (static_cast<unsigned>(__half_as_ushort(hv[1])) << 16);
      u.y = static_cast<unsigned>(__half_as_ushort(hv[2])) | (static_cast<unsigned>(__half_as_ushort(hv[3])) << 16);
      Eq[(static_cast<long>(c) * C::QP + q) * Kp + k] = u;
    }
  }
}

template <int P>
size_t s1_smem() {
  return sizeof(float) * 14 * Cfg<P>::N * Cfg<P>::NF;
}
template <int P>
size_t s2_smem() {
  return sizeof(float) * (13 * Cfg<P>::N * Cfg<P>::NF + Cfg<P>::EDGE);
}

}  // namespace

long packed_p_quads(int p) {
  switch (p) {
    case 0: return Cfg<0>::QP;
    case 1: return Cfg<1>::QP;
    case 2: return Cfg<2>::QP;
    case 3: return Cfg<3>::QP;
    default: return Cfg<4>::QP;
  }
}

// FP16 copy of the level's diagonal E blocks for the big-level smoother,
// scaled per element into [-1, 1] (half the bytes of FP32 in the HBM-bound
// stage 2; FP32 copies measured slower in round 1 at equal iterations)
void smooth_pack_e(Handle& h) {
#define CALL(P)                                                                                          \
  do {                                                                                                   \
    const long nq = 2L * Cfg<P>::QP * h.Kp;                                                              \
    if (!h.Eh.ptr) {                                                                                     \
      h.Eh.alloc(nq, &h.bytes);                                                                          \
      h.Escale.alloc(h.Kp, &h.bytes);                                                                    \
    }                                                                                                    \
    k_pack_eh<P><<<grid_of(h.Kp, 128), 128, 0, h.stream>>>(h.Kp, h.E.ptr, h.Escale.ptr, h.Eh.ptr);       \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void smooth_stage1(Handle& h, const double* x, int k0, int k1) {
  if (k1 < 0) k1 = h.K;
  if (k1 <= k0) return;
  const unsigned grid = grid_of(k1 - k0, 128);
#define CALL(P)                                                                                               \
  do {                                                                                                        \
    if (h.tz32.ptr)                                                                                           \
      launch_pdl(k_s1f<P, float>, grid, 128, s1_smem<P>(), h.stream, h.mesh(), h.dtab, x, h.tz32.ptr, k0, k1); \
    else                                                                                                      \
      launch_pdl(k_s1f<P, double>, grid, 128, s1_smem<P>(), h.stream, h.mesh(), h.dtab, x, h.tz.ptr, k0, k1); \
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
#define LAUNCH(P, M, TT, TZ)                                                                                      \
  launch_pdl(k_s2f<P, M, uint2, uint2, TT>, grid, 128, s2_smem<P>(), h.stream, h.mesh(), h.dtab, h.Eh.ptr,        \
             h.Escale.ptr, h.D.ptr, x, TZ, b, wm, dteta, dt, h.Ph.ptr, h.Pscale.ptr, om, out, cheb_beta, prev_zero, \
             k0, k1)
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
