// Block-Jacobi setup of the Schur operator, once per step and level
// (diagonal E blocks stored, off-diagonal ones matrix-free from D, E_D here).
//
//   P_k = wm M_k + dt (eta S_kk - sum_m sum_{j in {k} u nbr(k)} E^m_kj M_j^-1 B^m_jk)
//
// and its inverse, one N x N block per element.  M_j^-1 B^m_jk is a linear
// combination of the m_hat^-1-premultiplied reference tables (ldg_tables.cpp
// tmH, tmSd, tmSo) with per-element scalars, so the 8 block products fold
// into 8 "combined E x table" products: the diagonal slot mixes E^1, E^2 into
// one matrix per table (H^1, H^2, S_diag x3), each off-diagonal slot into one
// matrix against its S_off table.  Static blocks as in assembly.hpp:76-208;
// the reference itself has no preconditioner (system.hpp:190-205 factorises).
//
// Shape: a group of NG = N rounded up to a power of two lanes per element
// (2 elements per warp at p = 3, 4), lane i holding row i of P and of the
// augmented identity in registers; the tables sit in shared memory and are
// read as broadcasts.  Gauss-Jordan with partial pivoting without row swaps:
// the pivot row of each column is chosen among the rows not yet used and
// broadcast through shared memory; the lane that pivoted column c holds row c
// of P^-1 at the end.
#include <cuda_fp16.h>

#include <cmath>

#include "ldg_internal.hpp"
#include "ldg_pack.cuh"

namespace ldgb {

namespace {

template <int P>
struct Cfg {
  static constexpr int N = (P + 1) * (P + 2) / 2;
  static constexpr int NN = N * N;
  static constexpr int NP = (N % 2) ? N + 1 : N;
  static constexpr int NNP = N * NP;
  static constexpr int NG = N <= 1 ? 1 : (N <= 2 ? 2 : (N <= 4 ? 4 : (N <= 8 ? 8 : 16)));
  static constexpr int EPW = 32 / NG;  // elements per warp
  static constexpr int WARPS = 8;
  static constexpr int EPB = EPW * WARPS;
  static constexpr int Q = (3 * P + 2) / 2;  // edge rule of the off-diagonal E blocks
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

// OUT: 0 FP64 SoA, 1 FP32 SoA, 3 FP16 packed (ldg_pack.cuh)
// scaled per element.  S: the arithmetic of the products and the elimination
// -- FP32 for the FP16 smoother copy (OUT 3: the result is rounded to 11
// bits anyway; FP32 issues twice the FMAs per cycle and holds half the
// registers), FP64 otherwise.
// The block's diagonal E blocks are staged in shared memory first (one
// coalesced 128-byte segment per plane and 16 elements, every load of the
// block in flight at once): read straight from HBM by row-lanes of different
// elements, the 2 N^2 loads per lane touched a sector each (k_bjac_warp<4>
// was L1-bound at 1.44 ms for 518 MB).  The edge tables sit in shared memory
// too, and the neighbour's d_h at the edge points (Q dot products of length
// N) is computed once per element instead of once per row-lane.
// a[jj] += e * row[jj], jj < N, row 16-byte aligned in shared memory
template <typename S, int N, int NJ>
__device__ __forceinline__ void row_fma(const S* row, S e, S* a) {
  if constexpr (sizeof(S) == 4) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll
    for (int q = 0; q < NJ / 4; ++q) {
      const float4 v = r4[q];
      if (4 * q < N) a[4 * q] = fmaf(e, v.x, a[4 * q]);
      if (4 * q + 1 < N) a[4 * q + 1] = fmaf(e, v.y, a[4 * q + 1]);
      if (4 * q + 2 < N) a[4 * q + 2] = fmaf(e, v.z, a[4 * q + 2]);
      if (4 * q + 3 < N) a[4 * q + 3] = fmaf(e, v.w, a[4 * q + 3]);
    }
  } else {
    const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
    for (int q = 0; q < NJ / 2; ++q) {
      const double2 v = r2[q];
      if (2 * q < N) a[2 * q] = fma(e, v.x, a[2 * q]);
      if (2 * q + 1 < N) a[2 * q + 1] = fma(e, v.y, a[2 * q + 1]);
    }
  }
}

// the same for the first `lim` entries only (compile-time after unrolling)
template <typename S, int NJ>
__device__ __forceinline__ void row_fma_lim(const S* row, S e, S* a, int lim) {
  constexpr int VW = 16 / sizeof(S);
#pragma unroll
  for (int q = 0; q < NJ / VW; ++q) {
    if (q * VW >= lim) continue;
    if constexpr (sizeof(S) == 4) {
      const float4 v = reinterpret_cast<const float4*>(row)[q];
      if (4 * q < lim) a[4 * q] = fmaf(e, v.x, a[4 * q]);
      if (4 * q + 1 < lim) a[4 * q + 1] = fmaf(e, v.y, a[4 * q + 1]);
      if (4 * q + 2 < lim) a[4 * q + 2] = fmaf(e, v.z, a[4 * q + 2]);
      if (4 * q + 3 < lim) a[4 * q + 3] = fmaf(e, v.w, a[4 * q + 3]);
    } else {
      const double2 v = reinterpret_cast<const double2*>(row)[q];
      if (2 * q < lim) a[2 * q] = fma(e, v.x, a[2 * q]);
      if (2 * q + 1 < lim) a[2 * q + 1] = fma(e, v.y, a[2 * q + 1]);
    }
  }
}

template <int P, typename S>
struct BjacSmem {
  using C = Cfg<P>;
  static constexpr int EPAD = 2 * C::NN + 1;  // odd row: conflict-free row-lane reads
  static constexpr int EDGE = 12 * C::Q * C::N + C::Q;
  static constexpr size_t bytes() { return sizeof(S) * (static_cast<size_t>(C::EPB) * EPAD + EDGE); }
};

template <int P, int OUT, typename S = double>
__global__ void __launch_bounds__(256) k_bjac_warp(DevMesh m, DevTables T, const double* __restrict__ E,
                                                   const double* __restrict__ E_D, double wm, double dt, double eta,
                                                   void* __restrict__ out, float* __restrict__ out_scale,
                                                   uint2* __restrict__ Eq, float* __restrict__ Escale) {
  using C = Cfg<P>;
  using SM = BjacSmem<P, S>;
  constexpr int N = C::N, NN = C::NN, NP = C::NP, NNP = C::NNP, NG = C::NG, Q = C::Q;
  // tmH 2 | tmSd 3 | tmSo 9 transposed to [t][q][jj] rows of NJ (vector loads
  // over jj: one 128-bit broadcast load per 4 (FP32) / 2 (FP64) FMAs instead
  // of a scalar load per FMA -- the kernel was issue-bound on them)
  constexpr int VW = 16 / sizeof(S), NJ = (N + VW - 1) / VW * VW, TJ = N * NJ;
  __shared__ __align__(16) S s_tab[14 * TJ];
  __shared__ S s_piv[C::WARPS][C::EPW][2 * N + 2];
  __shared__ __align__(16) S s_g2[9 * Q * NJ];  // bjG2 [n*3+np][q][jj], rows of NJ
  extern __shared__ __align__(16) unsigned char bjac_smem[];
  S* s_E = reinterpret_cast<S*>(bjac_smem);     // [EPB][EPAD]: E^1_kk | E^2_kk rows of the block's elements
  S* s_pe = s_E + C::EPB * SM::EPAD;            // U^t [n][q][N]
  S* s_pth = s_pe + 3 * Q * N;                  // V^t [n][np][q][N]
  S* s_we = s_pth + 9 * Q * N;                  // [Q]
  const long Kp = m.Kp;
  const int kb = blockIdx.x * C::EPB;
  for (int x = threadIdx.x; x < 14 * TJ; x += blockDim.x) {
    const int t = x / TJ, q = (x % TJ) / NJ, jj = x % NJ;  // Tab_t[q][jj] = stored transpose [jj][q]
    s_tab[x] = jj < N ? static_cast<S>(T.base[T.tmH + t * NNP + jj * NP + q]) : S(0);
  }
  for (int x = threadIdx.x; x < 9 * Q * NJ; x += blockDim.x) {
    const int eq = x / NJ, jj = x % NJ;
    s_g2[x] = jj < N ? static_cast<S>(T.base[T.bjG2 + eq * N + jj]) : S(0);
  }
  for (int t = threadIdx.x; t < 3 * Q * N; t += blockDim.x) s_pe[t] = static_cast<S>(T.base[T.pe + t]);
  for (int t = threadIdx.x; t < 9 * Q * N; t += blockDim.x) s_pth[t] = static_cast<S>(T.base[T.pth + t]);
  for (int t = threadIdx.x; t < Q; t += blockDim.x) s_we[t] = static_cast<S>(T.base[T.we + t]);
  {
    // 8 loads in flight per thread (a rolled loop issued them one latency at a time)
    constexpr int TOT = 2 * NN * C::EPB, B = 8;
    for (int t0 = threadIdx.x; t0 < TOT; t0 += B * 256) {
      double vals[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int t = t0 + b * 256, v = t / C::EPB, e = t % C::EPB, ke = kb + e;
        vals[b] = (t < TOT && ke < m.K) ? __ldg(E + static_cast<long>(v) * Kp + ke) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int t = t0 + b * 256, v = t / C::EPB, e = t % C::EPB;
        if (t < TOT) s_E[e * SM::EPAD + v] = static_cast<S>(vals[b]);
      }
    }
  }
  __syncthreads();
  if constexpr (OUT == 3) {
    // The smoother's FP16 copy of the diagonal E blocks (ldg_pack.cuh quads, scaled per
    // element into [-1, 1]) leaves from the staged block: the same values the separate
    // packing kernel produced from a second and third pass over E (k_pack_eh: 183 us at
    // p = 4, 256^2), written as coalesced 8-byte stores, 16+ consecutive elements per plane.
    if (Eq) {
      using PC = SmCfg<P>;
      __shared__ float s_sc[C::EPB];
      constexpr int LPE = 256 / C::EPB;  // lanes per element (1 .. 16), consecutive threads
      {
        const int e = threadIdx.x / LPE, l = threadIdx.x % LPE;
        float mx = 0.f;
        for (int v = l; v < 2 * NN; v += LPE) mx = fmaxf(mx, fabsf(static_cast<float>(s_E[e * SM::EPAD + v])));
#pragma unroll
        for (int o = LPE / 2; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (l == 0) {
          const float sc = mx > 0.f ? mx : 1.0f;
          s_sc[e] = sc;
          if (kb + e < m.K) Escale[kb + e] = sc;
        }
      }
      __syncthreads();
      for (int t = threadIdx.x; t < 2 * PC::QP * C::EPB; t += 256) {
        const int plane = t / C::EPB, e = t % C::EPB, ke = kb + e;
        if (ke >= m.K) continue;
        const int c = plane / PC::QP, q = plane % PC::QP;
        const float inv = 1.0f / s_sc[e];
        __half hv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int v = 4 * q + r;
          int ii, jj;
          bool ok;
          if constexpr (PC::kFlat) {
            jj = v / N;
            ii = v % N;
            ok = v < NN;
          } else {
            const int gq = v / (PC::QC * 4), w = v % (PC::QC * 4);
            jj = gq * PC::CC + w / N;
            ii = w % N;
            ok = jj < N;
          }
          const float val = ok ? static_cast<float>(s_E[e * SM::EPAD + c * NN + ii * N + jj]) : 0.0f;
          hv[r] = __float2half_rn(val * inv);
        }
        uint2 u;
        u.x = static_cast<unsigned>(__half_as_ushort(hv[0])) | (static_cast<unsigned>(__half_as_ushort(hv[1])) << 16);
        u.y = static_cast<unsigned>(__half_as_ushort(hv[2])) | (static_cast<unsigned>(__half_as_ushort(hv[3])) << 16);
        Eq[(static_cast<long>(c) * PC::QP + q) * Kp + ke] = u;
      }
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / NG, i = lane % NG;
  const int el = warp * C::EPW + sub;
  const int k = kb + el;
  const bool live = k < m.K;
  const bool row = live && i < N;
  const int kk = live ? k : 0;
  const double* g = m.geom;
  const double* tb = T.base;
  const unsigned gmask = (NG == 32 ? 0xffffffffu : ((1u << NG) - 1u) << (NG * sub));  // this element's lanes

  // a[jj] = row i of P_k
  S a[N];
  const int ir = row ? i : 0;
  {
    const double two_a = 2.0 * g[kArea * Kp + kk];
    int kind[3];
#pragma unroll
    for (int n = 0; n < 3; ++n) kind[n] = m.kind[n * Kp + kk];
#pragma unroll
    for (int jj = 0; jj < N; ++jj) {
      double s = 0.0;
#pragma unroll
      for (int n = 0; n < 3; ++n)
        if (kind[n] == kInterior || kind[n] == kDirichlet) s += tb[T.sdiag + (ir * N + jj) * 3 + n];
      a[jj] = static_cast<S>(wm * two_a * tb[T.mhat + ir * N + jj] + dt * eta * s);
    }
  }
  // a -= dt sum E (M^-1 B), as combined-E rows against the tables:
  // a[jj] += sum_q e_t[q] Tab_t[q][jj] with Tab_t^t[jj][q] at jj*NP + q
  {
    // diagonal slot: E^1_k0, E^2_k0 against H^1, H^2, S_diag x3 (k's own geometry)
    const double inv2a = 1.0 / (2.0 * g[kArea * Kp + kk]);
    const double b11 = g[kB11 * Kp + kk], b12 = g[kB12 * Kp + kk], b21 = g[kB21 * Kp + kk], b22 = g[kB22 * Kp + kk];
    // B^1_kk = -(b22 H1 - b21 H2) + sum_n f_n nu^x_n |E_n| S_d,n;  B^2_kk = -(b11 H2 - b12 H1) + ... nu^y
    double c1d[5], c2d[5];  // coefficients of (tmH1, tmH2, tmSd0..2) for E^1 and E^2, with -dt and 1/(2|T|)
    const double sc = -dt * inv2a;
    c1d[0] = -b22 * sc;
    c1d[1] = b21 * sc;
    c2d[0] = b12 * sc;
    c2d[1] = -b11 * sc;
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      const int kd = m.kind[n * Kp + kk];
      const double f = kd == kInterior ? 0.5 : (kd == kNeumann ? 1.0 : 0.0);
      const double fl = f * g[(kLen0 + n) * Kp + kk] * sc;
      c1d[2 + n] = fl * g[(kNux0 + n) * Kp + kk];
      c2d[2 + n] = fl * g[(kNuy0 + n) * Kp + kk];
    }
    S c1[5], c2[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      c1[t] = static_cast<S>(c1d[t]);
      c2[t] = static_cast<S>(c2d[t]);
    }
    const S* erow = s_E + el * SM::EPAD + ir * N;
    if (T.rank_ok) {
      // h_hat(q, jj, m) = 0 unless deg phi_q > deg phi_jj (hierarchical basis): only the
      // columns below the first function of degree deg(q) are touched (28 of 60 chunks at p = 4)
#pragma unroll
      for (int q = 1; q < N; ++q) {
        const S e1 = erow[q];
        const S e2 = erow[NN + q];
        int dq = 0;
        while ((dq + 1) * (dq + 2) / 2 <= q) ++dq;
        const int lim = dq * (dq + 1) / 2;  // jj < lim
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const S e = c1[t] * e1 + c2[t] * e2;
          row_fma_lim<S, NJ>(s_tab + t * TJ + q * NJ, e, a, lim);
        }
      }
    }
#pragma unroll 1
    for (int q = 0; q < N; ++q) {
      const S e1 = erow[q];
      const S e2 = erow[NN + q];
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        if (t < 2 && T.rank_ok) continue;
        const S e = c1[t] * e1 + c2[t] * e2;
        row_fma<S, N, NJ>(s_tab + t * TJ + q * NJ, e, a);
      }
    }
    // off-diagonal slots: E^m_{k,j} against M_j^-1 B^m_{j,k} = (nu^m_j |E_j| / (4 |T_j|)) s_off(np, n).
    // E^m_{k,j} = co_m U diag(wd) V^T is matrix-free (ldg_offdiag.cuh): row i of
    // cx E^1 + cy E^2 is kappa sum_q U[i][q] wd[q] V[:, q], kappa = cx co_1 + cy co_2
#pragma unroll 1
    for (int s = 1; s < 4; ++s) {
      const int j = m.nbr[(s - 1) * Kp + kk];
      if (j < 0) continue;  // uniform over the element's lanes
      const int n = s - 1, np = m.nbrn[n * Kp + kk];
      const double h = -dt * 0.5 * g[(kLen0 + np) * Kp + j] / (2.0 * g[kArea * Kp + j]);
      const double cx = h * g[(kNux0 + np) * Kp + j], cy = h * g[(kNuy0 + np) * Kp + j];
      const double hl = 0.5 * g[(kLen0 + n) * Kp + kk];
      const double kappa = hl * (cx * g[(kNux0 + n) * Kp + kk] + cy * g[(kNuy0 + n) * Kp + kk]);
      const S* pth = s_pth + (n * 3 + np) * Q * N;  // V^t [q][.]
      const S* pe = s_pe + n * Q * N;               // U^t [q][.]
      // lane q < Q of the element: the neighbour's d_h at edge point q
      S dq = 0;
      if (i < Q) {
#pragma unroll
        for (int l = 0; l < N; ++l) dq = fma(static_cast<S>(E_D[l * Kp + j]), pth[i * N + l], dq);
      }
      S aq[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const S dv = __shfl_sync(gmask, dq, q, NG);
        aq[q] = static_cast<S>(kappa) * pe[q * N + ir] * s_we[q] * dv;
      }
      // row i of E_{k,j} (M_j^-1 B_{j,k}) = sum_q aq[q] (V^t M^-1 B)[q][.]: the rank-Qe row
      // space carried through the neighbour's block on the host (bjG2), Q row updates instead of N
      const S* g2 = s_g2 + (n * 3 + np) * Q * NJ;
#pragma unroll
      for (int q = 0; q < Q; ++q) row_fma<S, N, NJ>(g2 + q * NJ, aq[q], a);
    }
  }
  S v[N];  // row i of the augmented identity
#pragma unroll
  for (int jj = 0; jj < N; ++jj) v[jj] = (jj == i) ? S(1) : S(0);

  // Gauss-Jordan, partial pivoting over the rows not yet used
  bool used = !row;
  int my_col = -1;
  S* piv = s_piv[warp][sub];
#pragma unroll
  for (int c = 0; c < N; ++c) {
    S best = used ? S(-1) : fabs(a[c]);
    int who = i;
#pragma unroll
    for (int o = NG / 2; o > 0; o >>= 1) {
      const S ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int ow = __shfl_xor_sync(0xffffffffu, who, o);
      if (ob > best || (ob == best && ow < who)) {
        best = ob;
        who = ow;
      }
    }
    if (i == who && row) {
      const S inv = S(1) / a[c];
#pragma unroll
      for (int jj = 0; jj < N; ++jj) {
        a[jj] *= inv;
        v[jj] *= inv;
        piv[jj] = a[jj];
        piv[N + jj] = v[jj];
      }
      used = true;
      my_col = c;
    }
    __syncwarp();
    if (row && i != who) {
      const S f = a[c];
#pragma unroll
      for (int jj = 0; jj < N; ++jj) {
        a[jj] = fma(-f, piv[jj], a[jj]);
        v[jj] = fma(-f, piv[N + jj], v[jj]);
      }
    }
    __syncwarp();
  }
  if constexpr (OUT == 3) {  // FP16 packed, scaled per element by max |P^-1|
    S mx = 0;
    if (row)
#pragma unroll
      for (int jj = 0; jj < N; ++jj) mx = fmax(mx, fabs(v[jj]));
#pragma unroll
    for (int o = NG / 2; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const S sc = mx > S(0) ? mx : S(1);
    if (row) {
      if (i == 0) out_scale[k] = static_cast<float>(sc);
      const S inv = S(1) / sc;
#pragma unroll
      for (int jj = 0; jj < N; ++jj)
        static_cast<__half*>(out)[sm_packed_p_index<P>(my_col, jj, Kp, k)] = __float2half(static_cast<float>(v[jj] * inv));
    }
    return;
  }
  if (row) {  // this lane holds row my_col of P^-1
    const int r = my_col;
#pragma unroll
    for (int jj = 0; jj < N; ++jj) {
      if constexpr (OUT == 0) {
        static_cast<double*>(out)[static_cast<long>(r * N + jj) * Kp + k] = v[jj];
      } else if constexpr (OUT == 1) {
        static_cast<float*>(out)[static_cast<long>(r * N + jj) * Kp + k] = static_cast<float>(v[jj]);
      } else {
        static_cast<float*>(out)[sm_packed_p_index<P>(r, jj, Kp, k)] = static_cast<float>(v[jj]);
      }
    }
  }
}

}  // namespace

// Pinv (FP64 SoA), Pinv32 (FP32 SoA) or Ph + Pscale (FP16 packed, scaled per
// element) from the level's FP64 E
void launch_bjac(Handle& h, double wm, double dt, int out_kind) {
  void* out = out_kind == 0   ? static_cast<void*>(h.Pinv.ptr)
              : out_kind == 1 ? static_cast<void*>(h.Pinv32.ptr)
                              : static_cast<void*>(h.Ph.ptr);
  float* sc = out_kind == 3 ? h.Pscale.ptr : nullptr;
  if (out_kind == 3) smooth_pack_alloc(h);  // the kind-3 kernel also writes the FP16 copy of E
#define LAUNCH(P, O)                                                                                          \
  do {                                                                                                        \
    const size_t smem = BjacSmem<P, double>::bytes(); /* + static: always opt in beyond 48 KB */             \
    LDG_CUDA(cudaFuncSetAttribute(k_bjac_warp<P, O>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                                    static_cast<int>(smem)));                                                 \
    k_bjac_warp<P, O><<<grid, 256, smem, h.stream>>>(h.mesh(), h.dtab, h.E.ptr, h.D.ptr, wm, dt, h.prob.eta, out, \
                                                      sc, nullptr, nullptr);                                  \
  } while (0)
#define LAUNCH32(P, O)                                                                                        \
  do {                                                                                                        \
    const size_t smem = BjacSmem<P, float>::bytes();                                                          \
    LDG_CUDA(cudaFuncSetAttribute(k_bjac_warp<P, O, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                    static_cast<int>(smem)));                                                 \
    k_bjac_warp<P, O, float><<<grid, 256, smem, h.stream>>>(h.mesh(), h.dtab, h.E.ptr, h.D.ptr, wm, dt,       \
                                                             h.prob.eta, out, sc, h.Eh.ptr, h.Escale.ptr);    \
  } while (0)
#define CALL(P)                                                      \
  do {                                                               \
    const unsigned grid = grid_of(h.K, Cfg<P>::EPB);                 \
    switch (out_kind) {                                              \
      case 0: LAUNCH(P, 0); break;                                   \
      case 1: LAUNCH(P, 1); break;                                   \
      default: LAUNCH32(P, 3); break;                                \
    }                                                                \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
#undef LAUNCH
#undef LAUNCH32
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

}  // namespace ldgb
