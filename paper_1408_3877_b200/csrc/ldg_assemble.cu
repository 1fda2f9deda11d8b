// K2 projection, K5 right-hand side, K3 fused time-dependent assembly and
// K4 static blocks — one thread per triangle, element-interleaved layout
// (ldg_device.cuh), reference tables staged in shared memory.
//
//  K2  project            fields.hpp:53-82   (system.hpp:112-113 calls it for d, f)
//  K5  J_D^m, K_D, K_N, L  assembly.hpp:256-338, V of system.hpp:147-150
//  K3  E^m = -G^m + R^m + R_D^m
//        G^m              assembly.hpp:113-136 (tensor form, exact)
//        R^m, R_D^m       assembly.hpp:214-252, evaluated in rank-Q form:
//                         d_h is sampled at the Qe Gauss points of an edge
//                         rule exact for degree 3p, so each N x N block is a
//                         sum of Qe rank-one terms (N^2 Qe FMA instead of N^3);
//                         the integrand is polynomial, so this equals the
//                         reference's tensor contraction up to rounding.
//  K4  B^m = -H^m + Q^m + Q_N^m and S + S_D   assembly.hpp:76-208
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ldg_internal.hpp"

namespace ldgb {

namespace {

template <int P>
struct Cfg {
  static constexpr int N = (P + 1) * (P + 2) / 2;
  static constexpr int QE = (3 * P + 2) / 2;  // Gauss points exact for degree 3p
  static constexpr int QB = P + 1;            // rule_1d(2p+1)
};

inline unsigned grid_of(long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

__device__ __forceinline__ void map_point(const double* __restrict__ g, long Kp, int k, double r1, double r2,
                                          double* x1, double* x2) {
  // mesh.hpp:64-68, same operation order (no contraction)
  *x1 = __dadd_rn(__dadd_rn(__dmul_rn(g[kB11 * Kp + k], r1), __dmul_rn(g[kB12 * Kp + k], r2)), g[kA1x * Kp + k]);
  *x2 = __dadd_rn(__dadd_rn(__dmul_rn(g[kB21 * Kp + k], r1), __dmul_rn(g[kB22 * Kp + k], r2)), g[kA1y * Kp + k]);
}

__device__ __forceinline__ void edge_ref_point(int n, double s, double* x1, double* x2) {
  if (n == 0) {
    *x1 = 1.0 - s;
    *x2 = s;
  } else if (n == 1) {
    *x1 = 0.0;
    *x2 = 1.0 - s;
  } else {
    *x1 = s;
    *x2 = 0.0;
  }
}

__device__ __forceinline__ void stage_to_smem(double* dst, const double* __restrict__ src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// ---------------------------------------------------------------- K2
// rule = [x1(R) | x2(R) | w(R) | phi(R x N)], minv N x N.  Projects up to two
// functions at once onto elements [0, count).
// BASE: f0 = LDG_FN_BASE_D and f1 = LDG_FN_BASE_F (the BASELINE problem's
// per-step pair): the shared factors e^(x1+x2), sincos(7 x1), sincos(7 x2) are
// evaluated once per point and sin t, e^-t once per thread (the generic
// switch evaluates nine transcendentals per point) — same expressions, so
// the values agree with ldg_coeff_eval to rounding.
template <int N, bool BASE>
__global__ void __launch_bounds__(128) k_project(DevMesh m, int count, const double* __restrict__ rule, int R,
                                                 const double* __restrict__ minv, ldg_coeff f0, ldg_coeff f1,
                                                 int nfn, double t, double* __restrict__ out0,
                                                 double* __restrict__ out1) {
  extern __shared__ double sm[];
  double* s_rule = sm;
  double* s_minv = sm + R * (3 + N);
  stage_to_smem(s_rule, rule, R * (3 + N));
  stage_to_smem(s_minv, minv, N * N);
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const double* phi = s_rule + 3 * R;
  double a0[N], a1[N];
#pragma unroll
  for (int j = 0; j < N; ++j) a0[j] = a1[j] = 0.0;
  const double dt_fac = BASE ? 1.0 + 0.5 * sin(t) : 0.0, emt = BASE ? exp(-t) : 0.0;
  for (int r = 0; r < R; ++r) {
    double x1, x2;
    map_point(m.geom, m.Kp, k, s_rule[r], s_rule[R + r], &x1, &x2);
    const double w = s_rule[2 * R + r];
    double v0, v1 = 0.0;
    if constexpr (BASE) {
      double s1, c1, s2, c2;
      sincos(7.0 * x1, &s1, &c1);
      sincos(7.0 * x2, &s2, &c2);
      const double d = exp(x1 + x2) * dt_fac;
      v0 = w * d;
      v1 = w * (-emt + d * (98.0 * c1 * c2 + 7.0 * s1 * c2 + 7.0 * c1 * s2));
    } else {
      v0 = w * ldg_coeff_eval(f0.id, f0.p, t, x1, x2);
      if (nfn > 1) v1 = w * ldg_coeff_eval(f1.id, f1.p, t, x1, x2);
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      a0[j] += v0 * phi[r * N + j];
      a1[j] += v1 * phi[r * N + j];
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      s0 += s_minv[i * N + j] * a0[j];
      s1 += s_minv[i * N + j] * a1[j];
    }
    out0[i * m.Kp + k] = s0;
    if (nfn > 1) out1[i * m.Kp + k] = s1;
  }
}

// ---------------------------------------------------------------- K5
// which: 0 -> V = [-J1; -J2; eta K_D - K_N + L] (3 planes of N), 1 J1, 2 J2,
// 3 K_D, 4 K_N, 5 L (one plane of N each).  L = M F is written first; the
// boundary edges (a few elements) then add their terms in place, one edge at
// a time, so only N accumulators are live (the all-in-registers form needed
// 255 registers at p = 4 and ran at 2.6 TB/s).
template <int P>
__global__ void __launch_bounds__(128, 4) k_rhs(DevMesh m, DevTables T, ldg_coeff cd, ldg_coeff gn, double eta,
                                             double t, const double* __restrict__ D, const double* __restrict__ F,
                                             int which, double* __restrict__ out) {
  constexpr int N = Cfg<P>::N, QB = Cfg<P>::QB;
  __shared__ double s_m[N * N], s_pb[3 * QB * N], s_sb[QB], s_wb[QB];
  stage_to_smem(s_m, T.base + T.mhat, N * N);
  stage_to_smem(s_pb, T.base + T.pb, 3 * QB * N);
  stage_to_smem(s_sb, T.base + T.sb, QB);
  stage_to_smem(s_wb, T.base + T.wb, QB);
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m.K) return;
  const long Kp = m.Kp;
  const double* g = m.geom;
  {
    const bool need_l = which == 0 || which == 5;
    double f[N];
#pragma unroll
    for (int j = 0; j < N; ++j) f[j] = need_l ? F[j * Kp + k] : 0.0;
    const double two_area = 2.0 * g[kArea * Kp + k];
    double* lo = out + (which == 0 ? 2L * N * Kp : 0L);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double l = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) l += (two_area * s_m[i * N + j]) * f[j];
      lo[i * Kp + k] = l;
      if (which == 0) out[i * Kp + k] = out[(N + i) * Kp + k] = 0.0;
    }
  }
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kind = m.kind[n * Kp + k];
    if (kind != kDirichlet && kind != kNeumann) continue;
    const double len = g[(kLen0 + n) * Kp + k];
    double s[N];
#pragma unroll
    for (int i = 0; i < N; ++i) s[i] = 0.0;
#pragma unroll 1
    for (int q = 0; q < QB; ++q) {
      double r1, r2, x1, x2;
      edge_ref_point(n, s_sb[q], &r1, &r2);
      map_point(g, Kp, k, r1, r2, &x1, &x2);
      const double* ph = s_pb + (n * QB + q) * N;
      double cw;
      if (kind == kDirichlet) {
        cw = s_wb[q] * ldg_coeff_eval(cd.id, cd.p, t, x1, x2);
      } else {
        double dval = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) dval += D[l * Kp + k] * ph[l];
        cw = len * s_wb[q] * dval * ldg_coeff_eval(gn.id, gn.p, t, x1, x2);
      }
#pragma unroll
      for (int i = 0; i < N; ++i) s[i] += cw * ph[i];
    }
    // this edge's terms: J_D^m += nu^m |E| s, K_D += s (Dirichlet); K_N += s (Neumann)
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;  // coefficients for planes 0, 1, 2
    if (kind == kDirichlet) {
      const double j1 = g[(kNux0 + n) * Kp + k] * len, j2 = g[(kNuy0 + n) * Kp + k] * len;
      if (which == 0) {
        c0 = -j1;
        c1 = -j2;
        c2 = eta;
      } else {
        c0 = which == 1 ? j1 : (which == 2 ? j2 : (which == 3 ? 1.0 : 0.0));
      }
    } else {
      if (which == 0) c2 = -1.0;
      else c0 = which == 4 ? 1.0 : 0.0;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (c0 != 0.0) out[i * Kp + k] += c0 * s[i];
      if (c1 != 0.0) out[(N + i) * Kp + k] += c1 * s[i];
      if (c2 != 0.0) out[(2 * N + i) * Kp + k] += c2 * s[i];
    }
  }
}

// ---------------------------------------------------------------- K3
// out[(m*4 + s)*N*N + i*N + j][k]: s = 0 diagonal block, s = 1+n the block in
// column nbr[n].  MODE selects E = -G + R + R_D or one operator; kModeEdiag
// (the solver's per-step assembly) writes only the diagonal blocks,
// out[m*N*N + i*N + j][k].
template <int P, int MODE_>
__global__ void __launch_bounds__(128) k_assemble(DevMesh m, DevTables T, const double* __restrict__ D,
                                                  double* __restrict__ out) {
  constexpr bool kDiagOnly = MODE_ == kModeEdiag;
  constexpr int MODE = kDiagOnly ? kModeE : MODE_;
  constexpr int N = Cfg<P>::N, Q = Cfg<P>::QE, NN = N * N;
  extern __shared__ double sm[];
  double* s_g = sm;                    // [i][j][l][2]
  double* s_pe = s_g + 2 * N * NN;     // [n][q][i]
  double* s_pth = s_pe + 3 * Q * N;    // [n][np][q][j]
  double* s_we = s_pth + 9 * Q * N;    // [q]
  stage_to_smem(s_g, T.base + T.ghat, 2 * N * NN);
  stage_to_smem(s_pe, T.base + T.pe, 3 * Q * N);
  stage_to_smem(s_pth, T.base + T.pth, 9 * Q * N);
  stage_to_smem(s_we, T.base + T.we, Q);
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m.K) return;
  const long Kp = m.Kp;
  const double* g = m.geom;
  double dk[N];
#pragma unroll
  for (int l = 0; l < N; ++l) dk[l] = D[l * Kp + k];
  const double b11 = g[kB11 * Kp + k], b12 = g[kB12 * Kp + k];
  const double b21 = g[kB21 * Kp + k], b22 = g[kB22 * Kp + k];
  // edge weights c^m_n of the diagonal R terms and w_q d_h(gamma_n(s_q))
  double c1[3], c2[3], wd[3][Q];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    const int kind = m.kind[n * Kp + k];
    const double len = g[(kLen0 + n) * Kp + k];
    double f = 0.0;
    if (kind == kInterior && (MODE == kModeE || MODE == kModeR)) f = 0.5 * len;
    if (kind == kDirichlet && (MODE == kModeE || MODE == kModeRD)) f = len;
    c1[n] = f * g[(kNux0 + n) * Kp + k];
    c2[n] = f * g[(kNuy0 + n) * Kp + k];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double dv = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) dv += dk[l] * s_pe[(n * Q + q) * N + l];
      wd[n][q] = s_we[q] * dv;
    }
  }
  double* o1 = out;
  double* o2 = out + (kDiagOnly ? 1L : 4L) * NN * Kp;
  // diagonal blocks
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    double a[3][Q];
#pragma unroll
    for (int n = 0; n < 3; ++n)
#pragma unroll
      for (int q = 0; q < Q; ++q) a[n][q] = wd[n][q] * s_pe[(n * Q + q) * N + i];
#pragma unroll 1
    for (int j = 0; j < N; ++j) {
      double e1 = 0.0, e2 = 0.0;
      if (MODE == kModeE || MODE == kModeG) {
        const double* gij = s_g + (i * N + j) * N * 2;
        double g1 = 0.0, g2 = 0.0, G1, G2;
        if (MODE == kModeG) {
          // G^m alone (exports, ldg_assemble_dphi_phi_coeff): the reference's
          // operation order and rounding (assembly.hpp:122-129, no fused
          // multiply-add), so its exact zeros -- dropped from G's pattern -- match
#pragma unroll
          for (int l = 0; l < N; ++l) {
            g1 = __dadd_rn(g1, __dmul_rn(dk[l], gij[2 * l]));
            g2 = __dadd_rn(g2, __dmul_rn(dk[l], gij[2 * l + 1]));
          }
          G1 = __dsub_rn(__dmul_rn(b22, g1), __dmul_rn(b21, g2));
          G2 = __dsub_rn(__dmul_rn(b11, g2), __dmul_rn(b12, g1));
        } else {
#pragma unroll
          for (int l = 0; l < N; ++l) {
            g1 += dk[l] * gij[2 * l];
            g2 += dk[l] * gij[2 * l + 1];
          }
          G1 = b22 * g1 - b21 * g2;
          G2 = b11 * g2 - b12 * g1;
        }
        if (MODE == kModeE) {
          e1 = -G1;
          e2 = -G2;
        } else {
          e1 = G1;
          e2 = G2;
        }
      }
      if (MODE != kModeG) {
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          double r = 0.0;
#pragma unroll
          for (int q = 0; q < Q; ++q) r += a[n][q] * s_pe[(n * Q + q) * N + j];
          e1 += c1[n] * r;
          e2 += c2[n] * r;
        }
      }
      o1[static_cast<long>(i * N + j) * Kp + k] = e1;
      o2[static_cast<long>(i * N + j) * Kp + k] = e2;
    }
  }
  if constexpr (kDiagOnly) return;
  // off-diagonal blocks: neighbour coefficient, normal and length of the k- side
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kp = m.nbr[n * Kp + k];
    double* p1 = o1 + static_cast<long>(1 + n) * NN * Kp;
    double* p2 = o2 + static_cast<long>(1 + n) * NN * Kp;
    if (kp < 0 || MODE == kModeG || MODE == kModeRD) {
      for (int ij = 0; ij < NN; ++ij) {
        p1[ij * Kp + k] = 0.0;
        p2[ij * Kp + k] = 0.0;
      }
      continue;
    }
    const int np = m.nbrn[n * Kp + k];
    const double* pt = s_pth + (n * 3 + np) * Q * N;
    const double half_len = 0.5 * g[(kLen0 + n) * Kp + k];
    const double co1 = half_len * g[(kNux0 + n) * Kp + k];
    const double co2 = half_len * g[(kNuy0 + n) * Kp + k];
    double wdp[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double dv = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) dv += D[l * Kp + kp] * pt[q * N + l];
      wdp[q] = s_we[q] * dv;
    }
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
      double a[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) a[q] = wdp[q] * s_pe[(n * Q + q) * N + i];
#pragma unroll 1
      for (int j = 0; j < N; ++j) {
        double r = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) r += a[q] * pt[q * N + j];
        p1[static_cast<long>(i * N + j) * Kp + k] = co1 * r;
        p2[static_cast<long>(i * N + j) * Kp + k] = co2 * r;
      }
    }
  }
}

// K3, row form (kModeE / kModeEdiag, the production modes).  The kernel
// above walks (i, j) with short dependent FMA chains and loads one table
// entry per FMA; ncu at 1024^2, p = 4: 168 registers, 3 warps per scheduler,
// 9 cycles per issued instruction, short-scoreboard (shared-load latency)
// and fixed-latency (FMA chain) stalls on top — 3.7 TB/s.  Here a thread
// produces one block ROW i at a time for both m:
//   G:  acc^m[j] = sum_l D_l Ghat(i, j, l, m)     (table permuted to [i][l][j][m]:
//       one 128-bit broadcast load feeds the m = 1, 2 FMAs of one j)
//   E^m[j] = -(B-combination of acc)             (assembly.hpp:126-129)
//   R:  r[j] = sum_q (w_q d_h(gamma_n(s_q)) phi_i) phi_j   per edge n,
//       E^m[j] += c^m_n r[j]                      (rank-Qe form, see above)
//   off-diagonal rows likewise from the neighbour's D.
// 30 (G) or 15 (R) independent accumulators per row instead of 2-5, and the
// per-element constants (D_k, w_q d_h) live in shared memory (one conflict-free
// 64-bit load per use) so the registers hold the accumulators.
// CTA size of the row kernel at p = 4: 384 threads (<= 168 registers, no spills) and, for
// meshes that fit two rounds of 148 x 448 elements (the 256^2 level: 2.3 rounds of 384),
// 448 threads at 128 registers (0.290 -> 0.261 ms at 256^2; at 1024^2, all blocks, the
// 448-thread build was 7 % slower, so large meshes keep 384).
template <int P, bool WIDE = false>
struct Asm2 {
  static constexpr int N = Cfg<P>::N, Q = Cfg<P>::QE, NN = N * N;
  static constexpr int NP = (N % 2) ? N + 1 : N;  // padded table rows (16-byte aligned)
  // p = 4: one 384-thread CTA per SM (<= 168 registers, 12 warps; two
  // 128-thread CTAs were register- and shared-limited to 8); below, 128
  static constexpr int kThreads = P == 4 ? (WIDE ? 448 : 384) : 128;
  static constexpr int kMinBlocks = P == 4 ? 1 : 4;
  // shared: G [i][l][j][2] | pe [n][q][NP] | pth [n][np][q][NP] | we [Q] (even) | per-thread [N + 3Q][T]
  static constexpr int kG = 2 * N * NN, kPe = 3 * Q * NP, kPth = 9 * Q * NP, kWe = (Q + 1) / 2 * 2;
  static constexpr int kTab = kG + kPe + kPth + kWe;
  static constexpr int kPer = N + 3 * Q + 6;
  static constexpr size_t smem() { return sizeof(double) * (kTab + static_cast<size_t>(kPer) * kThreads); }
};

// acc[j] += a * row[j], j < N, row 16-byte aligned in shared memory
template <int N>
__device__ __forceinline__ void row_axpy(double a, const double* row, double* acc) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
  for (int q = 0; q < N / 2; ++q) {
    const double2 v = r2[q];
    acc[2 * q] = fma(a, v.x, acc[2 * q]);
    acc[2 * q + 1] = fma(a, v.y, acc[2 * q + 1]);
  }
  if (N & 1) acc[N - 1] = fma(a, row[N - 1], acc[N - 1]);
}

template <int P, int MODE, bool WIDE>
__device__ __forceinline__ void assemble_rows_element(const DevMesh& m, const double* __restrict__ D,
                                                      double* __restrict__ out, const double* s_g,
                                                      const double* s_pe, const double* s_pth,
                                                      const double* s_we, double* per, int k) {
  using A = Asm2<P, WIDE>;
  constexpr int N = A::N, Q = A::Q, NN = A::NN, NP = A::NP;
  constexpr bool kDiagOnly = MODE == kModeEdiag;
  const long Kp = m.Kp;
  const double* g = m.geom;
  auto dk = [&](int l) -> double& { return per[l * A::kThreads]; };
  auto wd = [&](int n, int q) -> double& { return per[(N + n * Q + q) * A::kThreads]; };
  // c^m_n of the diagonal R terms (rolled edge loops index them)
  auto cm = [&](int mm, int n) -> double& { return per[(N + 3 * Q + mm * 3 + n) * A::kThreads]; };
#pragma unroll
  for (int l = 0; l < N; ++l) dk(l) = D[l * Kp + k];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    const int kind = m.kind[n * Kp + k];
    const double len = g[(kLen0 + n) * Kp + k];
    const double f = kind == kInterior ? 0.5 * len : (kind == kDirichlet ? len : 0.0);
    cm(0, n) = f * g[(kNux0 + n) * Kp + k];
    cm(1, n) = f * g[(kNuy0 + n) * Kp + k];
#pragma unroll 1
    for (int q = 0; q < Q; ++q) {
      double dv = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) dv = fma(dk(l), s_pe[(n * Q + q) * NP + l], dv);
      wd(n, q) = s_we[q] * dv;
    }
  }
  const double b11 = g[kB11 * Kp + k], b12 = g[kB12 * Kp + k];
  const double b21 = g[kB21 * Kp + k], b22 = g[kB22 * Kp + k];
  double* o1 = out;
  double* o2 = out + (kDiagOnly ? 1L : 4L) * NN * Kp;
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    double e1[N], e2[N];
#pragma unroll
    for (int j = 0; j < N; ++j) e1[j] = e2[j] = 0.0;
#pragma unroll 3
    for (int l = 0; l < N; ++l) {
      const double d = dk(l);
      const double2* row = reinterpret_cast<const double2*>(s_g + (i * N + l) * 2 * N);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double2 v = row[j];
        e1[j] = fma(d, v.x, e1[j]);
        e2[j] = fma(d, v.y, e2[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {  // E^m = -G^m: G^1 = b22 g1 - b21 g2, G^2 = b11 g2 - b12 g1
      const double g1 = e1[j], g2 = e2[j];
      e1[j] = fma(b21, g2, -b22 * g1);
      e2[j] = fma(b12, g1, -b11 * g2);
    }
#pragma unroll 1
    for (int n = 0; n < 3; ++n) {
      const double c1 = cm(0, n), c2 = cm(1, n);
      if (c1 == 0.0 && c2 == 0.0) continue;
      double r[N];
#pragma unroll
      for (int j = 0; j < N; ++j) r[j] = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double* pr = s_pe + (n * Q + q) * NP;
        row_axpy<N>(wd(n, q) * pr[i], pr, r);
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        e1[j] = fma(c1, r[j], e1[j]);
        e2[j] = fma(c2, r[j], e2[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      o1[static_cast<long>(i * N + j) * Kp + k] = e1[j];
      o2[static_cast<long>(i * N + j) * Kp + k] = e2[j];
    }
  }
  if constexpr (kDiagOnly) return;
  // off-diagonal blocks (assembly.hpp:238-247): neighbour coefficient, normal
  // and length of the k- side.  Per edge: the neighbour's D into the (no
  // longer needed) D_k slots, its edge samples w_q d_{k+}(theta(s_q)) into the
  // diagonal's slots, c^m into cm (0 on boundary edges: zero blocks).  The
  // row loop runs outside the edge loop so the compiler cannot hoist an
  // edge's whole pth table into registers across rows.
  int npk = 0;
#pragma unroll 1
  for (int n = 0; n < 3; ++n) {
    const int kp = m.nbr[n * Kp + k];
    if (kp < 0) {
      for (int q = 0; q < Q; ++q) wd(n, q) = 0.0;
      cm(0, n) = cm(1, n) = 0.0;
      continue;
    }
    const int np = m.nbrn[n * Kp + k];
    npk |= np << (2 * n);
    const double* pt = s_pth + (n * 3 + np) * Q * NP;
#pragma unroll
    for (int l = 0; l < N; ++l) dk(l) = D[l * Kp + kp];
#pragma unroll 1
    for (int q = 0; q < Q; ++q) {
      double dv = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) dv = fma(dk(l), pt[q * NP + l], dv);
      wd(n, q) = s_we[q] * dv;
    }
    const double half_len = 0.5 * g[(kLen0 + n) * Kp + k];
    cm(0, n) = half_len * g[(kNux0 + n) * Kp + k];
    cm(1, n) = half_len * g[(kNuy0 + n) * Kp + k];
  }
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
#pragma unroll 1
    for (int n = 0; n < 3; ++n) {
      const double* pt = s_pth + (n * 3 + ((npk >> (2 * n)) & 3)) * Q * NP;
      double r[N];
#pragma unroll
      for (int j = 0; j < N; ++j) r[j] = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) row_axpy<N>(wd(n, q) * s_pe[(n * Q + q) * NP + i], pt + q * NP, r);
      const double co1 = cm(0, n), co2 = cm(1, n);
      double* p1 = o1 + static_cast<long>(1 + n) * NN * Kp;
      double* p2 = o2 + static_cast<long>(1 + n) * NN * Kp;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        p1[static_cast<long>(i * N + j) * Kp + k] = co1 * r[j];
        p2[static_cast<long>(i * N + j) * Kp + k] = co2 * r[j];
      }
    }
  }
}

// Persistent: the grid is sized to the resident CTAs and each CTA loops over
// blocks of kThreads elements, so the ~65 KB of tables are staged once per
// CTA (staged per 128 elements they cost ~15 % of the run in exposed L2
// latency at p = 4).
template <int P, int MODE, bool WIDE>
__global__ void __launch_bounds__(Asm2<P, WIDE>::kThreads, Asm2<P, WIDE>::kMinBlocks) k_assemble_rows(DevMesh m, DevTables T,
                                                                        const double* __restrict__ D,
                                                                        double* __restrict__ out) {
  using A = Asm2<P, WIDE>;
  constexpr int N = A::N, Q = A::Q, NP = A::NP;
  extern __shared__ __align__(16) double sm[];
  double* s_g = sm;                 // [i][l][j][m]
  double* s_pe = s_g + A::kG;       // [n][q][NP]
  double* s_pth = s_pe + A::kPe;    // [n][np][q][NP]
  double* s_we = s_pth + A::kPth;   // [q]
  double* s_per = s_we + A::kWe;    // [v][tid]: v < N D_k, then w_q d_h on edge n at N + n Q + q
  {
    const double* gsrc = T.base + T.ghat;  // [i][j][l][m]
#pragma unroll 8
    for (int t = threadIdx.x; t < A::kG; t += blockDim.x) {
      const int mm = t & 1, j = (t >> 1) % N, il = (t >> 1) / N, l = il % N, i = il / N;
      s_g[t] = __ldg(gsrc + ((i * N + j) * N + l) * 2 + mm);
    }
    for (int t = threadIdx.x; t < 3 * Q * NP; t += blockDim.x) {
      const int j = t % NP, nq = t / NP;
      s_pe[t] = j < N ? T.base[T.pe + nq * N + j] : 0.0;
    }
    for (int t = threadIdx.x; t < 9 * Q * NP; t += blockDim.x) {
      const int j = t % NP, nq = t / NP;
      s_pth[t] = j < N ? T.base[T.pth + nq * N + j] : 0.0;
    }
    for (int t = threadIdx.x; t < Q; t += blockDim.x) s_we[t] = T.base[T.we + t];
  }
  __syncthreads();
  const int tid = threadIdx.x;
  double* per = s_per + tid;
  for (int k = blockIdx.x * blockDim.x + tid; k - tid < m.K; k += gridDim.x * blockDim.x) {
    if (k < m.K) assemble_rows_element<P, MODE, WIDE>(m, D, out, s_g, s_pe, s_pth, s_we, per, k);
  }
}

// ---------------------------------------------------------------- K4
// Static blocks.  kStB: out = B^1 | B^2 (2 x 4 slots); kStS: S + S_D (4 slots);
// export modes write one operator (2 comps for H/Q/QN, 1 for M/S/SD).
template <int P>
__global__ void __launch_bounds__(128) k_static(DevMesh m, DevTables T, int mode, double* __restrict__ out) {
  constexpr int N = Cfg<P>::N, NN = N * N;
  __shared__ double s_m[NN], s_h[2 * NN], s_sd[3 * NN], s_so[9 * NN];
  stage_to_smem(s_m, T.base + T.mhat, NN);
  stage_to_smem(s_h, T.base + T.hhat, 2 * NN);
  stage_to_smem(s_sd, T.base + T.sdiag, 3 * NN);
  stage_to_smem(s_so, T.base + T.soff, 9 * NN);
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m.K) return;
  const long Kp = m.Kp;
  const double* g = m.geom;
  const double b11 = g[kB11 * Kp + k], b12 = g[kB12 * Kp + k];
  const double b21 = g[kB21 * Kp + k], b22 = g[kB22 * Kp + k];
  int kind[3], np[3];
  double len[3], nu[2][3];
  for (int n = 0; n < 3; ++n) {
    kind[n] = m.kind[n * Kp + k];
    np[n] = m.nbrn[n * Kp + k];
    len[n] = g[(kLen0 + n) * Kp + k];
    nu[0][n] = g[(kNux0 + n) * Kp + k];
    nu[1][n] = g[(kNuy0 + n) * Kp + k];
  }
  const int ncomp = (mode == kStB || mode == kStH || mode == kStQ || mode == kStQN) ? 2 : 1;
  for (int c = 0; c < ncomp; ++c) {
    double* o = out + static_cast<long>(c) * 4 * NN * Kp;
    // diagonal
    for (int ij = 0; ij < NN; ++ij) {
      const double h1 = s_h[2 * ij], h2 = s_h[2 * ij + 1];
      // the reference's rounding (assembly.hpp:100-101, no fused multiply-add):
      // its exact zeros -- dropped from H's pattern -- come out as exact zeros here
      const double H = (c == 0) ? __dsub_rn(__dmul_rn(b22, h1), __dmul_rn(b21, h2))
                                : __dsub_rn(__dmul_rn(b11, h2), __dmul_rn(b12, h1));
      double v = 0.0;
      switch (mode) {
        case kStM: v = 2.0 * g[kArea * Kp + k] * s_m[ij]; break;
        case kStH: v = H; break;
        case kStB: v = -H; break;
        default: break;
      }
      for (int n = 0; n < 3; ++n) {
        const double sd = s_sd[ij * 3 + n];
        const bool in = kind[n] == kInterior, di = kind[n] == kDirichlet, ne = kind[n] == kNeumann;
        if ((mode == kStB || mode == kStQ) && in) v += 0.5 * nu[c][n] * len[n] * sd;
        if ((mode == kStB || mode == kStQN) && ne) v += nu[c][n] * len[n] * sd;
        if ((mode == kStS || mode == kStSint) && in) v += sd;
        if ((mode == kStS || mode == kStSD) && di) v += sd;
      }
      o[static_cast<long>(ij) * Kp + k] = v;
    }
    // off-diagonal
    for (int n = 0; n < 3; ++n) {
      double* on = o + static_cast<long>(1 + n) * NN * Kp;
      const bool in = kind[n] == kInterior;
      const double cq = 0.5 * nu[c][n] * len[n];
      for (int ij = 0; ij < NN; ++ij) {
        double v = 0.0;
        if (in) {
          const double so = s_so[(ij * 3 + n) * 3 + np[n]];
          if (mode == kStB || mode == kStQ) v = cq * so;
          if (mode == kStS || mode == kStSint) v = -so;
        }
        on[static_cast<long>(ij) * Kp + k] = v;
      }
    }
  }
}

template <int P>
size_t assemble_smem() {
  constexpr int N = Cfg<P>::N, Q = Cfg<P>::QE;
  return sizeof(double) * (2 * N * N * N + 3 * Q * N + 9 * Q * N + Q);
}

// Row kernel for the production modes at p = 4 (C3, 1024^2: 6.0 vs 8.6 ms,
// 5.2 TB/s); at p = 2, 3 the (i, j) kernel measured 3-8 % faster (1.25 vs
// 1.36 ms, 3.20 vs 3.32 ms for the whole C3-style call at 1024^2).
// LDG_ASM_V1=1 forces the (i, j) kernel, =0 the row kernel (A/B runs).
bool asm_v1(int p) {
  static const int env = [] {
    const char* e = std::getenv("LDG_ASM_V1");
    return e ? std::atoi(e) : -1;
  }();
  return env < 0 ? p < 4 : env != 0;
}

template <int P, int MODE, bool WIDE>
void launch_assemble_rows(Handle& h, double* out, int sms) {
  using A = Asm2<P, WIDE>;
  const size_t smem = A::smem();
  auto kern = k_assemble_rows<P, MODE, WIDE>;
  static int grid_cap = 0;
  if (!grid_cap) {
    int per_sm = 0;
    LDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    LDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, A::kThreads, smem));
    grid_cap = std::max(1, sms * per_sm);
  }
  const unsigned grid = std::min<unsigned>(grid_of(h.K, A::kThreads), static_cast<unsigned>(grid_cap));
  kern<<<grid, A::kThreads, smem, h.stream>>>(h.mesh(), h.dtab, h.D.ptr, out);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

template <int P, int MODE>
void launch_assemble_p(Handle& h, double* out) {
  if constexpr (MODE == kModeE || MODE == kModeEdiag) {
    if (!asm_v1(P)) {
      // the wide CTA when the mesh fits two rounds of it on the SMs (Asm2)
      static int sms = 0;
      if (!sms) {
        int dev = 0;
        LDG_CUDA(cudaGetDevice(&dev));
        LDG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      }
      if (P == 4 && h.K <= 2L * sms * Asm2<P, true>::kThreads && h.K > 2L * sms * Asm2<P, false>::kThreads)
        launch_assemble_rows<P, MODE, true>(h, out, sms);
      else
        launch_assemble_rows<P, MODE, false>(h, out, sms);
      return;
    }
  }
  const size_t smem = assemble_smem<P>();
  auto kern = k_assemble<P, MODE>;
  static bool configured = false;
  if (!configured) {
    LDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = true;
  }
  kern<<<grid_of(h.K, 128), 128, smem, h.stream>>>(h.mesh(), h.dtab, h.D.ptr, out);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

template <int P>
void launch_assemble_mode(Handle& h, int mode, double* out) {
  switch (mode) {
    case kModeE: launch_assemble_p<P, kModeE>(h, out); break;
    case kModeEdiag: launch_assemble_p<P, kModeEdiag>(h, out); break;
    case kModeG: launch_assemble_p<P, kModeG>(h, out); break;
    case kModeR: launch_assemble_p<P, kModeR>(h, out); break;
    default: launch_assemble_p<P, kModeRD>(h, out); break;
  }
}

template <int N>
void launch_project_n(Handle& h, const ldg_coeff& f0, const ldg_coeff* f1, double t, const double* rule, int R,
                      double* out0, double* out1, int count) {
  const size_t smem = sizeof(double) * (R * (3 + N) + N * N);
  const bool base = f1 && f0.id == LDG_FN_BASE_D && f1->id == LDG_FN_BASE_F;
  auto kern = base ? k_project<N, true> : k_project<N, false>;
  LDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<grid_of(count, 128), 128, smem, h.stream>>>(h.mesh(), count, rule, R, h.dtab.base + h.dtab.minv, f0,
                                                     f1 ? *f1 : f0, f1 ? 2 : 1, t, out0, out1);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

}  // namespace

void upload_rule(Handle& h, int q_ord, DBuf<double>& buf, int* R) {
  const Rule2D r = rule_2d(q_ord);
  const int n = static_cast<int>(r.w.size());
  std::vector<double> host(static_cast<size_t>(n) * (3 + h.N));
  for (int i = 0; i < n; ++i) {
    host[i] = r.x1[i];
    host[n + i] = r.x2[i];
    host[2 * n + i] = r.w[i];
    for (int j = 0; j < h.N; ++j) host[3 * n + i * h.N + j] = basis_value(j, r.x1[i], r.x2[i]);
  }
  buf.alloc(host.size(), nullptr);
  LDG_CUDA(cudaMemcpy(buf.ptr, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice));
  *R = n;
}

void launch_project(Handle& h, const ldg_coeff& fn, double t, const double* rule_dev, int R, double* out,
                    int count) {
  switch (h.N) {
    case 1: launch_project_n<1>(h, fn, nullptr, t, rule_dev, R, out, nullptr, count); break;
    case 3: launch_project_n<3>(h, fn, nullptr, t, rule_dev, R, out, nullptr, count); break;
    case 6: launch_project_n<6>(h, fn, nullptr, t, rule_dev, R, out, nullptr, count); break;
    case 10: launch_project_n<10>(h, fn, nullptr, t, rule_dev, R, out, nullptr, count); break;
    default: launch_project_n<15>(h, fn, nullptr, t, rule_dev, R, out, nullptr, count); break;
  }
}

void launch_project_df(Handle& h, double t, const double* rule_dev, int R) {
  const ldg_coeff& d = h.prob.d;
  const ldg_coeff& f = h.prob.f;
  switch (h.N) {
    case 1: launch_project_n<1>(h, d, &f, t, rule_dev, R, h.D.ptr, h.F.ptr, h.Kg); break;
    case 3: launch_project_n<3>(h, d, &f, t, rule_dev, R, h.D.ptr, h.F.ptr, h.Kg); break;
    case 6: launch_project_n<6>(h, d, &f, t, rule_dev, R, h.D.ptr, h.F.ptr, h.Kg); break;
    case 10: launch_project_n<10>(h, d, &f, t, rule_dev, R, h.D.ptr, h.F.ptr, h.Kg); break;
    default: launch_project_n<15>(h, d, &f, t, rule_dev, R, h.D.ptr, h.F.ptr, h.Kg); break;
  }
}

void launch_rhs_which(Handle& h, double t, int which, double* out) {
  const unsigned grid = grid_of(h.K, 128);
  const DevMesh m = h.mesh();
  const ldg_coeff cd = h.prob.c_d, gn = h.prob.g_n;
  switch (h.p) {
    case 0: k_rhs<0><<<grid, 128, 0, h.stream>>>(m, h.dtab, cd, gn, h.prob.eta, t, h.D.ptr, h.F.ptr, which, out); break;
    case 1: k_rhs<1><<<grid, 128, 0, h.stream>>>(m, h.dtab, cd, gn, h.prob.eta, t, h.D.ptr, h.F.ptr, which, out); break;
    case 2: k_rhs<2><<<grid, 128, 0, h.stream>>>(m, h.dtab, cd, gn, h.prob.eta, t, h.D.ptr, h.F.ptr, which, out); break;
    case 3: k_rhs<3><<<grid, 128, 0, h.stream>>>(m, h.dtab, cd, gn, h.prob.eta, t, h.D.ptr, h.F.ptr, which, out); break;
    default: k_rhs<4><<<grid, 128, 0, h.stream>>>(m, h.dtab, cd, gn, h.prob.eta, t, h.D.ptr, h.F.ptr, which, out); break;
  }
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_rhs(Handle& h, double t) { launch_rhs_which(h, t, 0, h.Vv.ptr); }

void launch_assemble(Handle& h, int mode, double* out) {
  switch (h.p) {
    case 0: launch_assemble_mode<0>(h, mode, out); break;
    case 1: launch_assemble_mode<1>(h, mode, out); break;
    case 2: launch_assemble_mode<2>(h, mode, out); break;
    case 3: launch_assemble_mode<3>(h, mode, out); break;
    default: launch_assemble_mode<4>(h, mode, out); break;
  }
}

void launch_static(Handle& h, int mode, double* out) {
  const unsigned grid = grid_of(h.K, 128);
  const DevMesh m = h.mesh();
  switch (h.p) {
    case 0: k_static<0><<<grid, 128, 0, h.stream>>>(m, h.dtab, mode, out); break;
    case 1: k_static<1><<<grid, 128, 0, h.stream>>>(m, h.dtab, mode, out); break;
    case 2: k_static<2><<<grid, 128, 0, h.stream>>>(m, h.dtab, mode, out); break;
    case 3: k_static<3><<<grid, 128, 0, h.stream>>>(m, h.dtab, mode, out); break;
    default: k_static<4><<<grid, 128, 0, h.stream>>>(m, h.dtab, mode, out); break;
  }
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

}  // namespace ldgb
