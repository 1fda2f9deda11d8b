// Multigrid smoother kernels for the small (coarse) levels.
//
// A coarse level holds a few thousand elements or fewer, so a launch is pure
// latency: with one thread per (element, row) the time is a thread's serial
// chain of ~8 dependent block-row products (8-15 us per kernel measured on
// levels of 8..2048 elements at p = 4).  Here every (element, row) item gets
// 8 lanes: for the stage-2 residual lane l = (m, slot) streams one of the 8
// E blocks of the row, lanes 0..6 also take one of the 7 static-table products
// (M, S_diag x3, S_off x3); for stage 1 lane l takes one of the 8 static
// products (H x2, S_diag x3, S_off x3).  The chain is one block row (N FMAs,
// loads issued together) plus a 3-step shuffle reduction.  A CTA holds every
// row of EPC elements, so the damped block-Jacobi update of a sweep runs in
// the same kernel on the residual in shared memory.
//
// Operands: E and P^-1 as FP32 SoA copies (E32, Pinv32), vectors FP64,
// arithmetic FP64 (these levels are latency-bound; precision is free).
// Reference operators as in ldg_apply.cu / ldg_rows.cu (assembly.hpp:76-208).
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>

#include "ldg_internal.hpp"
#include "ldg_offdiag.cuh"

namespace ldgb {

namespace {

template <int P>
struct Cfg {
  static constexpr int N = (P + 1) * (P + 2) / 2;
  static constexpr int NN = N * N;
  static constexpr int NP = (N % 2) ? N + 1 : N;
  static constexpr int NNP = N * NP;
  // elements per CTA: ~512 threads of 8 lanes x N rows, a multiple of 4 (a
  // warp = 4 consecutive elements of one row: table reads broadcast); small
  // CTAs leave each thread the registers to issue all its loads up front
  static constexpr int EPC = (512 / (8 * N)) / 4 * 4 > 0 ? (512 / (8 * N)) / 4 * 4 : 4;
  static constexpr int THREADS = EPC * N * 8;
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

struct Item {
  int lane, i, ke, k;
  bool live;
};

// item of thread t (< THREADS) in virtual block vb, elements [k0, K)
template <int P>
__device__ __forceinline__ Item item_of(int K, int k0, int vb, int t) {
  using C = Cfg<P>;
  Item it;
  it.lane = t & 7;
  const int q = t >> 3;
  it.i = q / C::EPC;
  it.ke = q % C::EPC;
  it.k = k0 + vb * C::EPC + it.ke;
  it.live = it.k < K;
  return it;
}

__device__ __forceinline__ double lane_sum8(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

// (T x[.][col])_i, T^t[j][i] at tab + j*NP + i.  All 2N loads are issued
// before the FMA chain: these kernels are a handful of dependent load rounds
// (with the loads interleaved into the chain ptxas left ~2 in flight and a
// 8-element level took ~11 us per launch).
template <int N, int NP>
__device__ __forceinline__ double trow(const double* __restrict__ tab, int i, const double* __restrict__ x, long Kp,
                                       int col) {
  double tv[N], xv[N];
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

// tout^m_i = (1/2|T|) (mhat^-1 B^m x)_i with the premultiplied tables
template <int P>
__device__ __forceinline__ void s1_body(const DevMesh& m, const DevTables& T, const double* __restrict__ x,
                                        double* __restrict__ tout, int vb, int t) {
  using C = Cfg<P>;
  constexpr int N = C::N, NP = C::NP, NNP = C::NNP;
  const Item it = item_of<P>(m.K, 0, vb, t);
  const int k = it.live ? it.k : 0, i = it.i, l = it.lane;  // dead items compute on element 0, never store
  const long Kp = m.Kp;
  const double* g = m.geom;
  const double* tb = T.base;
  double u1 = 0.0, u2 = 0.0;
  if (l < 2) {
    const double d = trow<N, NP>(tb + T.tmH + l * NNP, i, x, Kp, k);
    const double b11 = g[kB11 * Kp + k], b12 = g[kB12 * Kp + k], b21 = g[kB21 * Kp + k], b22 = g[kB22 * Kp + k];
    u1 = l == 0 ? -b22 * d : b21 * d;
    u2 = l == 0 ? b12 * d : -b11 * d;
  } else if (l < 5) {
    const int n = l - 2;
    const int kind = m.kind[n * Kp + k];
    const double len = g[(kLen0 + n) * Kp + k];
    const double f = kind == kInterior ? 0.5 * len : (kind == kNeumann ? len : 0.0);
    if (f != 0.0) {
      const double d = trow<N, NP>(tb + T.tmSd + n * NNP, i, x, Kp, k);
      u1 = f * g[(kNux0 + n) * Kp + k] * d;
      u2 = f * g[(kNuy0 + n) * Kp + k] * d;
    }
  } else {
    const int n = l - 5;
    const int kp = m.nbr[n * Kp + k];
    if (kp >= 0) {
      const double d = trow<N, NP>(tb + T.tmSo + (n * 3 + m.nbrn[n * Kp + k]) * NNP, i, x, Kp, kp);
      const double hl = 0.5 * g[(kLen0 + n) * Kp + k];
      u1 = hl * g[(kNux0 + n) * Kp + k] * d;
      u2 = hl * g[(kNuy0 + n) * Kp + k] * d;
    }
  }
  u1 = lane_sum8(u1);
  u2 = lane_sum8(u2);
  if (it.live && l == 0) {
    const double inv2a = 1.0 / (2.0 * g[kArea * Kp + k]);
    tout[i * Kp + k] = inv2a * u1;
    tout[(N + i) * Kp + k] = inv2a * u2;
  }
}

template <int P>
__global__ void __launch_bounds__(Cfg<P>::THREADS, 1) k_s1_small(DevMesh m, DevTables T, const double* __restrict__ x,
                                                              double* __restrict__ tout) {
  pdl_wait();
  pdl_trigger();
  s1_body<P>(m, T, x, tout, blockIdx.x, threadIdx.x);
}

// r_i = b_i - [wm M x + dt (eta (S + S_D) x - sum_m E^m t^m)]_i, then
//   MODE 0: out = r;  MODE 1: out = x + omega P^-1 r
template <int P, int MODE>
__device__ __forceinline__ void s2_body(const DevMesh& m, const DevTables& T, const float* __restrict__ E,
                                        const double* __restrict__ D, const double* x, const double* __restrict__ tz,
                                        const double* __restrict__ b, double wm, double dteta, double dt,
                                        const float* __restrict__ Pinv, double omega, double* out, int k0, int kend,
                                        double (*s_r)[Cfg<P>::EPC], int vb, int t) {
  using C = Cfg<P>;
  constexpr int N = C::N, NN = C::NN, NP = C::NP, NNP = C::NNP, Q = C::Q;
  const Item it = item_of<P>(kend, k0, vb, t);  // (in place for one colour: see k_s2f)
  const int k = it.k, i = it.i, l = it.lane;
  const long Kp = m.Kp;
  double part = 0.0;
  if (it.live) {
    const double* g = m.geom;
    const double* tb = T.base;
    {  // lane (c, s): E^c[s] row i against t^c of the slot's column; the diagonal
       // block stored, the off-diagonal ones matrix-free (ldg_offdiag.cuh)
      const int c = l >> 2, s = l & 3;
      const int col = s == 0 ? k : m.nbr[(s - 1) * Kp + k];
      const double* tc = tz + static_cast<long>(c) * N * Kp + col;
      if (s == 0) {
        const float* blk = E + (static_cast<long>(c) * NN + i * N) * Kp + k;
        float ev[N];
        double tv[N];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          ev[j] = blk[j * Kp];
          tv[j] = tc[j * Kp];
        }
        double e = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) e = fma(static_cast<double>(ev[j]), tv[j], e);
        part = dt * e;
      } else if (col >= 0) {
        const int n = s - 1;
        const double co = 0.5 * g[(kLen0 + n) * Kp + k] * g[((c == 0 ? kNux0 : kNuy0) + n) * Kp + k];
        double dv[N], uv[N], z[Q];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          dv[j] = D[j * Kp + col];
          uv[j] = tc[j * Kp];
        }
        offdiag_z<N, Q, double>(
            tb + T.pth + (n * 3 + m.nbrn[n * Kp + k]) * Q * N, tb + T.we, [&](int j) { return dv[j]; },
            [&](int j) { return uv[j]; }, z);
        part = dt * co * offdiag_row<N, Q, double>(tb + T.pe + n * Q * N, z, i);
      }
    }
    if (l == 0) {
      part -= wm * 2.0 * g[kArea * Kp + k] * trow<N, NP>(tb + T.tM, i, x, Kp, k);
    } else if (l < 4) {
      const int n = l - 1;
      const int kind = m.kind[n * Kp + k];
      if (kind == kInterior || kind == kDirichlet) part -= dteta * trow<N, NP>(tb + T.tSd + n * NNP, i, x, Kp, k);
    } else if (l < 7) {
      const int n = l - 4;
      const int kp = m.nbr[n * Kp + k];
      if (kp >= 0) part += dteta * trow<N, NP>(tb + T.tSo + (n * 3 + m.nbrn[n * Kp + k]) * NNP, i, x, Kp, kp);
    }
  }
  part = lane_sum8(part);
  if constexpr (MODE == 0) {
    if (it.live && l == 0) out[i * Kp + k] = b[i * Kp + k] + part;
  } else {
    if (it.live && l == 0) s_r[i][it.ke] = b[i * Kp + k] + part;
    __syncthreads();
    double d = 0.0;
    if (it.live) {
      const float* row = Pinv + static_cast<long>(i) * N * Kp + k;
      for (int j = l; j < N; j += 8) d = fma(static_cast<double>(row[j * Kp]), s_r[j][it.ke], d);
    }
    d = lane_sum8(d);
    if (it.live && l == 0) out[i * Kp + k] = fma(omega, d, x[i * Kp + k]);
    __syncthreads();  // s_r is reused by the next virtual block (tail kernel)
  }
}

template <int P, int MODE>
__global__ void __launch_bounds__(Cfg<P>::THREADS, 1) k_s2_small(DevMesh m, DevTables T, const float* __restrict__ E,
                                                              const double* __restrict__ D, const double* x,
                                                              const double* __restrict__ tz,
                                                              const double* __restrict__ b, double wm, double dteta,
                                                              double dt, const float* __restrict__ Pinv,
                                                              double omega, double* out, int k0, int kend) {
  __shared__ double s_r[Cfg<P>::N][Cfg<P>::EPC];
  pdl_wait();
  pdl_trigger();
  s2_body<P, MODE>(m, T, E, D, x, tz, b, wm, dteta, dt, Pinv, omega, out, k0, kend, s_r, blockIdx.x, threadIdx.x);
}

// out = omega P^-1 b
template <int P>
__device__ __forceinline__ void bj_body(int K, long Kp, const float* __restrict__ Pinv, const double* __restrict__ b,
                                        double omega, double* __restrict__ out, int vb, int t) {
  constexpr int N = Cfg<P>::N;
  const Item it = item_of<P>(K, 0, vb, t);
  const int k = it.live ? it.k : 0, i = it.i, l = it.lane;
  const float* row = Pinv + static_cast<long>(i) * N * Kp + k;
  double d = 0.0;
  for (int j = l; j < N; j += 8) d = fma(static_cast<double>(row[j * Kp]), b[j * Kp + k], d);
  d = lane_sum8(d);
  if (it.live && l == 0) out[i * Kp + k] = omega * d;
}

template <int P>
__global__ void __launch_bounds__(Cfg<P>::THREADS, 1) k_bj_small(int K, long Kp, const float* __restrict__ Pinv,
                                                              const double* __restrict__ b, double omega,
                                                              double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  bj_body<P>(K, Kp, Pinv, b, omega, out, blockIdx.x, threadIdx.x);
}

// ------------------------------------------------- dense coarse operator
// Column c of the level operator applied to the unit vector e_c (SoA index
// c = i * Kp + k), for the dense coarsest-level solve (ldg_dense.cu): the
// stage bodies above with blockIdx.y = column, stage 2 in residual mode with
// b = 0, so column c of `out` is -S_c e_c.
template <int P>
__global__ void __launch_bounds__(Cfg<P>::THREADS, 1) k_s1_batch(DevMesh m, DevTables T, const double* X,
                                                              double* Tz, long stride) {
  const long c = blockIdx.y;
  s1_body<P>(m, T, X + c * stride, Tz + 2 * c * stride, blockIdx.x, threadIdx.x);
}

template <int P>
__global__ void __launch_bounds__(Cfg<P>::THREADS, 1) k_s2_batch(DevMesh m, DevTables T, const float* __restrict__ E,
                                                              const double* __restrict__ D, const double* X,
                                                              const double* Tz, const double* zero, double wm,
                                                              double dteta, double dt, double* out, long stride) {
  __shared__ double s_r[Cfg<P>::N][Cfg<P>::EPC];
  const long c = blockIdx.y;
  s2_body<P, 0>(m, T, E, D, X + c * stride, Tz + 2 * c * stride, zero, wm, dteta, dt, nullptr, 0.0, out + c * stride,
                0, m.K, s_r, blockIdx.x, threadIdx.x);
}

// ---------------------------------------------------------------- tail
// The coarsest levels (a few dozen elements) of a V-cycle in ONE thread block:
// every phase (sweep stages, residual, restriction, prolongation) is a loop
// of the bodies above over the level's virtual blocks, separated by
// __syncthreads, so the level data stays in this SM's L1 and no launch or
// grid drain sits between the ~30 dependent phases (separate launches cost
// 6-7 us each on these levels, mostly dependent L2 round trips).
constexpr int kTailMax = 6;

struct TailLevel {
  DevMesh m;
  const float* E32;
  const float* Pinv32;
  const double* D;
  double *x, *s, *b, *r, *tz;
  const int* children;  // this level as the coarse side of the transfer from the level above
  const float* Pm;
  int dim;
};

struct TailArgs {
  TailLevel lv[kTailMax];
  int nlev;
  double wm, dt, dteta, omega;
  int pre, post, coarse_min;
};

// CL > 1: the same phases spread over a thread-block cluster of CL CTAs (one
// per SM of a GPC), virtual blocks dealt round-robin, the phases separated by
// cluster barriers (release/acquire at cluster scope, after a device fence
// for the global-memory level data) instead of __syncthreads: CL SMs of
// issue rate for the p >= 2 levels, still no launch between phases.
template <int P, int CL>
__global__ void __launch_bounds__(Cfg<P>::THREADS, 1) k_tail(TailArgs a, DevTables T) {
  using C = Cfg<P>;
  constexpr int N = C::N, NN = C::NN;
  __shared__ double s_r[N][C::EPC];
  pdl_wait();
  pdl_trigger();
  const int t = threadIdx.x;
  int rank = 0;
  if constexpr (CL > 1) rank = static_cast<int>(cooperative_groups::this_cluster().block_rank());
  const int gt = rank * blockDim.x + t, gstride = CL * blockDim.x;
  auto bar = [&]() {
    if constexpr (CL > 1) {
      __threadfence();
      cooperative_groups::this_cluster().sync();
    } else {
      __syncthreads();
    }
  };
  auto nvb = [](int K) { return (K + C::EPC - 1) / C::EPC; };
  auto zero = [&](const TailLevel& L, const double* b, double* out) {
    for (int vb = rank; vb < nvb(L.m.K); vb += CL) bj_body<P>(L.m.K, L.m.Kp, L.Pinv32, b, a.omega, out, vb, t);
    bar();
  };
  auto stage1 = [&](const TailLevel& L, const double* x) {
    for (int vb = rank; vb < nvb(L.m.K); vb += CL) s1_body<P>(L.m, T, x, L.tz, vb, t);
    bar();
  };
  auto stage2 = [&](const TailLevel& L, int mode, const double* x, const double* b, double* out) {
    for (int vb = rank; vb < nvb(L.m.K); vb += CL) {
      if (mode == 0)
        s2_body<P, 0>(L.m, T, L.E32, L.D, x, L.tz, b, a.wm, a.dteta, a.dt, L.Pinv32, a.omega, out, 0, L.m.K, s_r, vb,
                      t);
      else
        s2_body<P, 1>(L.m, T, L.E32, L.D, x, L.tz, b, a.wm, a.dteta, a.dt, L.Pinv32, a.omega, out, 0, L.m.K, s_r, vb,
                      t);
    }
    bar();
  };
  auto sweep = [&](const TailLevel& L, const double* xi, double* xo) {
    stage1(L, xi);
    stage2(L, 1, xi, L.b, xo);
  };
  // C.b = P^T F.r  (ldg_mg.cu k_restrict)
  auto restrict_ = [&](const TailLevel& F, const TailLevel& Cl) {
    const long Kpc = Cl.m.Kp, Kpf = F.m.Kp;
    for (int it = gt; it < N * Cl.m.K; it += gstride) {
      const int kc = it % Cl.m.K, j = it / Cl.m.K;
      double acc = 0.0;
      for (int sl = 0; sl < 4; ++sl) {
        const int k = Cl.children[sl * Kpc + kc];
        const float* Ps = Cl.Pm + (static_cast<long>(sl) * NN + j) * Kpc + kc;
#pragma unroll
        for (int i = 0; i < N; ++i) acc = fma(static_cast<double>(Ps[static_cast<long>(i) * N * Kpc]), F.r[i * Kpf + k], acc);
      }
      Cl.b[j * Kpc + kc] = acc;
    }
    bar();
  };
  // xf += P C.x  (ldg_mg.cu k_prolong_add)
  auto prolong = [&](const TailLevel& F, const TailLevel& Cl, double* xf) {
    const long Kpc = Cl.m.Kp, Kpf = F.m.Kp;
    for (int it = gt; it < 4 * N * Cl.m.K; it += gstride) {
      const int kc = it % Cl.m.K, rest = it / Cl.m.K, sl = rest % 4, i = rest / 4;
      const int k = Cl.children[sl * Kpc + kc];
      const float* Ps = Cl.Pm + (static_cast<long>(sl) * NN + static_cast<long>(i) * N) * Kpc + kc;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) acc = fma(static_cast<double>(Ps[static_cast<long>(j) * Kpc]), Cl.x[j * Kpc + kc], acc);
      xf[i * Kpf + k] += acc;
    }
    bar();
  };

  double* cur[kTailMax];
  for (int l = 0; l + 1 < a.nlev; ++l) {  // down
    const TailLevel& L = a.lv[l];
    const int sweeps = (a.pre - 1) + a.post;
    cur[l] = (sweeps % 2) ? L.s : L.x;
    zero(L, L.b, cur[l]);
    for (int sw = 0; sw < a.pre - 1; ++sw) {
      double* o = cur[l] == L.x ? L.s : L.x;
      sweep(L, cur[l], o);
      cur[l] = o;
    }
    stage1(L, cur[l]);
    stage2(L, 0, cur[l], L.b, L.r);
    restrict_(L, a.lv[l + 1]);
  }
  {  // coarsest
    const TailLevel& L = a.lv[a.nlev - 1];
    const int sweeps = max(a.coarse_min, 2 * L.dim) - 1;
    double* c = (sweeps % 2) ? L.s : L.x;
    zero(L, L.b, c);
    for (int sw = 0; sw < sweeps; ++sw) {
      double* o = c == L.x ? L.s : L.x;
      sweep(L, c, o);
      c = o;
    }
  }
  for (int l = a.nlev - 2; l >= 0; --l) {  // up
    const TailLevel& L = a.lv[l];
    prolong(L, a.lv[l + 1], cur[l]);
    for (int sw = 0; sw < a.post; ++sw) {
      double* o = cur[l] == L.x ? L.s : L.x;
      sweep(L, cur[l], o);
      cur[l] = o;
    }
  }
}

}  // namespace

void small_stage1(Handle& h, const double* x) {
#define CALL(P)                                                                                          \
  launch_pdl(k_s1_small<P>, grid_of(h.K, Cfg<P>::EPC), Cfg<P>::THREADS, 0, h.stream, h.mesh(), h.dtab, x, h.tz.ptr)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void small_stage2(Handle& h, int mode, const double* x, const double* b, double wm, double dt, double omega,
                  double* out, int k0, int kend) {
  const double dteta = dt * h.prob.eta;
  if (kend < 0) kend = h.K;
#define CALL(P)                                                                                                \
  do {                                                                                                         \
    const unsigned grid = grid_of(kend - k0, Cfg<P>::EPC);                                                     \
    if (mode == 0)                                                                                             \
      launch_pdl(k_s2_small<P, 0>, grid, Cfg<P>::THREADS, 0, h.stream, h.mesh(), h.dtab, h.E32.ptr, h.D.ptr, x, \
                 h.tz.ptr, b, wm, dteta, dt, h.Pinv32.ptr, omega, out, k0, kend);                             \
    else                                                                                                       \
      launch_pdl(k_s2_small<P, 1>, grid, Cfg<P>::THREADS, 0, h.stream, h.mesh(), h.dtab, h.E32.ptr, h.D.ptr, x, \
                 h.tz.ptr, b, wm, dteta, dt, h.Pinv32.ptr, omega, out, k0, kend);                             \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

// out[:, c] = -S_c e_c for c < ncols (X = identity, stride = N * Kp; Tz: 2
// stride values per column; zero: stride zeros)
void small_dense_columns(Handle& h, const double* X, double* Tz, const double* zero, double wm, double dt, double* out,
                         int ncols) {
  const long stride = h.vec_len();
  const double dteta = dt * h.prob.eta;
#define CALL(P)                                                                                              \
  do {                                                                                                       \
    const dim3 grid(grid_of(h.K, Cfg<P>::EPC), ncols);                                                       \
    k_s1_batch<P><<<grid, Cfg<P>::THREADS, 0, h.stream>>>(h.mesh(), h.dtab, X, Tz, stride);                  \
    k_s2_batch<P><<<grid, Cfg<P>::THREADS, 0, h.stream>>>(h.mesh(), h.dtab, h.E32.ptr, h.D.ptr, X, Tz, zero, \
                                                          wm, dteta, dt, out, stride);                       \
  } while (0)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  h.launches += 2;
}

void small_zero(Handle& h, const double* b, double omega, double* out) {
#define CALL(P)                                                                                              \
  launch_pdl(k_bj_small<P>, grid_of(h.K, Cfg<P>::EPC), Cfg<P>::THREADS, 0, h.stream, h.K, h.Kp, h.Pinv32.ptr, b, \
             omega, out)
  LDG_DISPATCH_P(h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

}  // namespace ldgb

namespace ldgb {

// CTAs of the tail kernel's cluster (LDG_TAIL_CLUSTER: 1, 4, 8 or 16).
// Measured V-cycle at 256^2 (p = 0 / 2 / 4): one block 273 / 513 / 1437 us;
// clusters of 8 or 16 on the same levels 292 / 525 / 1438 us (the cluster
// barrier + fence per phase and the level data leaving the one SM's L1 cost
// more than the extra issue rate buys); with the p >= 2 levels below 600 or
// 2048 elements in the tail as well 295 / 542-573 / 1490-1595 us.  Off.
int tail_cluster() {
  static const int cl = [] {
    const char* e = std::getenv("LDG_TAIL_CLUSTER");
    const int v = e ? std::atoi(e) : 1;
    return (v == 4 || v == 8 || v == 16) ? v : 1;
  }();
  return cl;
}

// one cluster of `cl` CTAs, programmatic stream serialisation as launch_pdl
template <typename... KArgs, typename... Args>
void launch_cluster(void (*kern)(KArgs...), int cl, int threads, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cl;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  LDG_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// The V-cycle below level `top` (inclusive) of h's hierarchy in one block
// (see k_tail); x of the top level receives the result, b its right-hand side.
void small_tail_vcycle(Handle& h0, int top, double wm, double dt, double omega, int pre, int post, int coarse_min) {
  TailArgs a{};
  const int nl = 1 + static_cast<int>(h0.coarse.size());
  a.nlev = nl - top;
  if (a.nlev < 1 || a.nlev > kTailMax) throw Error(LDG_EINVAL, "tail V-cycle: level count out of range");
  for (int l = 0; l < a.nlev; ++l) {
    Handle& L = *h0.coarse[top + l - 1];
    TailLevel& t = a.lv[l];
    t.m = L.mesh();
    t.E32 = L.E32.ptr;
    t.Pinv32 = L.Pinv32.ptr;
    t.D = L.D.ptr;
    t.x = L.mg_x.ptr;
    t.s = L.mg_s.ptr;
    t.b = L.mg_b.ptr;
    t.r = L.mg_r.ptr;
    t.tz = L.tz.ptr;
    t.children = L.mg_children.ptr;
    t.Pm = L.mg_P.ptr;
    t.dim = L.dim;
  }
  a.wm = wm;
  a.dt = dt;
  a.dteta = dt * h0.prob.eta;
  a.omega = omega;
  a.pre = pre;
  a.post = post;
  a.coarse_min = coarse_min;
  const Handle& top_h = *h0.coarse[top - 1];  // all tail levels share its degree (p-coarsening, ldg_mg.cu)
  const int cl = tail_cluster();
#define CALL(P)                                                                                \
  do {                                                                                         \
    if (cl == 16) {                                                                            \
      static bool np = false;                                                                  \
      if (!np) {                                                                               \
        LDG_CUDA(cudaFuncSetAttribute(k_tail<P, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)); \
        np = true;                                                                             \
      }                                                                                        \
      launch_cluster(k_tail<P, 16>, 16, Cfg<P>::THREADS, h0.stream, a, top_h.dtab);            \
    } else if (cl == 8) {                                                                      \
      launch_cluster(k_tail<P, 8>, 8, Cfg<P>::THREADS, h0.stream, a, top_h.dtab);              \
    } else if (cl == 4) {                                                                      \
      launch_cluster(k_tail<P, 4>, 4, Cfg<P>::THREADS, h0.stream, a, top_h.dtab);              \
    } else {                                                                                   \
      launch_pdl(k_tail<P, 1>, 1, Cfg<P>::THREADS, 0, h0.stream, a, top_h.dtab);               \
    }                                                                                          \
  } while (0)
  LDG_DISPATCH_P(top_h.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++h0.launches;
}

}  // namespace ldgb
