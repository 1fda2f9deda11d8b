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
                  double* out) {
  const double dteta = dt * h.prob.eta;
  const int k0 = 0, kend = h.K;
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
