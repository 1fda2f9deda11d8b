// K6 block-SpMV kernels and K7 Krylov solve of one implicit-Euler step.
//
// The reference factorises W + dt A with SparseLU every step and checks
// ||lhs y - rhs|| / max(||rhs||, 1) <= 1e-10 (system.hpp:155-205).  Here the
// flux rows are eliminated exactly — their diagonal blocks are the block-
// diagonal mass matrix, Z^m = M^-1 (V_Z^m - B^m C) — and BiCGStab runs on the
// Schur system of the primary variable,
//     S_c C = [wM + dt(eta S - sum_m E^m M^-1 B^m)] C
//           = wM C^n + dt (V_C - sum_m E^m M^-1 V_Z^m),
// applied matrix-free in two block-SpMV passes (stage 1: t^m = M^-1 B^m x,
// stage 2: y = wMx + dt(eta S x - sum_m E^m t^m)).  The reference residual
// contract is then checked on the full 3KN system with the full block-SpMV.
#include <cmath>
#include <vector>

#include "ldg_internal.hpp"

namespace ldgb {

namespace {

inline unsigned grid_of(long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

__global__ void k_lincomb3(long n, double a, const double* x, double b, const double* y, double c, const double* z,
                           double* out) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    double v = a * x[i];
    if (y) v += b * y[i];
    if (z) v += c * z[i];
    out[i] = v;
  }
}

__global__ void k_axpby(long n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}

constexpr int kRedBlocks = 296;  // 2 x 148 SMs
constexpr int kMaxDots = 4;

struct DotArgs {
  const double* x[kMaxDots];
  const double* y[kMaxDots];
};

// Deterministic two-pass reduction: fixed grid, fixed per-block order.
__global__ void __launch_bounds__(256) k_dots_partial(long n, int nd, DotArgs a, double* __restrict__ part) {
  double s[kMaxDots] = {0.0, 0.0, 0.0, 0.0};
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    for (int d = 0; d < nd; ++d) s[d] += a.x[d][i] * a.y[d][i];
  __shared__ double sh[kMaxDots][8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int d = 0; d < nd; ++d) {
    double v = s[d];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[d][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < nd) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += sh[threadIdx.x][w];
    part[threadIdx.x * kRedBlocks + blockIdx.x] = v;
  }
}

__global__ void k_dots_final(int nd, const double* __restrict__ part, double* __restrict__ out) {
  const int d = threadIdx.x;
  if (d >= nd) return;
  double v = 0.0;
  for (int b = 0; b < kRedBlocks; ++b) v += part[d * kRedBlocks + b];
  out[d] = v;
}

// SoA [nvec][N][Kp] <-> k-major [nvec][K][N]
__global__ void k_soa_to_kmajor(int K, int N, long Kp, int nvec, const double* __restrict__ soa,
                                double* __restrict__ km) {
  const long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  const long total = static_cast<long>(nvec) * K * N;
  if (idx >= total) return;
  const long v = idx / (static_cast<long>(K) * N);
  const long r = idx % (static_cast<long>(K) * N);
  const long k = r / N, j = r % N;
  km[idx] = soa[(v * N + j) * Kp + k];
}

__global__ void k_kmajor_to_soa(int K, int N, long Kp, int nvec, const double* __restrict__ km,
                                double* __restrict__ soa) {
  const long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  const long total = static_cast<long>(nvec) * K * N;
  if (idx >= total) return;
  const long v = idx / (static_cast<long>(K) * N);
  const long r = idx % (static_cast<long>(K) * N);
  const long k = r / N, j = r % N;
  soa[(v * N + j) * Kp + k] = km[idx];
}

#define LDG_DISPATCH_P(p, CALL) \
  switch (p) {                  \
    case 0: { CALL(0); break; } \
    case 1: { CALL(1); break; } \
    case 2: { CALL(2); break; } \
    case 3: { CALL(3); break; } \
    default: { CALL(4); break; } \
  }

}  // namespace
void launch_lincomb3(Handle& h, long n, double a, const double* x, double b, const double* y, double c,
                     const double* z, double* out) {
  k_lincomb3<<<kRedBlocks * 4, 256, 0, h.stream>>>(n, a, x, b, y, c, z, out);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_axpby(Handle& h, long n, double a, const double* x, double b, double* y) {
  k_axpby<<<kRedBlocks * 4, 256, 0, h.stream>>>(n, a, x, b, y);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_dots(Handle& h, long n, int nd, const double* const* xs, const double* const* ys, double* out_host) {
  DotArgs a{};
  for (int d = 0; d < nd; ++d) {
    a.x[d] = xs[d];
    a.y[d] = ys[d];
  }
  k_dots_partial<<<kRedBlocks, 256, 0, h.stream>>>(n, nd, a, h.red.ptr);
  k_dots_final<<<1, 32, 0, h.stream>>>(nd, h.red.ptr, h.red.ptr + kMaxDots * kRedBlocks);
  LDG_CUDA(cudaGetLastError());
  h.launches += 2;
  LDG_CUDA(cudaMemcpyAsync(h.red_host, h.red.ptr + kMaxDots * kRedBlocks, sizeof(double) * nd,
                           cudaMemcpyDeviceToHost, h.stream));
  LDG_CUDA(cudaStreamSynchronize(h.stream));
  for (int d = 0; d < nd; ++d) out_host[d] = h.red_host[d];
}

void launch_soa_to_kmajor(Handle& h, const double* soa, int nvec, double* km) {
  const long total = static_cast<long>(nvec) * h.K * h.N;
  k_soa_to_kmajor<<<grid_of(total, 256), 256, 0, h.stream>>>(h.K, h.N, h.Kp, nvec, soa, km);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_kmajor_to_soa(Handle& h, const double* km, int nvec, double* soa) {
  const long total = static_cast<long>(nvec) * h.K * h.N;
  k_kmajor_to_soa<<<grid_of(total, 256), 256, 0, h.stream>>>(h.K, h.N, h.Kp, nvec, km, soa);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

size_t reduction_scratch() { return static_cast<size_t>(kMaxDots) * kRedBlocks + kMaxDots; }

// ------------------------------------------------------------------ driver

void assemble_step(Handle& h, double t) {
  launch_project_df(h, t, h.rule_ptr(), h.rule_R());        // K2: d, f (system.hpp:112-113)
  launch_rhs(h, t);                                          // K5: V (system.hpp:142-150)
  launch_assemble(h, kModeE, h.E.ptr);                       // K3: E^m (system.hpp:115-117)
  h.assembled = true;
  h.t_assembled = t;
}

namespace {

double norm2(Handle& h, const double* x, long n) {
  const double* xs[1] = {x};
  double r;
  launch_dots(h, n, 1, xs, xs, &r);
  return std::sqrt(r);
}

// Schur operator: y = wm M x + dt (eta S x - sum E^m M^-1 B^m x)
void schur_apply(Handle& h, double wm, double dt, const double* x, double* y) {
  launch_stage1(h, nullptr, 0.0, x, 1.0, h.tz.ptr);
  launch_stage2(h, x, wm, dt * h.prob.eta, h.tz.ptr, dt, nullptr, 0.0, y);
}

void precond(Handle& h, int pc, double wm, double dt, const double* x, double* y) {
  if (pc == 2)
    mg_vcycle(h, wm, dt, x, y);
  else if (pc == 1)
    launch_bjac_apply(h, x, y);
  else
    LDG_CUDA(cudaMemcpyAsync(y, x, sizeof(double) * h.vec_len(), cudaMemcpyDeviceToDevice, h.stream));
}

}  // namespace

// One linear solve with the operators of the last assemble_step: wm = 1, dt
// for W + dt A (euler_step), wm = 0, dt = 1 for A (solve_stationary).
// Y holds the previous state on entry and the solution on exit.
int solve_step(Handle& h, double wm, double dt, const ldg_solver_opts& o, ldg_step_stats* st) {
  const long n = h.vec_len();
  const long n3 = 3 * n;
  double* Y = h.Y.ptr;
  double* C = Y + 2 * n;
  const double* VZ = h.Vv.ptr;
  const double* VC = h.Vv.ptr + 2 * n;
  LDG_CUDA(cudaMemcpyAsync(h.Yold.ptr, Y, sizeof(double) * n3, cudaMemcpyDeviceToDevice, h.stream));
  const double* Cold = h.Yold.ptr + 2 * n;

  // Schur right-hand side b = wm M C^n + dt (V_C - sum E^m M^-1 V_Z^m)
  launch_stage1(h, VZ, 1.0, nullptr, 0.0, h.tz.ptr);
  launch_stage2(h, wm != 0.0 ? Cold : nullptr, wm, 0.0, h.tz.ptr, dt, VC, dt, h.kr_b.ptr);

  // full right-hand side of the reference system: r = W Y^n + dt V
  LDG_CUDA(cudaMemcpyAsync(h.full_r.ptr, h.Vv.ptr, sizeof(double) * n3, cudaMemcpyDeviceToDevice, h.stream));
  launch_axpby(h, n3, 0.0, h.full_r.ptr, dt, h.full_r.ptr);
  if (wm != 0.0) launch_stage2(h, Cold, wm, 0.0, nullptr, 0.0, VC, dt, h.full_r.ptr + 2 * n);
  const double rhs_norm = norm2(h, h.full_r.ptr, n3);
  const double contract = o.contract_tol > 0.0 ? o.contract_tol : 1e-10;

  // precond: 0 none, 1 block-Jacobi, 2 multigrid with the smoother on FP32
  // copies of E / block inverses (mixed precision), 3 multigrid all-FP64
  int pc = o.precond;
  if (pc >= 2 && !mg_build(h)) pc = 1;  // no FK hierarchy (general mesh): block-Jacobi
  if (pc >= 1) launch_bjac_setup(h, wm, dt);
  if (pc >= 2) {
    h.mg_f32 = pc == 2;
    pc = 2;
    mg_setup_step(h, h.t_assembled, wm, dt);
  }

  const double bnorm = norm2(h, h.kr_b.ptr, n);
  // stopping test on the Schur residual: the user's rtol/atol, tightened so
  // that the full-system contract (Schur residual = C-row residual) holds
  double tol = std::max(o.rtol * bnorm, o.atol);
  if (o.check_residual) {
    const double tc = 0.25 * contract * std::max(rhs_norm, 1.0);
    tol = tol > 0.0 ? std::min(tol, tc) : tc;
  }
  if (!(tol > 0.0)) tol = 1e-300;

  // BiCGStab (right preconditioned), x = C warm-started from C^n
  double* r = h.kr_r.ptr;
  double* rh = h.kr_rh.ptr;
  double* p = h.kr_p.ptr;
  double* v = h.kr_v.ptr;
  double* s = h.kr_s.ptr;
  double* t = h.kr_t.ptr;
  double* ph = h.kr_ph.ptr;
  double* sh = h.kr_sh.ptr;
  int applies = 0;
  schur_apply(h, wm, dt, C, r);
  ++applies;
  launch_axpby(h, n, 1.0, h.kr_b.ptr, -1.0, r);  // r = b - A x
  LDG_CUDA(cudaMemcpyAsync(rh, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, h.stream));
  LDG_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * n, h.stream));
  LDG_CUDA(cudaMemsetAsync(v, 0, sizeof(double) * n, h.stream));
  double rho = 1.0, alpha = 1.0, omega = 1.0;
  // three host synchronisations per iteration: (rh,v); (t,s),(t,t),(s,s); (r,r),(rh,r)
  double rr_rhr[2];
  {
    const double* xs[2] = {r, rh};
    const double* ys[2] = {r, r};
    launch_dots(h, n, 2, xs, ys, rr_rhr);
  }
  double rnorm = std::sqrt(rr_rhr[0]);
  double rho1 = rr_rhr[1];
  int it = 0;
  bool converged = rnorm <= tol;
  while (!converged && it < o.maxit) {
    ++it;
    if (rho1 == 0.0 || !std::isfinite(rho1)) {
      // breakdown: restart with the current residual as shadow vector
      LDG_CUDA(cudaMemcpyAsync(rh, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, h.stream));
      LDG_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * n, h.stream));
      LDG_CUDA(cudaMemsetAsync(v, 0, sizeof(double) * n, h.stream));
      rho = alpha = omega = 1.0;
      rho1 = rnorm * rnorm;
      if (rho1 == 0.0) break;
    }
    const double beta = (rho1 / rho) * (alpha / omega);
    launch_lincomb3(h, n, 1.0, r, beta, p, -beta * omega, v, p);  // p = r + beta (p - omega v)
    precond(h, pc, wm, dt, p, ph);
    schur_apply(h, wm, dt, ph, v);
    ++applies;
    double rv;
    {
      const double* xs[1] = {rh};
      const double* ys[1] = {v};
      launch_dots(h, n, 1, xs, ys, &rv);
    }
    alpha = rho1 / rv;
    launch_lincomb3(h, n, 1.0, r, -alpha, v, 0.0, nullptr, s);  // s = r - alpha v
    precond(h, pc, wm, dt, s, sh);
    schur_apply(h, wm, dt, sh, t);
    ++applies;
    double ts[3];
    {
      const double* xs[3] = {t, t, s};
      const double* ys[3] = {s, t, s};
      launch_dots(h, n, 3, xs, ys, ts);
    }
    if (std::sqrt(ts[2]) <= tol) {  // converged on s: x += alpha p^
      launch_lincomb3(h, n, 1.0, C, alpha, ph, 0.0, nullptr, C);
      rnorm = std::sqrt(ts[2]);
      converged = true;
      break;
    }
    omega = ts[1] != 0.0 ? ts[0] / ts[1] : 0.0;
    launch_lincomb3(h, n, 1.0, C, alpha, ph, omega, sh, C);  // x += alpha p^ + omega s^
    launch_lincomb3(h, n, 1.0, s, -omega, t, 0.0, nullptr, r);  // r = s - omega t
    {
      const double* xs[2] = {r, rh};
      const double* ys[2] = {r, r};
      launch_dots(h, n, 2, xs, ys, rr_rhr);
    }
    rnorm = std::sqrt(rr_rhr[0]);
    rho = rho1;
    rho1 = rr_rhr[1];
    if (!std::isfinite(rnorm)) break;
    converged = rnorm <= tol;
    if (omega == 0.0) break;
  }

  // flux recovery Z^m = M^-1 (V_Z^m - B^m C), written into Y[0 .. 2n)
  launch_stage1(h, VZ, 1.0, C, -1.0, Y);

  // reference residual contract on the full system (system.hpp:198-203)
  launch_full_apply(h, Y, wm, dt, h.full_y.ptr);
  launch_axpby(h, n3, -1.0, h.full_r.ptr, 1.0, h.full_y.ptr);
  const double res = norm2(h, h.full_y.ptr, n3) / std::max(rhs_norm, 1.0);
  if (st) {
    st->iterations += it;
    st->applies += applies;
    st->schur_relres = bnorm > 0.0 ? rnorm / bnorm : rnorm;
    st->residual = res;
  }
  if (o.check_residual && !(res <= contract)) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "linear solve residual %.6e exceeds tolerance (eta = %f, p = %d; BiCGStab %d iterations, "
             "Schur residual %.3e)",
             res, h.prob.eta, h.p, it, rnorm);
    throw Error(LDG_ENOCONV, buf);
  }
  return it;
}

}  // namespace ldgb
