// K7 driver: the implicit-Euler solve of one step over a Team of ranks
// (one rank on one GPU, strips over several GPUs with NCCL, or several
// virtual ranks on one GPU for validating the decomposition).
//
// The reference factorises W + dt A with SparseLU every step and checks
// ||lhs y - rhs|| / max(||rhs||, 1) <= 1e-10 (system.hpp:155-205).  Here the
// flux rows are eliminated exactly — their diagonal blocks are the block-
// diagonal mass matrix, Z^m = M^-1 (V_Z^m - B^m C) — and BiCGStab runs on the
// Schur system of the primary variable,
//     S_c C = [wM + dt(eta S - sum_m E^m M^-1 B^m)] C
//           = wM C^n + dt (V_C - sum_m E^m M^-1 V_Z^m),
// applied in two block-SpMV passes (stage 1: t^m = M^-1 B^m x, stage 2:
// y = wMx + dt(eta S x - sum_m E^m t^m)), preconditioned by a geometric
// multigrid V-cycle (ldg_mg.cu builds the levels).  The reference residual
// contract is checked on the full 3KN system afterwards.
//
// Exchange points: before stage 1 the ghost column of x, before
// stage 2 the ghost column of t^1, t^2 (and of Y before the full apply);
// every reduction is a sum over local ranks then one ncclAllReduce.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <optional>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <string>
#include <vector>

#include "ldg_internal.hpp"

namespace ldgb {

size_t reduction_scratch();
void launch_dots_async(Handle& h, int nd, const double* const* xs, const double* const* ys);
double* dots_result(Handle& h);

namespace {

// V-cycle parameters (LDG_MG_PRE0 / POST0 / PRE1 / POST1 override the level-0/1 sweeps in tuning runs)
double env_or(const char* name, double dflt) {
  const char* s = std::getenv(name);
  return s ? std::atof(s) : dflt;
}
// Sweeps (pre counts the residual-free first sweep from x = 0), per degree
// of the finest level.  Level-0 sweeps stream at ~60 % of HBM bandwidth
// while the coarse levels are latency-bound, so smoothing sits on level 0:
// V(5,5) there and V(2,1) below measured 6.1/8.9/17.9/33.8/68.4 ms/step at
// 256^2, p = 0..4, against 5.6/11.4/24.8/45/95 with V(2,2) everywhere.  With
// the p-coarsened hierarchy and Chebyshev level 0 the per-degree optimum
// (scripts/gpu_envs_perp.sh, stable to 0.1 ms) is level 0 V(6,6) / V(4,5) /
// V(4,6) / V(5,6) / V(5,6) and level 1 V(2,1) except V(1,1) at p = 4
// (ms/step 5.17 / 7.47 / 11.11 / 20.11 / 38.49 against 5.59 / 7.67 / 11.88 /
// 20.55 / 41.09 with V(5,5) + V(2,1)).
// Damped block-Jacobi weight and the sweeps of the levels below level 1,
// re-tuned after p-coarsening and Chebyshev level 0 made the coarse levels
// cheap relative to their effect (5-step C2 bench, all degrees): coarse
// V(2,1) with omega 0.7 1.775e8 DOF-updates/s; V(2,2) + 0.7 1.943e8; V(2,2)
// + 0.8 1.989e8 (p = 0..4: 4.8 / 6.4 / 8.7 / 15.0 / 34.2 ms); V(2,2) + 0.9
// 4.4 / 5.9 / 8.7 / 15.3 / 36.3 ms; V(3,2), V(2,3), V(3,3), V(4,4), V(1,1)
// all lower.  omega per finest degree: 0.9 for p <= 1, 0.8 above — on
// unjittered meshes solved by one rank.  Jittered meshes keep 0.7: with 0.8
// BASELINE config 4 (2048^2, jitter 0.2h, p = 3) went from 22 to 24
// iterations, and a 2-rank strip run at p = 1 with 0.9 (the per-kernel
// coarse levels, no single-block tail) from 42 to 184 iterations over 3
// steps; multi-rank teams keep 0.7 too.
constexpr double kOmegaP[5] = {0.9, 0.9, 0.8, 0.8, 0.8};
constexpr double kOmegaSafe = 0.7;
// Chebyshev interval of level 0 (below, sweep_cheb):
// upper end of the interval = safety x the power-iteration estimate: 1.08
// (5-step C2 bench: 1.15 p = 2 15.4 iterations / 11.2 ms, 1.05 and 1.08
// 15.0 / 10.9 ms, other degrees unchanged; 1.0 diverges towards 21
// iterations at p = 0).  Ratio 20 (10: p = 4 20 iterations; 30: +1 at p <= 3).
// (plain meshes, set_omega; jittered meshes / strips keep 1.15: config 4
// went from 22 to 24 iterations with 1.08 and coarse V(2,2))
double kChebSafety = 1.15;
// coarse post-sweeps: 2 on plain meshes (above), 1 on jittered meshes / strips
// (config 4 with 2: 24 instead of 22 iterations, 1.39 instead of 1.25 s/step)
int kPost = 1;  // set with kOmega
double kOmega = kOmegaSafe;  // set per team at the top of every V-cycle (vcycle, l = 0)
void set_omega(const Team& T) {
  const Handle& h = T.h0();
  const int p = h.p < 0 ? 0 : (h.p > 4 ? 4 : h.p);
  const bool plain = h.jitter == 0.0 && h.dim > 0 && T.size == 1 && T.nlocal() == 1;
  kOmega = plain ? kOmegaP[p] : kOmegaSafe;
  kPost = plain ? 2 : 1;
  // (p = 4 with the extrapolated start and the 4 -> 2 -> 1 chain: 1.04 gave
  // 19.71 -> 19.29 ms per step; at p = 0 it cost 0.14 ms, 1.00 diverges
  // towards 21 iterations at p = 0)
  kChebSafety = plain ? (p == 4 ? 1.04 : 1.08) : 1.15;
}
constexpr int kPre = 2;           // coarse levels
constexpr int kCoarseSweeps = 2;  // at least, on the coarsest level
// level 0 re-swept with the retuned coarse levels (5-step C2 bench): p = 1
// V(5,6) 5.6 ms / 10 iterations (V(4,5) 5.8 / 11), p = 4 V(5,7) 33.7 / 15
// (V(5,6) 34.2 / 16); p = 0, 2, 3 unchanged (V(4,4), V(3,5), V(4,5),
// V(6,6) elsewhere all slower; symmetric counts lose up to 2x at p = 3).
// With the extrapolated Krylov start (fewer, so relatively more valuable,
// V-cycles) re-swept on the 5-step C2 bench (ms per step p = 0..4): V(6,6) /
// V(5,6) / V(4,6) / V(5,6) / V(5,7) 4.68 / 4.83 / 6.85 / 11.31 / 23.78;
// V(6,7) everywhere 4.79 / 4.73 / 7.00 / 11.24 / 23.51; V(5,6) everywhere
// 4.98 / 4.82 / 6.62 / 11.32 / 23.56; V(4,5), V(3,5), V(4,6) all slower.
constexpr int kPre0P[5] = {6, 6, 5, 6, 6}, kPost0P[5] = {6, 7, 6, 7, 7};
// level 1 V(1,1) except V(2,1) at p = 3 (with the retuned coarse levels:
// p = 0..2 4.3 / 5.8 / 8.5 ms against 4.4 / 5.9 / 8.7 with V(2,1); V(2,2),
// V(3,2) slower)
constexpr int kPre1P[5] = {1, 1, 1, 2, 1}, kPost1P[5] = {1, 1, 1, 1, 1};
int sweeps_of(const char* env, const int* table, int p) {
  const char* s = std::getenv(env);
  return s ? std::atoi(s) : table[p < 0 ? 0 : (p > 4 ? 4 : p)];
}
int pre_of(int p, int l) {
  return l == 0 ? sweeps_of("LDG_MG_PRE0", kPre0P, p) : (l == 1 ? sweeps_of("LDG_MG_PRE1", kPre1P, p) : kPre);
}
int post_of(int p, int l) {
  return l == 0 ? sweeps_of("LDG_MG_POST0", kPost0P, p) : (l == 1 ? sweeps_of("LDG_MG_POST1", kPost1P, p) : kPost);
}

#define LDG_NCCL(call)                                                                          \
  do {                                                                                          \
    ncclResult_t r_ = (call);                                                                   \
    if (r_ != ncclSuccess) throw Error(LDG_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

Handle& level_of(Handle& h, int l) { return l == 0 ? h : *h.coarse[l - 1]; }

// named per-rank vectors: a Team operation names a vector, each rank
// resolves it to its own buffer
enum Vec : int {
  kR, kRh, kP, kV, kS, kT, kPh, kSh, kB, kC, kY, kTz, kMgX, kMgB, kMgR, kMgS, kMgZ, kVz, kVc, kFullR, kFullY, kCold,
  kYold, kNone
};

// FGMRES basis vectors: V_j = kGmV0 + j, Z_j = kGmZ0 + j
constexpr int kGmV0 = 1000, kGmZ0 = 2000;
Vec gmV(int j) { return static_cast<Vec>(kGmV0 + j); }
Vec gmZ(int j) { return static_cast<Vec>(kGmZ0 + j); }

double* vp(Handle& h, Vec v) {
  const long n = h.vec_len();
  if (v >= kGmZ0) return h.gm_Z.ptr + (v - kGmZ0) * n;
  if (v >= kGmV0) return h.gm_V.ptr + (v - kGmV0) * n;
  switch (v) {
    case kR: return h.kr_r.ptr;
    case kRh: return h.kr_rh.ptr;
    case kP: return h.kr_p.ptr;
    case kV: return h.kr_v.ptr;
    case kS: return h.kr_s.ptr;
    case kT: return h.kr_t.ptr;
    case kPh: return h.kr_ph.ptr;
    case kSh: return h.kr_sh.ptr;
    case kB: return h.kr_b.ptr;
    case kC: return h.Y.ptr + 2 * n;
    case kY: return h.Y.ptr;
    case kTz: return h.tz.ptr;
    case kMgX: return h.mg_x.ptr;
    case kMgB: return h.mg_b.ptr;
    case kMgR: return h.mg_r.ptr;
    case kMgS: return h.mg_s.ptr;
    case kMgZ: return h.mg_zero.ptr;
    case kVz: return h.Vv.ptr;
    case kVc: return h.Vv.ptr + 2 * n;
    case kFullR: return h.full_r.ptr;
    case kFullY: return h.full_y.ptr;
    case kCold: return h.Yold.ptr + 2 * n;
    case kYold: return h.Yold.ptr;
    default: return nullptr;
  }
}

// ---------------------------------------------------------------- exchange

void copy_cols(double* dst, long dpitch, const double* src, long spitch, long width, long rows, cudaStream_t s) {
  LDG_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * dpitch, src, sizeof(double) * spitch, sizeof(double) * width,
                             rows, cudaMemcpyDeviceToDevice, s));
}

bool cudaStreamIsCapturing_(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  LDG_CUDA(cudaStreamIsCapturing(s, &st));
  return st != cudaStreamCaptureStatusNone;
}

// Ghost-column refresh of vector v (ncomp blocks of N planes) on level
// `level` of every local rank, split for overlap with computation:
// halo_begin copies the ghosts of local neighbours (virtual ranks: device
// copies, complete in stream order) and posts the exchange with remote ones
// (owned boundary columns packed on the main stream, ncclSend/Recv on the
// team's comm stream); halo_end joins the comm stream and unpacks.  Returns
// whether a remote exchange is in flight.
bool halo_begin(Team& T, int level, Vec v, int ncomp) {
  if (T.size == 1) return false;
  bool remote = false;
  for (int r = 0; r < T.nlocal(); ++r) {
    Handle& L = level_of(*T.ranks[r], level);
    const int g = T.first + r;
    const long rows = static_cast<long>(ncomp) * L.N;
    if (L.ghost_left) {
      if (Handle* nb = T.local(g - 1)) {
        Handle& R = level_of(*nb, level);
        copy_cols(vp(L, v) + L.ghost_left_off(), L.Kp, vp(R, v) + R.own_right_off(), R.Kp, L.dim, rows, T.stream);
      } else {
        remote = true;
      }
    }
    if (L.ghost_right) {
      if (Handle* nb = T.local(g + 1)) {
        Handle& R = level_of(*nb, level);
        copy_cols(vp(L, v) + L.ghost_right_off(), L.Kp, vp(R, v) + R.own_left_off(), R.Kp, L.dim, rows, T.stream);
      } else {
        remote = true;
      }
    }
  }
  if (!remote) return false;
  auto* comm = static_cast<ncclComm_t>(T.nccl);
  if (!comm) throw Error(LDG_ENCCL, "ranks without a communicator");
  if (T.nlocal() != 1) throw Error(LDG_ENCCL, "remote halo: one rank per process expected");
  if (!T.comm_stream) {
    if (cudaStreamIsCapturing_(T.stream)) throw Error(LDG_ENCCL, "comm stream created during graph capture");
    LDG_CUDA(cudaStreamCreateWithFlags(&T.comm_stream, cudaStreamNonBlocking));
    for (auto& e : T.comm_ev) LDG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  Handle& L = level_of(T.h0(), level);
  const int g = T.first;
  const long rows = static_cast<long>(ncomp) * L.N;
  const long cnt = rows * L.dim;
  const bool left = L.ghost_left != 0, right = L.ghost_right != 0;
  if (static_cast<long>(T.send_l.n) < cnt) {
    // sized once for the largest exchange (3 components on level 0): the
    // V-cycle graphs bake these pointers, so they must never move
    if (cudaStreamIsCapturing_(T.stream)) throw Error(LDG_ENCCL, "halo staging allocated during graph capture");
    const long cap = std::max(cnt, 3L * T.h0().N * T.h0().dim);
    for (DBuf<double>* b : {&T.send_l, &T.send_r, &T.recv_l, &T.recv_r}) b->alloc(cap, nullptr);
  }
  if (left) copy_cols(T.send_l.ptr, L.dim, vp(L, v) + L.own_left_off(), L.Kp, L.dim, rows, T.stream);
  if (right) copy_cols(T.send_r.ptr, L.dim, vp(L, v) + L.own_right_off(), L.Kp, L.dim, rows, T.stream);
  LDG_CUDA(cudaEventRecord(T.comm_ev[0], T.stream));
  LDG_CUDA(cudaStreamWaitEvent(T.comm_stream, T.comm_ev[0], 0));
  LDG_NCCL(ncclGroupStart());
  if (left) {
    LDG_NCCL(ncclSend(T.send_l.ptr, cnt, ncclDouble, g - 1, comm, T.comm_stream));
    LDG_NCCL(ncclRecv(T.recv_l.ptr, cnt, ncclDouble, g - 1, comm, T.comm_stream));
  }
  if (right) {
    LDG_NCCL(ncclSend(T.send_r.ptr, cnt, ncclDouble, g + 1, comm, T.comm_stream));
    LDG_NCCL(ncclRecv(T.recv_r.ptr, cnt, ncclDouble, g + 1, comm, T.comm_stream));
  }
  LDG_NCCL(ncclGroupEnd());
  LDG_CUDA(cudaEventRecord(T.comm_ev[1], T.comm_stream));
  return true;
}

void halo_end(Team& T, int level, Vec v, int ncomp) {
  LDG_CUDA(cudaStreamWaitEvent(T.stream, T.comm_ev[1], 0));
  Handle& L = level_of(T.h0(), level);
  const long rows = static_cast<long>(ncomp) * L.N;
  if (L.ghost_left) copy_cols(vp(L, v) + L.ghost_left_off(), L.Kp, T.recv_l.ptr, L.dim, L.dim, rows, T.stream);
  if (L.ghost_right) copy_cols(vp(L, v) + L.ghost_right_off(), L.Kp, T.recv_r.ptr, L.dim, L.dim, rows, T.stream);
}

void halo(Team& T, int level, Vec v, int ncomp) {
  if (halo_begin(T, level, v, ncomp)) halo_end(T, level, v, ncomp);
}

// Owned elements of a strip whose stencil reaches no ghost: the lowers of
// column a touch the ghost uppers of column a - 1, the uppers of column b - 1
// the ghost lowers of column b; everything in between is interior.
int interior_lo(const Handle& L) { return L.ghost_left ? L.dim : 0; }
int interior_hi(const Handle& L) { return L.ghost_right ? L.K - L.dim : L.K; }

// A stage on `level` whose input v needs fresh ghost columns.  On strips with
// thread-per-element kernels (ranged == true) the interior elements run while
// the halo is in flight and the boundary columns after it lands (virtual
// ranks take the same split, so one GPU exercises the element ranges);
// otherwise the whole level after the halo.  launch(L, k0, k1), k1 = -1: all.
template <typename F>
void staged(Team& T, int level, Vec v, int ncomp, bool ranged, F launch) {
  if (T.size == 1) {
    each(T, level, [&](Handle& L) { launch(L, 0, -1); });
    return;
  }
  const bool pending = halo_begin(T, level, v, ncomp);
  if (!ranged) {
    if (pending) halo_end(T, level, v, ncomp);
    each(T, level, [&](Handle& L) { launch(L, 0, -1); });
    return;
  }
  each(T, level, [&](Handle& L) { launch(L, interior_lo(L), interior_hi(L)); });
  if (pending) halo_end(T, level, v, ncomp);
  each(T, level, [&](Handle& L) {
    launch(L, 0, interior_lo(L));
    launch(L, interior_hi(L), L.K);
  });
}

// Launches per-rank partial dots (launch(h) issues launch_dots_async), then
// sums over local ranks in a fixed order (deterministic) and across
// processes with one ncclAllReduce.
template <typename F>
void reduce_dots(Team& T, int nd, F launch, double* out, int level = 0) {
  if (nd > kMaxRed || T.nlocal() > kMaxLocalRanks) throw Error(LDG_EINVAL, "reduction too large");
  for (auto& rp : T.ranks) launch(level_of(*rp, level));
  if (T.nlocal() == 1) {
    // one rank per process (or one GPU): the partials stay on the device, one
    // in-place ncclAllReduce across the processes, one read of the sums
    double* part = dots_result(level_of(T.h0(), level));
    if (T.nccl && T.size > 1)
      LDG_NCCL(ncclAllReduce(part, part, nd, ncclDouble, ncclSum, static_cast<ncclComm_t>(T.nccl), T.stream));
    LDG_CUDA(cudaMemcpyAsync(T.red_host, part, sizeof(double) * nd, cudaMemcpyDeviceToHost, T.stream));
  } else {
    // virtual ranks of one process: summed on the host in rank order
    // (deterministic), then across processes
    // rank r's partial sums in slot r + 1 of the scratch (slot 0: the result)
    for (int r = 0; r < T.nlocal(); ++r)
      LDG_CUDA(cudaMemcpyAsync(T.red_all.ptr + kMaxRed * (r + 1), dots_result(level_of(*T.ranks[r], level)),
                               sizeof(double) * nd,
                               cudaMemcpyDeviceToDevice, T.stream));
    LDG_CUDA(cudaMemcpyAsync(T.red_host + kMaxRed, T.red_all.ptr + kMaxRed, sizeof(double) * kMaxRed * T.nlocal(),
                             cudaMemcpyDeviceToHost, T.stream));
    LDG_CUDA(cudaStreamSynchronize(T.stream));
    for (int d = 0; d < nd; ++d) {
      double s = 0.0;
      for (int r = 0; r < T.nlocal(); ++r) s += T.red_host[kMaxRed * (r + 1) + d];
      T.red_host[d] = s;
    }
    if (T.nccl && T.size > T.nlocal()) {
      LDG_CUDA(cudaMemcpyAsync(T.red_all.ptr, T.red_host, sizeof(double) * nd, cudaMemcpyHostToDevice, T.stream));
      LDG_NCCL(ncclAllReduce(T.red_all.ptr, T.red_all.ptr, nd, ncclDouble, ncclSum,
                             static_cast<ncclComm_t>(T.nccl), T.stream));
      LDG_CUDA(cudaMemcpyAsync(T.red_host, T.red_all.ptr, sizeof(double) * nd, cudaMemcpyDeviceToHost, T.stream));
    }
  }
  LDG_CUDA(cudaStreamSynchronize(T.stream));
  for (int d = 0; d < nd; ++d) out[d] = T.red_host[d];
}

// Sum over all ranks of nd dot products of level-0 vectors (owned entries).
void dots(Team& T, int nd, const Vec* xs, const Vec* ys, double* out) {
  reduce_dots(
      T, nd,
      [&](Handle& h) {
        const double* px[4];
        const double* py[4];
        for (int d = 0; d < nd; ++d) {
          px[d] = vp(h, xs[d]);
          py[d] = vp(h, ys[d]);
        }
        launch_dots_async(h, nd, px, py);
      },
      out);
}

// squared 2-norm of a 3-block (Z1, Z2, C) vector
double sq_norm3(Team& T, Vec v) {
  double s[3];
  reduce_dots(
      T, 3,
      [&](Handle& h) {
        const long n = h.vec_len();
        const double* p[3] = {vp(h, v), vp(h, v) + n, vp(h, v) + 2 * n};
        launch_dots_async(h, 3, p, p);
      },
      s);
  return s[0] + s[1] + s[2];
}

double norm(Team& T, Vec x) {
  double r;
  dots(T, 1, &x, &x, &r);
  return std::sqrt(r);
}

// 2-norm of a level-l vector (owned entries, all ranks)
double norm_level(Team& T, int l, Vec x) {
  double r;
  reduce_dots(
      T, 1,
      [&](Handle& L) {
        const double* px = vp(L, x);
        launch_dots_async(L, 1, &px, &px);
      },
      &r, l);
  return std::sqrt(r);
}

template <typename F>
void each(Team& T, int level, F f) {
  for (auto& rp : T.ranks) f(level_of(*rp, level));
}

// ---------------------------------------------------------------- operators

// y = a1 (wM x) + b1 dt eta S x - g1 dt sum E^m t^m(x) + d1 w   (tz = M^-1 B x computed here)
void schur_like(Team& T, int level, bool f32, Vec x, double alpha, double beta, double gamma, Vec w, double delta,
                Vec y) {
  (void)f32;  // the FP32 smoother has its own kernels (f_stage1 / f_stage2)
  const bool ranged = !level_uses_rows(level_of(T.h0(), level));
  staged(T, level, x, 1, ranged,
         [&](Handle& L, int k0, int k1) { launch_stage1(L, nullptr, 0.0, vp(L, x), 1.0, L.tz.ptr, k0, k1); });
  staged(T, level, kTz, 2, ranged, [&](Handle& L, int k0, int k1) {
    launch_stage2(L, vp(L, x), alpha, beta, L.tz.ptr, gamma, vp(L, w), delta, vp(L, y), k0, k1);
  });
}

void schur_apply(Team& T, double wm, double dt, Vec x, Vec y) {
  schur_like(T, 0, false, x, wm, dt * T.h0().prob.eta, dt, kNone, 0.0, y);
}

// r = b - A x on a multigrid level
void residual(Team& T, int level, bool f32, double wm, double dt, Vec b, Vec x, Vec r) {
  schur_like(T, level, f32, x, -wm, -dt * T.h0().prob.eta, -dt, b, 1.0, r);
}

void bjac_axpy(Handle& L, bool f32, const double* x, double omega, double beta, double* y) {
  if (f32)
    launch_bjac_axpy_f32(L, x, omega, beta, y);
  else
    launch_bjac_axpy(L, x, omega, beta, y);
}

void smooth(Team& T, int level, bool f32, double wm, double dt, Vec b, Vec x) {
  residual(T, level, f32, wm, dt, b, x, kMgR);
  each(T, level, [&](Handle& L) { bjac_axpy(L, f32, L.mg_r.ptr, kOmega, 1.0, vp(L, x)); });
}

int levels(Team& T) { return 1 + static_cast<int>(T.h0().coarse.size()); }

// multigrid setup on side streams overlapping the right-hand side (LDG_SETUP_OVERLAP=0 off)
bool setup_overlap() {
  static const bool on = env_or("LDG_SETUP_OVERLAP", 1) != 0;
  return on;
}

// order of the in-time extrapolated start of the Euler solves (team_solve):
// 0 = C^n, 1 = linear, ... 4 (LDG_EXTRAP for tuning runs).  Measured on the
// 5-step C2 bench (ms per sweep step / FGMRES iterations at p = 4): C^n 81.4 /
// 18.0, linear 71.7 / 15.8, quadratic 61.3 / 13.0, cubic 55.9 / 11.2, quartic
// 52.0 / 10.2, quintic 51.7 / 10.0.
// Per degree, from the 20-step C2 bench (the 5-step one has too little
// history to tell; ms per step p = 0..4, order 4 / 5 / 6 / 7 / 8):
//   p = 0  2.84 / 2.72 / 2.64 / 2.51 / 2.61
//   p = 1  3.37 / 3.04 / 2.81 / 2.66 / 2.77
//   p = 2  5.32 / 4.31 / 3.92 / 3.68 / 3.84
//   p = 3  9.11 / 7.31 / 6.66 / 6.72 / 7.04
//   p = 4 18.87 / 15.11 / 12.92 / 13.13 / 13.73
// (sweep step 39.5 ms at order 4 -> 28.4 ms with the table).  The start only
// changes the iteration count: every solve stops on the same relative
// residual, and a poor extrapolation (non-smooth data) costs iterations, not
// accuracy.
constexpr int kExtrapP[5] = {7, 7, 7, 6, 6};
int extrap_order(int p) {
  static const int o = static_cast<int>(env_or("LDG_EXTRAP", -1));
  const int v = o >= 0 ? o : kExtrapP[p < 0 ? 0 : (p > 4 ? 4 : p)];
  return v > kExtrapMax ? kExtrapMax : v;
}

// The mixed-precision (f32) smoother runs every level through three
// operations: stage 1, stage 2 with the block-Jacobi update (x ping-ponging
// between two buffers) and the residual-free first sweep.  Kernel shape by
// level size: packed-stream thread-per-element kernels with the update fused
// (ldg_smooth.cu) on large levels, the row-parallel kernels (ldg_rows.cu) on
// mid-size levels (coalesced streams of data that no longer sit in L2), and
// the lane-split kernels with the update fused (ldg_small.cu) on the small,
// latency-bound levels.
bool fused(Team& T, int l, bool f32) {
  (void)T;
  (void)l;
  return f32;
}

enum Tier { kBig, kMid, kSmall };
Tier tier(const Handle& L) {
  if (!level_uses_rows(L)) return kBig;
  return level_is_small(L) ? kSmall : kMid;
}

void f_stage1(Handle& L, Vec x, int k0 = 0, int k1 = -1, bool chained = false) {
  switch (tier(L)) {
    case kBig: smooth_stage1(L, vp(L, x), k0, k1, chained); break;
    case kMid: rows_stage1(L, nullptr, 0.0, vp(L, x), 1.0, L.tz.ptr); break;
    default: small_stage1(L, vp(L, x)); break;
  }
}

void f_stage2(Handle& L, int mode, Vec x, Vec b, double wm, double dt, Vec out, int k0 = 0, int k1 = -1) {
  switch (tier(L)) {
    case kBig: smooth_stage2(L, mode, vp(L, x), vp(L, b), wm, dt, kOmega, vp(L, out), 0.0, 0, k0, k1); break;
    case kSmall: small_stage2(L, mode, vp(L, x), vp(L, b), wm, dt, kOmega, vp(L, out)); break;
    default: {
      const double eta = L.prob.eta;
      double* r = mode == 0 ? vp(L, out) : L.mg_r.ptr;
      rows_stage2<float>(L, L.E32.ptr, vp(L, x), -wm, -dt * eta, L.tz.ptr, -dt, vp(L, b), 1.0, r);
      if (mode == 1) {
        LDG_CUDA(cudaMemcpyAsync(vp(L, out), vp(L, x), sizeof(double) * L.vec_len(), cudaMemcpyDeviceToDevice,
                                 L.stream));
        rows_bjac<float>(L, L.Pinv32.ptr, r, kOmega, 1.0, vp(L, out));
      }
      break;
    }
  }
}

void f_zero(Handle& L, Vec b, Vec out) {
  switch (tier(L)) {
    case kBig: smooth_zero(L, vp(L, b), kOmega, vp(L, out)); break;
    case kMid: rows_bjac<float>(L, L.Pinv32.ptr, vp(L, b), kOmega, 0.0, vp(L, out)); break;
    default: small_zero(L, vp(L, b), kOmega, vp(L, out)); break;
  }
}

bool ranged_level(Team& T, int l) { return tier(level_of(T.h0(), l)) == kBig; }

// r = b - S_c x (fused levels)
// chained: x is the output of the sweep launched just before on this level
// (its stage 2 left the x traces, ldg_smooth.cu)
void residual_f(Team& T, int l, double wm, double dt, Vec b, Vec x, Vec r, bool chained = false) {
  const bool rg = ranged_level(T, l);
  staged(T, l, x, 1, rg, [&](Handle& L, int k0, int k1) { f_stage1(L, x, k0, k1, chained); });
  staged(T, l, kTz, 2, rg, [&](Handle& L, int k0, int k1) { f_stage2(L, 0, x, b, wm, dt, r, k0, k1); });
}

// xo = xi + omega P^-1 (b - S_c xi) (fused levels)
void sweep_f(Team& T, int l, double wm, double dt, Vec b, Vec xi, Vec xo, bool chained = false) {
  const bool rg = ranged_level(T, l);
  staged(T, l, xi, 1, rg, [&](Handle& L, int k0, int k1) { f_stage1(L, xi, k0, k1, chained); });
  staged(T, l, kTz, 2, rg, [&](Handle& L, int k0, int k1) { f_stage2(L, 1, xi, b, wm, dt, xo, k0, k1); });
}

// second Gram-Schmidt pass when the first removed more than (1 - eta) of |w|^2
constexpr double kReorthEta = 0.5;

// Chebyshev smoothing on level 0 when it runs the fused thread kernels: the
// damped Jacobi sweeps replaced by Chebyshev steps for P^-1 S_c on
// [lmax / 20, lmax], lmax from a power iteration when the V-cycle graph is
// captured.  Same kernels (the step's extra term reads x_{k-1} from the
// ping-pong partner).  Measured against Jacobi level-0 sweeps in round 1
// (ratio 10: p = 4 20 iterations; 30: +1 at p <= 3).
constexpr double kChebRatio = 20.0;
constexpr int kChebPower = 30;  // power iterations
bool cheb_level(Team& T, int l) { return l == 0 && l + 1 < levels(T) && tier(level_of(T.h0(), l)) == kBig; }

struct Cheb {
  double theta, delta, sigma, rho;
  explicit Cheb(double lmax) {
    const double hi = kChebSafety * lmax, lo = hi / kChebRatio;
    theta = 0.5 * (hi + lo);
    delta = 0.5 * (hi - lo);
    sigma = theta / delta;
    rho = 1.0 / sigma;
  }
  // coefficients of step k (k = 0 starts the recurrence)
  void step(int k, double* alpha, double* beta) {
    if (k == 0) {
      rho = 1.0 / sigma;
      *alpha = 1.0 / theta;
      *beta = 0.0;
      return;
    }
    const double rn = 1.0 / (2.0 * sigma - rho);
    *alpha = 2.0 * rn / delta;
    *beta = rn * rho;
    rho = rn;
  }
};

void sweep_cheb(Team& T, int l, double wm, double dt, Vec b, Vec xi, Vec xo, double alpha, double beta,
                bool prev_zero, bool chained) {
  staged(T, l, xi, 1, true, [&](Handle& L, int k0, int k1) { f_stage1(L, xi, k0, k1, chained); });
  staged(T, l, kTz, 2, true, [&](Handle& L, int k0, int k1) {
    smooth_stage2(L, 1, vp(L, xi), vp(L, b), wm, dt, alpha, vp(L, xo), beta, prev_zero ? 1 : 0, k0, k1);
  });
}

void lincomb(Team& T, double a, Vec x, double b, Vec y, double c, Vec z, Vec out);

// largest eigenvalue of P^-1 S_c on level 0 by power iteration from a fixed
// pseudo-random vector (an underestimate lets the Chebyshev polynomial amplify
// the modes above it; a start from kP lacks the high-frequency modes)
double estimate_lmax(Team& T, int l, double wm, double dt) {
  each(T, l, [&](Handle& L) {
    if (!L.mg_zero.ptr) L.mg_zero.alloc(L.vec_len(), &L.bytes);
    if (!L.red.ptr) L.red.alloc(reduction_scratch(), &L.bytes);
    launch_fill_hash(L, vp(L, kMgS));  // all modes present
  });
  double nv = norm_level(T, l, kMgS), lam = 0.0;
  for (int it = 0; it < kChebPower && nv > 0.0; ++it) {
    each(T, l, [&](Handle& L) {
      launch_lincomb3(L, L.vec_len(), 1.0 / nv, vp(L, kMgS), 0.0, nullptr, 0.0, nullptr, vp(L, kMgS));
    });
    residual_f(T, l, wm, dt, kMgZ, kMgS, kMgR);                                     // r = -S_c v
    each(T, l, [&](Handle& L) { smooth_zero(L, vp(L, kMgR), -1.0, vp(L, kMgS)); });  // v <- P^-1 S_c v
    nv = norm_level(T, l, kMgS);
    lam = nv;
  }
  return lam;
}

// One V-cycle on level l: x = V(b).  Fused levels alternate x with the
// level's scratch vector; the first (residual-free) sweep writes whichever
// buffer makes the last sweep land in x.
// Strip teams: the coarsest strip level solved on every rank's replica of its
// whole mesh (ldg_dense.cu replica_candidate): the owned rows of b from all
// ranks (one ncclAllGather, or device copies between virtual ranks), a
// redundant dense solve, the owned rows of x back.
void replica_solve(Team& T, int l, Vec b, Vec x) {
  Handle& L0 = level_of(T.h0(), l);
  const long cnt = static_cast<long>(L0.N) * L0.K;  // owned rows, equal on every rank
  for (int r = 0; r < T.nlocal(); ++r) {
    Handle& L = level_of(*T.ranks[r], l);
    LDG_CUDA(cudaMemcpy2DAsync(T.rep_send.ptr + r * cnt, sizeof(double) * L.K, vp(L, b), sizeof(double) * L.Kp,
                               sizeof(double) * L.K, L.N, cudaMemcpyDeviceToDevice, T.stream));
  }
  if (T.nlocal() == T.size) {  // every rank local: the gather is a copy
    LDG_CUDA(cudaMemcpyAsync(T.rep_recv.ptr, T.rep_send.ptr, sizeof(double) * cnt * T.size, cudaMemcpyDeviceToDevice,
                             T.stream));
  } else {
    if (T.nlocal() != 1 || !T.nccl) throw Error(LDG_ENCCL, "replicated coarse solve: one rank per process expected");
    LDG_NCCL(ncclAllGather(T.rep_send.ptr, T.rep_recv.ptr, cnt, ncclDouble, static_cast<ncclComm_t>(T.nccl),
                           T.stream));
  }
  for (int r = 0; r < T.nlocal(); ++r) {
    Handle& top = *T.ranks[r];
    Handle& R = *top.replica;
    Handle& L = level_of(top, l);
    launch_rep_scatter(R, T.size, L.strip_w(), T.rep_recv.ptr);
    dense_solve(R, R.mg_b.ptr, R.mg_x.ptr);
    launch_rep_gather(R, L, T.first + r, vp(L, x));
  }
}

void vcycle(Team& T, int l, bool f32, double wm, double dt, Vec b, Vec x) {
  if (l == 0) set_omega(T);
  if (l > 0 && l == T.h0().replica_level) {
    replica_solve(T, l, b, x);
    return;
  }
  if (l > 0 && l == T.h0().dense_level) {  // dense coarsest level (ldg_dense.cu): x = S_c^-1 b
    Handle& L = level_of(T.h0(), l);
    dense_solve(L, vp(L, b), vp(L, x));
    return;
  }
  const bool coarsest = l == levels(T) - 1;
  // the coarsest level is 2x2 on one rank; strips stop coarsening earlier
  // (every rank keeps a column), so a larger coarsest grid gets more sweeps
  const Handle& Ll = level_of(T.h0(), l);
  const int ldim = Ll.dim > 0 ? Ll.dim : static_cast<int>(std::sqrt(0.5 * Ll.K));  // general meshes: ~sqrt(K/2)
  const int sweeps = coarsest ? std::max(kCoarseSweeps, 2 * ldim) - 1 : (pre_of(T.h0().p, l) - 1) + post_of(T.h0().p, l);
  if (fused(T, l, f32) && cheb_level(T, l) && !coarsest) {
    Cheb ch(level_of(T.h0(), l).cheb_lmax);
    double a, be;
    Vec cur = (sweeps % 2) ? kMgS : x;
    auto other = [&](Vec v) { return v == x ? kMgS : x; };
    ch.step(0, &a, &be);
    each(T, l, [&](Handle& L) { smooth_zero(L, vp(L, b), a, vp(L, cur)); });
    for (int s = 0; s < pre_of(T.h0().p, l) - 1; ++s) {
      ch.step(s + 1, &a, &be);
      sweep_cheb(T, l, wm, dt, b, cur, other(cur), a, be, s == 0, s > 0);
      cur = other(cur);
    }
    residual_f(T, l, wm, dt, b, cur, kMgR, pre_of(T.h0().p, l) > 1);
    for (auto& rp : T.ranks) mg_restrict(level_of(*rp, l), level_of(*rp, l + 1));
    vcycle(T, l + 1, f32, wm, dt, kMgB, kMgX);
    for (auto& rp : T.ranks) mg_prolong_add(level_of(*rp, l), level_of(*rp, l + 1), vp(level_of(*rp, l), cur));
    for (int s = 0; s < post_of(T.h0().p, l); ++s) {
      ch.step(s, &a, &be);
      sweep_cheb(T, l, wm, dt, b, cur, other(cur), a, be, false, s > 0);
      cur = other(cur);
    }
    return;
  }
  if (fused(T, l, f32)) {
    Vec cur = (sweeps % 2) ? kMgS : x;
    auto other = [&](Vec v) { return v == x ? kMgS : x; };
    each(T, l, [&](Handle& L) { f_zero(L, b, cur); });
    const int pre = coarsest ? sweeps : pre_of(T.h0().p, l) - 1;
    for (int s = 0; s < pre; ++s) {
      sweep_f(T, l, wm, dt, b, cur, other(cur), s > 0);
      cur = other(cur);
    }
    if (coarsest) return;
    residual_f(T, l, wm, dt, b, cur, kMgR, pre > 0);
    for (auto& rp : T.ranks) mg_restrict(level_of(*rp, l), level_of(*rp, l + 1));
    vcycle(T, l + 1, f32, wm, dt, kMgB, kMgX);
    for (auto& rp : T.ranks) mg_prolong_add(level_of(*rp, l), level_of(*rp, l + 1), vp(level_of(*rp, l), cur));
    for (int s = 0; s < post_of(T.h0().p, l); ++s) {
      sweep_f(T, l, wm, dt, b, cur, other(cur), s > 0);
      cur = other(cur);
    }
    return;
  }
  each(T, l, [&](Handle& L) { bjac_axpy(L, f32, vp(L, b), kOmega, 0.0, vp(L, x)); });  // first sweep, x = 0
  if (coarsest) {
    for (int s = 0; s < sweeps; ++s) smooth(T, l, f32, wm, dt, b, x);
    return;
  }
  for (int s = 1; s < pre_of(T.h0().p, l); ++s) smooth(T, l, f32, wm, dt, b, x);
  residual(T, l, f32, wm, dt, b, x, kMgR);
  for (auto& rp : T.ranks) mg_restrict(level_of(*rp, l), level_of(*rp, l + 1));
  vcycle(T, l + 1, f32, wm, dt, kMgB, kMgX);
  for (auto& rp : T.ranks) mg_prolong_add(level_of(*rp, l), level_of(*rp, l + 1), vp(level_of(*rp, l), x));
  for (int s = 0; s < post_of(T.h0().p, l); ++s) smooth(T, l, f32, wm, dt, b, x);
}

int64_t team_launches(Team& T) {
  int64_t n = 0;
  for (auto& rp : T.ranks) {
    n += rp->launches;
    for (auto& c : rp->coarse) n += c->launches;
  }
  return n;
}

// The V-cycle is a fixed sequence of kernels, copies and (multi-GPU) NCCL
// halo calls with no host synchronisation: captured once per (b, x, wm, dt)
// into a CUDA graph and replayed.  Operator contents change every step in
// place; the graph only bakes pointers and the scalars.
void precond_mg(Team& T, bool f32, double wm, double dt, Vec b, Vec x) {
  Handle& h = T.h0();
  for (auto& g : h.vgraphs)
    if (g.b == vp(h, b) && g.x == vp(h, x) && g.wm == wm && g.dt == dt && (g.kernels < 0) == f32) {
      LDG_CUDA(cudaGraphLaunch(g.exec, T.stream));
      h.launches += g.kernels < 0 ? -g.kernels : g.kernels;
      return;
    }
  if (h.vgraphs.size() >= 8) mg_release(h);
  for (int l = 0; f32 && l < levels(T); ++l) {
    if (!cheb_level(T, l)) continue;
    const double lmax = estimate_lmax(T, l, wm, dt);  // (kernels run eagerly, before capture)
    for (auto& rp : T.ranks) level_of(*rp, l).cheb_lmax = lmax;
  }
  const int64_t before = team_launches(T);
  cudaGraph_t graph = nullptr;
  LDG_CUDA(cudaStreamBeginCapture(T.stream, cudaStreamCaptureModeThreadLocal));
  try {
    vcycle(T, 0, f32, wm, dt, b, x);
  } catch (...) {
    cudaStreamEndCapture(T.stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  LDG_CUDA(cudaStreamEndCapture(T.stream, &graph));
  Handle::VGraph g;
  g.b = vp(h, b);
  g.x = vp(h, x);
  g.wm = wm;
  g.dt = dt;
  const int64_t k = team_launches(T) - before;
  g.kernels = f32 ? -k : k;  // sign tags the precision variant
  const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  LDG_CUDA(e);
  h.vgraphs.push_back(g);
  LDG_CUDA(cudaGraphLaunch(g.exec, T.stream));
}

void precond(Team& T, int pc, bool f32, double wm, double dt, Vec b, Vec x) {
  if (pc == 2) return precond_mg(T, f32, wm, dt, b, x);
  each(T, 0, [&](Handle& h) {
    if (pc == 1)
      launch_bjac_apply(h, vp(h, b), vp(h, x));
    else
      LDG_CUDA(cudaMemcpyAsync(vp(h, x), vp(h, b), sizeof(double) * h.vec_len(), cudaMemcpyDeviceToDevice, T.stream));
  });
}

// precond: 0 none, 1 block-Jacobi, 2 multigrid with the smoother on FP32
// copies of E / block inverses (mixed precision), 3 multigrid all-FP64.
// Returns the preconditioner that runs (2 = multigrid, f32 tells which).
int prepare_precond(Team& T, int pc, double wm, double dt, bool* f32) {
  if (pc >= 2) {
    bool ok = true;
    for (auto& rp : T.ranks) ok = mg_build(*rp, T.size) && ok;
    if (!ok) pc = 1;  // no FK hierarchy (general mesh): block-Jacobi
    if (ok && T.h0().replica && !T.rep_recv.ptr) {  // gather staging (before any V-cycle capture)
      const Handle& C = *T.h0().coarse[T.h0().replica_level - 1];
      const long cnt = static_cast<long>(C.N) * C.K;
      T.rep_send.alloc(cnt * T.nlocal(), nullptr);
      T.rep_recv.alloc(cnt * T.size, nullptr);
    }
  }
  *f32 = pc == 2;
  if (pc == 1 || pc == 3) each(T, 0, [&](Handle& h) { launch_bjac_setup(h, wm, dt); });
  if (pc >= 2) {
    if (T.nlocal() == 1 && setup_overlap()) {
      // one rank: level 0's block-Jacobi inverses and the coarse levels'
      // rediscretisation run on two side streams, concurrently with each
      // other and with the Schur right-hand side on the main stream; the
      // Krylov loop waits for both (join_precond)
      Handle& h = T.h0();
      if (!T.setup_stream[0]) {
        // the coarse levels' chain of small latency-bound kernels gets the higher priority:
        // its CTAs take the SM slots the 8192-CTA block-Jacobi kernel of level 0 frees
        int least = 0, greatest = 0;
        LDG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        const int coarse_prio = env_or("LDG_SETUP_PRIO", 1) != 0 ? greatest : least;
        LDG_CUDA(cudaStreamCreateWithPriority(&T.setup_stream[0], cudaStreamNonBlocking, least));
        LDG_CUDA(cudaStreamCreateWithPriority(&T.setup_stream[1], cudaStreamNonBlocking, coarse_prio));
        for (auto& e : T.setup_ev) LDG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      LDG_CUDA(cudaEventRecord(T.setup_ev[0], T.stream));
      for (auto& st : T.setup_stream) LDG_CUDA(cudaStreamWaitEvent(st, T.setup_ev[0], 0));
      auto on_stream = [&](cudaStream_t st, auto&& fn) {  // the levels' launches go to st
        std::vector<Handle*> hs{&h};
        for (auto& c : h.coarse) hs.push_back(c.get());
        if (h.replica) hs.push_back(h.replica.get());
        std::vector<cudaStream_t> saved;
        for (Handle* x : hs) {
          saved.push_back(x->stream);
          x->stream = st;
        }
        auto restore = [&] {
          for (size_t i = 0; i < hs.size(); ++i) hs[i]->stream = saved[i];
        };
        try {
          fn();
        } catch (...) {
          restore();
          throw;
        }
        restore();
      };
      on_stream(T.setup_stream[0], [&] { mg_setup_top(h, wm, dt, *f32); });
      on_stream(T.setup_stream[1], [&] { mg_setup_coarse(h, h.t_assembled, wm, dt, *f32); });
      LDG_CUDA(cudaEventRecord(T.setup_ev[1], T.setup_stream[0]));
      LDG_CUDA(cudaEventRecord(T.setup_ev[2], T.setup_stream[1]));
      T.setup_pending = true;
    } else {
      for (auto& rp : T.ranks) mg_setup_step(*rp, rp->t_assembled, wm, dt, *f32);
    }
    pc = 2;
  }
  return pc;
}

// the main stream waits for the preconditioner set up on the side streams
void join_precond(Team& T) {
  if (!T.setup_pending) return;
  LDG_CUDA(cudaStreamWaitEvent(T.stream, T.setup_ev[1], 0));
  LDG_CUDA(cudaStreamWaitEvent(T.stream, T.setup_ev[2], 0));
  T.setup_pending = false;
}

void lincomb(Team& T, double a, Vec x, double b, Vec y, double c, Vec z, Vec out) {
  each(T, 0, [&](Handle& h) {
    launch_lincomb3(h, h.vec_len(), a, vp(h, x), b, y == kNone ? nullptr : vp(h, y), c,
                    z == kNone ? nullptr : vp(h, z), vp(h, out));
  });
}

// BiCGStab (right preconditioned) on the Schur system, x = C warm-started
// from C^n; three host synchronisations per iteration.
void bicgstab(Team& T, int pc, bool f32, double wm, double dt, const ldg_solver_opts& o, double tol, int* it_out,
              int* applies_out, double* rnorm_out) {
  int applies = 0;

  schur_apply(T, wm, dt, kC, kR);
  ++applies;
  lincomb(T, 1.0, kB, -1.0, kR, 0.0, kNone, kR);  // r = b - A x
  each(T, 0, [&](Handle& h) {
    const long n = h.vec_len();
    LDG_CUDA(cudaMemcpyAsync(h.kr_rh.ptr, h.kr_r.ptr, sizeof(double) * n, cudaMemcpyDeviceToDevice, T.stream));
    LDG_CUDA(cudaMemsetAsync(h.kr_p.ptr, 0, sizeof(double) * n, T.stream));
    LDG_CUDA(cudaMemsetAsync(h.kr_v.ptr, 0, sizeof(double) * n, T.stream));
  });
  double rho = 1.0, alpha = 1.0, omega = 1.0;
  // three host synchronisations per iteration: (rh,v); (t,s),(t,t),(s,s); (r,r),(rh,r)
  double rr_rhr[2];
  {
    const Vec xs[2] = {kR, kRh}, ys[2] = {kR, kR};
    dots(T, 2, xs, ys, rr_rhr);
  }
  double rnorm = std::sqrt(rr_rhr[0]);
  double rho1 = rr_rhr[1];
  int it = 0;
  bool converged = rnorm <= tol;
  while (!converged && it < o.maxit) {
    ++it;
    if (rho1 == 0.0 || !std::isfinite(rho1)) {
      // breakdown: restart with the current residual as shadow vector
      each(T, 0, [&](Handle& h) {
        const long n = h.vec_len();
        LDG_CUDA(cudaMemcpyAsync(h.kr_rh.ptr, h.kr_r.ptr, sizeof(double) * n, cudaMemcpyDeviceToDevice, T.stream));
        LDG_CUDA(cudaMemsetAsync(h.kr_p.ptr, 0, sizeof(double) * n, T.stream));
        LDG_CUDA(cudaMemsetAsync(h.kr_v.ptr, 0, sizeof(double) * n, T.stream));
      });
      rho = alpha = omega = 1.0;
      rho1 = rnorm * rnorm;
      if (rho1 == 0.0) break;
    }
    const double beta = (rho1 / rho) * (alpha / omega);
    lincomb(T, 1.0, kR, beta, kP, -beta * omega, kV, kP);  // p = r + beta (p - omega v)
    precond(T, pc, f32, wm, dt, kP, kPh);
    schur_apply(T, wm, dt, kPh, kV);
    ++applies;
    double rv;
    {
      const Vec xs[1] = {kRh}, ys[1] = {kV};
      dots(T, 1, xs, ys, &rv);
    }
    alpha = rho1 / rv;
    lincomb(T, 1.0, kR, -alpha, kV, 0.0, kNone, kS);  // s = r - alpha v
    precond(T, pc, f32, wm, dt, kS, kSh);
    schur_apply(T, wm, dt, kSh, kT);
    ++applies;
    double ts[3];
    {
      const Vec xs[3] = {kT, kT, kS}, ys[3] = {kS, kT, kS};
      dots(T, 3, xs, ys, ts);
    }
    if (std::sqrt(ts[2]) <= tol) {  // converged on s: x += alpha p^
      lincomb(T, 1.0, kC, alpha, kPh, 0.0, kNone, kC);
      rnorm = std::sqrt(ts[2]);
      converged = true;
      break;
    }
    omega = ts[1] != 0.0 ? ts[0] / ts[1] : 0.0;
    lincomb(T, 1.0, kC, alpha, kPh, omega, kSh, kC);  // x += alpha p^ + omega s^
    lincomb(T, 1.0, kS, -omega, kT, 0.0, kNone, kR);  // r = s - omega t
    {
      const Vec xs[2] = {kR, kRh}, ys[2] = {kR, kR};
      dots(T, 2, xs, ys, rr_rhr);
    }
    rnorm = std::sqrt(rr_rhr[0]);
    rho = rho1;
    rho1 = rr_rhr[1];
    if (!std::isfinite(rnorm)) break;
    converged = rnorm <= tol;
    if (omega == 0.0) break;
  }

  *it_out = it;
  *applies_out = applies;
  *rnorm_out = rnorm;
}

// Restarted flexible GMRES (right preconditioned, FGMRES(m)) on the Schur
// system: one V-cycle and one operator apply per iteration (BiCGStab needs
// two of each), and robust to a preconditioner that is not exactly linear
// (the FP32-arithmetic smoother).  Classical Gram-Schmidt with one
// reorthogonalisation pass, each pass one fused multi-dot (one host
// synchronisation) and one fused multi-axpy over the basis; the Hessenberg
// least-squares problem (Givens rotations) is solved on the host.
// LDG_TRACE_ITER=1: device time of the parts of each FGMRES iteration
// (copy in, V-cycle, copy out, operator, projections), summed and printed to
// stderr per solve (diagnostics)
struct IterTrace {
  bool on = env_or("LDG_TRACE_ITER", 0) != 0;
  cudaEvent_t ev[7] = {};  // 0..4 marks of the iteration, 5 after the projection, 6 the previous 5
  double sum[6] = {0, 0, 0, 0, 0, 0};
  int n = 0;
  IterTrace() {
    if (on)
      for (auto& e : ev) cudaEventCreate(&e);
  }
  ~IterTrace() {
    if (!on || n == 0) return;
    fprintf(stderr,
            "[ldg trace] %d its, ms/it: copy-in %.3f vcycle %.3f copy-out %.3f operator %.3f project+sync %.3f "
            "update+host %.3f\n",
            n, sum[0] / n, sum[1] / n, sum[2] / n, sum[3] / n, sum[4] / n, n > 1 ? sum[5] / (n - 1) : 0.0);
    for (auto& e : ev) cudaEventDestroy(e);
  }
  void add(cudaStream_t st) {  // after the projection's host synchronisation
    cudaEventRecord(ev[5], st);
    cudaEventSynchronize(ev[5]);
    float a;
    for (int q = 0; q < 5; ++q) {
      cudaEventElapsedTime(&a, ev[q], ev[q + 1]);
      sum[q] += a;
    }
    if (n > 0) {  // previous projection end -> this iteration's start
      cudaEventElapsedTime(&a, ev[6], ev[0]);
      sum[5] += a;
    }
    std::swap(ev[5], ev[6]);
    n++;
  }
};

// in-place sum over the processes of n device values (one rank per process)
void allreduce_dev(Team& T, double* v, int n) {
  if (T.nccl && T.size > T.nlocal())
    LDG_NCCL(ncclAllReduce(v, v, n, ncclDouble, ncclSum, static_cast<ncclComm_t>(T.nccl), T.stream));
}

// FGMRES(m) for one rank per process (the production shape): the
// Gram-Schmidt coefficients never leave the device inside an iteration
// (CGS2: h1 = V^T w with (w, w), w -= V h1, h2 = V^T w with (w, w),
// w = (w - V h2) / |.| by Pythagoras, the next V-cycle input written in the
// same pass), and the host runs one iteration behind: iteration j + 1 is
// queued before the host waits for iteration j's coefficient slot, unless
// the residual trend says j may already converge.  The GPU queue therefore
// stays non-empty across the host's Givens update and launch latency.
void fgmres_dev(Team& T, int pc, bool f32, double wm, double dt, const ldg_solver_opts& o, double tol, int m,
                int* it_out, int* applies_out, double* rnorm_out) {
  Handle& h0 = T.h0();
  constexpr int kSlot = 2 * kMaxRed + 1;  // h1 (j + 2) | h2 (j + 2) | hn
  if (h0.gs.n < static_cast<size_t>(m) * kSlot) h0.gs.alloc(static_cast<size_t>(m) * kSlot, &h0.bytes);
  auto copy = [&](Vec dst, Vec src) {
    LDG_CUDA(cudaMemcpyAsync(vp(h0, dst), vp(h0, src), sizeof(double) * h0.vec_len(), cudaMemcpyDeviceToDevice,
                             T.stream));
  };
  auto scale_into = [&](double a, Vec src, Vec dst) { lincomb(T, a, src, 0.0, kNone, 0.0, kNone, dst); };
  int applies = 0;
  // LDG_TRACE_ITER=1: per-iteration device spans (work vs gaps) on stderr
  static const bool trace = env_or("LDG_TRACE_ITER", 0) != 0;
  std::vector<cudaEvent_t> tev;
  cudaEvent_t t_entry = nullptr;
  if (trace) {
    LDG_CUDA(cudaEventCreate(&t_entry));
    LDG_CUDA(cudaEventRecord(t_entry, T.stream));
  }
  auto mark = [&] {
    if (!trace) return;
    cudaEvent_t e;
    LDG_CUDA(cudaEventCreate(&e));
    LDG_CUDA(cudaEventRecord(e, T.stream));
    tev.push_back(e);
  };
  auto launch_it = [&](int j) {  // the GPU work of iteration j; with pc == 2 kP holds V_j on entry
    mark();
    if (pc == 2) {
      precond(T, pc, f32, wm, dt, kP, kPh);
      copy(gmZ(j), kPh);
    } else {
      precond(T, pc, f32, wm, dt, gmV(j), gmZ(j));
    }
    schur_apply(T, wm, dt, gmZ(j), gmV(j + 1));
    ++applies;
    const double* v[kMaxRed];
    for (int d = 0; d <= j + 1; ++d) v[d] = vp(h0, gmV(d));
    double* slot = h0.gs.ptr + static_cast<long>(j) * kSlot;
    for (int pass = 0; pass < 2; ++pass) {
      double* c = slot + pass * kMaxRed;
      launch_mdots_to(h0, j + 2, v, vp(h0, gmV(j + 1)), c);
      allreduce_dev(T, c, j + 2);
      launch_maxpy_dev(h0, j + 1, v, c, pass == 1, vp(h0, gmV(j + 1)), pass == 1 && pc == 2 ? vp(h0, kP) : nullptr,
                       slot + 2 * kMaxRed);
    }
    LDG_CUDA(cudaMemcpyAsync(T.gs_host + static_cast<long>(j) * kSlot, slot, sizeof(double) * kSlot,
                             cudaMemcpyDeviceToHost, T.stream));
    LDG_CUDA(cudaEventRecord(T.gs_ev[j & 1], T.stream));
    mark();
  };

  int it = 0;
  double rnorm = 0.0;
  std::vector<double> H(static_cast<size_t>(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  auto Hij = [&](int i, int j) -> double& { return H[static_cast<size_t>(j) * (m + 1) + i]; };
  while (true) {
    schur_apply(T, wm, dt, kC, gmV(0));  // r = b - A x into V_0
    ++applies;
    lincomb(T, 1.0, kB, -1.0, gmV(0), 0.0, kNone, gmV(0));
    rnorm = norm(T, gmV(0));
    if (!(rnorm > tol) || !std::isfinite(rnorm) || it >= o.maxit) break;
    scale_into(1.0 / rnorm, gmV(0), gmV(0));
    if (pc == 2) copy(kP, gmV(0));
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = rnorm;
    launch_it(0);
    int launched = 1;  // iterations of this cycle queued on the stream
    double r1 = rnorm, r2 = 0.0;  // last two residual estimates (trend)
    int j = 0;
    bool done = false;
    for (; j < m; ++j) {
      const bool more = j + 1 < m && it + 1 < o.maxit;
      if (more && launched == j + 1) {  // queue j + 1 now unless j is predicted to converge
        const double rate = r2 > 0.0 ? std::min(r1 / r2, 1.0) : 0.5;
        if (r1 * rate > 4.0 * tol) {
          launch_it(j + 1);
          launched = j + 2;
        }
      }
      LDG_CUDA(cudaEventSynchronize(T.gs_ev[j & 1]));
      ++it;
      const double* slot = T.gs_host + static_cast<long>(j) * kSlot;
      const double *h1 = slot, *h2 = slot + kMaxRed;
      for (int i = 0; i <= j; ++i) Hij(i, j) = h1[i] + h2[i];
      double hn = slot[2 * kMaxRed];
      if (hn > 0.0 && !(hn > 1e-6 * std::sqrt(std::max(h1[j + 1], 0.0)))) {
        // cancellation guard: normalise V_{j+1} explicitly; a queued
        // iteration j + 1 started from the unnormalised vector and is redone
        const double s2 = norm(T, gmV(j + 1));
        if (s2 > 0.0) {
          hn *= s2;
          scale_into(1.0 / s2, gmV(j + 1), gmV(j + 1));
          if (pc == 2) copy(kP, gmV(j + 1));
          if (launched == j + 2) launch_it(j + 1);
        }
      }
      Hij(j + 1, j) = hn;
      for (int i = 0; i < j; ++i) {  // Givens rotations
        const double a = Hij(i, j), b = Hij(i + 1, j);
        Hij(i, j) = cs[i] * a + sn[i] * b;
        Hij(i + 1, j) = -sn[i] * a + cs[i] * b;
      }
      const double a = Hij(j, j), b = Hij(j + 1, j);
      const double r = std::hypot(a, b);
      cs[j] = r > 0.0 ? a / r : 1.0;
      sn[j] = r > 0.0 ? b / r : 0.0;
      Hij(j, j) = r;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rnorm = std::fabs(g[j + 1]);
      r2 = r1;
      r1 = rnorm;
      if (rnorm <= tol || hn == 0.0 || !std::isfinite(rnorm)) {
        ++j;
        done = true;
        break;
      }
      if (it >= o.maxit) {
        ++j;
        break;
      }
      if (j + 1 < m && launched == j + 1) {
        launch_it(j + 1);
        launched = j + 2;
      }
    }
    // x += Z y, H(0:j, 0:j) y = g(0:j) (a queued iteration past j is unused)
    for (int i = j - 1; i >= 0; --i) {
      double v = g[i];
      for (int k = i + 1; k < j; ++k) v -= Hij(i, k) * y[k];
      y[i] = Hij(i, i) != 0.0 ? v / Hij(i, i) : 0.0;
    }
    const double* z[kMaxRed];
    for (int d = 0; d < j; ++d) z[d] = vp(h0, gmZ(d));
    launch_maxpy(h0, j, z, y.data(), 1.0, vp(h0, kC));
    if (done && rnorm <= tol) break;
    if (it >= o.maxit || !std::isfinite(rnorm)) break;
  }
  if (trace && tev.size() >= 2) {
    LDG_CUDA(cudaStreamSynchronize(T.stream));
    float work = 0.f, gap = 0.f, a = 0.f, gmax = 0.f, pre = 0.f;
    cudaEventElapsedTime(&pre, t_entry, tev[0]);
    cudaEventDestroy(t_entry);
    for (size_t i = 0; i + 1 < tev.size(); i += 2) {
      cudaEventElapsedTime(&a, tev[i], tev[i + 1]);
      work += a;
      if (i + 2 < tev.size()) {
        cudaEventElapsedTime(&a, tev[i + 1], tev[i + 2]);
        gap += a;
        gmax = std::max(gmax, a);
      }
    }
    fprintf(stderr, "[ldg trace] %zu launches: before the first %.3f ms, work %.3f ms (%.3f/it), between %.3f ms (max %.3f)\n",
            tev.size() / 2, pre, work, work / (tev.size() / 2), gap, gmax);
    for (auto e : tev) cudaEventDestroy(e);
  }
  *it_out = it;
  *applies_out = applies;
  *rnorm_out = rnorm;
}

void fgmres(Team& T, int pc, bool f32, double wm, double dt, const ldg_solver_opts& o, double tol, int* it_out,
            int* applies_out, double* rnorm_out) {
  Handle& h0 = T.h0();
  IterTrace tr;
  int m = o.restart > 0 ? o.restart : 30;
  m = std::min(m, kMaxRed - 2);
  const int m_req = m;
  if (h0.gm_m > 0 && h0.gm_req == m_req) {
    m = h0.gm_m;  // sized on an earlier solve (cudaMemGetInfo stalled the host for milliseconds per step)
  } else {  // basis memory: (2m + 1) vectors per rank, within free device memory
    size_t free_b = 0, total_b = 0;
    LDG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double vec_b = 8.0 * h0.vec_len() * T.nlocal();
    const double have = h0.gm_m > 0 ? (2.0 * h0.gm_m + 1) * vec_b : 0.0;
    const double budget = 0.8 * (static_cast<double>(free_b) + have) - 2.0 * vec_b;
    const int mfit = static_cast<int>(budget / (2.0 * vec_b));
    m = std::max(2, std::min(m, mfit));
  }
  if (h0.gm_m != m) {
    for (auto& rp : T.ranks) {
      rp->gm_V.alloc(static_cast<size_t>(m + 1) * rp->vec_len(), &rp->bytes);
      rp->gm_Z.alloc(static_cast<size_t>(m) * rp->vec_len(), &rp->bytes);
      rp->gm_m = m;
      rp->gm_req = m_req;
    }
  }
  // one rank per process: device-resident Gram-Schmidt, host one iteration
  // behind (LDG_GS_HOST=1 selects the host-side variant below, which
  // virtual-rank teams use)
  if (T.nlocal() == 1) return fgmres_dev(T, pc, f32, wm, dt, o, tol, m, it_out, applies_out, rnorm_out);
  auto copy = [&](Vec dst, Vec src) {  // (ranks differ in ghost counts, hence in vector length)
    each(T, 0, [&](Handle& h) {
      LDG_CUDA(cudaMemcpyAsync(vp(h, dst), vp(h, src), sizeof(double) * h.vec_len(), cudaMemcpyDeviceToDevice,
                               T.stream));
    });
  };
  auto scale_into = [&](double a, Vec src, Vec dst) { lincomb(T, a, src, 0.0, kNone, 0.0, kNone, dst); };
  // per-rank fused projections over the basis V_0..V_{nb-1} (plus (w, w) if with_norm)
  auto project = [&](int nb, Vec w, bool with_norm, double* out) {
    reduce_dots(
        T, nb + (with_norm ? 1 : 0),
        [&](Handle& h) {
          const double* v[kMaxRed];
          for (int d = 0; d < nb; ++d) v[d] = vp(h, gmV(d));
          if (with_norm) v[nb] = vp(h, w);
          launch_mdots_async(h, nb + (with_norm ? 1 : 0), v, vp(h, w));
        },
        out);
  };
  auto subtract = [&](int nb, const double* c, Vec w) {  // w -= sum c_d V_d
    std::vector<double> neg(nb);
    for (int d = 0; d < nb; ++d) neg[d] = -c[d];
    each(T, 0, [&](Handle& h) {
      const double* v[kMaxRed];
      for (int d = 0; d < nb; ++d) v[d] = vp(h, gmV(d));
      launch_maxpy(h, nb, v, neg.data(), 1.0, vp(h, w));
    });
  };

  int applies = 0, it = 0, reorth = 0;
  double rnorm = 0.0;
  std::vector<double> H(static_cast<size_t>(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  auto Hij = [&](int i, int j) -> double& { return H[static_cast<size_t>(j) * (m + 1) + i]; };
  while (true) {
    // r = b - A x into V_0
    schur_apply(T, wm, dt, kC, gmV(0));
    ++applies;
    lincomb(T, 1.0, kB, -1.0, gmV(0), 0.0, kNone, gmV(0));
    rnorm = norm(T, gmV(0));
    if (!(rnorm > tol) || !std::isfinite(rnorm) || it >= o.maxit) break;
    scale_into(1.0 / rnorm, gmV(0), gmV(0));
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = rnorm;
    int j = 0;
    bool done = false;
    for (; j < m && it < o.maxit; ++j) {
      ++it;
      if (tr.on) LDG_CUDA(cudaEventRecord(tr.ev[0], T.stream));
      // Z_j = M^-1 V_j (the V-cycle graph is keyed on kP -> kPh)
      if (pc == 2) {
        copy(kP, gmV(j));
        if (tr.on) LDG_CUDA(cudaEventRecord(tr.ev[1], T.stream));
        precond(T, pc, f32, wm, dt, kP, kPh);
        if (tr.on) LDG_CUDA(cudaEventRecord(tr.ev[2], T.stream));
        copy(gmZ(j), kPh);
      } else {
        precond(T, pc, f32, wm, dt, gmV(j), gmZ(j));
      }
      if (tr.on) LDG_CUDA(cudaEventRecord(tr.ev[3], T.stream));
      schur_apply(T, wm, dt, gmZ(j), gmV(j + 1));
      if (tr.on) LDG_CUDA(cudaEventRecord(tr.ev[4], T.stream));
      ++applies;
      // classical Gram-Schmidt: h = V^T w (+ |w|^2), w -= V h; a second pass
      // only when the projection removed more than half of |w|^2 ("twice is
      // enough"), so the basis stays orthogonal to working precision
      double h1[kMaxRed], h2[kMaxRed];
      project(j + 1, gmV(j + 1), true, h1);
      subtract(j + 1, h1, gmV(j + 1));
      double ss = h1[j + 1];
      for (int i = 0; i <= j; ++i) {
        Hij(i, j) = h1[i];
        ss -= h1[i] * h1[i];
      }
      if (tr.on) tr.add(T.stream);  // (project() synchronised the stream: "project" includes that gap)
      if (!(ss > kReorthEta * h1[j + 1])) {
        project(j + 1, gmV(j + 1), true, h2);
        subtract(j + 1, h2, gmV(j + 1));
        ss = h2[j + 1];
        for (int i = 0; i <= j; ++i) {
          Hij(i, j) += h2[i];
          ss -= h2[i] * h2[i];
        }
        ++reorth;
      }
      double hn = ss > 0.0 ? std::sqrt(ss) : 0.0;
      if (!(hn > 1e-6 * std::sqrt(std::max(h1[j + 1], 0.0)))) hn = norm(T, gmV(j + 1));  // cancellation guard
      Hij(j + 1, j) = hn;
      if (hn > 0.0) scale_into(1.0 / hn, gmV(j + 1), gmV(j + 1));
      // Givens rotations
      for (int i = 0; i < j; ++i) {
        const double a = Hij(i, j), b = Hij(i + 1, j);
        Hij(i, j) = cs[i] * a + sn[i] * b;
        Hij(i + 1, j) = -sn[i] * a + cs[i] * b;
      }
      const double a = Hij(j, j), b = Hij(j + 1, j);
      const double r = std::hypot(a, b);
      cs[j] = r > 0.0 ? a / r : 1.0;
      sn[j] = r > 0.0 ? b / r : 0.0;
      Hij(j, j) = r;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rnorm = std::fabs(g[j + 1]);
      if (rnorm <= tol || hn == 0.0 || !std::isfinite(rnorm)) {
        ++j;
        done = true;
        break;
      }
    }
    // x += Z y, H(0:j, 0:j) y = g(0:j)
    for (int i = j - 1; i >= 0; --i) {
      double v = g[i];
      for (int k = i + 1; k < j; ++k) v -= Hij(i, k) * y[k];
      y[i] = Hij(i, i) != 0.0 ? v / Hij(i, i) : 0.0;
    }
    each(T, 0, [&](Handle& h) {
      const double* z[kMaxRed];
      for (int d = 0; d < j; ++d) z[d] = vp(h, gmZ(d));
      launch_maxpy(h, j, z, y.data(), 1.0, vp(h, kC));
    });
    if (done && rnorm <= tol) break;
    if (it >= o.maxit || !std::isfinite(rnorm)) break;
  }
  *it_out = it;
  *applies_out = applies;
  *rnorm_out = rnorm;
  (void)reorth;
}

}  // namespace

void team_assemble(Team& T, double t) {
  for (auto& rp : T.ranks) assemble_step(*rp, t);
}

// One linear solve with the operators of the last team_assemble: wm = 1, dt
// for W + dt A (euler_step), wm = 0, dt = 1 for A (solve_stationary).
// Y holds the previous state on entry and the solution on exit.
int team_solve(Team& T, double wm, double dt, const ldg_solver_opts& o, ldg_step_stats* st) {
  Handle& h0 = T.h0();
  // preconditioner setup first: it needs the step's operators only, so a
  // host-buffer state upload (ldg_euler_steps_host) overlaps it
  bool f32 = false;
  std::optional<NvtxRange> phase;  // NVTX: one range per phase of the solve
  phase.emplace("solve setup (preconditioner, Schur rhs)");
  const int pc = prepare_precond(T, o.precond, wm, dt, &f32);
  if (T.y_pending) {
    LDG_CUDA(cudaStreamWaitEvent(T.stream, T.in_ev[1], 0));
    T.y_pending = false;
  }
  // Krylov start: C^n, or for a continued time integration the Lagrange
  // extrapolation in time of C^n and the last steps' C (order
  // extrap_order(), limited on the device to the valid history).  The
  // stopping rule is relative to the right-hand side, so a smaller initial
  // residual saves iterations at the same final accuracy.
  const Handle& H0 = T.h0();
  const int order = wm != 0.0 && H0.hist_ok &&
                            std::fabs(H0.t - (H0.hist_time[0] + H0.hist_dt)) <= 1e-12 * std::max(1.0, std::fabs(H0.t))
                        ? extrap_order(H0.p)
                        : 0;
  double w[kExtrapMax][kExtrapMax + 1] = {};
  {
    // nodes t_n, t_{n-1}, ... (distinct when the device says the history is valid)
    const double tx = H0.t + dt;
    double tn[kExtrapMax + 1] = {H0.t};
    for (int j = 0; j < kExtrapMax; ++j) tn[j + 1] = H0.hist_time[j];
    for (int o = 1; o <= kExtrapMax; ++o)
      for (int j = 0; j <= o; ++j) {
        double l = 1.0;
        for (int m = 0; m <= o; ++m)
          if (m != j) l *= (tn[m] != tn[j]) ? (tx - tn[m]) / (tn[j] - tn[m]) : 0.0;
        w[o - 1][j] = l;
      }
  }
  each(T, 0, [&](Handle& h) {
    const long n = h.vec_len();
    LDG_CUDA(cudaMemcpyAsync(h.Yold.ptr, h.Y.ptr, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, T.stream));
    if (wm != 0.0 && extrap_order(h.p) > 0) {
      if (!h.hist_dev.ptr) {
        for (auto& b : h.Chist) b.alloc(n, &h.bytes);
        h.hist_dev.alloc(2, &h.bytes);  // zeroed: no history
      }
      const double* hv[kExtrapMax];
      for (int j = 0; j < kExtrapMax; ++j) hv[j] = h.Chist[j].ptr;
      launch_extrap(h, n, order, w, vp(h, kCold), hv, h.hist_dev.ptr, h.hist_same, vp(h, kC));
    }
    h.hist_ok = false;
    h.hist_same = nullptr;
    // Schur right-hand side b = wm M C^n + dt (V_C - sum E^m M^-1 V_Z^m): t = M^-1 V_Z (local)
    launch_stage1(h, h.Vv.ptr, 1.0, nullptr, 0.0, h.tz.ptr);
  });
  halo(T, 0, kTz, 2);
  each(T, 0, [&](Handle& h) {
    const long n = h.vec_len();
    launch_stage2(h, wm != 0.0 ? vp(h, kCold) : nullptr, wm, 0.0, h.tz.ptr, dt, vp(h, kVc), dt, h.kr_b.ptr);
    // full right-hand side of the reference system: r = W Y^n + dt V
    launch_lincomb3(h, 3 * n, dt, h.Vv.ptr, 0.0, nullptr, 0.0, nullptr, h.full_r.ptr);
    if (wm != 0.0) launch_stage2(h, vp(h, kCold), wm, 0.0, nullptr, 0.0, vp(h, kVc), dt, h.full_r.ptr + 2 * n);
  });
  const double rhs_norm = std::sqrt(sq_norm3(T, kFullR));
  const double contract = o.contract_tol > 0.0 ? o.contract_tol : 1e-10;

  const double bnorm = norm(T, kB);
  // stopping test on the Schur residual: the user's rtol/atol, tightened so
  // that the full-system contract (Schur residual = C-row residual) holds
  double tol = std::max(o.rtol * bnorm, o.atol);
  if (o.check_residual) {
    const double tc = 0.25 * contract * std::max(rhs_norm, 1.0);
    tol = tol > 0.0 ? std::min(tol, tc) : tc;
  }
  if (!(tol > 0.0)) tol = 1e-300;

  int applies = 0;
  int it = 0;
  double rnorm = 0.0;
  join_precond(T);
  LDG_CUDA(cudaEventRecord(h0.ev[3], T.stream));  // end of the per-solve setup
  phase.reset();
  phase.emplace(o.krylov == 0 ? "FGMRES (V-cycle + Schur operator per iteration)" : "BiCGStab");
  if (o.krylov == 0) {
    fgmres(T, pc, f32, wm, dt, o, tol, &it, &applies, &rnorm);
  } else {
    bicgstab(T, pc, f32, wm, dt, o, tol, &it, &applies, &rnorm);
  }

  LDG_CUDA(cudaEventRecord(h0.ev[4], T.stream));  // end of the Krylov loop
  phase.reset();
  phase.emplace("flux recovery + residual contract");
  // flux recovery Z^m = M^-1 (V_Z^m - B^m C), written into Y[0 .. 2n)

  halo(T, 0, kC, 1);
  each(T, 0, [&](Handle& h) { launch_stage1(h, h.Vv.ptr, 1.0, vp(h, kC), -1.0, h.Y.ptr); });

  if (T.early_out && T.in_stream && T.size == 1 && T.nlocal() == 1) {
    // the new state is final: its copy to the caller's host buffer overlaps the contract check
    Handle& h = T.h0();
    const size_t cnt = 3L * h.K * h.N;
    LDG_CUDA(cudaEventRecord(T.in_ev[2], T.stream));
    LDG_CUDA(cudaStreamWaitEvent(T.in_stream, T.in_ev[2], 0));
    launch_soa_to_kmajor(h, h.Y.ptr, 3, h.host_stage.ptr, T.in_stream);
    LDG_CUDA(cudaMemcpyAsync(T.early_out, h.host_stage.ptr, sizeof(double) * cnt, cudaMemcpyDeviceToHost,
                             T.in_stream));
    LDG_CUDA(cudaEventRecord(T.in_ev[3], T.in_stream));
    T.early_out_sent = true;
    T.early_out = nullptr;
  }
  // reference residual contract on the full system (system.hpp:198-203)
  halo(T, 0, kY, 3);
  each(T, 0, [&](Handle& h) {
    const long n3 = 3 * h.vec_len();
    launch_full_apply(h, h.Y.ptr, wm, dt, h.full_y.ptr);
    launch_lincomb3(h, n3, 1.0, h.full_y.ptr, -1.0, h.full_r.ptr, 0.0, nullptr, h.full_y.ptr);
  });
  const double res = std::sqrt(sq_norm3(T, kFullY)) / std::max(rhs_norm, 1.0);
  if (wm != 0.0 && extrap_order(h0.p) > 0) {  // C^n becomes the next step's C^{n-1}
    each(T, 0, [&](Handle& h) {
      double* hv[kExtrapMax];
      for (int j = 0; j < kExtrapMax; ++j) hv[j] = h.Chist[j].ptr;
      launch_hist_shift(h, h.vec_len(), vp(h, kCold), hv, h.hist_dev.ptr);
      for (int j = kExtrapMax - 1; j > 0; --j) h.hist_time[j] = h.hist_time[j - 1];
      h.hist_time[0] = h.t;
      h.hist_dt = dt;
      h.hist_ok = res <= contract;
    });
  }
  if (st) {
    st->iterations += it;
    st->applies += applies;
    st->schur_relres = bnorm > 0.0 ? rnorm / bnorm : rnorm;
    st->residual = res;
  }
  if (o.check_residual && !(res <= contract)) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "linear solve residual %.6e exceeds tolerance (eta = %f, p = %d; %s %d iterations, "
             "Schur residual %.3e)",
             res, h0.prob.eta, h0.p, o.krylov == 0 ? "FGMRES" : "BiCGStab", it, rnorm);
    throw Error(LDG_ENOCONV, buf);
  }
  return it;
}

// (W + dt A) Y on the team's current state buffers (used by exports/tests)
void team_full_apply(Team& T, double wm, double dt) {
  halo(T, 0, kY, 3);
  each(T, 0, [&](Handle& h) { launch_full_apply(h, h.Y.ptr, wm, dt, h.full_y.ptr); });
}

// Schur operator apply on level-0 buffers C -> kr_v (kernel timing)
void team_schur_apply_c(Team& T, double wm, double dt) { schur_apply(T, wm, dt, kC, kV); }

// The dominant kernel of the step for the roofline (kernel timing): stage 2
// of one level-0 smoothing sweep (fused block-Jacobi update), on the
// level's current operators, from kPh into the scratch vector.
void team_sweep_s2_prepare(Team& T, double wm, double dt) {
  bool f32 = false;
  prepare_precond(T, 2, wm, dt, &f32);
  join_precond(T);
  each(T, 0, [&](Handle& L) { f_stage1(L, kPh); });
}
void team_sweep_s2(Team& T, double wm, double dt) {
  each(T, 0, [&](Handle& L) { f_stage2(L, 1, kPh, kP, wm, dt, kMgS); });
}
// level 0 of vcycle(): (pre - 1) sweeps after the residual-free one, the
// residual before restriction, post sweeps
int team_s2_per_vcycle(Team& T) {
  const int p = T.h0().p;
  return pre_of(p, 0) + post_of(p, 0);
}

// Multigrid cost breakdown (kernel timing): one V-cycle of the FP32-smoother
// preconditioner and one smoothing sweep (residual + block-Jacobi) per level,
// each captured in a graph of `reps` repetitions and replayed once after a
// warm-up replay, so the figures carry the same launch gaps as the solve.
int team_time_mg(Team& T, double wm, double dt, int reps, double* ms_vcycle, double* ms_level, int max_levels) {
  bool f32 = false;
  if (prepare_precond(T, 2, wm, dt, &f32) != 2) return 0;
  join_precond(T);
  Handle& h = T.h0();
  const int nl = levels(T);
  auto graph_time = [&](auto&& body) {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    LDG_CUDA(cudaStreamBeginCapture(T.stream, cudaStreamCaptureModeThreadLocal));
    for (int r = 0; r < reps; ++r) body();
    LDG_CUDA(cudaStreamEndCapture(T.stream, &graph));
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    LDG_CUDA(e);
    LDG_CUDA(cudaGraphLaunch(exec, T.stream));  // warm-up
    LDG_CUDA(cudaEventRecord(h.ev[0], T.stream));
    LDG_CUDA(cudaGraphLaunch(exec, T.stream));
    LDG_CUDA(cudaEventRecord(h.ev[1], T.stream));
    LDG_CUDA(cudaEventSynchronize(h.ev[1]));
    cudaGraphExecDestroy(exec);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h.ev[0], h.ev[1]);
    return static_cast<double>(ms) / reps;
  };
  *ms_vcycle = graph_time([&] { vcycle(T, 0, f32, wm, dt, kP, kPh); });
  for (int l = 0; l < nl && l < max_levels; ++l) {
    const Vec b = l == 0 ? kP : kMgB, x = l == 0 ? kPh : kMgX;
    if (l > 0 && l == h.dense_level) {  // the dense coarsest level: one solve; the levels below are never visited
      Handle& L = level_of(h, l);
      ms_level[l] = graph_time([&] { dense_solve(L, vp(L, b), vp(L, x)); });
      return l + 1;
    }
    if (l > 0 && l == h.replica_level) {
      ms_level[l] = graph_time([&] { replica_solve(T, l, b, x); });
      return l + 1;
    }
    if (fused(T, l, f32))
      ms_level[l] = graph_time([&] { sweep_f(T, l, wm, dt, b, x, kMgS); });
    else
      ms_level[l] = graph_time([&] { smooth(T, l, f32, wm, dt, b, x); });
  }
  return nl;
}

// sum of squares of the owned entries of one vector per rank, over all ranks
double team_sum_sq(Team& T, const std::function<const double*(Handle&)>& v) {
  double s;
  reduce_dots(
      T, 1,
      [&](Handle& h) {
        const double* p[1] = {v(h)};
        launch_dots_async(h, 1, p, p);
      },
      &s);
  return s;
}

}  // namespace ldgb
