// The C ABI of include/ldg_b200.h: handle lifecycle, status/exception
// mapping, exports for parity, and kernel timing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ldg_internal.hpp"

namespace ldgb {
size_t reduction_scratch();
}

struct ldg_handle {
  ldgb::Handle h;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(ldg_handle* H, F&& fn) {
  try {
    fn();
    return LDG_OK;
  } catch (const ldgb::Error& e) {
    g_last_error = e.what();
    if (H) H->h.err = e.what();
    return e.status;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    if (H) H->h.err = e.what();
    return LDG_EINVAL;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    if (H) H->h.err = g_last_error;
    return LDG_ECUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    if (H) H->h.err = e.what();
    return LDG_ENOCONV;
  }
}

using ldgb::DBuf;
using ldgb::Error;
using ldgb::Handle;

void validate_problem(const ldg_problem* prob, int p) {
  if (!prob) throw Error(LDG_EINVAL, "problem description is NULL");
  if (p < 0 || p > ldgb::kMaxP) throw Error(LDG_EINVAL, "polynomial order must be zero to four");
  if (!(prob->eta > 0.0)) throw Error(LDG_EINVAL, "penalty eta must be positive");
  if (prob->n_bc < 0 || prob->n_bc > LDG_MAX_BC) throw Error(LDG_EINVAL, "too many boundary conditions");
  const ldg_coeff* fs[5] = {&prob->d, &prob->f, &prob->c_d, &prob->g_n, &prob->c0};
  for (const ldg_coeff* f : fs)
    if (f->id < 0 || f->id >= LDG_FN_COUNT) throw Error(LDG_EINVAL, "unknown coefficient function id");
}

void init_device_side(Handle& h, int p, const ldg_problem* prob) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(LDG_ECUDA, "no CUDA device available: the LDG path has no CPU fallback");
  h.p = p;
  h.N = ldgb::dofs_of(p);
  h.prob = *prob;
  LDG_CUDA(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking));
  for (auto& e : h.ev) LDG_CUDA(cudaEventCreate(&e));
  LDG_CUDA(cudaMallocHost(&h.red_host, 64 * sizeof(double)));
  h.tables = ldgb::build_tables(p);
  h.tab.alloc(h.tables.data.size(), &h.bytes);
  LDG_CUDA(cudaMemcpy(h.tab.ptr, h.tables.data.data(), sizeof(double) * h.tables.data.size(),
                      cudaMemcpyHostToDevice));
  const ldgb::TableLayout& L = h.tables.lay;
  h.dtab = ldgb::DevTables{h.tab.ptr, L.p, L.N, L.R, L.Qe, L.Qb, L.proj_phi, L.proj_w, L.proj_x, L.mhat,
                           L.minv, L.ghat, L.hhat, L.sdiag, L.soff, L.pe, L.pth, L.we, L.pb, L.sb, L.wb, L.total,
                           L.mono, L.NP, L.tH, L.tSd, L.tSo, L.tM, L.tMinv, L.tmH, L.tmSd, L.tmSo};
  ldgb::upload_rule(h, std::max(2 * p, 1), h.rule_elem, &h.rule_elem_R);
}

void alloc_step_buffers(Handle& h) {
  const long n = h.vec_len();
  const long NN = static_cast<long>(h.N) * h.N;
  h.D.alloc(n, &h.bytes);
  h.F.alloc(n, &h.bytes);
  h.E.alloc(8 * NN * h.Kp, &h.bytes);
  h.Vv.alloc(3 * n, &h.bytes);
  h.Y.alloc(3 * n, &h.bytes);
}

// Solver-side buffers and the static blocks, allocated on first use so an
// assembly-only run (BASELINE config 3) does not pay for them.
void ensure_solver(Handle& h) {
  if (h.Yold.ptr) return;
  const long n = h.vec_len();
  const long NN = static_cast<long>(h.N) * h.N;
  h.Yold.alloc(3 * n, &h.bytes);
  for (DBuf<double>* b : {&h.kr_r, &h.kr_rh, &h.kr_p, &h.kr_v, &h.kr_s, &h.kr_t, &h.kr_ph, &h.kr_sh, &h.kr_b})
    b->alloc(n, &h.bytes);
  h.tz.alloc(2 * n, &h.bytes);
  h.Pinv.alloc(NN * h.Kp, &h.bytes);
  h.full_r.alloc(3 * n, &h.bytes);
  h.full_y.alloc(3 * n, &h.bytes);
  h.red.alloc(ldgb::reduction_scratch(), &h.bytes);
  LDG_CUDA(cudaStreamSynchronize(h.stream));
}

void require_assembled(const Handle& h) {
  if (!h.assembled) throw Error(LDG_EINVAL, "no assembled operators: call ldg_assemble first");
}

// Device SoA blocks [ncomp][4][N*N][Kp] -> host copy
std::vector<double> blocks_to_host(Handle& h, const double* dev, int ncomp) {
  const size_t cnt = static_cast<size_t>(ncomp) * 4 * h.N * h.N * h.Kp;
  std::vector<double> out(cnt);
  LDG_CUDA(cudaMemcpyAsync(out.data(), dev, cnt * sizeof(double), cudaMemcpyDeviceToHost, h.stream));
  LDG_CUDA(cudaStreamSynchronize(h.stream));
  return out;
}

struct Coo {
  std::vector<int64_t> r, c;
  std::vector<double> v;
};

// Appends block slot s of element k: rows (ru*K + gid(k))*N + i, cols (cu*K + gid(col))*N + j.
void push_block(const Handle& h, const std::vector<int>& nbr_host, const double* blk, int k, int s, int ru,
                int cu, double scale, Coo& out) {
  const int N = h.N;
  int col = k;
  if (s > 0) {
    col = nbr_host[(s - 1) * h.Kp + k];
    if (col < 0) return;
  }
  const int64_t Kg = h.Kglobal;
  const int64_t grow = ru * Kg + h.gid[k], gcol = cu * Kg + h.gid[col];
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      out.r.push_back(grow * N + i);
      out.c.push_back(gcol * N + j);
      out.v.push_back(scale * blk[static_cast<size_t>(s * N * N + i * N + j) * h.Kp + k]);
    }
}

}  // namespace

extern "C" {

const char* ldg_last_error(const ldg_handle* H) {
  if (H && !H->h.err.empty()) return H->h.err.c_str();
  return g_last_error.c_str();
}

int ldg_reference_tensors(int n_local, double* m, double* h, double* g, double* sd, double* so, double* rd,
                          double* ro) {
  return guarded(nullptr, [&] {
    const ldgb::RefTensors t = ldgb::reference_tensors(n_local);
    auto put = [](const std::vector<double>& v, double* out) {
      if (out) std::copy(v.begin(), v.end(), out);
    };
    put(t.m, m);
    put(t.h, h);
    put(t.g, g);
    put(t.sd, sd);
    put(t.so, so);
    put(t.rd, rd);
    put(t.ro, ro);
  });
}

int ldg_set_device(int device) {
  return guarded(nullptr, [&] { LDG_CUDA(cudaSetDevice(device)); });
}

ldg_solver_opts ldg_default_solver_opts(void) {
  ldg_solver_opts o;
  o.rtol = 0.0;
  o.atol = 0.0;
  o.maxit = 20000;
  o.precond = 2;
  o.check_residual = 1;
  o.contract_tol = 1e-10;
  return o;
}

int ldg_create(const double* coords, int num_v, const int* v0t, int num_t, const int* id_e0t, int p,
               const ldg_problem* prob, ldg_handle** out) {
  if (!out) return LDG_EINVAL;
  *out = nullptr;
  auto H = std::make_unique<ldg_handle>();
  const int rc = guarded(nullptr, [&] {
    validate_problem(prob, p);
    init_device_side(H->h, p, prob);
    ldgb::build_general_mesh(H->h, coords, num_v, v0t, num_t, id_e0t);
    alloc_step_buffers(H->h);
    LDG_CUDA(cudaStreamSynchronize(H->h.stream));
  });
  if (rc == LDG_OK) *out = H.release();
  return rc;
}

int ldg_create_square(int dim, double jitter, uint64_t seed, int p, const ldg_problem* prob, ldg_handle** out) {
  if (!out) return LDG_EINVAL;
  *out = nullptr;
  auto H = std::make_unique<ldg_handle>();
  const int rc = guarded(nullptr, [&] {
    validate_problem(prob, p);
    init_device_side(H->h, p, prob);
    ldgb::build_square_mesh(H->h, dim, jitter, seed);
    alloc_step_buffers(H->h);
    LDG_CUDA(cudaStreamSynchronize(H->h.stream));
  });
  if (rc == LDG_OK) *out = H.release();
  return rc;
}

void ldg_destroy(ldg_handle* H) {
  if (!H) return;
  Handle& h = H->h;
  if (h.stream) cudaStreamSynchronize(h.stream);
  ldgb::mg_release(h);
  if (h.red_host) cudaFreeHost(h.red_host);
  for (auto& e : h.ev)
    if (e) cudaEventDestroy(e);
  cudaStream_t s = h.stream;
  delete H;  // DBuf destructors free device memory
  if (s) cudaStreamDestroy(s);
}

int ldg_get_info(const ldg_handle* H, ldg_info_t* out) {
  if (!H || !out) return LDG_EINVAL;
  const Handle& h = H->h;
  out->p = h.p;
  out->n_local = h.N;
  out->num_t = h.Kglobal;
  out->num_owned = h.K;
  out->num_ghost = h.Kg - h.K;
  out->num_v = h.V;
  out->rank = h.rank;
  out->size = h.size;
  out->bytes_device = h.bytes;
  out->launches = h.launches;
  for (const auto& c : h.coarse) out->launches += c->launches;
  return LDG_OK;
}

int ldg_mesh_lists(ldg_handle* H, double* coords, int* v0t, double* b, double* area, double* len, double* nu,
                   int* nbr, int* nbr_n, int* id_e0t) {
  if (!H) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    const long Kp = h.Kp;
    std::vector<double> g(static_cast<size_t>(ldgb::kGeomCount) * Kp);
    std::vector<int> nb(3 * Kp), nn(3 * Kp), bid(3 * Kp), vt(3L * h.Kg);
    LDG_CUDA(cudaMemcpy(g.data(), h.geom.ptr, sizeof(double) * g.size(), cudaMemcpyDeviceToHost));
    LDG_CUDA(cudaMemcpy(nb.data(), h.nbr.ptr, sizeof(int) * nb.size(), cudaMemcpyDeviceToHost));
    LDG_CUDA(cudaMemcpy(nn.data(), h.nbrn.ptr, sizeof(int) * nn.size(), cudaMemcpyDeviceToHost));
    LDG_CUDA(cudaMemcpy(bid.data(), h.bid.ptr, sizeof(int) * bid.size(), cudaMemcpyDeviceToHost));
    LDG_CUDA(cudaMemcpy(vt.data(), h.v0t.ptr, sizeof(int) * vt.size(), cudaMemcpyDeviceToHost));
    if (coords) LDG_CUDA(cudaMemcpy(coords, h.coords.ptr, sizeof(double) * 2 * h.V, cudaMemcpyDeviceToHost));
    for (int k = 0; k < h.K; ++k) {
      const int gk = h.gid[k];
      if (v0t)
        for (int i = 0; i < 3; ++i) v0t[3 * gk + i] = vt[3 * k + i];
      if (b) {
        b[4 * gk] = g[ldgb::kB11 * Kp + k];
        b[4 * gk + 1] = g[ldgb::kB12 * Kp + k];
        b[4 * gk + 2] = g[ldgb::kB21 * Kp + k];
        b[4 * gk + 3] = g[ldgb::kB22 * Kp + k];
      }
      if (area) area[gk] = g[ldgb::kArea * Kp + k];
      for (int n = 0; n < 3; ++n) {
        if (len) len[3 * gk + n] = g[(ldgb::kLen0 + n) * Kp + k];
        if (nu) {
          nu[6 * gk + 2 * n] = g[(ldgb::kNux0 + n) * Kp + k];
          nu[6 * gk + 2 * n + 1] = g[(ldgb::kNuy0 + n) * Kp + k];
        }
        const int kp = nb[n * Kp + k];
        if (nbr) nbr[3 * gk + n] = kp < 0 ? -1 : h.gid[kp];
        if (nbr_n) nbr_n[3 * gk + n] = nn[n * Kp + k];
        if (id_e0t) id_e0t[3 * gk + n] = bid[n * Kp + k];
      }
    }
  });
}

int ldg_project(ldg_handle* H, const ldg_coeff* fn, double t, int q_ord, double* out) {
  if (!H || !fn) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    if (fn->id < 0 || fn->id >= LDG_FN_COUNT) throw Error(LDG_EINVAL, "unknown coefficient function id");
    DBuf<double> rule, tmp, km;
    int R = 0;
    ldgb::upload_rule(h, q_ord, rule, &R);
    tmp.alloc(h.vec_len(), nullptr);
    km.alloc(static_cast<size_t>(h.K) * h.N, nullptr);
    ldgb::launch_project(h, *fn, t, rule.ptr, R, tmp.ptr, h.K);
    ldgb::launch_soa_to_kmajor(h, tmp.ptr, 1, km.ptr);
    LDG_CUDA(cudaMemcpyAsync(out, km.ptr, sizeof(double) * h.K * h.N, cudaMemcpyDeviceToHost, h.stream));
    LDG_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int ldg_assemble(ldg_handle* H, double t) {
  if (!H) return LDG_EINVAL;
  return guarded(H, [&] {
    ldgb::assemble_step(H->h, t);
    LDG_CUDA(cudaStreamSynchronize(H->h.stream));
  });
}

int ldg_export_operator(ldg_handle* H, int which, int64_t* nnz, int64_t* rows, int64_t* cols, double* vals,
                        int64_t cap) {
  if (!H || !nnz) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    if (which < 0 || which >= LDG_OP_COUNT) throw Error(LDG_EINVAL, "unknown operator");
    const bool needs_d = which == LDG_OP_G1 || which == LDG_OP_G2 || which == LDG_OP_R1 || which == LDG_OP_R2 ||
                         which == LDG_OP_RD1 || which == LDG_OP_RD2 || which == LDG_OP_A;
    if (needs_d) require_assembled(h);
    ensure_solver(h);
    std::vector<int> nb(3 * h.Kp);
    LDG_CUDA(cudaMemcpy(nb.data(), h.nbr.ptr, sizeof(int) * nb.size(), cudaMemcpyDeviceToHost));
    const long NN = static_cast<long>(h.N) * h.N;
    DBuf<double> tmp;
    Coo coo;
    auto emit = [&](const std::vector<double>& blk, int comp, bool off, int ru, int cu, double scale) {
      const double* base = blk.data() + static_cast<size_t>(comp) * 4 * NN * h.Kp;
      for (int k = 0; k < h.K; ++k)
        for (int s = 0; s < (off ? 4 : 1); ++s) push_block(h, nb, base, k, s, ru, cu, scale, coo);
    };
    if (which == LDG_OP_A) {
      // the static blocks exactly as the matrix-free kernels rebuild them (K4)
      tmp.alloc(8 * NN * h.Kp, nullptr);
      ldgb::launch_static(h, ldgb::kStM, tmp.ptr);
      const auto M = blocks_to_host(h, tmp.ptr, 1);
      ldgb::launch_static(h, ldgb::kStB, tmp.ptr);
      const auto B = blocks_to_host(h, tmp.ptr, 2);
      ldgb::launch_static(h, ldgb::kStS, tmp.ptr);
      const auto S = blocks_to_host(h, tmp.ptr, 1);
      const auto E = blocks_to_host(h, h.E.ptr, 2);
      emit(M, 0, false, 0, 0, 1.0);
      emit(B, 0, true, 0, 2, 1.0);
      emit(M, 0, false, 1, 1, 1.0);
      emit(B, 1, true, 1, 2, 1.0);
      emit(E, 0, true, 2, 0, 1.0);
      emit(E, 1, true, 2, 1, 1.0);
      emit(S, 0, true, 2, 2, h.prob.eta);
    } else {
      tmp.alloc(8 * NN * h.Kp, nullptr);
      int comp = 0;
      bool off = false;
      switch (which) {
        case LDG_OP_MASS: ldgb::launch_static(h, ldgb::kStM, tmp.ptr); break;
        case LDG_OP_H1: case LDG_OP_H2:
          ldgb::launch_static(h, ldgb::kStH, tmp.ptr);
          comp = which == LDG_OP_H2;
          break;
        case LDG_OP_Q1: case LDG_OP_Q2:
          ldgb::launch_static(h, ldgb::kStQ, tmp.ptr);
          comp = which == LDG_OP_Q2;
          off = true;
          break;
        case LDG_OP_QN1: case LDG_OP_QN2:
          ldgb::launch_static(h, ldgb::kStQN, tmp.ptr);
          comp = which == LDG_OP_QN2;
          break;
        case LDG_OP_S:
          ldgb::launch_static(h, ldgb::kStSint, tmp.ptr);
          off = true;
          break;
        case LDG_OP_SD: ldgb::launch_static(h, ldgb::kStSD, tmp.ptr); break;
        case LDG_OP_G1: case LDG_OP_G2:
          ldgb::launch_assemble(h, ldgb::kModeG, tmp.ptr);
          comp = which == LDG_OP_G2;
          break;
        case LDG_OP_R1: case LDG_OP_R2:
          ldgb::launch_assemble(h, ldgb::kModeR, tmp.ptr);
          comp = which == LDG_OP_R2;
          off = true;
          break;
        default:
          ldgb::launch_assemble(h, ldgb::kModeRD, tmp.ptr);
          comp = which == LDG_OP_RD2;
          break;
      }
      const auto blk = blocks_to_host(h, tmp.ptr, 2);
      emit(blk, comp, off, 0, 0, 1.0);
    }
    *nnz = static_cast<int64_t>(coo.v.size());
    if (rows && cols && vals) {
      if (cap < *nnz) throw Error(LDG_EINVAL, "export capacity too small");
      std::copy(coo.r.begin(), coo.r.end(), rows);
      std::copy(coo.c.begin(), coo.c.end(), cols);
      std::copy(coo.v.begin(), coo.v.end(), vals);
    }
  });
}

int ldg_export_vector(ldg_handle* H, int which, double* out, int64_t cap) {
  if (!H || !out) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    const long n = h.vec_len();
    const double* src = nullptr;
    int nvec = 1;
    DBuf<double> tmp;
    switch (which) {
      case LDG_VEC_D: require_assembled(h); src = h.D.ptr; break;
      case LDG_VEC_F: require_assembled(h); src = h.F.ptr; break;
      case LDG_VEC_JD1: case LDG_VEC_JD2: case LDG_VEC_KD: case LDG_VEC_KN: case LDG_VEC_L:
        require_assembled(h);
        tmp.alloc(n, nullptr);
        ldgb::launch_rhs_which(h, h.t_assembled, 1 + (which - LDG_VEC_JD1), tmp.ptr);
        src = tmp.ptr;
        break;
      case LDG_VEC_V: require_assembled(h); src = h.Vv.ptr; nvec = 3; break;
      case LDG_VEC_Y: src = h.Y.ptr; nvec = 3; break;
      default: throw Error(LDG_EINVAL, "unknown vector");
    }
    const int64_t cnt = static_cast<int64_t>(nvec) * h.K * h.N;
    if (cap < cnt) throw Error(LDG_EINVAL, "export capacity too small");
    DBuf<double> km;
    km.alloc(cnt, nullptr);
    ldgb::launch_soa_to_kmajor(h, src, nvec, km.ptr);
    LDG_CUDA(cudaMemcpyAsync(out, km.ptr, sizeof(double) * cnt, cudaMemcpyDeviceToHost, h.stream));
    LDG_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int ldg_initial_state(ldg_handle* H) {
  if (!H) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    LDG_CUDA(cudaMemsetAsync(h.Y.ptr, 0, sizeof(double) * 3 * h.vec_len(), h.stream));
    ldgb::launch_project(h, h.prob.c0, 0.0, h.rule_elem.ptr, h.rule_elem_R, h.Y.ptr + 2 * h.vec_len(), h.K);
    h.t = 0.0;
    LDG_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int ldg_set_state(ldg_handle* H, const double* y, double t) {
  if (!H || !y) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    const size_t cnt = 3L * h.K * h.N;
    DBuf<double> km;
    km.alloc(cnt, nullptr);
    LDG_CUDA(cudaMemcpyAsync(km.ptr, y, sizeof(double) * cnt, cudaMemcpyHostToDevice, h.stream));
    ldgb::launch_kmajor_to_soa(h, km.ptr, 3, h.Y.ptr);
    h.t = t;
    LDG_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int ldg_get_state(ldg_handle* H, double* y, double* t) {
  if (!H) return LDG_EINVAL;
  if (t) *t = H->h.t;
  if (!y) return LDG_OK;
  return ldg_export_vector(H, LDG_VEC_Y, y, 3L * H->h.K * H->h.N);
}

int ldg_euler_steps(ldg_handle* H, double dt, int nsteps, const ldg_solver_opts* opts, ldg_step_stats* st) {
  if (!H) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    if (!(dt > 0.0)) throw Error(LDG_EINVAL, "time step must be positive");
    ensure_solver(h);
    const ldg_solver_opts o = opts ? *opts : ldg_default_solver_opts();
    if (st) *st = ldg_step_stats{};
    for (int s = 0; s < nsteps; ++s) {
      const double t_next = h.t + dt;  // system.hpp:158
      LDG_CUDA(cudaEventRecord(h.ev[0], h.stream));
      ldgb::assemble_step(h, t_next);
      LDG_CUDA(cudaEventRecord(h.ev[1], h.stream));
      ldgb::solve_step(h, 1.0, dt, o, st);
      LDG_CUDA(cudaEventRecord(h.ev[2], h.stream));
      LDG_CUDA(cudaEventSynchronize(h.ev[2]));
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, h.ev[0], h.ev[1]);
      cudaEventElapsedTime(&b, h.ev[1], h.ev[2]);
      if (st) {
        st->ms_assemble += a;
        st->ms_solve += b;
      }
      h.t = t_next;
    }
  });
}

int ldg_euler_steps_host(ldg_handle* H, const double* y_in, double t, double dt, int nsteps, double* y_out,
                         const ldg_solver_opts* opts, ldg_step_stats* st, double* ms_total) {
  if (!H || !y_in || !y_out) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    if (!(dt > 0.0)) throw Error(LDG_EINVAL, "time step must be positive");
    ensure_solver(h);
    const ldg_solver_opts o = opts ? *opts : ldg_default_solver_opts();
    if (st) *st = ldg_step_stats{};
    const size_t cnt = 3L * h.K * h.N;
    if (!h.host_stage.ptr) h.host_stage.alloc(cnt, &h.bytes);
    LDG_CUDA(cudaEventRecord(h.ev[3], h.stream));
    LDG_CUDA(cudaMemcpyAsync(h.host_stage.ptr, y_in, sizeof(double) * cnt, cudaMemcpyHostToDevice, h.stream));
    ldgb::launch_kmajor_to_soa(h, h.host_stage.ptr, 3, h.Y.ptr);
    h.t = t;
    for (int s = 0; s < nsteps; ++s) {
      const double t_next = h.t + dt;
      LDG_CUDA(cudaEventRecord(h.ev[0], h.stream));
      ldgb::assemble_step(h, t_next);
      LDG_CUDA(cudaEventRecord(h.ev[1], h.stream));
      ldgb::solve_step(h, 1.0, dt, o, st);
      LDG_CUDA(cudaEventRecord(h.ev[2], h.stream));
      LDG_CUDA(cudaEventSynchronize(h.ev[2]));
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, h.ev[0], h.ev[1]);
      cudaEventElapsedTime(&b, h.ev[1], h.ev[2]);
      if (st) {
        st->ms_assemble += a;
        st->ms_solve += b;
      }
      h.t = t_next;
    }
    ldgb::launch_soa_to_kmajor(h, h.Y.ptr, 3, h.host_stage.ptr);
    LDG_CUDA(cudaMemcpyAsync(y_out, h.host_stage.ptr, sizeof(double) * cnt, cudaMemcpyDeviceToHost, h.stream));
    LDG_CUDA(cudaEventRecord(h.ev[2], h.stream));
    LDG_CUDA(cudaEventSynchronize(h.ev[2]));
    float tot = 0.f;
    cudaEventElapsedTime(&tot, h.ev[3], h.ev[2]);
    if (ms_total) *ms_total = tot;
  });
}

int ldg_solve_stationary(ldg_handle* H, double t, const ldg_solver_opts* opts, ldg_step_stats* st) {
  if (!H) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    ensure_solver(h);
    const ldg_solver_opts o = opts ? *opts : ldg_default_solver_opts();
    if (st) *st = ldg_step_stats{};
    ldgb::assemble_step(h, t);
    ldgb::solve_step(h, 0.0, 1.0, o, st);
    h.t = t;
    LDG_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int ldg_apply_lhs(ldg_handle* H, double dt, const double* x, double* y) {
  if (!H || !x || !y) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    require_assembled(h);
    ensure_solver(h);
    const size_t cnt = 3L * h.K * h.N;
    DBuf<double> km, xs, ys;
    km.alloc(cnt, nullptr);
    xs.alloc(3 * h.vec_len(), nullptr);
    ys.alloc(3 * h.vec_len(), nullptr);
    LDG_CUDA(cudaMemcpyAsync(km.ptr, x, sizeof(double) * cnt, cudaMemcpyHostToDevice, h.stream));
    ldgb::launch_kmajor_to_soa(h, km.ptr, 3, xs.ptr);
    ldgb::launch_full_apply(h, xs.ptr, 1.0, dt, ys.ptr);
    ldgb::launch_soa_to_kmajor(h, ys.ptr, 3, km.ptr);
    LDG_CUDA(cudaMemcpyAsync(y, km.ptr, sizeof(double) * cnt, cudaMemcpyDeviceToHost, h.stream));
    LDG_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int ldg_sync(ldg_handle* H) {
  if (!H) return LDG_EINVAL;
  return guarded(H, [&] { LDG_CUDA(cudaStreamSynchronize(H->h.stream)); });
}

int ldg_time_kernels(ldg_handle* H, double t, double dt, int reps, int flush, ldg_kernel_times* out) {
  if (!H || !out || reps < 1) return LDG_EINVAL;
  return guarded(H, [&] {
    Handle& h = H->h;
    ensure_solver(h);
    const size_t flush_n = (256ull << 20) / sizeof(double);  // 256 MB > 126 MB L2
    if (flush && !h.flush.ptr) h.flush.alloc(flush_n, nullptr);
    auto timed = [&](auto&& fn) {
      for (int w = 0; w < 2; ++w) fn();  // warm-up
      float total = 0.f;
      for (int r = 0; r < reps; ++r) {
        if (flush) LDG_CUDA(cudaMemsetAsync(h.flush.ptr, r & 0xff, flush_n * sizeof(double), h.stream));
        LDG_CUDA(cudaEventRecord(h.ev[0], h.stream));
        fn();
        LDG_CUDA(cudaEventRecord(h.ev[1], h.stream));
        LDG_CUDA(cudaEventSynchronize(h.ev[1]));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h.ev[0], h.ev[1]);
        total += ms;
      }
      return static_cast<double>(total) / reps;
    };
    out->reps = reps;
    out->ms_project = timed([&] {
      ldgb::launch_project_df(h, t, h.rule_elem.ptr, h.rule_elem_R);
      ldgb::launch_rhs(h, t);
    });
    out->ms_assemble = timed([&] { ldgb::launch_assemble(h, ldgb::kModeE, h.E.ptr); });
    h.assembled = true;
    h.t_assembled = t;
    out->ms_spmv = timed([&] { ldgb::launch_full_apply(h, h.Y.ptr, 1.0, dt, h.full_y.ptr); });
    out->ms_schur = timed([&] {
      ldgb::launch_stage1(h, nullptr, 0.0, h.Y.ptr + 2 * h.vec_len(), 1.0, h.tz.ptr);
      ldgb::launch_stage2(h, h.Y.ptr + 2 * h.vec_len(), 1.0, dt * h.prob.eta, h.tz.ptr, dt, nullptr, 0.0,
                          h.kr_v.ptr);
    });
  });
}

}  // extern "C"
