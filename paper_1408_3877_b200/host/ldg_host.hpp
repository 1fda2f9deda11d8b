// C++ host mirror of the reference's entry points over the C ABI of
// include/ldg_b200.h — the same class/function shapes as
// proj/include/ldg/system.hpp and fields.hpp, the same exception types
// (std::invalid_argument, ldg::b200::MeshError, std::runtime_error), so a
// caller written against ldg::LdgSystem (e.g. cmd_simulate, ldg_main.cpp:
// 174-222) switches by changing the namespace and the coefficient type.
//
// Header-only; link with -lldg_b200.  Not thread-safe per object (one
// LdgSystem per GPU/thread), like the handle it wraps.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "ldg_b200.h"

namespace ldg::b200 {

/// mesh.hpp:25-27
struct MeshError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// A compiled-in coefficient function (the device cannot call std::function,
/// fields.hpp:19); see include/ldg_b200_coeffs.h for the ids.
inline ldg_coeff coeff(int id, double p0 = 0.0, double p1 = 0.0, double p2 = 0.0, double p3 = 0.0) {
  ldg_coeff c;
  c.id = id;
  c.p[0] = p0;
  c.p[1] = p1;
  c.p[2] = p2;
  c.p[3] = p3;
  return c;
}

enum class Bc { kDirichlet, kNeumann };  // system.hpp:23

/// system.hpp:26-37
struct ProblemSpec {
  ldg_coeff d = coeff(LDG_FN_CONST, 1.0);
  ldg_coeff f = coeff(LDG_FN_ZERO);
  ldg_coeff c_d = coeff(LDG_FN_ZERO);
  ldg_coeff g_n = coeff(LDG_FN_ZERO);
  ldg_coeff c0 = coeff(LDG_FN_ZERO);
  double eta = 1.0;
  std::map<int, Bc> boundary;
  double t_end = 1.0;
  int num_steps = 1;
};

/// system.hpp:40-43
struct SystemState {
  std::vector<double> y;  // 3*K*N, ordered (Z1, Z2, C), k-major per block
  double t = 0.0;
};

/// SparseOperator (assembly.hpp:21): the arrays of a compressed column-major
/// Eigen::SparseMatrix<double> with int indices, maps onto
/// Eigen::Map<const Eigen::SparseMatrix<double>>(rows, cols, nnz, outer.data(), inner.data(), values.data()).
struct SparseOperator {
  int rows = 0, cols = 0;
  std::vector<int> outer;     // cols + 1 column pointers
  std::vector<int> inner;     // row index per stored entry, ascending within a column
  std::vector<double> values;
  long nonZeros() const { return static_cast<long>(values.size()); }
};

/// system.hpp:57-61
struct SystemBlocks {
  SparseOperator a;           // 3KN x 3KN, Eq. (5) block layout
  std::vector<double> v;      // [-J_D^1; -J_D^2; eta K_D - K_N + L]
};

/// RefTensors (reftensors.hpp:25-50): the same flat index layout.
struct RefTensors {
  int n = 0;
  std::vector<double> m, h, g, sd, so, rd, ro;
};

/// Block CSR of an operator: N x N row-major blocks, block rows in the
/// reference's element order.
struct BlockOperator {
  int n_local = 0;
  std::vector<int> rowptr, colind;
  std::vector<double> blocks;
};

namespace detail {

inline void check(int rc, const ldg_handle* h) {
  if (rc == LDG_OK) return;
  const std::string msg = ldg_last_error(h);
  switch (rc) {
    case LDG_EINVAL: throw std::invalid_argument(msg);
    case LDG_EMESH: throw MeshError(msg);
    default: throw std::runtime_error(msg);
  }
}

inline ldg_problem to_c(const ProblemSpec& s) {
  ldg_problem p{};
  p.d = s.d;
  p.f = s.f;
  p.c_d = s.c_d;
  p.g_n = s.g_n;
  p.c0 = s.c0;
  p.eta = s.eta;
  if (s.boundary.size() > LDG_MAX_BC) throw std::invalid_argument("too many boundary conditions");
  p.n_bc = 0;
  for (const auto& [id, kind] : s.boundary) {
    p.bc_id[p.n_bc] = id;
    p.bc_kind[p.n_bc] = kind == Bc::kDirichlet ? LDG_BC_DIRICHLET : LDG_BC_NEUMANN;
    ++p.n_bc;
  }
  return p;
}

struct HandleDeleter {
  void operator()(ldg_handle* h) const { ldg_destroy(h); }
};

}  // namespace detail

/// Device-resident LdgSystem (system.hpp:65-213).
class LdgSystem {
 public:
  /// domain_square(1/dim) (mesh.hpp:225-254) generated on the device.
  static LdgSystem square(int dim, int p, const ProblemSpec& spec, double jitter = 0.0, uint64_t seed = 0) {
    const ldg_problem pr = detail::to_c(spec);
    ldg_handle* h = nullptr;
    detail::check(ldg_create_square(dim, jitter, seed, p, &pr, &h), nullptr);
    return LdgSystem(h, spec);
  }

  /// generate_grid_data(coords, v0t) + the LdgSystem ctor; id_e0t (K x 3,
  /// optional) carries boundary IDs per (triangle, local edge).
  LdgSystem(const std::vector<std::array<double, 2>>& coords, const std::vector<std::array<int, 3>>& v0t, int p,
            const ProblemSpec& spec, const std::vector<std::array<int, 3>>* id_e0t = nullptr)
      : spec_(spec) {
    const ldg_problem pr = detail::to_c(spec);
    ldg_handle* h = nullptr;
    detail::check(ldg_create(coords.empty() ? nullptr : coords[0].data(), static_cast<int>(coords.size()),
                             v0t.empty() ? nullptr : v0t[0].data(), static_cast<int>(v0t.size()),
                             id_e0t ? (*id_e0t)[0].data() : nullptr, p, &pr, &h),
                  nullptr);
    h_.reset(h);
    load_info();
  }

  int n_local() const { return info_.n_local; }
  int num_t() const { return info_.num_t; }
  int block_dim() const { return info_.num_t * info_.n_local; }  // system.hpp:95
  const ProblemSpec& spec() const { return spec_; }
  ldg_handle* handle() const { return h_.get(); }

  /// project(mesh, func, t, q_ord, rt) (fields.hpp:53-82): K x N, k-major.
  std::vector<double> project(const ldg_coeff& fn, double t, int q_ord) const {
    std::vector<double> out(static_cast<size_t>(block_dim()));
    detail::check(ldg_project(h_.get(), &fn, t, q_ord, out.data()), h_.get());
    return out;
  }

  /// build_blocks(t) (system.hpp:110-152): assembles on the device (the
  /// operators stay in HBM for euler_step) and returns A in the reference's
  /// CSC storage with V.  Use assemble(t) to skip the host copy.
  SystemBlocks build_blocks(double t) const {
    assemble(t);
    SystemBlocks b;
    b.a = operator_csc(LDG_OP_A);
    b.v.resize(3u * static_cast<size_t>(block_dim()));
    detail::check(ldg_export_vector(h_.get(), LDG_VEC_V, b.v.data(), static_cast<int64_t>(b.v.size())), h_.get());
    return b;
  }

  /// The rt of the reference's LdgSystem(mesh, spec, rt) (system.hpp:67): the
  /// device operators are then built from the caller's tensors.
  void set_reference_tensors(const RefTensors& rt) const {
    if (rt.n != n_local()) throw std::invalid_argument("reference tensor size mismatch");
    detail::check(ldg_set_reference_tensors(h_.get(), rt.m.data(), rt.h.data(), rt.g.data(), rt.sd.data(),
                                            rt.so.data(), rt.rd.empty() ? nullptr : rt.rd.data(),
                                            rt.ro.empty() ? nullptr : rt.ro.data()),
                  h_.get());
  }

  /// The device half of build_blocks(t): projection, assembly, right-hand side.
  void assemble(double t) const { detail::check(ldg_assemble(h_.get(), t), h_.get()); }

  /// One operator of the last assemble() (enum ldg_operator) as the reference stores it.
  SparseOperator operator_csc(int which) const {
    const int n = (which == LDG_OP_A ? 3 : 1) * block_dim();
    return csc_call(n, [&](int64_t* nnz, int32_t* cp, int32_t* ri, double* v, int64_t cap) {
      return ldg_export_operator_csc(h_.get(), which, nnz, cp, ri, v, cap);
    });
  }

  /// The same operator as block CSR (N x N row-major blocks).
  BlockOperator operator_bsr(int which) const {
    BlockOperator b;
    b.n_local = n_local();
    int64_t nb = 0;
    detail::check(ldg_export_operator_bsr(h_.get(), which, &nb, nullptr, nullptr, nullptr, 0), h_.get());
    b.rowptr.resize(static_cast<size_t>((which == LDG_OP_A ? 3 : 1) * num_t()) + 1);
    b.colind.resize(static_cast<size_t>(nb));
    b.blocks.resize(static_cast<size_t>(nb) * n_local() * n_local());
    detail::check(ldg_export_operator_bsr(h_.get(), which, &nb, b.rowptr.data(), b.colind.data(), b.blocks.data(), nb),
                  h_.get());
    return b;
  }

  /// assemble_dphi_phi_coeff(mesh, rt, d_disc) (assembly.hpp:113-136) -> (G^1, G^2);
  /// d_disc is K x N, k-major.
  std::pair<SparseOperator, SparseOperator> assemble_dphi_phi_coeff(const std::vector<double>& d_disc) const {
    check_d(d_disc);
    auto g = [&](int m) {
      return csc_call(block_dim(), [&](int64_t* nnz, int32_t* cp, int32_t* ri, double* v, int64_t cap) {
        return ldg_assemble_dphi_phi_coeff(h_.get(), d_disc.data(), m, nnz, cp, ri, v, cap);
      });
    };
    return {g(1), g(2)};
  }

  /// assemble_edge_avg_coeff_nu(mesh, m, d_disc, sel_int, sel_dir, rt)
  /// (assembly.hpp:214-252) -> (R^m, R_D^m).
  std::pair<SparseOperator, SparseOperator> assemble_edge_avg_coeff_nu(int m, const std::vector<double>& d_disc) const {
    check_d(d_disc);
    auto r = [&](int dir) {
      return csc_call(block_dim(), [&](int64_t* nnz, int32_t* cp, int32_t* ri, double* v, int64_t cap) {
        return ldg_assemble_edge_avg_coeff_nu(h_.get(), d_disc.data(), m, dir, nnz, cp, ri, v, cap);
      });
    };
    return {r(0), r(1)};
  }

  /// system.hpp:99-107
  SystemState initial_state() const {
    detail::check(ldg_initial_state(h_.get()), h_.get());
    return state();
  }

  /// system.hpp:155-174: one implicit Euler step of length dt.
  SystemState euler_step(const SystemState& s, double dt, const ldg_solver_opts* opts = nullptr) const {
    if (s.y.size() != 3u * static_cast<size_t>(block_dim()))
      throw std::invalid_argument("state length does not match 3*K*N");
    SystemState next;
    next.y.resize(s.y.size());
    detail::check(ldg_euler_steps_host(h_.get(), s.y.data(), s.t, dt, 1, next.y.data(), opts, nullptr, nullptr),
                  h_.get());
    next.t = s.t + dt;
    return next;
  }

  /// nsteps steps on the device-resident state (no host copies in between).
  ldg_step_stats advance(double dt, int nsteps, const ldg_solver_opts* opts = nullptr) const {
    ldg_step_stats st{};
    detail::check(ldg_euler_steps(h_.get(), dt, nsteps, opts, &st), h_.get());
    return st;
  }

  SystemState state() const {
    SystemState s;
    s.y.resize(3u * static_cast<size_t>(block_dim()));
    detail::check(ldg_get_state(h_.get(), s.y.data(), &s.t), h_.get());
    return s;
  }

  /// system.hpp:177-185 -> (c, z1, z2), each K x N k-major.
  std::tuple<std::vector<double>, std::vector<double>, std::vector<double>> solve_stationary(
      double t = 0.0, const ldg_solver_opts* opts = nullptr) const {
    detail::check(ldg_solve_stationary(h_.get(), t, opts, nullptr), h_.get());
    const SystemState s = state();
    const size_t kn = static_cast<size_t>(block_dim());
    return {std::vector<double>(s.y.begin() + 2 * kn, s.y.end()), std::vector<double>(s.y.begin(), s.y.begin() + kn),
            std::vector<double>(s.y.begin() + kn, s.y.begin() + 2 * kn)};
  }

  /// l2_error(mesh, dof, exact, t, q_ord) (fields.hpp:100-123) of the
  /// device-resident state component (0 Z1, 1 Z2, 2 C).
  double l2_error(const ldg_coeff& exact, double t, int q_ord, int component = 2) const {
    double e = 0.0;
    detail::check(ldg_l2_error(h_.get(), component, &exact, t, q_ord, &e), h_.get());
    return e;
  }

  /// write_vtu (vtkout.hpp:42-108) of a state component (2 = C) from the
  /// device-resident state; returns the written path.
  std::string write_vtu(int component, const std::string& var_name, const std::string& basename,
                        int t_lvl) const {
    char path[4096];
    detail::check(ldg_write_vtu(h_.get(), component, var_name.c_str(), basename.c_str(), t_lvl, path,
                                static_cast<int>(sizeof(path))),
                  h_.get());
    return path;
  }

  /// to_lagrange(dof) (fields.hpp:87-97) of a state component: K x 3 (p <= 1)
  /// or K x 6, k-major; *nodes receives the column count.
  std::vector<double> to_lagrange(int component = 2, int* nodes = nullptr) const {
    const int m = info_.p <= 1 ? 3 : 6;
    std::vector<double> out(static_cast<size_t>(num_t()) * m);
    detail::check(ldg_to_lagrange(h_.get(), component, out.data(), nodes), h_.get());
    return out;
  }

 private:
  LdgSystem(ldg_handle* h, ProblemSpec spec) : h_(h), spec_(std::move(spec)) { load_info(); }
  void load_info() { detail::check(ldg_get_info(h_.get(), &info_), h_.get()); }
  void check_d(const std::vector<double>& d) const {
    if (d.size() != static_cast<size_t>(block_dim())) throw std::invalid_argument("coefficient matrix shape mismatch");
  }
  template <typename F>
  SparseOperator csc_call(int n, F&& call) const {
    SparseOperator op;
    op.rows = op.cols = n;
    int64_t nnz = 0;
    detail::check(call(&nnz, nullptr, nullptr, nullptr, 0), h_.get());
    op.outer.resize(static_cast<size_t>(n) + 1);
    op.inner.resize(static_cast<size_t>(nnz));
    op.values.resize(static_cast<size_t>(nnz));
    detail::check(call(&nnz, op.outer.data(), op.inner.data(), op.values.data(), nnz), h_.get());
    return op;
  }

  std::unique_ptr<ldg_handle, detail::HandleDeleter> h_;
  ProblemSpec spec_;
  ldg_info_t info_{};
};

}  // namespace ldg::b200
