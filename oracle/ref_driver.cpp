// TEST INFRASTRUCTURE ONLY — oracle/_ref/libldgref.so.
//
// A thin C ABI over the UNMODIFIED reference headers (/root/reference/proj/
// include/ldg, compiled in place against oracle/shim), so Python tests,
// tests/golden generation and bench.py's reference arm can call the
// reference's own code path:
//   domain_square / generate_grid_data / refine_uniform   (mesh.hpp:103-293)
//   build_ref_tensors                                      (reftensors.hpp:55)
//   project                                                (fields.hpp:53)
//   every assemble_* operator and vector                   (assembly.hpp:76-338)
//   LdgSystem::{build_blocks, euler_step, solve_stationary} (system.hpp:110-185)
//   l2_error, run_convergence                              (fields.hpp:100, convergence.hpp:77)
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
// legs load this library.  The product path never does.
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>

#include "ldg/assembly.hpp"
#include "ldg/convergence.hpp"
#include "ldg/fields.hpp"
#include "ldg/mesh.hpp"
#include "ldg/reftensors.hpp"
#include "ldg/system.hpp"
#include "../include/ldg_b200_coeffs.h"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const ldg::MeshError& e) {
    g_err = std::string("MeshError: ") + e.what();
    return 2;
  } catch (const std::runtime_error& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = std::string("exception: ") + e.what();
    return 9;
  }
}

ldg::ScalarFunc make_func(int id, const double* p) {
  std::array<double, 4> q{p[0], p[1], p[2], p[3]};
  return [id, q](double t, double x1, double x2) { return ldg_coeff_eval(id, q.data(), t, x1, x2); };
}

struct RefCase {
  ldg::Mesh* mesh = nullptr;  // borrowed: the caller keeps the mesh alive (system.hpp:207)
  ldg::ProblemSpec spec;
  std::unique_ptr<ldg::RefTensors> rt;
  std::unique_ptr<ldg::LdgSystem> sys;
  std::set<int> dir_ids, neu_ids;
  std::map<std::string, ldg::SparseOperator> ops;
  std::map<std::string, Eigen::VectorXd> vecs;
  std::map<std::string, ldg::DofMatrix> dofs;
};

void store_vec(RefCase* c, const std::string& name, const Eigen::VectorXd& v) { c->vecs[name] = v; }

}  // namespace

extern "C" {

const char* ldgref_last_error() { return g_err.c_str(); }

void ldgref_set_sparse_solver(Eigen::SparseSolverHook hook) { Eigen::sparse_solver_hook() = hook; }

// ------------------------------------------------------------------ mesh
void* ldgref_mesh_square(double h_max) {
  ldg::Mesh* m = nullptr;
  if (guarded([&] { m = new ldg::Mesh(ldg::domain_square(h_max)); })) return nullptr;
  return m;
}

// coords: nv x 2; v0t: nt x 3; id_e0t (nullable): nt x 3 boundary IDs applied
// to boundary edges (id_e[e0t[k][n]] = id_e0t[k][n]).
void* ldgref_mesh_create(int nv, const double* coords, int nt, const int* v0t, const int* id_e0t) {
  ldg::Mesh* m = nullptr;
  if (guarded([&] {
        std::vector<ldg::Point2> c(static_cast<size_t>(nv));
        for (int i = 0; i < nv; ++i) c[i] = {coords[2 * i], coords[2 * i + 1]};
        std::vector<std::array<int, 3>> t(static_cast<size_t>(nt));
        for (int k = 0; k < nt; ++k) t[k] = {v0t[3 * k], v0t[3 * k + 1], v0t[3 * k + 2]};
        auto* mm = new ldg::Mesh(ldg::generate_grid_data(std::move(c), std::move(t)));
        if (id_e0t) {
          for (int k = 0; k < nt; ++k)
            for (int n = 0; n < 3; ++n) {
              const int e = mm->e0t[k][n];
              if (mm->is_boundary_edge(e)) mm->id_e[e] = id_e0t[3 * k + n];
            }
          mm->sync_edge_ids();
        }
        m = mm;
      }))
    return nullptr;
  return m;
}

void* ldgref_mesh_refine(void* mesh) {
  ldg::Mesh* m = nullptr;
  if (guarded([&] { m = new ldg::Mesh(ldg::refine_uniform(*static_cast<ldg::Mesh*>(mesh))); }))
    return nullptr;
  return m;
}

void ldgref_mesh_free(void* mesh) { delete static_cast<ldg::Mesh*>(mesh); }

void ldgref_mesh_sizes(void* mesh, int* num_t, int* num_e, int* num_v) {
  const auto* m = static_cast<ldg::Mesh*>(mesh);
  *num_t = m->num_t;
  *num_e = m->num_e;
  *num_v = m->num_v;
}

// Per-element lists (all K-major): coords nv*2, v0t K*3, b K*4 (b11,b12,b21,b22),
// area K, len K*3, nu K*3*2, nbr K*3, nbr_n K*3 (-1 on boundary), id_e0t K*3.
void ldgref_mesh_lists(void* mesh, double* coords, int* v0t, double* b, double* area, double* len,
                       double* nu, int* nbr, int* nbr_n, int* id_e0t) {
  const auto* m = static_cast<ldg::Mesh*>(mesh);
  for (int i = 0; i < m->num_v; ++i) {
    coords[2 * i] = m->coord_v[i][0];
    coords[2 * i + 1] = m->coord_v[i][1];
  }
  for (int k = 0; k < m->num_t; ++k) {
    b[4 * k + 0] = m->b[k][0][0];
    b[4 * k + 1] = m->b[k][0][1];
    b[4 * k + 2] = m->b[k][1][0];
    b[4 * k + 3] = m->b[k][1][1];
    area[k] = m->area_t[k];
    for (int n = 0; n < 3; ++n) {
      v0t[3 * k + n] = m->v0t[k][n];
      len[3 * k + n] = m->area_e0t[k][n];
      nu[6 * k + 2 * n] = m->nu_e0t[k][n][0];
      nu[6 * k + 2 * n + 1] = m->nu_e0t[k][n][1];
      auto [kp, np] = m->neighbor(k, n);
      nbr[3 * k + n] = kp;
      nbr_n[3 * k + n] = np;
      id_e0t[3 * k + n] = m->id_e0t[k][n];
    }
  }
}

// ------------------------------------------------------------------ tensors
// Sizes: m n*n, h n*n*2, g n^3*2, sd n*n*3, so n*n*9, rd n^3*3, ro n^3*9.
int ldgref_ref_tensors(int n, double* m, double* h, double* g, double* sd, double* so, double* rd,
                       double* ro) {
  return guarded([&] {
    ldg::RefTensors t = ldg::build_ref_tensors(n);
    std::copy(t.m_hat_.begin(), t.m_hat_.end(), m);
    std::copy(t.h_hat_.begin(), t.h_hat_.end(), h);
    std::copy(t.g_hat_.begin(), t.g_hat_.end(), g);
    std::copy(t.s_diag_.begin(), t.s_diag_.end(), sd);
    std::copy(t.s_offdiag_.begin(), t.s_offdiag_.end(), so);
    std::copy(t.r_diag_.begin(), t.r_diag_.end(), rd);
    std::copy(t.r_offdiag_.begin(), t.r_offdiag_.end(), ro);
  });
}

// Quadrature rule tables: returns point count, fills up to cap entries.
int ldgref_quad_rule_2d(int q_ord, double* x1, double* x2, double* w, int cap) {
  ldg::QuadRule2D r = ldg::quad_rule_2d(q_ord);
  const int n = static_cast<int>(r.points.size());
  for (int i = 0; i < n && i < cap; ++i) {
    x1[i] = r.points[i][0];
    x2[i] = r.points[i][1];
    w[i] = r.weights[i];
  }
  return n;
}

int ldgref_quad_rule_1d(int q_ord, double* s, double* w, int cap) {
  int n = -1;
  if (guarded([&] {
        ldg::QuadRule1D r = ldg::quad_rule_1d(q_ord);
        n = static_cast<int>(r.points.size());
        for (int i = 0; i < n && i < cap; ++i) {
          s[i] = r.points[i];
          w[i] = r.weights[i];
        }
      }))
    return -1;
  return n;
}

// ------------------------------------------------------------------ projection
// out: K x N, k-major (vec_dof order, fields.hpp:26-31).
int ldgref_project(void* mesh, int n_local, int fn_id, const double* fn_p, double t, int q_ord,
                   double* out) {
  return guarded([&] {
    const auto* m = static_cast<ldg::Mesh*>(mesh);
    ldg::RefTensors rt = ldg::build_ref_tensors(n_local);
    ldg::DofMatrix d = ldg::project(*m, make_func(fn_id, fn_p), t, q_ord, rt);
    Eigen::VectorXd v = ldg::vec_dof(d);
    std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(v.size()));
  });
}

double ldgref_l2_error(void* mesh, int n_local, const double* dof_kmajor, int fn_id, const double* fn_p,
                       double t, int q_ord) {
  double r = -1.0;
  guarded([&] {
    const auto* m = static_cast<ldg::Mesh*>(mesh);
    Eigen::VectorXd v(static_cast<Eigen::Index>(m->num_t) * n_local);
    std::memcpy(v.data(), dof_kmajor, sizeof(double) * static_cast<size_t>(v.size()));
    r = ldg::l2_error(*m, ldg::unvec_dof(v, m->num_t, n_local), make_func(fn_id, fn_p), t, q_ord);
  });
  return r;
}

// ------------------------------------------------------------------ system case
// fn_ids[5] / fn_p[5*4]: d, f, c_d, g_n, c0.  bc_kinds: 0 Dirichlet, 1 Neumann.
void* ldgref_case_create(void* mesh, int n_local, double eta, const int* fn_ids, const double* fn_p,
                         const int* bc_ids, const int* bc_kinds, int nbc) {
  RefCase* c = nullptr;
  if (guarded([&] {
        auto cc = std::make_unique<RefCase>();
        cc->mesh = static_cast<ldg::Mesh*>(mesh);
        cc->spec.d = make_func(fn_ids[0], fn_p + 0);
        cc->spec.f = make_func(fn_ids[1], fn_p + 4);
        cc->spec.c_d = make_func(fn_ids[2], fn_p + 8);
        cc->spec.g_n = make_func(fn_ids[3], fn_p + 12);
        cc->spec.c0 = make_func(fn_ids[4], fn_p + 16);
        cc->spec.eta = eta;
        for (int i = 0; i < nbc; ++i) {
          cc->spec.boundary[bc_ids[i]] = bc_kinds[i] == 0 ? ldg::Bc::kDirichlet : ldg::Bc::kNeumann;
          (bc_kinds[i] == 0 ? cc->dir_ids : cc->neu_ids).insert(bc_ids[i]);
        }
        cc->rt = std::make_unique<ldg::RefTensors>(ldg::build_ref_tensors(n_local));
        cc->sys = std::make_unique<ldg::LdgSystem>(*cc->mesh, cc->spec, *cc->rt);
        c = cc.release();
      }))
    return nullptr;
  return c;
}

void ldgref_case_free(void* c) { delete static_cast<RefCase*>(c); }

// Assembles every operator and vector of build_blocks(t) through the
// reference free functions (system.hpp:110-152) and keeps them by name:
// ops  mass h1 h2 g1 g2 r1 rd1 r2 rd2 q1 qn1 q2 qn2 s sd A
// vecs jd1 jd2 kd kn l V     dofs D F
int ldgref_case_assemble(void* cv, double t) {
  auto* c = static_cast<RefCase*>(cv);
  return guarded([&] {
    const ldg::Mesh& m = *c->mesh;
    const ldg::RefTensors& rt = *c->rt;
    const int p = ldg::degree_from_dof_count(rt.n);
    const int q = std::max(2 * p, 1);
    auto si = ldg::select_interior(m);
    auto sd = ldg::select_boundary(m, c->dir_ids);
    auto sn = ldg::select_boundary(m, c->neu_ids);
    ldg::BasisQuadCache cache(rt.n);
    ldg::DofMatrix d = ldg::project(m, c->spec.d, t, q, rt);
    ldg::DofMatrix f = ldg::project(m, c->spec.f, t, q, rt);
    c->dofs["D"] = d;
    c->dofs["F"] = f;
    c->ops["mass"] = ldg::assemble_mass(m, rt);
    std::tie(c->ops["h1"], c->ops["h2"]) = ldg::assemble_dphi_phi(m, rt);
    std::tie(c->ops["g1"], c->ops["g2"]) = ldg::assemble_dphi_phi_coeff(m, rt, d);
    std::tie(c->ops["r1"], c->ops["rd1"]) = ldg::assemble_edge_avg_coeff_nu(m, 1, d, si, sd, rt);
    std::tie(c->ops["r2"], c->ops["rd2"]) = ldg::assemble_edge_avg_coeff_nu(m, 2, d, si, sd, rt);
    std::tie(c->ops["q1"], c->ops["qn1"]) = ldg::assemble_edge_avg_nu(m, 1, si, sn, rt);
    std::tie(c->ops["q2"], c->ops["qn2"]) = ldg::assemble_edge_avg_nu(m, 2, si, sn, rt);
    std::tie(c->ops["s"], c->ops["sd"]) = ldg::assemble_edge_jump(m, si, sd, rt);
    auto [j1, j2] = ldg::assemble_vec_dirichlet_nu(m, sd, c->spec.c_d, t, cache);
    store_vec(c, "jd1", j1);
    store_vec(c, "jd2", j2);
    store_vec(c, "kd", ldg::assemble_vec_dirichlet(m, sd, c->spec.c_d, t, cache));
    store_vec(c, "kn", ldg::assemble_vec_neumann(m, sn, d, c->spec.g_n, t, cache));
    store_vec(c, "l", ldg::assemble_vec_source(c->ops["mass"], f));
    ldg::SystemBlocks blocks = c->sys->build_blocks(t);
    c->ops["A"] = blocks.a;
    store_vec(c, "V", blocks.v);
  });
}

// The per-step coefficient operators for a caller's D (K x N, k-major):
// assemble_dphi_phi_coeff and assemble_edge_avg_coeff_nu (m = 1, 2) stored as
// "ug1", "ug2", "ur1", "urd1", "ur2", "urd2".
int ldgref_case_assemble_with_d(void* cv, const double* d_kmajor) {
  auto* c = static_cast<RefCase*>(cv);
  return guarded([&] {
    const ldg::Mesh& m = *c->mesh;
    const ldg::RefTensors& rt = *c->rt;
    Eigen::VectorXd y(static_cast<Eigen::Index>(m.num_t) * rt.n);
    std::memcpy(y.data(), d_kmajor, sizeof(double) * static_cast<size_t>(y.size()));
    const ldg::DofMatrix d = ldg::unvec_dof(y, m.num_t, rt.n);
    auto si = ldg::select_interior(m);
    auto sd = ldg::select_boundary(m, c->dir_ids);
    std::tie(c->ops["ug1"], c->ops["ug2"]) = ldg::assemble_dphi_phi_coeff(m, rt, d);
    std::tie(c->ops["ur1"], c->ops["urd1"]) = ldg::assemble_edge_avg_coeff_nu(m, 1, d, si, sd, rt);
    std::tie(c->ops["ur2"], c->ops["urd2"]) = ldg::assemble_edge_avg_coeff_nu(m, 2, d, si, sd, rt);
  });
}

// Operator export, CSC order.  Returns nnz (or -1); fills when arrays non-null.
long ldgref_case_op(void* cv, const char* name, int* rows, int* cols, double* vals) {
  auto* c = static_cast<RefCase*>(cv);
  auto it = c->ops.find(name);
  if (it == c->ops.end()) {
    g_err = std::string("unknown operator ") + name;
    return -1;
  }
  const ldg::SparseOperator& op = it->second;
  if (rows) {
    long p = 0;
    for (int j = 0; j < op.outerSize(); ++j)
      for (ldg::SparseOperator::InnerIterator e(op, j); e; ++e, ++p) {
        rows[p] = static_cast<int>(e.row());
        cols[p] = j;
        vals[p] = e.value();
      }
  }
  return static_cast<long>(op.nonZeros());
}

long ldgref_case_vec(void* cv, const char* name, double* out) {
  auto* c = static_cast<RefCase*>(cv);
  auto it = c->vecs.find(name);
  if (it != c->vecs.end()) {
    if (out) std::memcpy(out, it->second.data(), sizeof(double) * static_cast<size_t>(it->second.size()));
    return static_cast<long>(it->second.size());
  }
  auto jt = c->dofs.find(name);
  if (jt != c->dofs.end()) {
    Eigen::VectorXd v = ldg::vec_dof(jt->second);
    if (out) std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(v.size()));
    return static_cast<long>(v.size());
  }
  g_err = std::string("unknown vector ") + name;
  return -1;
}

int ldgref_case_initial_state(void* cv, double* y) {
  auto* c = static_cast<RefCase*>(cv);
  return guarded([&] {
    ldg::SystemState s = c->sys->initial_state();
    std::memcpy(y, s.y.data(), sizeof(double) * static_cast<size_t>(s.y.size()));
  });
}

// `steps` implicit Euler steps (system.hpp:155-174) from (y, t); writes the
// final state into y/t and the summed wall time of the euler_step calls,
// timed as ldg_main.cpp:199-214 does.
int ldgref_case_euler(void* cv, double* y, double* t, double dt, int steps, double* seconds) {
  auto* c = static_cast<RefCase*>(cv);
  return guarded([&] {
    const long n = 3L * c->mesh->num_t * c->rt->n;
    ldg::SystemState s;
    s.y = Eigen::VectorXd(n);
    std::memcpy(s.y.data(), y, sizeof(double) * static_cast<size_t>(n));
    s.t = *t;
    double total = 0.0;
    for (int i = 0; i < steps; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      s = c->sys->euler_step(s, dt);
      total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (!s.y.allFinite()) throw std::runtime_error("non-finite values after step");
    }
    std::memcpy(y, s.y.data(), sizeof(double) * static_cast<size_t>(n));
    *t = s.t;
    if (seconds) *seconds = total;
  });
}

// Times only build_blocks(t) (projection + per-step assembly + triplet merge).
int ldgref_case_time_build(void* cv, double t, int reps, double* seconds) {
  auto* c = static_cast<RefCase*>(cv);
  return guarded([&] {
    double total = 0.0;
    for (int i = 0; i < reps; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      ldg::SystemBlocks b = c->sys->build_blocks(t);
      total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (b.v.size() == 0) throw std::runtime_error("empty system");
    }
    *seconds = total;
  });
}

int ldgref_case_solve_stationary(void* cv, double t, double* cc, double* z1, double* z2) {
  auto* c = static_cast<RefCase*>(cv);
  return guarded([&] {
    auto [dc, d1, d2] = c->sys->solve_stationary(t);
    Eigen::VectorXd a = ldg::vec_dof(dc), b1 = ldg::vec_dof(d1), b2 = ldg::vec_dof(d2);
    std::memcpy(cc, a.data(), sizeof(double) * static_cast<size_t>(a.size()));
    std::memcpy(z1, b1.data(), sizeof(double) * static_cast<size_t>(b1.size()));
    std::memcpy(z2, b2.data(), sizeof(double) * static_cast<size_t>(b2.size()));
  });
}

// run_convergence (convergence.hpp:77-103): rows = n_orders*(j_max+1), each
// (p, j, h, K, error, alpha).
int ldgref_run_convergence(const int* orders, int n_orders, int j_max, double* rows) {
  return guarded([&] {
    std::vector<int> o(orders, orders + n_orders);
    auto r = ldg::run_convergence(o, j_max);
    for (size_t i = 0; i < r.size(); ++i) {
      rows[6 * i + 0] = r[i].p;
      rows[6 * i + 1] = r[i].j;
      rows[6 * i + 2] = r[i].h;
      rows[6 * i + 3] = r[i].num_t;
      rows[6 * i + 4] = r[i].error;
      rows[6 * i + 5] = r[i].alpha;
    }
  });
}

}  // extern "C"
