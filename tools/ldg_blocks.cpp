// build_blocks(t) (system.hpp:110-152) through the C++ host mirror: writes
// the returned SystemBlocks -- A in the reference's CSC storage
// (SparseOperator, assembly.hpp:21) and V -- and, given a coefficient file,
// the per-operator results assemble_dphi_phi_coeff / assemble_edge_avg_coeff_nu
// (assembly.hpp:113-136, 214-252) for that D, as raw little-endian arrays.
//
//   ldg_blocks dim p t out_prefix [d_file (K*N doubles, k-major) [rt_file]]
//
// rt_file: the caller's reference tensors m | h | g | sd | so (raw doubles,
// reftensors.hpp layout), passed to set_reference_tensors as the reference's
// LdgSystem(mesh, spec, rt) receives its rt.
//
// Files: <prefix>.A.{outer,inner}.i32 / .A.values.f64, <prefix>.V.f64 and,
// with d_file, <prefix>.{G1,G2,R1,RD1,R2,RD2}.{outer,inner}.i32 / .values.f64.
// The BASELINE problem on domain_square(1/dim).  Exit code 1 on any error.
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>
#include <vector>

#include "ldg_host.hpp"

namespace {

template <typename T>
void dump(const std::string& path, const std::vector<T>& v) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot write " + path);
  const size_t w = std::fwrite(v.data(), sizeof(T), v.size(), f);
  std::fclose(f);
  if (w != v.size()) throw std::runtime_error("short write " + path);
}

void dump_op(const std::string& prefix, const std::string& name, const ldg::b200::SparseOperator& op) {
  dump(prefix + "." + name + ".outer.i32", op.outer);
  dump(prefix + "." + name + ".inner.i32", op.inner);
  dump(prefix + "." + name + ".values.f64", op.values);
}

}  // namespace

int main(int argc, char** argv) {
  namespace lb = ldg::b200;
  if (argc < 5) {
    std::cerr << "usage: ldg_blocks dim p t out_prefix [d_file]\n";
    return 1;
  }
  try {
    const int dim = std::atoi(argv[1]), p = std::atoi(argv[2]);
    const double t = std::atof(argv[3]);
    const std::string prefix = argv[4];
    lb::ProblemSpec spec;
    spec.d = lb::coeff(LDG_FN_BASE_D);
    spec.f = lb::coeff(LDG_FN_BASE_F);
    spec.c_d = lb::coeff(LDG_FN_BASE_C);
    spec.c0 = lb::coeff(LDG_FN_BASE_C);
    spec.g_n = lb::coeff(LDG_FN_BASE_GN);
    spec.boundary = {{1, lb::Bc::kDirichlet}, {2, lb::Bc::kDirichlet}, {3, lb::Bc::kNeumann}, {4, lb::Bc::kNeumann}};
    lb::LdgSystem sys = lb::LdgSystem::square(dim, p, spec);
    if (argc > 6) {  // the caller's RefTensors: m | h | g | sd | so, raw doubles
      lb::RefTensors rt;
      const size_t n = static_cast<size_t>(sys.n_local());
      rt.n = static_cast<int>(n);
      rt.m.resize(n * n);
      rt.h.resize(2 * n * n);
      rt.g.resize(2 * n * n * n);
      rt.sd.resize(3 * n * n);
      rt.so.resize(9 * n * n);
      FILE* f = std::fopen(argv[6], "rb");
      bool ok = f != nullptr;
      for (auto* v : {&rt.m, &rt.h, &rt.g, &rt.sd, &rt.so})
        ok = ok && std::fread(v->data(), sizeof(double), v->size(), f) == v->size();
      if (f) std::fclose(f);
      if (!ok) throw std::invalid_argument("cannot read the reference tensor file");
      sys.set_reference_tensors(rt);
    }
    const lb::SystemBlocks b = sys.build_blocks(t);
    dump_op(prefix, "A", b.a);
    dump(prefix + ".V.f64", b.v);
    if (argc > 5) {
      std::vector<double> d(static_cast<size_t>(sys.block_dim()));
      FILE* f = std::fopen(argv[5], "rb");
      if (!f || std::fread(d.data(), sizeof(double), d.size(), f) != d.size())
        throw std::invalid_argument("cannot read the coefficient file");
      std::fclose(f);
      const auto g = sys.assemble_dphi_phi_coeff(d);
      dump_op(prefix, "G1", g.first);
      dump_op(prefix, "G2", g.second);
      for (int m = 1; m <= 2; ++m) {
        const auto r = sys.assemble_edge_avg_coeff_nu(m, d);
        dump_op(prefix, "R" + std::to_string(m), r.first);
        dump_op(prefix, "RD" + std::to_string(m), r.second);
      }
    }
    std::printf("ldg_blocks: K = %d, N = %d, nnz(A) = %ld\n", sys.num_t(), sys.n_local(), b.a.nonZeros());
  } catch (const std::exception& err) {
    std::cerr << "error: " << err.what() << "\n";
    return 1;
  }
  return 0;
}
