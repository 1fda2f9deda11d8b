// TEST INFRASTRUCTURE ONLY — oracle/_ref/ref_vtu.
//
// The UNMODIFIED reference's write_vtu (vtkout.hpp:42-108) as a standalone
// program: the reference's iostreams cannot run inside a Python process that
// has another libstdc++ loaded (numpy), so reflib.write_vtu calls this binary.
//   ref_vtu <h_max> <m> <lagrange.bin (K x m doubles, k-major)> <var> <basename> <t_lvl>
// writes <basename>.<t_lvl>.vtu on domain_square(h_max) (mesh.hpp:225-254) and
// prints the path.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ldg/mesh.hpp"
#include "ldg/vtkout.hpp"

int main(int argc, char** argv) {
  if (argc != 7) {
    std::fprintf(stderr, "usage: ref_vtu h_max m lagrange.bin var basename t_lvl\n");
    return 2;
  }
  const ldg::Mesh mesh = ldg::domain_square(std::atof(argv[1]));
  const int m = std::atoi(argv[2]);
  std::vector<double> lag(static_cast<size_t>(mesh.num_t) * m);
  FILE* f = std::fopen(argv[3], "rb");
  if (!f || std::fread(lag.data(), sizeof(double), lag.size(), f) != lag.size()) {
    std::fprintf(stderr, "cannot read %s\n", argv[3]);
    return 1;
  }
  std::fclose(f);
  ldg::VtuSnapshot snap;
  snap.mesh = &mesh;
  snap.lagrange = Eigen::MatrixXd(mesh.num_t, m);
  for (int k = 0; k < mesh.num_t; ++k)
    for (int i = 0; i < m; ++i) snap.lagrange(k, i) = lag[static_cast<size_t>(k) * m + i];
  snap.var_name = argv[4];
  snap.basename = argv[5];
  snap.t_lvl = std::atoi(argv[6]);
  std::printf("%s\n", ldg::write_vtu(snap).c_str());
  return 0;
}
