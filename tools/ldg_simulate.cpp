// The time loop of the reference CLI's `simulate` (proj/tools/ldg_main.cpp:
// 174-222) on the B200 path, through the C++ host mirror: build the system,
// project c0, run num_steps implicit-Euler steps, print per-step timing, and
// (with a basename) write `<basename>.<step>.vtu` of c at step 0 and every
// output_every steps (ldg_main.cpp:195-207, write_vtu of to_lagrange(c)).
//
//   ldg_simulate [dim=32] [p=2] [num_steps=20] [t_end=1] [--device-resident|--host]
//                [basename] [output_every=1]
//
// The problem is the BASELINE.json one (c = cos7x1 cos7x2 + e^-t,
// d = e^(x1+x2)(1 + 0.5 sin t), f derived, Dirichlet on all sides).
// Exit code 1 on any error, as the reference CLI (ldg_main.cpp:302-305).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>

#include "ldg_host.hpp"

int main(int argc, char** argv) {
  namespace lb = ldg::b200;
  int dim = argc > 1 ? std::atoi(argv[1]) : 32;
  int p = argc > 2 ? std::atoi(argv[2]) : 2;
  int num_steps = argc > 3 ? std::atoi(argv[3]) : 20;
  double t_end = argc > 4 ? std::atof(argv[4]) : 1.0;
  bool resident = argc > 5 && std::strcmp(argv[5], "--device-resident") == 0;
  const std::string basename = argc > 6 ? argv[6] : "";
  const int output_every = argc > 7 ? std::atoi(argv[7]) : 1;
  try {
    lb::ProblemSpec spec;
    spec.d = lb::coeff(LDG_FN_BASE_D);
    spec.f = lb::coeff(LDG_FN_BASE_F);
    spec.c_d = lb::coeff(LDG_FN_BASE_C);
    spec.c0 = lb::coeff(LDG_FN_BASE_C);
    spec.g_n = lb::coeff(LDG_FN_BASE_GN);
    spec.boundary = {{1, lb::Bc::kDirichlet}, {2, lb::Bc::kDirichlet}, {3, lb::Bc::kDirichlet},
                     {4, lb::Bc::kDirichlet}};
    if (num_steps < 1) throw std::runtime_error("num_steps must be at least 1");
    lb::LdgSystem sys = lb::LdgSystem::square(dim, p, spec);
    lb::SystemState state = sys.initial_state();
    if (!basename.empty()) sys.write_vtu(2, "c", basename, 0);
    const double dt = t_end / num_steps;
    const auto wall_start = std::chrono::steady_clock::now();
    for (int step = 1; step <= num_steps; ++step) {
      const auto t0 = std::chrono::steady_clock::now();
      if (resident) {
        sys.advance(dt, 1);
        state.t += dt;
      } else {
        state = sys.euler_step(state, dt);
        for (double v : state.y)
          if (!std::isfinite(v)) throw std::runtime_error("non-finite values after step " + std::to_string(step));
      }
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      std::printf("step %d/%d  t = %g  (%g ms)\n", step, num_steps, state.t, ms);
      if (!basename.empty() && output_every > 0 && step % output_every == 0)
        std::printf("  wrote %s\n", sys.write_vtu(2, "c", basename, step).c_str());
    }
    const double total =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - wall_start).count();
    std::printf("simulate: %d steps to t_end = %g in %g s (K = %d, N = %d)\n", num_steps, t_end, total,
                sys.num_t(), sys.n_local());
  } catch (const std::exception& err) {
    std::cerr << "error: " << err.what() << "\n";
    return 1;
  }
  return 0;
}
