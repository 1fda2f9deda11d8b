"""FGMRES iterations per step for a few mesh/BC variants (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mixed = {1: "D", 2: "N", 3: "N", 4: "D"}
alld = {1: "D", 2: "D", 3: "D", 4: "D"}
for name, bc, jit, dt in (("dirichlet nojit dt.05", alld, 0.0, 0.05), ("dirichlet nojit dt.1", alld, 0.0, 0.1),
                          ("mixed nojit dt.1", mixed, 0.0, 0.1), ("dirichlet jit.2 dt.1", alld, 0.2, 0.1),
                          ("mixed jit.2 dt.1", mixed, 0.2, 0.1), ("mixed jit.1 dt.1", mixed, 0.1, 0.1)):
    spec = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0, boundary=bc)
    s = ld.LdgSystem.square(dim, p, spec, jitter=jit, seed=0)
    s.initial_state()
    st = s.euler_steps(dt, 2, ld.SolverOptions())
    print(f"{name:24s} it/step {st['iterations'] / 2:6.1f}  ms/step {(st['ms_assemble'] + st['ms_solve']) / 2:7.1f}",
          flush=True)
    s.close()
