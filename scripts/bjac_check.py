"""Block-Jacobi setup check: FGMRES iterations with the block-Jacobi preconditioner alone
(precond = 1: the FP64 inverses) and with the multigrid (FP16 inverses) on a jittered
mixed-BC mesh, per degree.  Run against two builds (LDG_B200_LIB) to compare a kernel
change: the inverses are the same matrices, so the counts must agree."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1408_3877_b200 as ld

mixed = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0,
                       boundary={1: "D", 2: "N", 3: "N", 4: "D"})
for p in range(5):
    row = []
    for pc in (1, 2):
        s = ld.LdgSystem.square(48, p, mixed, jitter=0.2, seed=1)
        s.initial_state()
        st = s.euler_steps(0.05, 2, ld.SolverOptions(rtol=1e-12, precond=pc))
        y = s.get_state()[0]
        row.append((st["iterations"], float(np.linalg.norm(y))))
        s.close()
    print(f"p={p} bjac its {row[0][0]} |y| {row[0][1]:.15e}   mg its {row[1][0]} |y| {row[1][1]:.15e}")
