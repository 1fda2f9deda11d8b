"""Virtual-rank strips vs single rank under solver variants (diagnostic)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld

MIXED = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0,
                       boundary={1: "D", 2: "N", 3: "N", 4: "D"})
for nranks, p in ((2, 1), (4, 2), (2, 3), (4, 1)):
    for kr in (0, 1):
        for pc in (1, 2, 3):
            o = ld.SolverOptions(rtol=1e-13, precond=pc, krylov=kr, maxit=3000, check_residual=False)
            one = ld.LdgSystem.square(32, p, MIXED, jitter=0.2, seed=0)
            grp = ld.LdgSystem.square_group(32, p, MIXED, nranks, jitter=0.2, seed=0)
            one.initial_state()
            grp.initial_state()
            st1 = one.euler_steps(0.1, 1, o)
            st2 = grp.euler_steps(0.1, 1, o)
            y1, _ = one.get_state()
            y2, _ = grp.get_state()
            err = np.linalg.norm(y2 - y1) / np.linalg.norm(y1)
            print(f"ranks {nranks} p {p} krylov {kr} pc {pc}: it {st1['iterations']} vs {st2['iterations']}  "
                  f"res {st1['residual']:.1e} vs {st2['residual']:.1e}  err {err:.1e}", flush=True)
            one.close()
            grp.close()
