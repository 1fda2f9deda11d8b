"""FGMRES vs BiCGStab on the BASELINE problem and a jittered mixed-BC mesh."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 256
mixed = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0,
                       boundary={1: "D", 2: "N", 3: "N", 4: "D"})
cases = [("base", ld.BASELINE_SPEC, 0.0, 0.05, p) for p in range(5)] + [("mixed", mixed, 0.2, 0.1, 3)]
for name, spec, jit, dt, p in cases:
    line = f"{name} p={p}:"
    for kr, rs in ((1, 0), (0, 20), (0, 40), (0, 60)):
        s = ld.LdgSystem.square(dim, p, spec, jitter=jit, seed=0)
        s.initial_state()
        o = ld.SolverOptions(krylov=kr, restart=rs)
        s.euler_steps(dt, 1, o)
        st = s.euler_steps(dt, 2, o)
        ms = (st["ms_assemble"] + st["ms_solve"]) / 2
        line += f"  [{'bicg' if kr else 'gmres%d' % rs}] {ms:7.1f} ms it {st['iterations'] / 2:5.1f} ap {st['applies'] / 2:5.1f} res {st['residual']:.1e}"
        s.close()
    print(line, flush=True)
