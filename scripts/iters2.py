import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld
dim = int(sys.argv[1]); p = int(sys.argv[2])
spec = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0,
                      boundary={1: "D", 2: "N", 3: "N", 4: "D"})
s = ld.LdgSystem.square(dim, p, spec, jitter=0.2, seed=0)
s.initial_state()
st = s.euler_steps(0.1, 2, ld.SolverOptions())
print(os.environ.get("TAGX", ""), f"it/step {st['iterations'] / 2:6.1f}  ms/step {(st['ms_assemble'] + st['ms_solve']) / 2:7.1f}", flush=True)
