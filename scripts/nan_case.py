import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld
dim, p = int(sys.argv[1]), int(sys.argv[2])
spec = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0,
                      boundary={1: "D", 2: "N", 3: "N", 4: "D"})
s = ld.LdgSystem.square(dim, p, spec, jitter=0.0, seed=0)
s.initial_state()
try:
    st = s.euler_steps(0.1, 2, ld.SolverOptions())
    print(os.environ.get("TAGX", ""), "ok it/step", st["iterations"] / 2, flush=True)
except Exception as e:
    print(os.environ.get("TAGX", ""), "FAIL", str(e)[:120], flush=True)
