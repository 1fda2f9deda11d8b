import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld
dim, p = int(sys.argv[1]), int(sys.argv[2])
seq = sys.argv[3].split(",")
mixed = {1: "D", 2: "N", 3: "N", 4: "D"}
alld = {1: "D", 2: "D", 3: "D", 4: "D"}
for name in seq:
    bc = mixed if name == "m" else alld
    spec = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0, boundary=bc)
    s = ld.LdgSystem.square(dim, p, spec, jitter=0.0, seed=0)
    s.initial_state()
    try:
        st = s.euler_steps(0.1, int(os.environ.get("NSTEP", "2")), ld.SolverOptions())
        print(name, "ok it/step", st["iterations"] / 2, flush=True)
    except Exception as e:
        print(name, "FAIL", str(e)[:100], flush=True)
    s.close()
