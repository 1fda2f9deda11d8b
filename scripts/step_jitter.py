"""Per-step device times (CUDA events inside the library) to expose jitter."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld

for p in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,4").split(",")]:
    s = ld.LdgSystem.square(256, p, ld.BASELINE_SPEC)
    s.initial_state()
    s.euler_steps(0.05, 2, ld.SolverOptions())
    out = []
    for i in range(12):
        t0 = time.perf_counter()
        st = s.euler_steps(0.05, 1, ld.SolverOptions())
        wall = (time.perf_counter() - t0) * 1e3
        out.append(f"{st['ms_assemble'] + st['ms_solve']:.1f}/{wall:.1f}/{st['iterations']}")
    print(f"p={p}:", " ".join(out), flush=True)
    s.close()
