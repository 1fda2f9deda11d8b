"""Per-step phase breakdown (device events inside the library), median of 8 steps."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld

dim = int(os.environ.get("DIM", "256"))
OPTS = dict(restart=int(os.environ["RESTART"])) if "RESTART" in os.environ else {}
for p in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4").split(",")]:
    s = ld.LdgSystem.square(dim, p, ld.BASELINE_SPEC)
    s.initial_state()
    s.euler_steps(0.05, 2, ld.SolverOptions(**OPTS))
    rows = []
    for i in range(8):
        st = s.euler_steps(0.05, 1, ld.SolverOptions(**OPTS))
        fin = st["ms_solve"] - st["ms_setup"] - st["ms_krylov"]
        rows.append((st["ms_assemble"] + st["ms_solve"], st["ms_assemble"], st["ms_setup"], st["ms_krylov"], fin,
                     st["iterations"]))
    med = [statistics.median(r[c] for r in rows) for c in range(6)]
    kt = s.time_kernels(s.t, 0.05, reps=10, flush=False)
    print(f"p={p}: step {med[0]:.2f} ms = assemble {med[1]:.2f} + setup {med[2]:.2f} + krylov {med[3]:.2f} "
          f"({med[5]:.0f} it, {med[3] / med[5]:.3f} ms/it) + finish {med[4]:.2f};  vcycle {kt['ms_vcycle']:.3f} "
          f"schur {kt['ms_schur']:.3f} -> per-it other {med[3] / med[5] - kt['ms_vcycle'] - kt['ms_schur']:.3f} ms",
          flush=True)
    s.close()
