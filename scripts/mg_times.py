"""Multigrid cost breakdown per level (graph-replayed, L2 warm) for dim 256."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for p in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2,3,4").split(",")]:
    s = ld.LdgSystem.square(dim, p, ld.BASELINE_SPEC)
    s.initial_state()
    s.euler_steps(0.05, 1, ld.SolverOptions())
    t = s.time_kernels(s.t, 0.05, reps=10, flush=False)
    print(f"p={p} schur {t['ms_schur']*1e3:.1f} us  spmv {t['ms_spmv']*1e3:.1f} us  vcycle {t['ms_vcycle']*1e3:.1f} us")
    print("   smooth sweep per level (us):", " ".join(f"{v*1e3:.1f}" for v in t["ms_level"]))
    s.close()
