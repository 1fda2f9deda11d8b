"""Convergence study (convergence.hpp:77-103) solved on the device: FK(3*2^j),
manufactured stationary problem, L2 error of C with order 2p+2 on the device
(ldg_l2_error), estimated orders alpha."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1408_3877_b200 as ld

jmax = int(os.environ.get("JMAX", 6))
spec = ld.ProblemSpec(d="exp_sum", f="mms_f", c_d="mms_exact", g_n="mms_gn", c0="mms_exact", eta=1.0,
                      boundary={1: "N", 2: "D", 3: "N", 4: "D"})
print("p,j,h,K,error,alpha,iterations,ms")
for p in range(5):
    prev = None
    for j in range(jmax + 1):
        dim = 3 * 2 ** j
        s = ld.LdgSystem.square(dim, p, spec)
        t0 = time.perf_counter()
        s.solve_stationary(0.0, ld.SolverOptions(rtol=1e-13, maxit=100000))
        ms = (time.perf_counter() - t0) * 1e3
        e = s.l2_error("mms_exact", 0.0, 2 * p + 2)
        a = math.log(prev / e) / math.log(2.0) if prev else float("nan")
        print(f"{p},{j},{1.0 / dim:.6g},{s.num_t},{e:.6e},{a:.4f},{s.last_stats['iterations']},{ms:.1f}", flush=True)
        prev = e
        s.close()
