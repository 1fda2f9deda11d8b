"""Solver-tolerance study: state error of production stopping rules against a
tight solve (rtol 1e-14; pinned to the oracle's exact solve at 64^2 by
tests/test_gpu_parity_scale.py) on the C2 mesh, plus iterations per step.

python scripts/tol_study.py [dim] [steps]"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1408_3877_b200 as ld  # noqa: E402

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dt = 1.0 / 20
variants = {"default": ld.SolverOptions(), "contract_only": ld.SolverOptions(rtol=0.0),
            "rtol1e-13": ld.SolverOptions(rtol=1e-13), "rtol3e-14": ld.SolverOptions(rtol=3e-14),
            "rtol1e-14": ld.SolverOptions(rtol=1e-14, maxit=5000)}
out = {}
for p in range(5):
    s = ld.LdgSystem.square(dim, p, ld.BASELINE_SPEC)
    s.initial_state()
    y0, _ = s.get_state()
    ys = []
    s.set_state(y0, 0.0)
    for _ in range(steps):
        s.euler_steps(dt, 1, ld.SolverOptions(rtol=2e-15, maxit=400))
        ys.append(s.get_state()[0])
    row = {}
    for name, o in variants.items():
        s.set_state(y0, 0.0)
        errs, its = [], 0
        t0 = time.time()
        for i in range(steps):
            st = s.euler_steps(dt, 1, o)
            its += st["iterations"]
            rr = st["schur_relres"]
            y, _ = s.get_state()
            errs.append(float(np.linalg.norm(y - ys[i]) / np.linalg.norm(ys[i])))
        row[name] = {"max_rel_l2": max(errs), "iters_per_step": its / steps, "schur_relres": rr}
    out[p] = row
    print(p, json.dumps(row), flush=True)
    s.close()
