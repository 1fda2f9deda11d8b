"""Device-resident steps vs host-buffer steps (ldg_euler_steps_host) per p at 256^2:
device-event ms, wall ms and iterations of each, to explain the e2e gap."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1408_3877_b200 as ld

dim = int(os.environ.get("DIM", 256))
for p in [int(x) for x in os.environ.get("PS", "0,1,2,3,4").split(",")]:
    s = ld.LdgSystem.square(dim, p, ld.BASELINE_SPEC)
    s.initial_state()
    o = ld.SolverOptions()
    for _ in range(3):
        s.euler_steps(0.05, 1, o)
    dev, wall, its = [], [], []
    for _ in range(5):
        w0 = time.perf_counter()
        st = s.euler_steps(0.05, 1, o)
        wall.append((time.perf_counter() - w0) * 1e3)
        dev.append(st["ms_assemble"] + st["ms_solve"])
        its.append(st["iterations"])
    y, t = s.get_state()
    pin_in = torch.from_numpy(y).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    edev, ewall, eits = [], [], []
    for _ in range(5):
        w0 = time.perf_counter()
        st = s.euler_steps_host(pin_in.data_ptr(), t, 0.05, 1, pin_out.data_ptr(), o)
        ewall.append((time.perf_counter() - w0) * 1e3)
        edev.append(st["ms_total"])
        eits.append(st["iterations"])
        t += 0.05
        pin_in.copy_(pin_out)
    print(f"p={p} device ms {np.median(dev):.2f} wall {np.median(wall):.2f} it {np.mean(its):.1f} | "
          f"host-buffer ms {np.median(edev):.2f} wall {np.median(ewall):.2f} it {np.mean(eits):.1f}", flush=True)
    s.close()
