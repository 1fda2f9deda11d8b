"""Device-resident step vs host-buffer step (ldg_euler_steps_host) from the SAME
state (same iterations) per p at 256^2: the pure host<->device overhead."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1408_3877_b200 as ld

dim = int(os.environ.get("DIM", 256))
for p in [int(x) for x in os.environ.get("PS", "0,1,2,3,4").split(",")]:
    s = ld.LdgSystem.square(dim, p, ld.BASELINE_SPEC)
    s.initial_state()
    o = ld.SolverOptions()
    s.euler_steps(0.05, 3, o)
    y0, t0 = s.get_state()
    pin_in = torch.from_numpy(y0).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    dev, hb, its = [], [], []
    for _ in range(6):
        s.set_state(y0, t0)
        st = s.euler_steps(0.05, 1, o)
        dev.append(st["ms_assemble"] + st["ms_solve"])
        st2 = s.euler_steps_host(pin_in.data_ptr(), t0, 0.05, 1, pin_out.data_ptr(), o)
        hb.append(st2["ms_total"])
        its.append((st["iterations"], st2["iterations"]))
    y1, _ = s.get_state()
    assert np.array_equal(pin_out.numpy(), y1)
    mb = y0.nbytes / 1e6
    print(f"p={p} device {np.median(dev):.2f} ms | host-buffer {np.median(hb):.2f} ms | overhead "
          f"{np.median(hb) - np.median(dev):.2f} ms for {mb:.1f} MB each way | its {its[-1]}", flush=True)
    s.close()
