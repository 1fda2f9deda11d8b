"""One implicit-Euler step of the LDG path for ncu (run under
`ncu --profile-from-start off ...`): warm-up steps outside the profiled
range (multigrid build, graph capture), then exactly one profiled step."""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=256)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--dt", type=float, default=0.05)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--assemble-only", action="store_true")
    ap.add_argument("--blocks", action="store_true", help="BASELINE config 3 call (all 8 blocks + projection + rhs)")
    ap.add_argument("--precond", type=int, default=2)
    args = ap.parse_args()
    import torch

    import paper_1408_3877_b200 as ld

    s = ld.LdgSystem.square(args.dim, args.p, ld.BASELINE_SPEC)
    s.initial_state()
    opts = ld.SolverOptions(precond=args.precond)
    if args.blocks:
        for i in range(args.warmup):
            print("warm-up assemble_blocks ms", s.assemble_blocks(0.05 * (i + 1)))
    elif args.assemble_only:
        for i in range(args.warmup):
            s.assemble(0.05 * (i + 1))
    else:
        s.euler_steps(args.dt, args.warmup, opts)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    if args.blocks:
        st = {"ms": s.assemble_blocks(1.0)}
    elif args.assemble_only:
        s.assemble(1.0)
        st = {}
    else:
        st = s.euler_steps(args.dt, 1, opts)
    s.sync()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled step:", st)


if __name__ == "__main__":
    main()
