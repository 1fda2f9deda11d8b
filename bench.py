#!/usr/bin/env python
"""Benchmark of the LDG per-step hot path (BASELINE.json metric).

metric  DOF-updates/s (assembly + solve per implicit-Euler step)
        = sum over the step of 3*K*N / device time of the step
workload (default, BASELINE configs[1] = "C2"): Friedrichs-Keller 256x256
        (K = 131072), p swept 0..4, the analytic c, d(t), f(t) of
        BASELINE.json, dt = 1/20 (20 steps to T = 1).  One bench "step" is one
        implicit-Euler step of every p in the sweep (each p its own system).
value   device time (CUDA events on the library's stream) with the state
        resident in HBM; e2e = the same steps through the host-buffer C ABI
        call (ldg_euler_steps_host: H2D + steps + D2H inside the timed region).

`python bench.py --impl reference` times the reference's own CPU path
(oracle/_ref/libldgref.so = the unmodified reference headers + Eigen shim,
SciPy SuperLU as its SparseLU) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DOF-updates/s (assembly+solve per step)"
UNIT = "DOF-updates/s"

WORKLOADS = {
    # name: (dim, p list, dt, jitter, boundary, description)
    "c2": (256, [0, 1, 2, 3, 4], 1.0 / 20, 0.0, {1: "D", 2: "D", 3: "D", 4: "D"},
           "C2: FK 256x256 (K=131072), p=0..4 sweep, implicit Euler dt=1/20, all-Dirichlet BASELINE problem"),
    "c1": (16, [1], 1.0 / 100, 0.0, {1: "D", 2: "D", 3: "D", 4: "D"},
           "C1: FK 16x16 (K=512), p=1, dt=1/100, all-Dirichlet BASELINE problem"),
    "c3": (1024, [4], 0.0, 0.0, {1: "D", 2: "D", 3: "D", 4: "D"},
           "C3: assembly-only stress, FK 1024x1024 (K=2097152), p=4: projection of d, f, right-hand side and "
           "all 8 time-dependent C-row blocks per element each step"),
    "c4": (2048, [3], 1.0 / 10, 0.2, {1: "D", 2: "N", 3: "N", 4: "D"},
           "C4: FK 2048x2048 jittered +-0.2h (seed 0), p=3, dt=1/10, D on x1=0,x2=0, N elsewhere"),
    "c5": (4096, [2], 1.0 / 5, 0.0, {1: "D", 2: "D", 3: "D", 4: "D"},
           "C5: FK 4096x4096 (K=33.5M), p=2, dt=1/5"),
}


# weak scaling: the rank count at which the workload's own mesh is reached
# (C4 is quoted on 8 GPUs; C5's weak series is dim = 4096 sqrt(P/8))
WEAK_ANCHOR = {"c4": 8, "c5": 8}


def n_of(p):
    return (p + 1) * (p + 2) // 2


def e_int(dim):
    return 3 * dim * dim - 2 * dim


def packed_quads(p):
    """float4-sized quads of one packed N x N block (paper_1408_3877_b200/csrc/ldg_pack.cuh)."""
    n = n_of(p)
    if p <= 1:
        return (n * n + 3) // 4
    cc = 2 if n % 2 == 0 else 4
    ncol = (n + cc - 1) // cc * cc
    return ncol * n // 4


def bytes_schur(dim, p):
    """Compulsory bytes of one Schur-operator apply (k_stage1 + k_stage2):
    the stored diagonal blocks E^1_kk, E^2_kk (FP64; the off-diagonal E blocks are
    evaluated from D, the static M, B^m, S from shared-memory tables), the vectors
    x (read by both stages), t^1, t^2 (written, read), D (read), y (written) and the
    per-element geometry/topology (area, 3 lengths, 6 normal components, B (4);
    3 nbr, 3 nbrn, 3 kind)."""
    K, N = 2 * dim * dim, n_of(p)
    blocks = 2 * N * N * K
    vectors = (2 + 4 + 1 + 1) * K * N
    geometry = 2 * 14 * K
    return 8 * (blocks + vectors + geometry) + 4 * 2 * 9 * K


def bytes_sweep_s2(dim, p):
    """Compulsory bytes of the level-0 smoother stage 2 with the fused block-Jacobi
    update (k_s2f, FP16 packed E diagonal blocks and P^-1, each with a per-element
    scale): E 2 blocks x quads x 8 B, P quads x 8 B, 2 scales, vectors x, t (2),
    D, b, out (FP64), geometry (10 doubles) and topology (9 ints); from p = 3 on the
    edge-trace form (see below)."""
    K, N = 2 * dim * dim, n_of(p)
    q = packed_quads(p)
    if p >= 3:
        # edge-trace form (ldg_smooth.cu, kTraceMinP): no D and no edge geometry; instead the
        # traces x, -(c1 t1 + c2 t2), d_h at the Qe points of the 3 edges (FP32), the area
        qe = (3 * p + 2) // 2
        return K * (3 * q * 8 + 2 * 4 + 8 * 5 * N + 4 * 9 * qe + 8 * 1 + 4 * 9)
    return K * (2 * q * 8 + q * 8 + 2 * 4 + 8 * 6 * N + 8 * 10 + 4 * 9)


def bytes_asm(dim, p):
    """Assembly as run by the solver (kModeEdiag): writes the 2 diagonal blocks,
    reads D: 8*2*N^2*K + 8*K*N (+ geometry).  SURVEY.md §8d's B_asm assumes all
    8 blocks are written (8*2*N^2*(K + 2 E_int) + 8*K*N); see bytes_asm_survey."""
    K, N = 2 * dim * dim, n_of(p)
    return 8 * 2 * N * N * K + 8 * K * N + 8 * 16 * K


def bytes_asm_survey(dim, p):
    """8*2*N^2*(K + 2 E_int) + 8*K*N."""
    K, N = 2 * dim * dim, n_of(p)
    return 8 * 2 * N * N * (K + 2 * e_int(dim)) + 8 * K * N


def bytes_full_compulsory(dim, p):
    """Compulsory bytes of the full (W + dt A) Y apply as implemented: diagonal E
    blocks streamed, off-diagonal ones from D, static blocks from tables, Y (3
    vectors), D, out (3 vectors), geometry/topology."""
    K, N = 2 * dim * dim, n_of(p)
    return 8 * (2 * N * N * K + 7 * K * N + 14 * K) + 36 * K


def bytes_spmv(dim, p):
    """8 N^2 nb + 4 nb + 4 (3K+1) + 2*8*3KN, nb = 7K + 10 E_int."""
    K, N = 2 * dim * dim, n_of(p)
    nb = 7 * K + 10 * e_int(dim)
    return 8 * N * N * nb + 4 * nb + 4 * (3 * K + 1) + 2 * 8 * 3 * K * N


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_prefix, p, dim):
    """dram__bytes_read + dram__bytes_write of the first matching launch (the
    level-0 one: largest grid) in the committed ncu --set full summary
    (profiles/*_ncu_traffic.json, scripts/ncu_traffic.py), or None."""
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_traffic.json")), reverse=True):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        if d.get("p") != p or d.get("dim") != dim:
            continue
        ks = [k for k in d["kernels"] if k["kernel"].startswith(kernel_prefix) and k.get("dram_bytes")]
        if ks:
            k = max(ks, key=lambda k: k.get("launch__grid_size") or 0)
            return k["dram_bytes"], f"{os.path.basename(path)}: {k['kernel']} grid {k['grid']}"
    return None, None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region.

    The nvidia-smi process is started before the warm-up (its start-up, a
    driver/NVML initialisation, stalls the GPU's first launches by several ms)
    and only the samples taken after mark() -- the start of the timed region --
    are reported."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None
        self._thread = None
        self._mark = 0

    def mark(self):
        self._mark = len(self.samples)

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                           "--format=csv,noheader,nounits", "-lms", "200"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._proc = None
            return self
        self._thread = threading.Thread(target=self._read, daemon=True)
        self._thread.start()
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        if self._thread is not None:
            self._thread.join(timeout=5)
        if len(self.samples) > self._mark:
            self.samples = self.samples[self._mark:]
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[2 + i]
                          and "Not" not in s[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


REF_FUNCS = dict(d=(9, []), f=(10, []), c_d=(8, []), g_n=(11, []), c0=(8, []))
# degrees the reference's SparseLU can factor on the C2 mesh (256^2) on one
# host core: measured in the build container (1 Xeon core, 62 GB) one
# implicit-Euler step took 21.7 s at p = 0 and 423 s at p = 1; at p = 2
# (2.36M unknowns) SuperLU with COLAMD ordering -- the ordering of Eigen's
# SparseLU -- ran out of the 62 GB host memory ("Not enough memory to perform
# factorization"), and p = 3, 4 are larger still.
REF_P_DEFAULT = {"c2": [0, 1]}
CPU_SAMPLE = {"c2": ([0], 1), "c1": ([1], 100)}
REF_STEPS = {"c1": 100}  # reference arm: implicit-Euler steps per degree (C1: the whole 100-step run)  # our line's cpu_baseline: (degrees, steps)
REF_P_INFEASIBLE = ("p >= 2 not run: the reference's SparseLU of the 3KN system (2.36M unknowns at p = 2) "
                    "exhausted 62 GB of host memory in the build container; p = 3, 4 are larger")


def ref_worker(p, dim, dt, steps, jitter, bc):
    """One process, one degree: `steps` implicit-Euler steps of the reference
    (oracle/_ref = the unmodified headers + Eigen shim, SciPy SuperLU as its
    SparseLU) from the initial state, timed around euler_step with
    steady_clock as ldg_main.cpp:199-214 does.  Prints one JSON line."""
    from oracle import reflib as R

    if not R.available():
        raise RuntimeError("oracle/_ref/libldgref.so missing")
    import scipy.sparse.linalg  # noqa: F401  (the SparseLU stand-in: imported before the timed region)

    boundary = {int(k): v for k, v in bc.items()}
    warm = R.RefCase(R.RefMesh.square(0.5), n_of(p), 1.0, REF_FUNCS, boundary)  # untimed: loads SuperLU
    warm.euler(warm.initial_state(), 0.0, dt, 1)
    if jitter > 0.0:
        from oracle import ldg_oracle as O

        coords, v0t = O.fk_lists(dim)
        coords = O.fk_jittered_coords(dim, jitter, 0)
        mesh = R.RefMesh.create(coords, v0t.astype("int32"))
    else:
        mesh = R.RefMesh.square(1.0 / dim)
    n = n_of(p)
    case = R.RefCase(mesh, n, 1.0, REF_FUNCS, boundary)
    y = case.initial_state()
    y, t, sec = case.euler(y, 0.0, dt, steps)
    print(json.dumps({"p": p, "K": mesh.num_t, "N": n, "steps": steps, "seconds": sec,
                      "dof": 3 * mesh.num_t * n * steps}), flush=True)


def reference_runs(workload, ps, steps, cap_s):
    """Runs ref_worker for every p concurrently, one process (one host core)
    each, killed at cap_s seconds.  Returns {p: result dict | {"status": why}}."""
    dim, _, dt, jitter, boundary, _ = WORKLOADS[workload]
    procs = {}
    for p in ps:
        cmd = [sys.executable, os.path.abspath(__file__), "--ref-worker", str(p), "--steps", str(steps),
               "--workload", workload]
        procs[p] = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                                    env=dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1"))
    out = {}
    t_end = time.time() + cap_s
    for p, pr in procs.items():
        try:
            so, se = pr.communicate(timeout=max(1.0, t_end - time.time()))
            line = [x for x in so.splitlines() if x.startswith("{")]
            out[p] = json.loads(line[-1]) if pr.returncode == 0 and line else {
                "status": f"failed (rc {pr.returncode}): {se.strip().splitlines()[-1] if se.strip() else ''}"}
        except subprocess.TimeoutExpired:
            pr.kill()
            pr.communicate()
            out[p] = {"status": f"not finished within the {cap_s:.0f} s cap"}
    return out, dim


def reference_summary(res, dim, workload):
    done = {p: r for p, r in res.items() if "seconds" in r}
    if not done:
        raise RuntimeError(f"no reference degree finished: {res}")
    dof = sum(r["dof"] for r in done.values())
    sec = sum(r["seconds"] for r in done.values())
    per_p = {str(p): ({"seconds_per_step": r["seconds"] / r["steps"], "dof_updates_per_s": r["dof"] / r["seconds"]}
                      if "seconds" in r else r) for p, r in sorted(res.items())}
    try:
        cpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        model = next((ln.split(":", 1)[1].strip() for ln in cpu.splitlines() if ln.startswith("Model name")), "?")
    except Exception:  # pragma: no cover
        model = "?"
    sample = (f"reference (oracle/_ref: unmodified headers + Eigen shim, SciPy SuperLU with COLAMD as its SparseLU) "
              f"on the {workload.upper()} mesh FK {dim}x{dim} (K={2 * dim * dim}), p={sorted(done)}, "
              f"{next(iter(done.values()))['steps']} implicit-Euler step(s) each from the initial state, "
              f"one single-threaded process per degree on its own core (host: {model}, nproc {os.cpu_count()}); "
              f"value = sum of DOF updates / sum of per-degree step times (one core)")
    return dof / sec, sec, sample, per_p, sorted(done)


C3_METRIC, C3_UNIT = "assembled BSR bytes/s (time-dependent C-row blocks, SURVEY.md §8d)", "B/s"


def reference_sample_c3(steps, warmup):
    """Reference build_blocks (system.hpp:110-152) on FK 64x64 at p=4: assembled
    time-dependent BSR bytes (SURVEY §8d formula) per second."""
    from oracle import reflib as R

    dim, p = 64, 4
    funcs = dict(d=(9, []), f=(10, []), c_d=(8, []), g_n=(11, []), c0=(8, []))
    if not R.available():
        raise RuntimeError("oracle/_ref/libldgref.so missing")
    mesh = R.RefMesh.square(1.0 / dim)
    case = R.RefCase(mesh, n_of(p), 1.0, funcs, {1: "D", 2: "D", 3: "D", 4: "D"})
    case.time_build(0.0, max(warmup, 0) or 1)
    sec = case.time_build(0.1, steps)
    sample = (f"reference build_blocks (unmodified headers + Eigen shim): FK {dim}x{dim} (K={2 * dim * dim}), p={p}, "
              f"{steps} calls (projection, all operators as triplets, CSC merge)")
    return bytes_asm_survey(dim, p) * steps / sec, sec, sample


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    if args.workload == "c3":
        value, sec, sample = reference_sample_c3(args.steps, args.warmup)
        line = {"impl": "reference", "metric": C3_METRIC, "value": value, "unit": C3_UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (analytic BASELINE.json problem)",
                "config": {"workload": WORKLOADS["c3"][5] + " [reference: bounded sample, see cpu_baseline]"},
                "cpu_baseline": {"value": value, "unit": C3_UNIT, "cores": 1, "kind": "reference", "sample": sample},
                "e2e": {"value": value, "unit": C3_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    ps = ([int(x) for x in args.ref_p.split(",")] if args.ref_p else
          REF_P_DEFAULT.get(args.workload, WORKLOADS[args.workload][1]))
    # the reference is CPU-only and deterministic: one timed step per degree
    # is the bounded sample (its p = 1 step alone takes ~7 min); no warm-up
    res, dim = reference_runs(args.workload, ps, REF_STEPS.get(args.workload, 1), args.ref_cap)
    value, sec, sample, per_p, done = reference_summary(res, dim, args.workload)
    cfg = config_of(args.workload, dim, WORKLOADS[args.workload][1], WORKLOADS[args.workload][2], 1)
    cfg["p_measured"] = done
    cfg["per_p"] = per_p
    if args.workload == "c2" and not args.ref_p:
        cfg["p_not_run"] = REF_P_INFEASIBLE
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec / REF_STEPS.get(args.workload, 1),  # one step of every measured p
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic BASELINE.json problem)", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_of(workload, dim, ps, dt, world):
    """The `config` both arms report for a workload (same keys, same values)."""
    return {"workload": WORKLOADS[workload][5], "dim": dim, "K": 2 * dim * dim, "p": ps, "dt": dt,
            "parallelism": f"strips{world} (NCCL halos + allreduce)" if world > 1 else "single"}


def run_assembly_c3(args):
    """BASELINE config 3: projection + right-hand side + the full time-dependent
    C-row BSR (8 blocks per element) every step, device-resident output."""
    world, rank, local = dist_env()
    import torch

    import paper_1408_3877_b200 as ld

    ld.set_device(local)
    dim, ps, _, _, boundary, desc = WORKLOADS["c3"]
    p = ps[0]
    spec = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0,
                          boundary=boundary)
    s = ld.LdgSystem.square(dim, p, spec)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=f"cuda:{local}")
    clocks = ClockSampler(local)
    if not args.no_clocks:
        clocks.start()
    for i in range(args.warmup):
        s.assemble_blocks(0.01 * (i + 1))
    torch.cuda.synchronize()
    clocks.mark()
    total_ms = 0.0
    launches0 = s.info()["launches"]
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        total_ms += s.assemble_blocks(0.1 * (i + 1))
    clk = clocks.stop()
    launches = s.info()["launches"] - launches0
    bsr = bytes_asm_survey(dim, p)
    value = bsr * args.steps / (total_ms * 1e-3)
    peak, peak_src = hbm_peak()
    kern = s.time_kernels(0.5, 0.05, reps=3, flush=True)  # the solver's diagonal-block assembly, for reference
    traffic, traffic_src = ncu_traffic("k_assemble_rows<4, 0", p, dim)
    cpu = None
    if not args.no_cpu_baseline:
        try:
            v, sec, sample = reference_sample_c3(1, 1)
            cpu = {"value": v, "unit": C3_UNIT, "cores": 1, "kind": "reference", "sample": sample}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": C3_UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {e}"}
    line = {
        "metric": C3_METRIC, "value": value, "unit": C3_UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: analytic d(t), f(t) of BASELINE.json; FK mesh generated on device",
        "config": {"workload": desc, "dim": dim, "K": 2 * dim * dim, "p": p,
                   "bytes_per_step": bsr, "l2": "flushed (256 MB write) before every timed step"},
        "e2e": {"value": None, "unit": C3_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "note": "the assembled blocks stay on the device (30 GB per step); the reference's build_blocks "
                        "result is its host CSC"},
        "gpu_launches": launches,
        "roofline": {"kernel": "projection + rhs + k_assemble_rows<4, kModeE> (all 8 blocks), one call",
                     "bound": "hbm", "achieved": value / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": value / 1e9 / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "traffic_note": "DRAM bytes of the assembly kernel alone (87 % of the call); the call's "
                                     "algorithmic bytes are bytes_per_step", "peak_source": peak_src,
                     "solver_assembly_diagonal_blocks_ms": kern["ms_assemble"]},
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    s.close()
    return 0


def run_ours(args):
    if args.workload == "c3":
        return run_assembly_c3(args)
    world, rank, local = dist_env()
    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    import paper_1408_3877_b200 as ld
    from paper_1408_3877_b200 import strips

    ld.set_device(local)
    dim1, ps, dt, jitter, boundary, desc = WORKLOADS[args.workload]
    if args.p is not None:
        ps = [int(x) for x in args.p.split(",")]
    # strips of one FK(dim) mesh: weak scaling keeps the elements per GPU of the
    # workload's anchor (C4/C5: their 8-GPU size), strong
    # scaling keeps the mesh
    dim = strips.scaled_dim(dim1, world, args.scaling, WEAK_ANCHOR.get(args.workload, 1))
    spec = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0,
                          boundary=boundary)
    opts = ld.SolverOptions()
    if args.krylov is not None:
        opts.krylov = args.krylov
    if args.restart is not None:
        opts.restart = args.restart
    def make(p):
        if world > 1:
            ids = [ld.nccl_unique_id() if rank == 0 else None]
            torch.distributed.broadcast_object_list(ids, src=0)
            s = ld.LdgSystem.square_dist(dim, p, spec, rank, world, ids[0], jitter=jitter, seed=0)
        else:
            s = ld.LdgSystem.square(dim, p, spec, jitter=jitter, seed=0)
        return s

    systems = [make(p) for p in ps]
    for s in systems:
        s.initial_state()
    dof_step = sum(3 * s.num_t * s.n for s in systems)  # whole-job DOF per step (global K)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local)
    if not args.no_clocks:
        clocks.start()
    # warm-up (W full steps)
    for _ in range(args.warmup):
        for s in systems:
            s.euler_steps(dt, 1, opts)
    barrier()
    # e2e runs the host-buffer C ABI call (the call a caller's time loop
    # makes).  Twins: the same time integration from t = 0 on second systems
    # driven through host buffers, so their timed steps are the device-timed
    # steps (same states, solver history, iterations) -- when a second copy
    # fits in HBM; otherwise the systems continue their own integration
    # through host buffers after the device-timed steps (one untimed host step
    # first, so the timed ones continue the caller's loop).
    used = sum(s.info()["bytes_device"] for s in systems)
    free = torch.cuda.mem_get_info(local)[0]
    twin_mode = free > 1.2 * used + (4 << 30)
    if world > 1:  # the same decision on every rank (the twins' creation is collective)
        flag = torch.tensor([1 if twin_mode else 0], device=f"cuda:{local}")
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
        twin_mode = bool(flag.item())
    twins = [make(p) for p in ps] if twin_mode else systems
    twin_io = []
    for s in twins:
        if twin_mode:
            y0, t0 = s.initial_state()
        else:
            y0, t0 = None, None
        twin_io.append([y0, None, t0])

    def twin_step(i):
        if twin_io[i][0] is not None and not isinstance(twin_io[i][0], torch.Tensor):
            twin_io[i][0] = torch.from_numpy(twin_io[i][0]).pin_memory()
            twin_io[i][1] = torch.empty_like(twin_io[i][0]).pin_memory()
        pin_in, pin_out, t = twin_io[i]
        st = twins[i].euler_steps_host(pin_in.data_ptr(), t, dt, 1, pin_out.data_ptr(), opts)
        pin_in.copy_(pin_out)
        twin_io[i][2] = t + dt
        return st

    if twin_mode:
        for _ in range(args.warmup):
            for i in range(len(ps)):
                twin_step(i)
    barrier()
    clocks.mark()
    launches0 = sum(s.info()["launches"] for s in systems)
    per_p = {p: dict(ms=0.0, ms_asm=0.0, ms_solve=0.0, ms_setup=0.0, ms_krylov=0.0, iters=0, applies=0, residual=0.0)
             for p in ps}
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        for p, s in zip(ps, systems):
            st = s.euler_steps(dt, 1, opts)
            r = per_p[p]
            r["ms_asm"] += st["ms_assemble"]
            r["ms_solve"] += st["ms_solve"]
            r["ms_setup"] += st["ms_setup"]
            r["ms_krylov"] += st["ms_krylov"]
            r["ms"] += st["ms_assemble"] + st["ms_solve"]
            r["iters"] += st["iterations"]
            r["applies"] += st["applies"]
            r["residual"] = max(r["residual"], st["residual"])
    barrier()
    clk = clocks.stop()
    launches = sum(s.info()["launches"] for s in systems) - launches0
    total_ms = max_over_ranks(sum(r["ms"] for r in per_p.values()))
    value = dof_step * args.steps / (total_ms * 1e-3)

    # e2e through the host-buffer C ABI call (each rank copies its owned rows):
    # the twins run the same K steps as the device-timed systems above
    if not twin_mode:
        for i, s in enumerate(systems):  # continue each system's integration through host buffers
            y, t = s.get_state()
            twin_io[i] = [y, None, t]
            twin_step(i)
    e2e_ms = 0.0
    h2d = 0
    e2e_iters = 0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        for i in range(len(ps)):
            st = twin_step(i)
            e2e_ms += st["ms_total"]
            e2e_iters += st["iterations"]
    h2d = sum(io[0].numel() * io[0].element_size() for io in twin_io)
    e2e_ms = max_over_ranks(e2e_ms)
    e2e_value = dof_step * args.steps / (e2e_ms * 1e-3)

    # per-kernel timing for the roofline (CUDA events on the library's stream, L2 flushed)
    peak, peak_src = hbm_peak()
    kern = {}
    for p, s in zip(ps, systems):
        kern[p] = s.time_kernels(s.t, dt, reps=5, flush=True)
    kloc = dim if world == 1 else None  # per-rank byte counts below assume one GPU
    # dominant kernel: stage 2 of the level-0 multigrid smoother (k_s2f;
    # s2_per_vcycle launches per V-cycle = level-0 sweeps + the residual, one
    # V-cycle per FGMRES iteration), taken at the p where it holds the largest
    # share of the step
    shares = {p: kern[p]["ms_sweep_s2"] * kern[p]["s2_per_vcycle"] * per_p[p]["iters"] / max(total_ms, 1e-9)
              for p in ps}
    pd = max(shares, key=shares.get)
    roof = None
    if kloc is not None:
        bs = bytes_sweep_s2(dim, pd)
        achieved = bs / (kern[pd]["ms_sweep_s2"] * 1e-3) / 1e9
        traffic, traffic_src = ncu_traffic("k_s2f<%d, 1" % pd, pd, dim)
        roof = {"kernel": f"k_s2f (level-0 smoother stage 2 + block-Jacobi update, FP16 E), p={pd}",
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                "share_of_step_est": shares[pd], "bytes_per_launch": bs,
                "others": {str(p): {"sweep_s2_GBps": bytes_sweep_s2(dim, p) / (kern[p]["ms_sweep_s2"] * 1e-3) / 1e9,
                                    "schur_apply_GBps": bytes_schur(dim, p) / (kern[p]["ms_schur"] * 1e-3) / 1e9,
                                    "assemble_GBps": bytes_asm(dim, p) / (kern[p]["ms_assemble"] * 1e-3) / 1e9,
                                    "full_apply_compulsory_GBps": bytes_full_compulsory(dim, p)
                                    / (kern[p]["ms_spmv"] * 1e-3) / 1e9,
                                    "full_apply_effective_GBps_survey_formula": bytes_spmv(dim, p)
                                    / (kern[p]["ms_spmv"] * 1e-3) / 1e9,
                                    "assemble_effective_GBps_survey_formula": bytes_asm_survey(dim, p)
                                    / (kern[p]["ms_assemble"] * 1e-3) / 1e9,
                                    "ms": kern[p]} for p in ps}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded sample of the same workload: the lowest degree of the sweep on
        # the same mesh (one reference step: ~22 s at 256^2, p = 0)
        cps, csteps = CPU_SAMPLE.get(args.workload, (None, 1))
        try:
            if cps is None:
                raise RuntimeError("not run: the reference cannot assemble/factor this mesh on one host core "
                                   "(SURVEY.md §8d)")
            res, rdim = reference_runs(args.workload, cps, csteps, args.ref_cap)
            v, sec, sample, _, _ = reference_summary(res, rdim, args.workload)
            cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "reference", "sample": sample}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"{e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: analytic c, d(t), f(t) of BASELINE.json; FK mesh generated on device",
            "config": dict(config_of(args.workload, dim, ps, dt, world), **{
                       "l2": "flushed (256 MB write) before every timed step; p>=2 working sets exceed L2",
                       "solver": "default ldg_solver_opts: FGMRES(30) on the exact Schur complement to a relative "
                                 "Schur residual of 1e-14 (states within 1e-10 relative L2 of the reference's direct "
                                 "solve: tests/test_gpu_parity_scale.py) plus the reference residual contract 1e-10; "
                                 "p-coarsened geometric multigrid preconditioner (level 0 Chebyshev, coarse levels "
                                 "damped block-Jacobi, mixed-precision smoother)",
                       "per_p": {str(p): {"ms_per_step": per_p[p]["ms"] / args.steps,
                                          "ms_assemble": per_p[p]["ms_asm"] / args.steps,
                                          "ms_solve": per_p[p]["ms_solve"] / args.steps,
                                          "ms_solve_setup": per_p[p]["ms_setup"] / args.steps,
                                          "ms_krylov": per_p[p]["ms_krylov"] / args.steps,
                                          "iterations_per_step": per_p[p]["iters"] / args.steps,
                                          "max_residual": per_p[p]["residual"],
                                          "dof_updates_per_s": 3 * 2 * dim * dim * n_of(p) * args.steps /
                                          (per_p[p]["ms"] * 1e-3)} for p in ps}}),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d,
                    "iterations": e2e_iters, "device_iterations": sum(r["iters"] for r in per_p.values()),
                    "note": ("ldg_euler_steps_host on a twin system integrating the same steps from t = 0 "
                             if twin_mode else
                             "ldg_euler_steps_host continuing each system's integration after the device-timed "
                             "steps (a second copy does not fit in HBM) ")
                            + "(pinned host state in, host state out, copies inside the timed region)"},
            "gpu_launches": launches,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    for s in systems + (twins if twin_mode else []):
        s.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--p", default=None, help="comma-separated degrees (overrides the workload's sweep)")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="N > 1: weak = fixed elements per GPU (the workload's anchor size), strong = fixed mesh "
                         "(default: strong for C4/C5, whose meshes are quoted for the whole job, weak otherwise)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="skip the nvidia-smi sampler (diagnostics only)")
    ap.add_argument("--krylov", type=int, default=None, help="0 FGMRES (default), 1 BiCGStab")
    ap.add_argument("--restart", type=int, default=None, help="FGMRES restart length")
    ap.add_argument("--ref-p", default=None, help="reference arm: comma-separated degrees (default: the feasible ones)")
    ap.add_argument("--ref-cap", type=float, default=900.0, help="reference arm: wall-clock cap in seconds")
    ap.add_argument("--ref-worker", type=int, default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.scaling is None:
        args.scaling = "strong" if args.workload in WEAK_ANCHOR else "weak"
    if args.ref_worker is not None:
        dim, _, dt, jitter, boundary, _ = WORKLOADS[args.workload]
        ref_worker(args.ref_worker, dim, dt, args.steps, jitter, boundary)
        return 0
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
