"""Parity of the sm_100a path (through the C ABI) with the reference.

Golden fixtures (tests/golden, generated from the unmodified reference by
make_golden.py) pin the small cases; the CPU oracle (oracle/ldg_oracle.py)
checks mid-size meshes; size-independent properties cover the BASELINE
sizes.  Tolerances are those of north_star / SURVEY.md §8d: operators within
1e-12 of max|ref| on the union pattern, states within 1e-10 relative L2.
"""
from __future__ import annotations

import numpy as np
import pytest

from ldg_testutil import CASES, N_TO_P, coo, op_rel_err, spec_from_golden, vec_rel_err

pytestmark = pytest.mark.gpu

OP_TOL = 1e-12
STATE_TOL = 1e-10


def _system(g, ld):
    funcs, boundary = spec_from_golden(g)
    spec = ld.ProblemSpec(d=funcs["d"], f=funcs["f"], c_d=funcs["c_d"], g_n=funcs["g_n"], c0=funcs["c0"],
                          eta=1.0, boundary=boundary)
    p = N_TO_P[int(g["n_local"])]
    return ld.LdgSystem.from_mesh(g["coords"], g["v0t"], p, spec, id_e0t=g["id_in"])


@pytest.fixture(scope="module")
def ld():
    import paper_1408_3877_b200 as ld

    ld.load_library()
    return ld


TIGHT = dict(rtol=1e-14, atol=0.0, maxit=50000, precond=1)


@pytest.mark.parametrize("case", CASES)
def test_mesh_lists(case, golden, ld):
    g = golden(case)
    s = _system(g, ld)
    L = s.mesh_lists()
    np.testing.assert_array_equal(L["nbr"], g["mesh_nbr"])
    np.testing.assert_array_equal(L["nbr_n"], g["mesh_nbr_n"])
    bnd = g["mesh_nbr"] < 0
    np.testing.assert_array_equal(L["id_e0t"][bnd], g["mesh_id_e0t"][bnd])
    np.testing.assert_array_equal(L["b"], g["mesh_b"])
    np.testing.assert_array_equal(L["area"], g["mesh_area"])
    np.testing.assert_allclose(L["len"], g["mesh_len"], rtol=4e-16, atol=0)
    np.testing.assert_allclose(L["nu"], g["mesh_nu"], rtol=0, atol=4e-16)


def test_device_generated_square_mesh(golden, ld):
    """domain_square(1/16) generated on the device equals the reference lists."""
    g = golden("c1_fk16_p1")
    s = ld.LdgSystem.square(16, 1, ld.BASELINE_SPEC)
    L = s.mesh_lists()
    np.testing.assert_array_equal(L["coords"], g["coords"])
    np.testing.assert_array_equal(L["v0t"], g["v0t"])
    np.testing.assert_array_equal(L["nbr"], g["mesh_nbr"])
    np.testing.assert_array_equal(L["nbr_n"], g["mesh_nbr_n"])
    np.testing.assert_array_equal(L["id_e0t"][g["mesh_nbr"] < 0], g["mesh_id_e0t"][g["mesh_nbr"] < 0])


def test_device_jitter_matches_fixture(golden, ld):
    """Config-4 jitter (splitmix64 stream) is bit-identical to the coordinates the reference saw."""
    g = golden("jitter8_p2")
    funcs, boundary = spec_from_golden(g)
    spec = ld.ProblemSpec(**funcs, eta=1.0, boundary=boundary)
    s = ld.LdgSystem.square(8, 2, spec, jitter=0.2, seed=0)
    L = s.mesh_lists()
    np.testing.assert_array_equal(L["coords"], g["coords"])
    np.testing.assert_array_equal(L["nbr"], g["mesh_nbr"])


@pytest.mark.parametrize("case", CASES)
def test_operators(case, golden, ld):
    g = golden(case)
    s = _system(g, ld)
    s.assemble(float(g["t_ops"]))
    kn = s.block_dim
    names = sorted({k[3:-2] for k in g if k.startswith("op_") and k.endswith("_r")})
    assert names
    for name in names:
        n = 3 * kn if name == "A" else kn
        ref = coo(g[f"op_{name}_r"], g[f"op_{name}_c"], g[f"op_{name}_v"], n)
        dev = coo(*s.operator(name), n)
        err = op_rel_err(dev, ref)
        assert err <= OP_TOL, f"{case}: operator {name} rel err {err:.3e}"


@pytest.mark.parametrize("case", CASES)
def test_vectors(case, golden, ld):
    g = golden(case)
    s = _system(g, ld)
    s.assemble(float(g["t_ops"]))
    for name in ("D", "F", "jd1", "jd2", "kd", "kn", "l", "V"):
        dev = s.vector(name)
        ref = g[f"vec_{name}"]
        err = vec_rel_err(dev, ref)
        assert err <= OP_TOL, f"{case}: vector {name} rel err {err:.3e}"


@pytest.mark.parametrize("case", CASES)
def test_initial_state(case, golden, ld):
    g = golden(case)
    s = _system(g, ld)
    y0, t0 = s.initial_state()
    assert t0 == 0.0
    assert vec_rel_err(y0, g["y0"]) <= OP_TOL


@pytest.mark.parametrize("case", ["c1_fk16_p1", "jitter8_p2", "fk6_p4", "fk8_p0", "fk8_p3"])
def test_euler_states(case, golden, ld):
    """Implicit Euler states after the fixture's step counts (system.hpp:155-174)."""
    g = golden(case)
    s = _system(g, ld)
    y, t = s.initial_state()
    dt = float(g["dt"])
    steps = sorted(int(k[1:]) for k in g if k.startswith("y") and k[1:].isdigit() and k != "y0")
    done = 0
    for n in steps:
        st = s.euler_steps(dt, n - done, ld.SolverOptions(**TIGHT))
        done = n
        assert st["residual"] <= 1e-10
        y, t = s.get_state()
        ref = g[f"y{n}"]
        rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        assert rel <= STATE_TOL, f"{case}: state after {n} steps rel L2 {rel:.3e}"
    assert abs(t - done * dt) < 1e-12


def test_c1_hundred_steps_default_solver(golden, ld):
    """BASELINE config 1 end to end with the default (production) solver options."""
    g = golden("c1_fk16_p1")
    s = ld.LdgSystem.square(16, 1, ld.BASELINE_SPEC)
    s.initial_state()
    st = s.euler_steps(0.01, 100)
    y, t = s.get_state()
    rel = np.linalg.norm(y - g["y100"]) / np.linalg.norm(g["y100"])
    assert rel <= STATE_TOL, rel
    assert st["residual"] <= 1e-10


@pytest.mark.parametrize("p", [0, 1, 2, 3, 4])
def test_multigrid_matches_block_jacobi(p, ld):
    """The geometric-multigrid preconditioner changes the iteration count, not the
    answer: same state as block-Jacobi within the solve tolerance, far fewer iterations."""
    res = {}
    for pc in (1, 2, 3):  # block-Jacobi, multigrid (FP32 smoother copies), multigrid (FP64)
        s = ld.LdgSystem.square(32, p, ld.BASELINE_SPEC, jitter=0.0)
        s.initial_state()
        st = s.euler_steps(0.05, 2, ld.SolverOptions(rtol=1e-13, precond=pc))
        assert st["residual"] <= 1e-10
        res[pc] = (s.get_state()[0], st["iterations"])
    y1, it1 = res[1]
    for pc in (2, 3):
        y2, it2 = res[pc]
        assert np.linalg.norm(y2 - y1) / np.linalg.norm(y1) <= 1e-9
        assert it2 * 3 < it1, (pc, it1, it2)


def test_multigrid_jittered_mesh(ld):
    """Config-4 style jittered FK mesh with mixed boundary conditions: multigrid
    (coarse levels subsample the jittered vertices) agrees with block-Jacobi."""
    spec = ld.ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0,
                          boundary={1: "D", 2: "N", 3: "N", 4: "D"})
    out = []
    for pc in (1, 2):
        s = ld.LdgSystem.square(32, 3, spec, jitter=0.2, seed=0)
        s.initial_state()
        st = s.euler_steps(0.1, 1, ld.SolverOptions(rtol=1e-13, precond=pc))
        assert st["residual"] <= 1e-10
        out.append(s.get_state()[0])
    assert np.linalg.norm(out[1] - out[0]) / np.linalg.norm(out[0]) <= 1e-9


def test_apply_lhs_matches_reference_operator(golden, ld):
    """The full block-SpMV (W + dt A) y against the reference's assembled A."""
    g = golden("jitter8_p2")
    s = _system(g, ld)
    t = float(g["t_ops"])
    s.assemble(t)
    kn = s.block_dim
    A = coo(g["op_A_r"], g["op_A_c"], g["op_A_v"], 3 * kn)
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, 3 * kn)
    dt = 0.05
    M = coo(g["op_mass_r"], g["op_mass_c"], g["op_mass_v"], kn) if "op_mass_r" in g else None
    y = s.apply_lhs(dt, x)
    ref = dt * (A @ x)
    if M is None:
        s2 = s.operator("mass")
        M = coo(*s2, kn)
    ref[2 * kn:] += M @ x[2 * kn:]
    assert vec_rel_err(y, ref) <= 1e-13


def test_stationary_solve(golden, ld):
    """solve_stationary (system.hpp:177-185) on the refined 1/3 square, manufactured problem."""
    g = golden("stationary_mms_p2")
    spec = ld.ProblemSpec(d="exp_sum", f="mms_f", c_d="mms_exact", g_n="mms_gn", c0="mms_exact", eta=1.0,
                          boundary={1: "N", 2: "D", 3: "N", 4: "D"})
    s = ld.LdgSystem.from_mesh(g["coords"], g["v0t"], 2, spec, id_e0t=g["id_in"])
    c, z1, z2 = s.solve_stationary(0.0, ld.SolverOptions(rtol=1e-14, maxit=100000))
    for dev, ref in ((c, g["c"]), (z1, g["z1"]), (z2, g["z2"])):
        rel = np.linalg.norm(dev.ravel() - ref) / np.linalg.norm(ref)
        assert rel <= 1e-9, rel


def test_reference_exceptions(ld):
    spec = ld.ProblemSpec(boundary={1: "D", 2: "D", 4: "D"})  # ID 3 unmapped
    with pytest.raises(ValueError, match="boundary ID 3"):
        ld.LdgSystem.square(2, 1, spec)
    with pytest.raises(ValueError, match="eta"):
        ld.LdgSystem.square(2, 1, ld.ProblemSpec(eta=0.0, boundary={1: "D", 2: "D", 3: "D", 4: "D"}))
    with pytest.raises(ld.MeshError):
        ld.LdgSystem.from_mesh([[0, 0], [1, 0], [0, 1]], [[0, 2, 1]], 1,
                               ld.ProblemSpec(boundary={0: "D"}))  # clockwise
    s = ld.LdgSystem.square(2, 1, ld.BASELINE_SPEC)
    s.initial_state()
    with pytest.raises(ValueError, match="time step"):
        s.euler_steps(0.0, 1)
    with pytest.raises(ValueError):
        ld.LdgSystem.square(2, 5, ld.BASELINE_SPEC)


def test_cpp_host_mirror_simulate(ld):
    """The C++ host mirror (paper_1408_3877_b200/host/ldg_host.hpp) driving the
    reference's simulate loop, host-buffer and device-resident variants."""
    import os
    import subprocess

    import tempfile

    sim = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "ldg_simulate")
    for extra in (["--host"], ["--device-resident"]):
        with tempfile.TemporaryDirectory() as d:
            base = os.path.join(d, "c")
            r = subprocess.run([sim, "16", "1", "10", "1.0"] + extra + [base, "5"], capture_output=True, text=True,
                               timeout=300)
            assert r.returncode == 0, r.stderr
            assert "simulate: 10 steps" in r.stdout
            # the reference's output cadence (ldg_main.cpp:195-207): step 0, then every output_every steps
            assert sorted(os.listdir(d)) == ["c.0.vtu", "c.10.vtu", "c.5.vtu"]
            assert open(base + ".10.vtu").read().count("\n") > 3 * 512


def test_consecutive_handles_fp16_smoother(ld):
    """Buffers allocated lazily by one handle's first solve must be zeroed
    before its kernels use them: the zeroing ran on the legacy default stream
    without ordering against the library's non-blocking stream, and a second
    handle at 512^2, p = 3 got FP16 smoother copies full of inf (regression)."""
    for _ in range(2):
        s = ld.LdgSystem.square(512, 3, ld.BASELINE_SPEC)
        s.initial_state()
        st = s.euler_steps(0.1, 1, ld.SolverOptions())
        assert st["residual"] <= 1e-10 and st["iterations"] < 40, st
        s.close()
