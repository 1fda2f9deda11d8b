"""The drop-in boundary's operator formats against the reference (SURVEY §8a
row a12, §8b): CSC exactly as the reference's Eigen SparseMatrix stores it
(same column pointers, same row indices, values within 1e-12), block CSR in
reference element order, the per-operator entry points taking a caller's D
(assembly.hpp:113-136, 214-252), and build_blocks through the C++ host mirror
(tools/ldg_blocks, SystemBlocks of system.hpp:110-152).

The reference side is oracle/_ref (the unmodified reference compiled against
the Eigen shim); the pattern comparison needs it, so these tests skip when it
was not built."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from oracle import ldg_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = dict(d=(9, []), f=(10, []), c_d=(8, []), g_n=(11, []), c0=(8, []))
MIXED = {1: "D", 2: "D", 3: "N", 4: "N"}
OPS = ["mass", "h1", "h2", "g1", "g2", "r1", "rd1", "r2", "rd2", "q1", "qn1", "q2", "qn2", "s", "sd", "A"]
# (dim, p, jitter)
CASES = {"fk16_p2": (16, 2, 0.0), "fk8_p4": (8, 4, 0.0), "jitter12_p3": (12, 3, 0.2), "fk32_p1": (32, 1, 0.0)}
T_OPS = 0.3


def _reflib():
    from oracle import reflib as R

    if not R.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return R


@pytest.fixture(scope="module")
def ld():
    import paper_1408_3877_b200 as ld

    ld.load_library()
    return ld


def _ids(coords, v0t):
    K = v0t.shape[0]
    ids = np.zeros((K, 3), np.int32)
    for n in range(3):
        a, b = coords[v0t[:, (n + 1) % 3]], coords[v0t[:, (n + 2) % 3]]
        mx, my = 0.5 * (a[:, 0] + b[:, 0]), 0.5 * (a[:, 1] + b[:, 1])
        i = np.zeros(K, np.int32)
        i = np.where(np.abs(my) < 1e-12, 1, i)
        i = np.where((i == 0) & (np.abs(mx - 1.0) < 1e-12), 2, i)
        i = np.where((i == 0) & (np.abs(my - 1.0) < 1e-12), 3, i)
        i = np.where((i == 0) & (np.abs(mx) < 1e-12), 4, i)
        ids[:, n] = i
    return ids


def _pair(name, ld):
    dim, p, jitter = CASES[name]
    R = _reflib()
    coords, v0t = O.fk_lists(dim)
    if jitter:
        coords = O.fk_jittered_coords(dim, jitter, 0)
    v0t = v0t.astype(np.int32)
    mesh = R.RefMesh.create(coords, v0t, _ids(coords, v0t))
    case = R.RefCase(mesh, O.local_dof_count(p), 1.0, BASE, MIXED)
    case.assemble(T_OPS)
    spec = ld.ProblemSpec(**BASE, eta=1.0, boundary=MIXED)
    s = ld.LdgSystem.square(dim, p, spec, jitter=jitter, seed=0)
    # the reference's own RefTensors, as its LdgSystem(mesh, spec, rt) receives them
    s.set_reference_tensors(R.ref_tensors(O.local_dof_count(p)))
    s.assemble(T_OPS)
    return s, case, mesh


def _same_csc(dev, ref_cp, ref_ri, ref_v, what):
    np.testing.assert_array_equal(dev.indptr, ref_cp, err_msg=f"{what}: column pointers")
    np.testing.assert_array_equal(dev.indices, ref_ri, err_msg=f"{what}: row indices")
    scale = np.abs(ref_v).max() if ref_v.size else 1.0
    err = np.abs(dev.data - ref_v).max() if ref_v.size else 0.0
    assert err <= 1e-12 * max(scale, 1e-300), f"{what}: value error {err:.3e} (max {scale:.3e})"


@pytest.mark.parametrize("name", sorted(CASES))
def test_csc_export_is_the_reference_storage(name, ld):
    """ldg_export_operator_csc == the reference's compressed CSC arrays for every
    operator of build_blocks, A included (assembly.hpp:21-22,62-67; system.hpp:137-140)."""
    s, case, _ = _pair(name, ld)
    for op in OPS:
        cp, ri, v = case.op_csc(op)
        _same_csc(s.operator_csc(op), cp, ri, v, f"{name}/{op}")


@pytest.mark.parametrize("name", ["fk16_p2", "jitter12_p3"])
def test_csc_export_with_library_tensors(name, ld):
    """Without the caller's tensors (the library's own build_ref_tensors, equal to
    the reference's to ~1e-14 but not bit for bit): A's pattern is still the
    reference's (its M blocks drop the same exact zeros; every other block of A
    is stored whole), values within 1e-12."""
    dim, p, jitter = CASES[name]
    s0, case, _ = _pair(name, ld)
    spec = ld.ProblemSpec(**BASE, eta=1.0, boundary=MIXED)
    s = ld.LdgSystem.square(dim, p, spec, jitter=jitter, seed=0)
    s.assemble(T_OPS)
    for op in ("A", "mass", "s", "sd", "q1", "qn2", "r1", "rd2"):
        _same_csc(s.operator_csc(op), *case.op_csc(op), f"{name}/{op} (library tensors)")


@pytest.mark.parametrize("name", sorted(CASES))
def test_bsr_export_matches_reference(name, ld):
    """Block CSR of A: block rows in reference order, the reference's block pattern,
    N x N row-major blocks whose entries equal the reference's (zeros where it stores none)."""
    s, case, mesh = _pair(name, ld)
    n = s.n
    rp, ci, blocks = s.operator_bsr("A")
    r, c, v = case.op("A")
    ref_blocks = {}
    for rr, cc, vv in zip(r // n, c // n, np.arange(len(v))):
        ref_blocks.setdefault((int(rr), int(cc)), []).append(vv)
    assert rp[-1] == len(ref_blocks) == len(ci)
    scale = np.abs(v).max()
    for b in range(3 * s.num_t):
        cols = ci[rp[b]:rp[b + 1]]
        assert np.all(np.diff(cols) > 0)
        for q, col in enumerate(cols):
            idx = ref_blocks[(b, int(col))]
            ref = np.zeros((n, n))
            ref[r[idx] % n, c[idx] % n] = v[idx]
            assert np.abs(blocks[rp[b] + q] - ref).max() <= 1e-12 * scale


@pytest.mark.parametrize("name", ["fk16_p2", "jitter12_p3", "fk8_p4"])
def test_per_operator_entry_points_with_caller_d(name, ld):
    """assemble_dphi_phi_coeff / assemble_edge_avg_coeff_nu with a random caller D
    (not the projection of d): same CSC arrays as the reference's functions."""
    s, case, mesh = _pair(name, ld)
    D = np.random.default_rng(5).uniform(-1.0, 2.0, (s.num_t, s.n))
    case.assemble_with_d(D)
    g1, g2 = s.assemble_dphi_phi_coeff(D)
    for dev, ref in ((g1, "ug1"), (g2, "ug2")):
        _same_csc(dev, *case.op_csc(ref), f"{name}/{ref}")
    for m in (1, 2):
        r, rd = s.assemble_edge_avg_coeff_nu(m, D)
        _same_csc(r, *case.op_csc(f"ur{m}"), f"{name}/ur{m}")
        _same_csc(rd, *case.op_csc(f"urd{m}"), f"{name}/urd{m}")
    # the handle's own assembly is untouched
    cp, ri, v = case.op_csc("g1")
    _same_csc(s.operator_csc("g1"), cp, ri, v, f"{name}/g1 after")
    with pytest.raises(ValueError):
        s.assemble_edge_avg_coeff_nu(3, D)


def test_cpp_mirror_build_blocks_returns_reference_csc(ld, tmp_path):
    """tools/ldg_blocks: SystemBlocks{A, V} = build_blocks(t) and the per-operator
    calls through paper_1408_3877_b200/host/ldg_host.hpp, against the reference."""
    R = _reflib()
    exe = os.path.join(ROOT, "tools", "ldg_blocks")
    assert os.path.exists(exe), "build() must produce tools/ldg_blocks"
    dim, p = 12, 2
    mesh = R.RefMesh.square(1.0 / dim)
    case = R.RefCase(mesh, O.local_dof_count(p), 1.0, BASE, MIXED)
    case.assemble(T_OPS)
    D = np.random.default_rng(9).uniform(0.5, 1.5, mesh.num_t * O.local_dof_count(p))
    dfile = tmp_path / "d.bin"
    D.tofile(dfile)
    rt = R.ref_tensors(O.local_dof_count(p))
    rtfile = tmp_path / "rt.bin"
    np.concatenate([rt[k] for k in ("m", "h", "g", "sd", "so")]).tofile(rtfile)
    pre = str(tmp_path / "out")
    res = subprocess.run([exe, str(dim), str(p), repr(T_OPS), pre, str(dfile), str(rtfile)], capture_output=True,
                         text=True, timeout=300)
    assert res.returncode == 0, res.stderr

    def load(name):
        import scipy.sparse as sp

        cp = np.fromfile(f"{pre}.{name}.outer.i32", np.int32)
        ri = np.fromfile(f"{pre}.{name}.inner.i32", np.int32)
        v = np.fromfile(f"{pre}.{name}.values.f64", np.float64)
        return sp.csc_matrix((v, ri, cp), shape=(len(cp) - 1, len(cp) - 1))

    _same_csc(load("A"), *case.op_csc("A"), "C++ build_blocks A")
    Vref = case.vec("V")
    assert np.abs(np.fromfile(f"{pre}.V.f64") - Vref).max() <= 1e-12 * np.abs(Vref).max()
    case.assemble_with_d(D)
    for dev, ref in (("G1", "ug1"), ("G2", "ug2"), ("R1", "ur1"), ("RD1", "urd1"), ("R2", "ur2"), ("RD2", "urd2")):
        _same_csc(load(dev), *case.op_csc(ref), f"C++ {dev}")
