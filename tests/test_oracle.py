"""CPU oracle (oracle/ldg_oracle.py) pinned against the reference.

Two pins: (1) known-answer values and properties restated from the
reference's own unit tests (proj/tests/test_*.cpp), and (2) the golden
fixtures in tests/golden, produced by the unmodified reference compiled
against the Eigen shim (tests/golden/make_golden.py).  No GPU needed.
"""
from __future__ import annotations

import os

import math

import numpy as np
import pytest

from ldg_testutil import CASES, coo, op_rel_err, spec_from_golden, vec_rel_err
from oracle import ldg_oracle as O


# ----------------------------------------------------------------- known answers

def test_basis_orthonormal_and_gradients():
    """test_basis.cpp: orthonormality at full order; acceptance criterion 7 (FD gradients)."""
    pts, w = O.quad_rule_2d(8)
    phi = O.phi_table(15, pts[:, 0], pts[:, 1])
    gram = np.einsum("r,ri,rj->ij", w, phi, phi)
    assert np.abs(gram - np.eye(15)).max() < 1e-12
    rng = np.random.default_rng(2024)
    h = 1e-6
    x1 = rng.uniform(0.05, 0.95, 200)
    x2 = rng.uniform(0.05, 0.95, 200) * (1.0 - x1)
    for i in range(1, 16):
        fd1 = (O.basis_fn(i, x1 + h, x2) - O.basis_fn(i, x1 - h, x2)) / (2 * h)
        fd2 = (O.basis_fn(i, x1, x2 + h) - O.basis_fn(i, x1, x2 - h)) / (2 * h)
        assert np.abs(fd1 - O.basis_grad(i, 1, x1, x2)).max() < 1e-5
        assert np.abs(fd2 - O.basis_grad(i, 2, x1, x2)).max() < 1e-5
    assert float(O.basis_fn(2, 1.0, 0.0)) == pytest.approx(-4.0)
    assert float(O.basis_grad(6, 2, 0.0, 0.0)) == pytest.approx(-12.0 * math.sqrt(5.0))
    with pytest.raises(IndexError):
        O.basis_fn(16, 0.0, 0.0)


def test_quadrature_exact_positive_interior():
    """acceptance.cpp:109-156 (criterion 3)."""
    for o in range(18):
        s, w = O.quad_rule_1d(o)
        assert np.all(w > 0) and np.all((s > 0) & (s < 1))
        order = 2 * s.size - 1
        for a in range(order + 1):
            assert abs(np.sum(w * s ** a) * (a + 1) - 1.0) < 1e-12
    for o in range(13):
        pts, w = O.quad_rule_2d(o)
        assert np.all(w > 0) and np.all(pts > 0) and np.all(pts.sum(1) < 1)
        for a in range(max(o, 1) + 1):
            for b in range(max(o, 1) + 1 - a):
                exact = math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
                assert abs(np.sum(w * pts[:, 0] ** a * pts[:, 1] ** b) - exact) <= 1e-12 * exact
    with pytest.raises(ValueError):
        O.quad_rule_1d(18)


def test_theta_maps_involution():
    """acceptance criterion 8: edge maps are involutions that reverse orientation."""
    for nm in range(1, 4):
        for npl in range(1, 4):
            s = np.linspace(0, 1, 20)
            x = O.gamma_map(nm, s)
            y = O.theta_map(npl, nm, O.theta_map(nm, npl, x))
            assert np.abs(y - x).max() < 1e-15
            assert np.abs(O.theta_map(nm, npl, O.gamma_map(nm, 0.0)) - O.gamma_map(npl, 1.0)).max() < 1e-15


def test_reference_tensor_spot_values():
    """test_reftensors.cpp:9-41"""
    for n in (1, 3, 6, 10, 15):
        assert np.abs(O.build_ref_tensors(n).m_hat - np.eye(n)).max() < 1e-12
    t1 = O.build_ref_tensors(1)
    assert np.all(t1.g_hat == 0.0) and np.all(t1.h_hat == 0.0)
    assert t1.s_diag[0, 0, :] == pytest.approx([2.0] * 3, rel=1e-14)
    assert t1.r_diag[0, 0, 0, :] == pytest.approx([2.0 * math.sqrt(2.0)] * 3, rel=1e-14)
    assert np.allclose(t1.r_offdiag[0, 0, 0], 2.0 * math.sqrt(2.0), rtol=1e-14)
    t3 = O.build_ref_tensors(3)
    assert t3.h_hat[1, 0, 0] == pytest.approx(-3.0 * math.sqrt(2.0), rel=1e-13)


def two_triangle():
    s3 = math.sqrt(3.0)
    m = O.generate_grid_data([[0.0, -1.0], [s3, 0.0], [0.0, 1.0], [-s3, 0.0]], [[3, 0, 2], [0, 1, 2]])
    bnd = m.t0e[:, 1] == -1
    m.id_e[bnd] = np.where(m.bary_e[bnd, 1] < 0.0, 1, 2)
    m.sync_edge_ids()
    return m


def test_assembly_spot_values():
    """test_assembly.cpp:34-109"""
    two = two_triangle()
    rt = O.build_ref_tensors(1)
    mass = O.assemble_mass(two, rt).toarray()
    assert mass[0, 0] == pytest.approx(2.0 * math.sqrt(3.0), rel=1e-14)
    si, sb = O.select_interior(two), O.select_boundary(two, {1, 2})
    s, sd = O.assemble_edge_jump(two, si, sb, rt)
    assert np.abs(s.toarray() - np.array([[2.0, -2.0], [-2.0, 2.0]])).max() < 1e-13
    assert np.abs(sd.toarray() - np.diag([4.0, 4.0])).max() < 1e-13
    q1, qn1 = O.assemble_edge_avg_nu(two, 1, si, np.zeros_like(si), rt)
    assert np.abs(q1.toarray() - np.array([[2.0, 2.0], [-2.0, -2.0]])).max() < 1e-13
    q2, _ = O.assemble_edge_avg_nu(two, 2, si, np.zeros_like(si), rt)
    assert np.abs(q2.toarray()).max() < 1e-13
    assert qn1.nnz == 0 or np.abs(qn1.toarray()).max() == 0.0

    tri = O.generate_grid_data([[0.0, 0.0], [2.0, 0.0], [0.0, 2.0]], [[0, 1, 2]])
    south = np.array([[abs(tri.bary_e[tri.e0t[0, n], 1]) < 1e-12 for n in range(3)]])
    one = O.coeff((1, [1.0]))
    j1, j2 = O.assemble_vec_dirichlet_nu(tri, south, one, 0.0, 1)
    assert abs(j1[0]) < 1e-14 and j2[0] == pytest.approx(-2.0 * math.sqrt(2.0), rel=1e-14)
    kd = O.assemble_vec_dirichlet(tri, np.array([[False, True, True]]), one, 0.0, 1)
    assert kd[0] == pytest.approx(2.0 * math.sqrt(2.0), rel=1e-13)
    kn = O.assemble_vec_neumann(tri, south, np.array([[1.0 / math.sqrt(2.0)]]), one, 0.0, 1)
    assert kn[0] == pytest.approx(2.0 * math.sqrt(2.0), rel=1e-13)


def test_coefficient_linearity():
    """test_assembly.cpp:111-134: d = 0 -> G = 0; d = 1 -> G = H and R^1 = Q^1."""
    sq = O.domain_square(0.5)
    for n in (3, 6):
        rt = O.build_ref_tensors(n)
        si, sdir = O.select_interior(sq), O.select_boundary(sq, {2, 4})
        g1, g2 = O.assemble_dphi_phi_coeff(sq, rt, np.zeros((sq.num_t, n)))
        assert np.abs(g1.toarray()).max() == 0.0 and np.abs(g2.toarray()).max() == 0.0
        one = np.zeros((sq.num_t, n))
        one[:, 0] = 1.0 / math.sqrt(2.0)
        g1, g2 = O.assemble_dphi_phi_coeff(sq, rt, one)
        h1, h2 = O.assemble_dphi_phi(sq, rt)
        assert np.abs((g1 - h1).toarray()).max() < 1e-12 and np.abs((g2 - h2).toarray()).max() < 1e-12
        r1, _ = O.assemble_edge_avg_coeff_nu(sq, 1, one, si, sdir, rt)
        q1, _ = O.assemble_edge_avg_nu(sq, 1, si, np.zeros_like(si), rt)
        assert np.abs((r1 - q1).toarray()).max() < 1e-12


def test_system_properties():
    """test_system.cpp: zero data, eta scaling, flux decoupling, polynomial consistency, fixed point."""
    sq = O.domain_square(0.5)
    zero_b = {1: "D", 2: "D", 3: "D", 4: "D"}
    rt3 = O.build_ref_tensors(3)
    spec = O.ProblemSpec(d=(1, [1.0]), boundary=zero_b)
    c, z1, z2 = O.LdgSystem(sq, spec, rt3).solve_stationary()
    assert max(np.abs(c).max(), np.abs(z1).max(), np.abs(z2).max()) < 1e-12
    with pytest.raises(ValueError):
        O.LdgSystem(sq, O.ProblemSpec(boundary={1: "D", 2: "D", 4: "D"}), rt3)
    with pytest.raises(ValueError):
        O.LdgSystem(sq, O.ProblemSpec(eta=0.0, boundary=zero_b), rt3)
    s1 = O.LdgSystem(sq, O.ProblemSpec(d=(1, [1.0]), c_d=(2, [0.0, 1.0, 1.0]), boundary=zero_b), rt3)
    s2 = O.LdgSystem(sq, O.ProblemSpec(d=(1, [1.0]), c_d=(2, [0.0, 1.0, 1.0]), eta=2.0, boundary=zero_b), rt3)
    a1, v1 = s1.build_blocks(0.0)
    a2, v2 = s2.build_blocks(0.0)
    kn = s1.block_dim
    diff = (a2 - a1).toarray()
    assert np.abs(diff[: 2 * kn]).max() < 1e-14
    assert np.abs(diff[2 * kn:, 2 * kn:] - a1.toarray()[2 * kn:, 2 * kn:]).max() < 1e-12
    assert np.abs(v2[2 * kn:] - 2.0 * v1[2 * kn:]).max() < 1e-12
    A = a1.toarray()
    assert np.abs(A[:kn, kn:2 * kn]).max() == 0.0 and np.abs(A[kn:2 * kn, :kn]).max() == 0.0
    exact = O.coeff((2, [1.0, 1.0, 1.0]))
    for p in (1, 2, 3, 4):
        rt = O.build_ref_tensors(O.local_dof_count(p))
        s = O.LdgSystem(sq, O.ProblemSpec(d=(1, [1.0]), c_d=(2, [1.0, 1.0, 1.0]), boundary=zero_b), rt)
        c, z1, z2 = s.solve_stationary()
        assert O.l2_error(sq, c, exact, 0.0, 2 * p + 2) < 1e-9
        assert O.l2_error(sq, z1, O.coeff((1, [-1.0])), 0.0, 2 * p + 2) < 1e-9
    rt = O.build_ref_tensors(6)
    s = O.LdgSystem(sq, O.ProblemSpec(d=(1, [1.0]), c_d=(2, [1.0, 1.0, 1.0]), c0=(2, [1.0, 1.0, 1.0]),
                                      boundary=zero_b), rt)
    c, z1, z2 = s.solve_stationary()
    y = np.concatenate([z1.ravel(), z2.ravel(), c.ravel()])
    y1, _ = s.euler_step(y, 0.0, 0.1)
    assert np.abs(y1 - y).max() < 1e-9


def test_mass_conservation_neumann():
    """test_system.cpp:125-156 / acceptance criterion 6."""
    sq = O.domain_square(0.5)
    rt = O.build_ref_tensors(3)
    spec = O.ProblemSpec(d=(12, []), c0=(13, []), boundary={1: "N", 2: "N", 3: "N", 4: "N"})
    s = O.LdgSystem(sq, spec, rt)
    y, t = s.initial_state()
    ones = np.zeros((sq.num_t, 3))
    ones[:, 0] = 1.0 / math.sqrt(2.0)
    ones = ones.ravel()
    kn = s.block_dim
    prev = ones @ (s.mass @ y[2 * kn:])
    for _ in range(10):
        y, t = s.euler_step(y, t, 0.05)
        now = ones @ (s.mass @ y[2 * kn:])
        assert abs(now - prev) < 1e-11 * abs(prev)
        prev = now


# ----------------------------------------------------------------- golden pins

def test_tensors_and_rules_match_golden(golden):
    g = golden("tensors")
    for n in (1, 3, 6, 10, 15):
        t = O.build_ref_tensors(n)
        for key, arr in (("m", t.m_hat), ("h", t.h_hat), ("g", t.g_hat), ("sd", t.s_diag), ("so", t.s_offdiag),
                         ("rd", t.r_diag), ("ro", t.r_offdiag)):
            assert np.abs(arr.ravel() - g[f"N{n}_{key}"]).max() < 1e-14, (n, key)
    for o in range(13):
        pts, w = O.quad_rule_2d(o)
        np.testing.assert_array_equal(pts, g[f"rule2d_{o}_x"])
        np.testing.assert_array_equal(w, g[f"rule2d_{o}_w"])
    for o in range(18):
        s, w = O.quad_rule_1d(o)
        np.testing.assert_array_equal(s, g[f"rule1d_{o}_s"])
        np.testing.assert_array_equal(w, g[f"rule1d_{o}_w"])


def _oracle_system(g):
    funcs, boundary = spec_from_golden(g)
    m = O.generate_grid_data(g["coords"], g["v0t"])
    bnd = m.t0e[m.e0t, 1] == -1
    ids = np.where(bnd, g["id_in"], 0)
    for k in range(m.num_t):
        for n in range(3):
            if bnd[k, n]:
                m.id_e[m.e0t[k, n]] = ids[k, n]
    m.sync_edge_ids()
    spec = O.ProblemSpec(**funcs, eta=1.0, boundary=boundary)
    return m, O.LdgSystem(m, spec, O.build_ref_tensors(int(g["n_local"])))


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_golden(case, golden):
    g = golden(case)
    m, s = _oracle_system(g)
    np.testing.assert_array_equal(m.b.reshape(-1, 4), g["mesh_b"])
    np.testing.assert_array_equal(m.area_t, g["mesh_area"])
    np.testing.assert_array_equal(m.nbr, g["mesh_nbr"])
    np.testing.assert_array_equal(m.nbr_n, g["mesh_nbr_n"])
    assert np.abs(m.nu_e0t - g["mesh_nu"]).max() <= 2e-16
    t = float(g["t_ops"])
    ops = s.build_operators(t)
    A, V = s.build_blocks(t)
    ops["A"] = A
    kn = s.block_dim
    for name in sorted({k[3:-2] for k in g if k.startswith("op_") and k.endswith("_r")}):
        n = 3 * kn if name == "A" else kn
        ref = coo(g[f"op_{name}_r"], g[f"op_{name}_c"], g[f"op_{name}_v"], n)
        assert op_rel_err(ops[name].tocsr(), ref) <= 1e-13, name
    for name in ("jd1", "jd2", "kd", "kn", "l"):
        assert vec_rel_err(np.ravel(ops[name]), g[f"vec_{name}"]) <= 1e-13, name
    assert vec_rel_err(np.ravel(ops["D"]), g["vec_D"]) <= 1e-13
    assert vec_rel_err(V, g["vec_V"]) <= 1e-13
    y0, _ = s.initial_state()
    assert vec_rel_err(y0, g["y0"]) <= 1e-13


@pytest.mark.parametrize("case", ["c1_fk16_p1", "jitter8_p2", "fk8_p0"])
def test_oracle_euler_matches_golden(case, golden):
    g = golden(case)
    _, s = _oracle_system(g)
    y, t = s.initial_state()
    dt = float(g["dt"])
    steps = sorted(int(k[1:]) for k in g if k.startswith("y") and k[1:].isdigit() and k != "y0")
    last = min(steps[-1], 10)
    for i in range(1, last + 1):
        y, t = s.euler_step(y, t, dt)
        if i in steps:
            ref = g[f"y{i}"]
            assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 1e-12


@pytest.mark.parametrize("case", ["c1_fk16_p1", "jitter8_p2", "fk8_p0", "fk8_p3", "fk6_p4"])
def test_oracle_schur_euler_matches_reference_lu(case, golden):
    """The exact block-elimination solve (euler_step_schur, the 64^2 parity
    oracle) reproduces the reference's SparseLU states (golden fixtures)."""
    g = golden(case)
    _, s = _oracle_system(g)
    y, t = s.initial_state()
    dt = float(g["dt"])
    steps = sorted(int(k[1:]) for k in g if k.startswith("y") and k[1:].isdigit() and k != "y0")
    last = min(steps[-1], 10)
    for i in range(1, last + 1):
        y, t = s.euler_step_schur(y, t, dt)
        if i in steps:
            ref = g[f"y{i}"]
            assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 1e-12


def test_jitter_generator_matches_golden(golden):
    g = golden("jitter8_p2")
    np.testing.assert_array_equal(O.fk_jittered_coords(8, 0.2, 0), g["coords"])


def test_convergence_ladder_matches_golden(golden):
    """convergence.hpp:77-103 on p = 0..2, j <= 2 (the reference rows pin j <= 3)."""
    ref = golden("convergence")["rows"]
    rows = np.array(O.run_convergence([0, 1, 2], 2))
    for r in rows:
        match = ref[(ref[:, 0] == r[0]) & (ref[:, 1] == r[1])][0]
        assert r[3] == match[3]
        assert abs(r[4] - match[4]) <= 1e-9 * match[4]
    # order (p+1) on the finest pinned level (acceptance.cpp:77-93 thresholds at j = 3)
    fin = ref[(ref[:, 1] == 3) & (ref[:, 0] >= 2)]
    for p, alpha in zip(fin[:, 0], fin[:, 5]):
        assert abs(alpha - (p + 1.0)) <= 0.25, (p, alpha)


@pytest.mark.parametrize("h_max,m", [(0.25, 3), (0.5, 6), (1.0 / 3.0, 6)])
def test_write_vtu_restatement_matches_reference(h_max, m, tmp_path):
    """The oracle's write_vtu (vtkout.hpp:42-108) writes the reference's file
    byte for byte (the reference writer runs as oracle/_ref/ref_vtu)."""
    from oracle import reflib as R

    if not os.path.exists(os.path.join(os.path.dirname(R.LIB_PATH), "ref_vtu")):
        pytest.skip("oracle/_ref/ref_vtu not built (make -C oracle)")
    mesh = O.domain_square(h_max)
    rng = np.random.default_rng(7)
    lag = rng.standard_normal((mesh.num_t, m)) * 10.0 ** rng.integers(-6, 6, (mesh.num_t, m))
    a = R.write_vtu(h_max, lag, "c", str(tmp_path / "ref"), 2)
    b = O.write_vtu(mesh, lag, "c", str(tmp_path / "ora"), 2)
    assert open(a).read() == open(b).read()


@pytest.mark.parametrize("p", range(5))
def test_edge_tensors_are_rank_qe_quadrature_sums(p):
    """The identities behind the rank-Q_e operator and smoother kernels,
    on the restated reference tensors (pinned to the reference's above): with the
    Q_e = (3p + 2) // 2 point Gauss rule on the edge, U_n[q, i] = phi_i(gamma_n(s_q)) and
    V_{n,np}[q, j] = phi_j(theta_{n,np}(gamma_n(s_q))),
        s_diag[:, :, n] = U_n^T W U_n,   s_offdiag[:, :, n, np] = U_n^T W V_{n,np},
    the neighbour's trace points are this element's in reverse order, and h_hat[i, j, m]
    vanishes unless deg phi_i > deg phi_j (hierarchical modal basis)."""
    n = O.local_dof_count(p)
    rt = O.build_ref_tensors(n)
    q = (3 * p + 2) // 2
    s, w = O.gauss_legendre_unit(q)
    assert np.allclose(s[::-1], 1.0 - s, atol=1e-15)
    tol = 1e-13 * max(1.0, np.abs(rt.s_diag).max())
    for nm in range(1, 4):
        g = O.gamma_map(nm, s)
        U = O.phi_table(n, g[:, 0], g[:, 1])
        assert np.abs(np.einsum("r,ri,rj->ij", w, U, U) - rt.s_diag[:, :, nm - 1]).max() <= tol
        for np_ in range(1, 4):
            th = O.theta_map(nm, np_, g)
            V = O.phi_table(n, th[:, 0], th[:, 1])
            assert np.abs(np.einsum("r,ri,rj->ij", w, U, V) - rt.s_offdiag[:, :, nm - 1, np_ - 1]).max() <= tol
            # the same physical points seen from the neighbour's edge np, reversed
            gn = O.gamma_map(np_, s[::-1])
            assert np.abs(O.phi_table(n, gn[:, 0], gn[:, 1]) - V).max() <= tol
    deg = [d for d in range(p + 1) for _ in range(d + 1)]
    for i in range(n):
        for j in range(n):
            if deg[i] <= deg[j]:
                assert np.abs(rt.h_hat[i, j, :]).max() <= tol, (i, j)
