"""Generates tests/golden/*.npz from the UNMODIFIED reference.

Run in the build container (needs /root/reference and oracle/_ref/libldgref.so,
built by `make -C oracle`):  python tests/golden/make_golden.py
The fixtures are small (<= a few MB) and committed; the GPU box never reads
/root/reference.  Each file records the reference outputs of one case:
mesh lists, reference tensors, every operator of build_blocks (COO, CSC
order), the per-step vectors, and states after implicit-Euler steps.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ldg_oracle as O  # noqa: E402
from oracle import reflib as R  # noqa: E402

OPS = ["mass", "h1", "h2", "g1", "g2", "r1", "rd1", "r2", "rd2", "q1", "qn1", "q2", "qn2", "s", "sd", "A"]
VECS = ["D", "F", "jd1", "jd2", "kd", "kn", "l", "V"]

# coefficient sets: (d, f, c_d, g_n, c0)
TEST_FUNCS = dict(d=(3, []), f=(4, []), c_d=(2, [1.0, 1.0, -2.0]), g_n=(2, [0.0, 0.0, 1.0]), c0=(5, []))
BASE_FUNCS = dict(d=(9, []), f=(10, []), c_d=(8, []), g_n=(11, []), c0=(8, []))


def two_triangle():
    """test_assembly.cpp:16-26 (IDs by the sign of the edge barycentre)."""
    s3 = np.sqrt(3.0)
    coords = np.array([[0.0, -1.0], [s3, 0.0], [0.0, 1.0], [-s3, 0.0]])
    v0t = np.array([[3, 0, 2], [0, 1, 2]], np.int32)
    ids = np.zeros((2, 3), np.int32)
    for k in range(2):
        for n in range(3):
            a, b = coords[v0t[k, (n + 1) % 3]], coords[v0t[k, (n + 2) % 3]]
            ids[k, n] = 1 if 0.5 * (a[1] + b[1]) < 0.0 else 2
    return coords, v0t, ids


def square_ids(coords, v0t):
    """domain_square boundary IDs (mesh.hpp:245-252) per (k, n)."""
    K = v0t.shape[0]
    ids = np.zeros((K, 3), np.int32)
    for n in range(3):
        a, b = coords[v0t[:, (n + 1) % 3]], coords[v0t[:, (n + 2) % 3]]
        mx, my = 0.5 * (a[:, 0] + b[:, 0]), 0.5 * (a[:, 1] + b[:, 1])
        tol = 1e-12
        i = np.zeros(K, np.int32)
        i = np.where(np.abs(my) < tol, 1, i)
        i = np.where((i == 0) & (np.abs(mx - 1.0) < tol), 2, i)
        i = np.where((i == 0) & (np.abs(my - 1.0) < tol), 3, i)
        i = np.where((i == 0) & (np.abs(mx) < tol), 4, i)
        ids[:, n] = i
    return ids


def dump_case(name, mesh, coords, v0t, ids, n_local, funcs, boundary, t_ops, steps=(), dt=0.0, ops=OPS):
    out = dict(n_local=n_local, t_ops=t_ops, dt=dt, coords=coords, v0t=v0t, id_in=ids,
               bc_ids=np.array(list(boundary.keys()), np.int32),
               bc_kinds=np.array([0 if v == "D" else 1 for v in boundary.values()], np.int32))
    for key in ("d", "f", "c_d", "g_n", "c0"):
        fid, p = funcs[key]
        out[f"fn_{key}"] = np.array([fid] + list(p) + [0.0] * (4 - len(p)), np.float64)
    L = mesh.lists()
    for k in ("b", "area", "len", "nu", "nbr", "nbr_n", "id_e0t"):
        out[f"mesh_{k}"] = L[k]
    case = R.RefCase(mesh, n_local, 1.0, funcs, boundary)
    case.assemble(t_ops)
    for op in ops:
        r, c, v = case.op(op)
        out[f"op_{op}_r"], out[f"op_{op}_c"], out[f"op_{op}_v"] = r, c, v
    for vec in VECS:
        out[f"vec_{vec}"] = case.vec(vec)
    y = case.initial_state()
    out["y0"] = y
    t = 0.0
    done = 0
    for s in steps:
        y, t, _ = case.euler(y, t, dt, s - done)
        done = s
        out[f"y{s}"] = y
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "K", mesh.num_t, "keys", len(out))


def main():
    # reference tensors and rules
    tens = {}
    for n in (1, 3, 6, 10, 15):
        for k, v in R.ref_tensors(n).items():
            tens[f"N{n}_{k}"] = v
    for o in range(0, 13):
        pts, w = R.quad_rule_2d(o)
        tens[f"rule2d_{o}_x"], tens[f"rule2d_{o}_w"] = pts, w
    for o in range(0, 18):
        s, w = R.quad_rule_1d(o)
        tens[f"rule1d_{o}_s"], tens[f"rule1d_{o}_w"] = s, w
    np.savez_compressed(os.path.join(HERE, "tensors.npz"), **tens)
    print("tensors", len(tens))

    coords, v0t, ids = two_triangle()
    for n in (1, 3, 6):
        mesh = R.RefMesh.create(coords, v0t, ids)
        dump_case(f"two_tri_N{n}", mesh, coords, v0t, ids, n, TEST_FUNCS, {1: "D", 2: "N"}, 0.0)

    c2, t2 = O.fk_lists(2)
    for n in (3, 6, 10):
        mesh = R.RefMesh.square(0.5)
        dump_case(f"square2_N{n}", mesh, c2, t2, square_ids(c2, t2), n, TEST_FUNCS,
                  {1: "N", 2: "D", 3: "N", 4: "D"}, 0.0)

    # BASELINE config 1 (CPU-runnable): 16x16 FK, p = 1, all Dirichlet, dt = 0.01, 100 steps
    c16, t16 = O.fk_lists(16)
    mesh = R.RefMesh.square(1.0 / 16.0)
    dump_case("c1_fk16_p1", mesh, c16, t16, square_ids(c16, t16), 3, BASE_FUNCS,
              {1: "D", 2: "D", 3: "D", 4: "D"}, 0.01, steps=(1, 10, 100), dt=0.01, ops=["A"])

    # config-4 style: jittered 8x8 FK, p = 2, Dirichlet on x1=0 / x2=0, Neumann elsewhere
    cj = O.fk_jittered_coords(8, 0.2, 0)
    _, tj = O.fk_lists(8)
    idj = square_ids(cj, tj)
    mesh = R.RefMesh.create(cj, tj, idj)
    dump_case("jitter8_p2", mesh, cj, tj, idj, 6, BASE_FUNCS, {1: "D", 2: "N", 3: "N", 4: "D"}, 0.1,
              steps=(1, 5), dt=0.1, ops=["A", "g1", "r2", "rd1", "qn2", "s", "sd", "q1"])

    # p = 4 on a 6x6 FK mesh
    c6, t6 = O.fk_lists(6)
    mesh = R.RefMesh.square(1.0 / 6.0)
    dump_case("fk6_p4", mesh, c6, t6, square_ids(c6, t6), 15, BASE_FUNCS, {1: "D", 2: "D", 3: "D", 4: "D"},
              0.05, steps=(1, 3), dt=0.05, ops=["A", "g2", "r1", "rd2"])

    # p = 0 and p = 3 on 8x8
    c8, t8 = O.fk_lists(8)
    for n, tag in ((1, "p0"), (10, "p3")):
        mesh = R.RefMesh.square(1.0 / 8.0)
        dump_case(f"fk8_{tag}", mesh, c8, t8, square_ids(c8, t8), n, BASE_FUNCS,
                  {1: "D", 2: "N", 3: "N", 4: "D"}, 0.2, steps=(2,), dt=0.1, ops=["A"])

    # stationary manufactured problem and the convergence ladder (convergence.hpp:77-103)
    rows = R.run_convergence([0, 1, 2, 3], 3)
    np.savez_compressed(os.path.join(HERE, "convergence.npz"), rows=rows)
    print("convergence rows", rows.shape)
    mesh = R.RefMesh.square(1.0 / 3.0).refine()
    L = mesh.lists()
    mms = dict(d=(3, []), f=(6, []), c_d=(5, []), g_n=(7, []), c0=(5, []))
    case = R.RefCase(mesh, 6, 1.0, mms, {1: "N", 2: "D", 3: "N", 4: "D"})
    c, z1, z2 = case.solve_stationary(0.0)
    np.savez_compressed(os.path.join(HERE, "stationary_mms_p2.npz"), coords=L["coords"], v0t=L["v0t"],
                        id_in=L["id_e0t"], c=c, z1=z1, z2=z2)
    print("stationary", c.shape)


if __name__ == "__main__":
    main()
