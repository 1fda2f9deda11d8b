"""TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/_ref/libldgref.so.

libldgref.so is the UNMODIFIED reference (/root/reference/proj/include/ldg)
compiled against the in-repo Eigen/doctest shims (oracle/Makefile).  This
module exposes it to tests/, tests/golden generation and bench.py's
reference arm.  Its SparseLU stand-in is SciPy's SuperLU (installed as the
shim's solver hook), so the reference's `solve_checked` (system.hpp:190-205)
runs a supernodal sparse LU like Eigen's SparseLU does.  The product package
never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libldgref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_SOLVER = C.CFUNCTYPE(C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _dp, _dp)

_lib = None
_hook = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _scipy_solver(n, nnz, colptr, rowind, values, rhs, x):
    try:
        import scipy.sparse as sp
        import scipy.sparse.linalg as spla

        cp = np.ctypeslib.as_array(colptr, shape=(n + 1,)).copy()
        ri = np.ctypeslib.as_array(rowind, shape=(nnz,)).copy()
        va = np.ctypeslib.as_array(values, shape=(nnz,)).copy()
        b = np.ctypeslib.as_array(rhs, shape=(n,)).copy()
        a = sp.csc_matrix((va, ri, cp), shape=(n, n))
        sol = spla.splu(a, permc_spec="COLAMD").solve(b)
        out = np.ctypeslib.as_array(x, shape=(n,))
        out[:] = sol
        return 0
    except Exception:  # pragma: no cover - reported as a factorization failure
        return 1


def lib():
    global _lib, _hook
    if _lib is not None:
        return _lib
    if not available():
        raise RuntimeError(f"reference oracle library missing: {LIB_PATH} (run `make -C oracle`)")
    L = C.CDLL(LIB_PATH)
    L.ldgref_last_error.restype = C.c_char_p
    L.ldgref_set_sparse_solver.argtypes = [_SOLVER]
    L.ldgref_mesh_square.restype = C.c_void_p
    L.ldgref_mesh_square.argtypes = [C.c_double]
    L.ldgref_mesh_create.restype = C.c_void_p
    L.ldgref_mesh_create.argtypes = [C.c_int, _dp, C.c_int, _ip, _ip]
    L.ldgref_mesh_refine.restype = C.c_void_p
    L.ldgref_mesh_refine.argtypes = [C.c_void_p]
    L.ldgref_mesh_free.argtypes = [C.c_void_p]
    L.ldgref_mesh_sizes.argtypes = [C.c_void_p, _ip, _ip, _ip]
    L.ldgref_mesh_lists.argtypes = [C.c_void_p, _dp, _ip, _dp, _dp, _dp, _dp, _ip, _ip, _ip]
    L.ldgref_ref_tensors.argtypes = [C.c_int] + [_dp] * 7
    L.ldgref_quad_rule_2d.argtypes = [C.c_int, _dp, _dp, _dp, C.c_int]
    L.ldgref_quad_rule_1d.argtypes = [C.c_int, _dp, _dp, C.c_int]
    L.ldgref_project.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_double, C.c_int, _dp]
    L.ldgref_l2_error.restype = C.c_double
    L.ldgref_l2_error.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, _dp, C.c_double, C.c_int]
    L.ldgref_case_create.restype = C.c_void_p
    L.ldgref_case_create.argtypes = [C.c_void_p, C.c_int, C.c_double, _ip, _dp, _ip, _ip, C.c_int]
    L.ldgref_case_free.argtypes = [C.c_void_p]
    L.ldgref_case_assemble.argtypes = [C.c_void_p, C.c_double]
    L.ldgref_case_assemble_with_d.argtypes = [C.c_void_p, _dp]
    L.ldgref_case_op.restype = C.c_long
    L.ldgref_case_op.argtypes = [C.c_void_p, C.c_char_p, _ip, _ip, _dp]
    L.ldgref_case_vec.restype = C.c_long
    L.ldgref_case_vec.argtypes = [C.c_void_p, C.c_char_p, _dp]
    L.ldgref_case_initial_state.argtypes = [C.c_void_p, _dp]
    L.ldgref_case_euler.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, _dp]
    L.ldgref_case_time_build.argtypes = [C.c_void_p, C.c_double, C.c_int, _dp]
    L.ldgref_case_solve_stationary.argtypes = [C.c_void_p, C.c_double, _dp, _dp, _dp]
    L.ldgref_run_convergence.argtypes = [_ip, C.c_int, C.c_int, _dp]
    _hook = _SOLVER(_scipy_solver)
    L.ldgref_set_sparse_solver(_hook)
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        raise RuntimeError(lib().ldgref_last_error().decode())


class RefMesh:
    """Reference `Mesh` (mesh.hpp:35-98) held by the oracle library."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError(lib().ldgref_last_error().decode())
        self.h = handle
        nt, ne, nv = C.c_int(), C.c_int(), C.c_int()
        lib().ldgref_mesh_sizes(self.h, C.byref(nt), C.byref(ne), C.byref(nv))
        self.num_t, self.num_e, self.num_v = nt.value, ne.value, nv.value

    @classmethod
    def square(cls, h_max: float) -> "RefMesh":
        return cls(lib().ldgref_mesh_square(h_max))

    @classmethod
    def create(cls, coords, v0t, id_e0t=None) -> "RefMesh":
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        v0t = np.ascontiguousarray(v0t, dtype=np.int32)
        ids = None if id_e0t is None else np.ascontiguousarray(id_e0t, dtype=np.int32)
        return cls(lib().ldgref_mesh_create(coords.shape[0], _d(coords), v0t.shape[0], _i(v0t),
                                            None if ids is None else _i(ids)))

    def refine(self) -> "RefMesh":
        return RefMesh(lib().ldgref_mesh_refine(self.h))

    def lists(self) -> dict:
        K, V = self.num_t, self.num_v
        out = dict(coords=np.zeros((V, 2)), v0t=np.zeros((K, 3), np.int32), b=np.zeros((K, 4)),
                   area=np.zeros(K), len=np.zeros((K, 3)), nu=np.zeros((K, 3, 2)),
                   nbr=np.zeros((K, 3), np.int32), nbr_n=np.zeros((K, 3), np.int32),
                   id_e0t=np.zeros((K, 3), np.int32))
        lib().ldgref_mesh_lists(self.h, _d(out["coords"]), _i(out["v0t"]), _d(out["b"]), _d(out["area"]),
                                _d(out["len"]), _d(out["nu"]), _i(out["nbr"]), _i(out["nbr_n"]),
                                _i(out["id_e0t"]))
        return out

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ldgref_mesh_free(self.h)
            self.h = None


def write_vtu(h_max: float, lagrange, var_name: str, basename: str, t_lvl: int) -> str:
    """The reference's write_vtu (vtkout.hpp:42-108) on domain_square(h_max),
    run as oracle/_ref/ref_vtu (its iostreams cannot share this process with
    numpy's libstdc++)."""
    import subprocess
    import tempfile

    lag = np.ascontiguousarray(lagrange, dtype=np.float64)
    with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as f:
        f.write(lag.tobytes())
        path = f.name
    try:
        res = subprocess.run([os.path.join(HERE, "_ref", "ref_vtu"), repr(float(h_max)), str(lag.shape[1]), path,
                              var_name, basename, str(int(t_lvl))], capture_output=True, text=True, check=True)
    finally:
        os.unlink(path)
    return res.stdout.strip()


def ref_tensors(n: int) -> dict:
    arrs = dict(m=np.zeros(n * n), h=np.zeros(n * n * 2), g=np.zeros(n ** 3 * 2), sd=np.zeros(n * n * 3),
                so=np.zeros(n * n * 9), rd=np.zeros(n ** 3 * 3), ro=np.zeros(n ** 3 * 9))
    _check(lib().ldgref_ref_tensors(n, *[_d(arrs[k]) for k in ("m", "h", "g", "sd", "so", "rd", "ro")]))
    return arrs


def quad_rule_2d(q_ord: int):
    x1, x2, w = np.zeros(256), np.zeros(256), np.zeros(256)
    n = lib().ldgref_quad_rule_2d(q_ord, _d(x1), _d(x2), _d(w), 256)
    return np.stack([x1[:n], x2[:n]], 1), w[:n]


def quad_rule_1d(q_ord: int):
    s, w = np.zeros(64), np.zeros(64)
    n = lib().ldgref_quad_rule_1d(q_ord, _d(s), _d(w), 64)
    if n < 0:
        raise ValueError(lib().ldgref_last_error().decode())
    return s[:n], w[:n]


def _fn(fn):
    fid, p = fn
    arr = np.zeros(4)
    arr[: len(p)] = p
    return int(fid), arr


def project(mesh: RefMesh, n_local: int, fn, t: float, q_ord: int) -> np.ndarray:
    fid, p = _fn(fn)
    out = np.zeros(mesh.num_t * n_local)
    _check(lib().ldgref_project(mesh.h, n_local, fid, _d(p), t, q_ord, _d(out)))
    return out


def l2_error(mesh: RefMesh, n_local: int, dof_kmajor, fn, t: float, q_ord: int) -> float:
    fid, p = _fn(fn)
    dof = np.ascontiguousarray(dof_kmajor, dtype=np.float64)
    return lib().ldgref_l2_error(mesh.h, n_local, _d(dof), fid, _d(p), t, q_ord)


class RefCase:
    """Reference `LdgSystem` (system.hpp:65-213) plus every assembled operator."""

    def __init__(self, mesh: RefMesh, n_local: int, eta: float, funcs, boundary: dict):
        self.mesh, self.n = mesh, n_local
        ids = np.zeros(5, np.int32)
        ps = np.zeros(20)
        for i, key in enumerate(("d", "f", "c_d", "g_n", "c0")):
            fid, p = _fn(funcs[key])
            ids[i], ps[4 * i:4 * i + 4] = fid, p
        bc_ids = np.array(list(boundary.keys()), np.int32)
        bc_kinds = np.array([0 if v in ("D", "dirichlet", 0) else 1 for v in boundary.values()], np.int32)
        self.h = lib().ldgref_case_create(mesh.h, n_local, eta, _i(ids), _d(ps), _i(bc_ids), _i(bc_kinds),
                                          len(bc_ids))
        if not self.h:
            raise RuntimeError(lib().ldgref_last_error().decode())

    def assemble(self, t: float):
        _check(lib().ldgref_case_assemble(self.h, t))

    def assemble_with_d(self, d_kmajor):
        """assemble_dphi_phi_coeff / assemble_edge_avg_coeff_nu (m = 1, 2) for a
        caller's D (K x N, k-major): operators "ug1", "ug2", "ur1", "urd1", "ur2", "urd2"."""
        d = np.ascontiguousarray(d_kmajor, dtype=np.float64).reshape(-1)
        _check(lib().ldgref_case_assemble_with_d(self.h, _d(d)))

    def op_csc(self, name: str):
        """(colptr, rowind, values) of an operator exactly as the reference stores it."""
        r, c, v = self.op(name)
        n = self.mesh.num_t * self.n * (3 if name == "A" else 1)
        colptr = np.zeros(n + 1, np.int64)
        np.add.at(colptr, c.astype(np.int64) + 1, 1)
        return np.cumsum(colptr), r, v

    def op(self, name: str):
        """Returns (rows, cols, vals) in CSC order."""
        nnz = lib().ldgref_case_op(self.h, name.encode(), None, None, None)
        if nnz < 0:
            raise KeyError(lib().ldgref_last_error().decode())
        r, c, v = np.zeros(nnz, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz)
        lib().ldgref_case_op(self.h, name.encode(), _i(r), _i(c), _d(v))
        return r, c, v

    def vec(self, name: str) -> np.ndarray:
        n = lib().ldgref_case_vec(self.h, name.encode(), None)
        if n < 0:
            raise KeyError(lib().ldgref_last_error().decode())
        out = np.zeros(n)
        lib().ldgref_case_vec(self.h, name.encode(), _d(out))
        return out

    def initial_state(self) -> np.ndarray:
        y = np.zeros(3 * self.mesh.num_t * self.n)
        _check(lib().ldgref_case_initial_state(self.h, _d(y)))
        return y

    def euler(self, y, t: float, dt: float, steps: int = 1):
        y = np.array(y, dtype=np.float64, copy=True)
        tt = np.array([t], dtype=np.float64)
        sec = np.zeros(1)
        _check(lib().ldgref_case_euler(self.h, _d(y), _d(tt), dt, steps, _d(sec)))
        return y, float(tt[0]), float(sec[0])

    def time_build(self, t: float, reps: int = 1) -> float:
        sec = np.zeros(1)
        _check(lib().ldgref_case_time_build(self.h, t, reps, _d(sec)))
        return float(sec[0])

    def solve_stationary(self, t: float = 0.0):
        kn = self.mesh.num_t * self.n
        c, z1, z2 = np.zeros(kn), np.zeros(kn), np.zeros(kn)
        _check(lib().ldgref_case_solve_stationary(self.h, t, _d(c), _d(z1), _d(z2)))
        return c, z1, z2

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ldgref_case_free(self.h)
            self.h = None


def run_convergence(orders, j_max: int) -> np.ndarray:
    o = np.ascontiguousarray(orders, dtype=np.int32)
    rows = np.zeros(6 * len(o) * (j_max + 1))
    _check(lib().ldgref_run_convergence(_i(o), len(o), j_max, _d(rows)))
    return rows.reshape(-1, 6)
