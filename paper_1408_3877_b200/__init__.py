"""B200-native LDG diffusion path (arXiv 1408.3877, FESTUNG Part I).

Python host mirror of the reference's entry points (proj/include/ldg), bound
through ctypes to the C ABI of include/ldg_b200.h (libldg_b200.so, built
in-tree by __graft_entry__.build()).  There is no CPU fallback: every call
runs the sm_100a kernels, and loading fails loudly when the library or a GPU
is missing.

Reference interface -> this module
  generate_grid_data / domain_square   LdgSystem.from_mesh / LdgSystem.square
  LdgSystem(mesh, spec, rt) ctor       ditto (static operators, selectors)
  project(mesh, f, t, q_ord, rt)       LdgSystem.project
  build_blocks(t)                      LdgSystem.build_blocks / assemble
  assemble_* operators                 LdgSystem.operator(name)
  initial_state / euler_step           LdgSystem.initial_state / euler_step
  solve_stationary                     LdgSystem.solve_stationary
  l2_error / to_lagrange (fields.hpp)  LdgSystem.l2_error / to_lagrange
  write_vtu (vtkout.hpp)               LdgSystem.write_vtu
Exceptions follow the reference: ValueError for std::invalid_argument,
MeshError for ldg::MeshError, RuntimeError for solver failures.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["FN", "ProblemSpec", "LdgSystem", "MeshError", "SolverOptions", "library_path", "load_library",
           "OPERATORS", "VECTORS", "BASELINE_SPEC"]

HERE = os.path.dirname(os.path.abspath(__file__))


def library_path() -> str:
    # LDG_B200_LIB: an alternative build of the same library (kernel-tuning
    # experiments in scripts/); the in-tree build otherwise
    return os.environ.get("LDG_B200_LIB") or os.path.join(HERE, "libldg_b200.so")


class MeshError(RuntimeError):
    """ldg::MeshError (mesh.hpp:25-27)."""


# coefficient ids of include/ldg_b200_coeffs.h
FN = dict(zero=0, const=1, poly=2, exp_sum=3, cos7x1_x2=4, mms_exact=5, mms_f=6, mms_gn=7, base_c=8, base_d=9,
          base_f=10, base_gn=11, sin_x1x2=12, cos3x1_plus_x2=13, mms_z1=14, mms_z2=15, sin3x1_x2sq=16,
          exp_x1_minus_x2=17)

OPERATORS = ["mass", "h1", "h2", "g1", "g2", "r1", "rd1", "r2", "rd2", "q1", "qn1", "q2", "qn2", "s", "sd", "A"]
VECTORS = ["D", "F", "jd1", "jd2", "kd", "kn", "l", "V", "Y"]


class _Coeff(C.Structure):
    _fields_ = [("id", C.c_int), ("p", C.c_double * 4)]


class _Problem(C.Structure):
    _fields_ = [("d", _Coeff), ("f", _Coeff), ("c_d", _Coeff), ("g_n", _Coeff), ("c0", _Coeff),
                ("eta", C.c_double), ("n_bc", C.c_int), ("bc_id", C.c_int * 16), ("bc_kind", C.c_int * 16)]


class _Opts(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("maxit", C.c_int), ("precond", C.c_int),
                ("check_residual", C.c_int), ("contract_tol", C.c_double), ("krylov", C.c_int),
                ("restart", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("applies", C.c_int), ("schur_relres", C.c_double),
                ("residual", C.c_double), ("ms_assemble", C.c_double), ("ms_solve", C.c_double),
                ("ms_setup", C.c_double), ("ms_krylov", C.c_double)]


class _Info(C.Structure):
    _fields_ = [("p", C.c_int), ("n_local", C.c_int), ("num_t", C.c_int), ("num_owned", C.c_int),
                ("num_ghost", C.c_int), ("num_v", C.c_int), ("rank", C.c_int), ("size", C.c_int),
                ("bytes_device", C.c_int64), ("launches", C.c_int64)]


class _Times(C.Structure):
    _fields_ = [("ms_project", C.c_double), ("ms_assemble", C.c_double), ("ms_spmv", C.c_double),
                ("ms_schur", C.c_double), ("reps", C.c_int), ("levels", C.c_int), ("ms_vcycle", C.c_double),
                ("ms_level", C.c_double * 8), ("ms_sweep_s2", C.c_double), ("s2_per_vcycle", C.c_int)]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_int64)
_H = C.c_void_p
_lib = None

# The C ABI: name -> (restype, argtypes).  tests/test_capi.py checks that the
# library exports exactly what include/ldg_b200.h declares.
_SIGNATURES = {
    "ldg_reference_tensors": (C.c_int, [C.c_int] + [_dp] * 7),
    "ldg_rank_form_supported": (C.c_int, [C.c_int] + [_dp] * 5 + [C.POINTER(C.c_int)]),
    "ldg_set_device": (C.c_int, [C.c_int]),
    "ldg_set_reference_tensors": (C.c_int, [_H] + [_dp] * 7),
    "ldg_create": (C.c_int, [_dp, C.c_int, _ip, C.c_int, _ip, C.c_int, C.POINTER(_Problem), C.POINTER(_H)]),
    "ldg_create_square": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_int, C.POINTER(_Problem),
                                    C.POINTER(_H)]),
    "ldg_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "ldg_create_square_dist": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_int, C.POINTER(_Problem), C.c_int,
                                         C.c_int, C.c_char_p, C.POINTER(_H)]),
    "ldg_create_square_group": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_int, C.POINTER(_Problem), C.c_int,
                                          C.POINTER(_H)]),
    "ldg_destroy": (None, [_H]),
    "ldg_last_error": (C.c_char_p, [_H]),
    "ldg_get_info": (C.c_int, [_H, C.POINTER(_Info)]),
    "ldg_mesh_lists": (C.c_int, [_H, _dp, _ip, _dp, _dp, _dp, _dp, _ip, _ip, _ip]),
    "ldg_project": (C.c_int, [_H, C.POINTER(_Coeff), C.c_double, C.c_int, _dp]),
    "ldg_assemble": (C.c_int, [_H, C.c_double]),
    "ldg_assemble_blocks": (C.c_int, [_H, C.c_double, _dp]),
    "ldg_export_operator": (C.c_int, [_H, C.c_int, _lp, _lp, _lp, _dp, C.c_int64]),
    "ldg_export_vector": (C.c_int, [_H, C.c_int, _dp, C.c_int64]),
    "ldg_export_operator_csc": (C.c_int, [_H, C.c_int, _lp, _ip, _ip, _dp, C.c_int64]),
    "ldg_export_operator_bsr": (C.c_int, [_H, C.c_int, _lp, _ip, _ip, _dp, C.c_int64]),
    "ldg_assemble_dphi_phi_coeff": (C.c_int, [_H, _dp, C.c_int, _lp, _ip, _ip, _dp, C.c_int64]),
    "ldg_assemble_edge_avg_coeff_nu": (C.c_int, [_H, _dp, C.c_int, C.c_int, _lp, _ip, _ip, _dp, C.c_int64]),
    "ldg_initial_state": (C.c_int, [_H]),
    "ldg_set_state": (C.c_int, [_H, _dp, C.c_double]),
    "ldg_get_state": (C.c_int, [_H, _dp, _dp]),
    "ldg_default_solver_opts": (_Opts, []),
    "ldg_euler_steps": (C.c_int, [_H, C.c_double, C.c_int, C.POINTER(_Opts), C.POINTER(_Stats)]),
    "ldg_euler_steps_host": (C.c_int, [_H, C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_void_p,
                                       C.POINTER(_Opts), C.POINTER(_Stats), _dp]),
    "ldg_solve_stationary": (C.c_int, [_H, C.c_double, C.POINTER(_Opts), C.POINTER(_Stats)]),
    "ldg_l2_error": (C.c_int, [_H, C.c_int, C.POINTER(_Coeff), C.c_double, C.c_int, _dp]),
    "ldg_to_lagrange": (C.c_int, [_H, C.c_int, _dp, C.POINTER(C.c_int)]),
    "ldg_write_vtu": (C.c_int, [_H, C.c_int, C.c_char_p, C.c_char_p, C.c_int, C.c_char_p, C.c_int]),
    "ldg_apply_lhs": (C.c_int, [_H, C.c_double, _dp, _dp]),
    "ldg_apply_schur": (C.c_int, [_H, C.c_double, _dp, _dp]),
    "ldg_time_kernels": (C.c_int, [_H, C.c_double, C.c_double, C.c_int, C.c_int, C.POINTER(_Times)]),
    "ldg_sync": (C.c_int, [_H]),
}


def load_library():
    """Loads libldg_b200.so (no fallback: raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not os.path.exists(path):
        raise ImportError(f"libldg_b200.so not built ({path}); run __graft_entry__.build() — "
                          "the LDG path has no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def rank_form_supported(n_local: int, tensors: dict | None = None) -> bool:
    """Host-only: may the operator kernels use the rank-Q_e edge form with these reference
    tensors (None: the library's own)?  See ldg_rank_form_supported in include/ldg_b200.h."""
    lib = load_library()
    ok = C.c_int(-1)
    if tensors is None:
        args = [None] * 5
    else:
        keep = [np.ascontiguousarray(tensors[k], dtype=np.float64).ravel() for k in ("m", "h", "g", "sd", "so")]
        args = [a.ctypes.data_as(_dp) for a in keep]
    rc = lib.ldg_rank_form_supported(int(n_local), *args, C.byref(ok))
    _raise(rc, lib.ldg_last_error(None).decode())
    return bool(ok.value)


def reference_tensors(n_local: int) -> dict:
    """The library's host-built reference tensors (build_ref_tensors, reftensors.hpp:55); no GPU needed."""
    n = int(n_local)
    arrs = dict(m=np.zeros(n * n), h=np.zeros(n * n * 2), g=np.zeros(n ** 3 * 2), sd=np.zeros(n * n * 3),
                so=np.zeros(n * n * 9), rd=np.zeros(n ** 3 * 3), ro=np.zeros(n ** 3 * 9))
    lib = load_library()
    rc = lib.ldg_reference_tensors(n, *[arrs[k].ctypes.data_as(_dp) for k in ("m", "h", "g", "sd", "so", "rd",
                                                                             "ro")])
    _raise(rc, lib.ldg_last_error(None).decode())
    return arrs


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, every rank passes it to square_dist)."""
    lib = load_library()
    buf = C.create_string_buffer(128)
    _raise(lib.ldg_nccl_unique_id(buf), lib.ldg_last_error(None).decode())
    return buf.raw


def set_device(device: int) -> None:
    """cudaSetDevice in the library's runtime (one process per GPU)."""
    lib = load_library()
    _raise(lib.ldg_set_device(int(device)), lib.ldg_last_error(None).decode())


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _coeff(fn) -> _Coeff:
    if isinstance(fn, (str, int)):
        fn = (fn, [])
    fid, params = fn
    if isinstance(fid, str):
        fid = FN[fid]
    c = _Coeff()
    c.id = int(fid)
    for i, v in enumerate(list(params)[:4]):
        c.p[i] = float(v)
    return c


@dataclass
class ProblemSpec:
    """ProblemSpec (system.hpp:26-37); coefficients are (id, params) or names of FN."""
    d: object = ("const", [1.0])
    f: object = "zero"
    c_d: object = "zero"
    g_n: object = "zero"
    c0: object = "zero"
    eta: float = 1.0
    boundary: dict = field(default_factory=dict)  # id -> "D" | "N"
    t_end: float = 1.0
    num_steps: int = 1

    def to_c(self) -> _Problem:
        pr = _Problem()
        pr.d, pr.f, pr.c_d, pr.g_n, pr.c0 = (_coeff(x) for x in (self.d, self.f, self.c_d, self.g_n, self.c0))
        pr.eta = float(self.eta)
        if len(self.boundary) > 16:
            raise ValueError("too many boundary conditions")
        pr.n_bc = len(self.boundary)
        for i, (bid, kind) in enumerate(sorted(self.boundary.items())):
            pr.bc_id[i] = int(bid)
            pr.bc_kind[i] = 0 if kind in ("D", "dirichlet", 0) else 1
        return pr


# The BASELINE.json problem: c = cos7x1 cos7x2 + e^-t,
# d = e^(x1+x2)(1 + 0.5 sin t), f derived, Dirichlet everywhere.
BASELINE_SPEC = ProblemSpec(d="base_d", f="base_f", c_d="base_c", g_n="base_gn", c0="base_c", eta=1.0,
                            boundary={1: "D", 2: "D", 3: "D", 4: "D"})


@dataclass
class SolverOptions:
    rtol: float = 1e-14  # ldg_default_solver_opts(): relative Schur residual (states within 1e-10 of the reference)
    atol: float = 0.0
    maxit: int = 20000
    precond: int = 2  # 0 none, 1 block-Jacobi, 2 geometric multigrid (p-coarsened, FK meshes; else 1)
    check_residual: bool = True
    contract_tol: float = 1e-10
    krylov: int = 0  # 0 FGMRES(restart), 1 BiCGStab
    restart: int = 30

    def to_c(self) -> _Opts:
        o = _Opts()
        o.rtol, o.atol, o.maxit, o.precond = self.rtol, self.atol, self.maxit, self.precond
        o.check_residual, o.contract_tol = int(self.check_residual), self.contract_tol
        o.krylov, o.restart = self.krylov, self.restart
        return o


def _raise(rc: int, msg: str):
    if rc == 0:
        return
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise MeshError(msg)
    raise RuntimeError(msg)


class LdgSystem:
    """Device-resident LdgSystem (system.hpp:65-213) of one GPU."""

    def __init__(self, handle, spec: ProblemSpec, p: int):
        self._h = handle
        self.spec = spec
        self.p = p
        info = self.info()
        self.num_t = info["num_t"]
        self.n = info["n_local"]
        self.t = 0.0

    # ---- construction --------------------------------------------------
    @classmethod
    def square(cls, dim: int, p: int, spec: ProblemSpec, jitter: float = 0.0, seed: int = 0) -> "LdgSystem":
        lib = load_library()
        h = _H()
        pr = spec.to_c()
        rc = lib.ldg_create_square(int(dim), float(jitter), int(seed), int(p), C.byref(pr), C.byref(h))
        _raise(rc, lib.ldg_last_error(None).decode())
        return cls(h, spec, p)

    @classmethod
    def square_group(cls, dim: int, p: int, spec: ProblemSpec, nranks: int, jitter: float = 0.0,
                     seed: int = 0) -> "LdgSystem":
        """The strip decomposition with all `nranks` ranks on this GPU (virtual ranks)."""
        lib = load_library()
        h = _H()
        pr = spec.to_c()
        rc = lib.ldg_create_square_group(int(dim), float(jitter), int(seed), int(p), C.byref(pr), int(nranks),
                                         C.byref(h))
        _raise(rc, lib.ldg_last_error(None).decode())
        return cls(h, spec, p)

    @classmethod
    def square_dist(cls, dim: int, p: int, spec: ProblemSpec, rank: int, size: int, nccl_id: bytes | None,
                    jitter: float = 0.0, seed: int = 0) -> "LdgSystem":
        """Rank `rank` of `size` (one process per GPU, NCCL halos and allreduce)."""
        lib = load_library()
        h = _H()
        pr = spec.to_c()
        rc = lib.ldg_create_square_dist(int(dim), float(jitter), int(seed), int(p), C.byref(pr), int(rank),
                                        int(size), nccl_id, C.byref(h))
        _raise(rc, lib.ldg_last_error(None).decode())
        return cls(h, spec, p)

    @classmethod
    def from_mesh(cls, coords, v0t, p: int, spec: ProblemSpec, id_e0t=None) -> "LdgSystem":
        lib = load_library()
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        v0t = np.ascontiguousarray(v0t, dtype=np.int32)
        ids = None if id_e0t is None else np.ascontiguousarray(id_e0t, dtype=np.int32)
        h = _H()
        pr = spec.to_c()
        rc = lib.ldg_create(_d(coords), coords.shape[0], _i(v0t), v0t.shape[0], None if ids is None else _i(ids),
                            int(p), C.byref(pr), C.byref(h))
        _raise(rc, lib.ldg_last_error(None).decode())
        return cls(h, spec, p)

    def close(self):
        if getattr(self, "_h", None):
            load_library().ldg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != 0:
            _raise(rc, load_library().ldg_last_error(self._h).decode())

    # ---- info -----------------------------------------------------------
    def info(self) -> dict:
        inf = _Info()
        self._check(load_library().ldg_get_info(self._h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in _Info._fields_}

    @property
    def block_dim(self) -> int:
        return self.num_t * self.n

    def mesh_lists(self) -> dict:
        K, V = self.num_t, self.info()["num_v"]
        out = dict(coords=np.zeros((V, 2)), v0t=np.zeros((K, 3), np.int32), b=np.zeros((K, 4)), area=np.zeros(K),
                   len=np.zeros((K, 3)), nu=np.zeros((K, 3, 2)), nbr=np.zeros((K, 3), np.int32),
                   nbr_n=np.zeros((K, 3), np.int32), id_e0t=np.zeros((K, 3), np.int32))
        self._check(load_library().ldg_mesh_lists(self._h, _d(out["coords"]), _i(out["v0t"]), _d(out["b"]),
                                                  _d(out["area"]), _d(out["len"]), _d(out["nu"]),
                                                  _i(out["nbr"]), _i(out["nbr_n"]), _i(out["id_e0t"])))
        return out

    # ---- per-step path --------------------------------------------------
    def project(self, fn, t: float, q_ord: int | None = None) -> np.ndarray:
        """project(mesh, func, t, q_ord, rt) (fields.hpp:53-82) -> K x N."""
        if q_ord is None:
            q_ord = max(2 * self.p, 1)
        out = np.zeros(self.num_t * self.n)
        c = _coeff(fn)
        self._check(load_library().ldg_project(self._h, C.byref(c), float(t), int(q_ord), _d(out)))
        return out.reshape(self.num_t, self.n)

    def assemble(self, t: float):
        """The device half of build_blocks(t) (system.hpp:110-152)."""
        self._check(load_library().ldg_assemble(self._h, float(t)))

    def assemble_blocks(self, t: float) -> float:
        """All 8 time-dependent C-row blocks per element as the reference assembles
        them, with the projection of d, f and the right-hand side (BASELINE config 3);
        returns the device time in ms."""
        ms = C.c_double()
        self._check(load_library().ldg_assemble_blocks(self._h, float(t), C.byref(ms)))
        return ms.value

    def operator(self, name: str):
        """COO (rows, cols, vals) of one operator at the last assemble time."""
        which = OPERATORS.index(name)
        lib = load_library()
        nnz = C.c_int64()
        self._check(lib.ldg_export_operator(self._h, which, C.byref(nnz), None, None, None, 0))
        r, c, v = np.zeros(nnz.value, np.int64), np.zeros(nnz.value, np.int64), np.zeros(nnz.value)
        self._check(lib.ldg_export_operator(self._h, which, C.byref(nnz), r.ctypes.data_as(_lp),
                                            c.ctypes.data_as(_lp), _d(v), nnz.value))
        return r, c, v

    def set_reference_tensors(self, rt: dict):
        """The caller's RefTensors (the rt of LdgSystem(mesh, spec, rt), system.hpp:67):
        dict with m, h, g, sd, so (and optionally rd, ro) in the reference layout."""
        arrs = {k: np.ascontiguousarray(rt[k], dtype=np.float64) for k in ("m", "h", "g", "sd", "so")}
        opt = {k: (np.ascontiguousarray(rt[k], dtype=np.float64) if k in rt else None) for k in ("rd", "ro")}
        self._check(load_library().ldg_set_reference_tensors(
            self._h, *[_d(arrs[k]) for k in ("m", "h", "g", "sd", "so")],
            *[(_d(opt[k]) if opt[k] is not None else None) for k in ("rd", "ro")]))

    def _csc_call(self, n: int, call):
        """Two-phase CSC export: call(nnz, colptr, rowind, vals, cap) -> scipy csc_matrix."""
        import scipy.sparse as sp

        nnz = C.c_int64()
        self._check(call(C.byref(nnz), None, None, None, 0))
        cp = np.zeros(n + 1, np.int32)
        ri, v = np.zeros(nnz.value, np.int32), np.zeros(nnz.value)
        self._check(call(C.byref(nnz), _i(cp), _i(ri), _d(v), nnz.value))
        return sp.csc_matrix((v, ri, cp), shape=(n, n))

    def operator_csc(self, name: str):
        """An operator in the reference's storage (Eigen CSC, assembly.hpp:21-22)
        as a scipy csc_matrix with the same colptr / rowind / values."""
        which = OPERATORS.index(name)
        n = (3 if name == "A" else 1) * self.block_dim
        lib = load_library()
        return self._csc_call(n, lambda *a: lib.ldg_export_operator_csc(self._h, which, *a))

    def operator_bsr(self, name: str):
        """(rowptr, colind, blocks[nb, N, N]) block CSR in reference element order."""
        which = OPERATORS.index(name)
        nbr = (3 if name == "A" else 1) * self.num_t
        lib = load_library()
        nb = C.c_int64()
        self._check(lib.ldg_export_operator_bsr(self._h, which, C.byref(nb), None, None, None, 0))
        rp, ci = np.zeros(nbr + 1, np.int32), np.zeros(nb.value, np.int32)
        v = np.zeros(nb.value * self.n * self.n)
        self._check(lib.ldg_export_operator_bsr(self._h, which, C.byref(nb), _i(rp), _i(ci), _d(v), nb.value))
        return rp, ci, v.reshape(nb.value, self.n, self.n)

    def assemble_dphi_phi_coeff(self, d_disc):
        """(G^1, G^2) = assemble_dphi_phi_coeff(mesh, rt, d_disc) (assembly.hpp:113-136)
        for a caller's K x N coefficient matrix; scipy CSC."""
        d = np.ascontiguousarray(d_disc, dtype=np.float64).reshape(-1)
        if d.size != self.block_dim:
            raise ValueError("coefficient matrix shape mismatch")
        lib = load_library()
        return tuple(self._csc_call(self.block_dim, lambda *a, m=m: lib.ldg_assemble_dphi_phi_coeff(
            self._h, _d(d), m, *a)) for m in (1, 2))

    def assemble_edge_avg_coeff_nu(self, m: int, d_disc):
        """(R^m, R_D^m) = assemble_edge_avg_coeff_nu(mesh, m, d_disc, sel_int, sel_dir, rt)
        (assembly.hpp:214-252); scipy CSC."""
        d = np.ascontiguousarray(d_disc, dtype=np.float64).reshape(-1)
        if d.size != self.block_dim:
            raise ValueError("coefficient matrix shape mismatch")
        lib = load_library()
        return tuple(self._csc_call(self.block_dim, lambda *a, w=w: lib.ldg_assemble_edge_avg_coeff_nu(
            self._h, _d(d), int(m), w, *a)) for w in (0, 1))

    def vector(self, name: str) -> np.ndarray:
        which = VECTORS.index(name)
        n = (3 if name in ("V", "Y") else 1) * self.block_dim
        out = np.zeros(n)
        self._check(load_library().ldg_export_vector(self._h, which, _d(out), n))
        return out

    def build_blocks(self, t: float):
        """SystemBlocks (A, V) of system.hpp:110-152: A (3KN x 3KN) in the reference's
        CSC storage (scipy csc_matrix), V the stacked right-hand side."""
        self.assemble(t)
        return self.operator_csc("A"), self.vector("V")

    def initial_state(self):
        """system.hpp:99-107 -> (y, t)."""
        self._check(load_library().ldg_initial_state(self._h))
        self.t = 0.0
        return self.get_state()

    def set_state(self, y, t: float):
        y = np.ascontiguousarray(y, dtype=np.float64)
        if y.size != 3 * self.block_dim:
            raise ValueError("state length does not match 3*K*N")
        self._check(load_library().ldg_set_state(self._h, _d(y), float(t)))
        self.t = float(t)

    def get_state(self):
        y = np.zeros(3 * self.block_dim)
        t = C.c_double()
        self._check(load_library().ldg_get_state(self._h, _d(y), C.byref(t)))
        return y, t.value

    def euler_steps(self, dt: float, nsteps: int, opts: SolverOptions | None = None) -> dict:
        """nsteps implicit Euler steps on the device-resident state (system.hpp:155-174)."""
        o = (opts or SolverOptions()).to_c()
        st = _Stats()
        self._check(load_library().ldg_euler_steps(self._h, float(dt), int(nsteps), C.byref(o), C.byref(st)))
        self.t = self.get_time()
        return {k: getattr(st, k) for k, _ in _Stats._fields_}

    def get_time(self) -> float:
        t = C.c_double()
        self._check(load_library().ldg_get_state(self._h, None, C.byref(t)))
        return t.value

    def euler_step(self, y, t: float, dt: float, opts: SolverOptions | None = None):
        """SystemState euler_step(state, dt) with host vectors -> (y_next, t_next)."""
        self.set_state(y, t)
        self.euler_steps(dt, 1, opts)
        return self.get_state()

    def euler_steps_host(self, y_in_ptr: int, t: float, dt: float, nsteps: int, y_out_ptr: int,
                         opts: SolverOptions | None = None) -> dict:
        """Host-buffer euler_step through the C ABI (copies inside; device-timed).
        y_in_ptr / y_out_ptr are host addresses of 3KN doubles (k-major), ideally pinned."""
        o = (opts or SolverOptions()).to_c()
        st = _Stats()
        ms = C.c_double()
        self._check(load_library().ldg_euler_steps_host(self._h, C.c_void_p(y_in_ptr), float(t), float(dt),
                                                        int(nsteps), C.c_void_p(y_out_ptr), C.byref(o),
                                                        C.byref(st), C.byref(ms)))
        self.t = float(t) + nsteps * float(dt)
        out = {k: getattr(st, k) for k, _ in _Stats._fields_}
        out["ms_total"] = ms.value
        return out

    def solve_stationary(self, t: float = 0.0, opts: SolverOptions | None = None):
        """system.hpp:177-185 -> (c, z1, z2) as K x N."""
        o = (opts or SolverOptions()).to_c()
        st = _Stats()
        self._check(load_library().ldg_solve_stationary(self._h, float(t), C.byref(o), C.byref(st)))
        y, _ = self.get_state()
        kn = self.block_dim
        K, n = self.num_t, self.n
        self.last_stats = {k: getattr(st, k) for k, _ in _Stats._fields_}
        return y[2 * kn:].reshape(K, n), y[:kn].reshape(K, n), y[kn:2 * kn].reshape(K, n)

    _COMPONENTS = dict(z1=0, z2=1, c=2)

    def l2_error(self, exact, t: float, q_ord: int, component: str = "c") -> float:
        """l2_error(mesh, dof, exact, t, q_ord) (fields.hpp:100-123) of a component
        of the device-resident state ('c', 'z1' or 'z2')."""
        err = C.c_double()
        c = _coeff(exact)
        self._check(load_library().ldg_l2_error(self._h, self._COMPONENTS[component], C.byref(c), float(t),
                                                int(q_ord), C.byref(err)))
        return err.value

    def write_vtu(self, component: str = "c", var_name: str = "u", basename: str = "out", t_lvl: int = 0) -> str:
        """write_vtu (vtkout.hpp:42-108) of a state component from the device;
        returns the path `<basename>.<t_lvl>.vtu`."""
        buf = C.create_string_buffer(4096)
        self._check(load_library().ldg_write_vtu(self._h, self._COMPONENTS[component], var_name.encode(),
                                                 basename.encode(), int(t_lvl), buf, 4096))
        return buf.value.decode()

    def to_lagrange(self, component: str = "c") -> np.ndarray:
        """to_lagrange(dof) (fields.hpp:87-97) of a state component -> K x 3 (p <= 1) or K x 6."""
        m = 3 if self.p <= 1 else 6
        out = np.zeros(self.num_t * m)
        nodes = C.c_int()
        self._check(load_library().ldg_to_lagrange(self._h, self._COMPONENTS[component], _d(out), C.byref(nodes)))
        assert nodes.value == m
        return out.reshape(self.num_t, m)

    def apply_lhs(self, dt: float, x) -> np.ndarray:
        """(W + dt A) x with the operators of the last assemble."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        self._check(load_library().ldg_apply_lhs(self._h, float(dt), _d(x), _d(y)))
        return y

    def apply_schur(self, dt: float, c) -> np.ndarray:
        """S_c c = [M + dt(eta(S + S_D) - sum_m E^m M^-1 B^m)] c (KN vector) with the
        operators of the last assemble: the Krylov solve's operator."""
        c = np.ascontiguousarray(c, dtype=np.float64)
        if c.size != self.block_dim:
            raise ValueError("vector length does not match K*N")
        y = np.zeros_like(c)
        self._check(load_library().ldg_apply_schur(self._h, float(dt), _d(c), _d(y)))
        return y

    def time_kernels(self, t: float, dt: float, reps: int = 10, flush: bool = True) -> dict:
        tm = _Times()
        self._check(load_library().ldg_time_kernels(self._h, float(t), float(dt), int(reps), int(flush),
                                                    C.byref(tm)))
        out = {k: getattr(tm, k) for k, _ in _Times._fields_}
        out["ms_level"] = list(tm.ms_level)[: tm.levels]
        return out

    def sync(self):
        self._check(load_library().ldg_sync(self._h))
