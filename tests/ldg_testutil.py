"""Shared helpers for the parity tests (comparison on the union pattern)."""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

CASES = ["two_tri_N1", "two_tri_N3", "two_tri_N6", "square2_N3", "square2_N6", "square2_N10", "c1_fk16_p1",
         "jitter8_p2", "fk6_p4", "fk8_p0", "fk8_p3"]

N_TO_P = {1: 0, 3: 1, 6: 2, 10: 3, 15: 4}


def coo(r, c, v, n):
    return sp.coo_matrix((v, (np.asarray(r, np.int64), np.asarray(c, np.int64))), shape=(n, n)).tocsr()


def op_rel_err(a, b) -> float:
    """max|a - b| / max|b| on the union pattern (SURVEY.md §8d parity criterion);
    absolute when the reference operator is identically zero."""
    d = (a - b).tocsr()
    err = np.abs(d.data).max() if d.nnz else 0.0
    scale = np.abs(b.data).max() if b.nnz else 0.0
    return err / scale if scale > 0 else err


def vec_rel_err(a, b) -> float:
    scale = np.abs(b).max()
    err = np.abs(a - b).max() if a.size else 0.0
    return err / scale if scale > 0 else err


def spec_from_golden(g: dict):
    """(d, f, c_d, g_n, c0) coefficient tuples and the boundary map stored in a fixture."""
    funcs = {}
    for key in ("d", "f", "c_d", "g_n", "c0"):
        a = g[f"fn_{key}"]
        funcs[key] = (int(a[0]), [float(x) for x in a[1:5]])
    boundary = {int(i): ("D" if int(k) == 0 else "N") for i, k in zip(g["bc_ids"], g["bc_kinds"])}
    return funcs, boundary
