"""Host-side plan of the strip decomposition of Friedrichs-Keller meshes
 — the Python statement of what the library's
build_square_strip / halo / mg_depth do in C++ (csrc/ldg_mesh.cu,
ldg_team.cu, ldg_mg.cu), used by bench.py to size multi-GPU runs and by the
CPU (gloo) tests of the distributed algorithm.

FK(dim) (mesh.hpp:225-254) numbers all lower triangles (ix, iy) as
ix*dim + iy, then all upper ones as dim^2 + ix*dim + iy.  Rank r of `size`
owns element columns [a, b) = [r*dim//size, (r+1)*dim//size): in reference
numbering two contiguous ranges.  Lower (a, iy) touches upper (a-1, iy) and
upper (b-1, iy) touches lower (b, iy); every other neighbour is in the same
column, so one ghost column per side closes the stencil.
"""
from __future__ import annotations

import math

import numpy as np


def strip_bounds(dim: int, size: int, rank: int) -> tuple[int, int]:
    return rank * dim // size, (rank + 1) * dim // size


def local_elements(dim: int, a: int, b: int) -> np.ndarray:
    """Global element ids in the library's local order: owned lowers,
    owned uppers, ghost uppers of column a-1, ghost lowers of column b."""
    iy = np.arange(dim)
    cols = np.arange(a, b)
    lowers = (cols[:, None] * dim + iy[None, :]).ravel()
    uppers = dim * dim + lowers
    parts = [lowers, uppers]
    if a > 0:
        parts.append(dim * dim + (a - 1) * dim + iy)
    if b < dim:
        parts.append(b * dim + iy)
    return np.concatenate(parts)


def owned_count(dim: int, a: int, b: int) -> int:
    return 2 * (b - a) * dim


def halo_plan(dim: int, size: int, rank: int) -> dict:
    """Local index ranges exchanged with the neighbours (ghost receive ranges
    and the owned columns the neighbours receive)."""
    a, b = strip_bounds(dim, size, rank)
    w = b - a
    gl = dim if a > 0 else 0
    plan = {"own_left": (0, dim), "own_right": ((2 * w - 1) * dim, 2 * w * dim)}
    if rank > 0:
        plan["ghost_left"] = (2 * w * dim, 2 * w * dim + dim)
    if rank < size - 1:
        plan["ghost_right"] = (2 * w * dim + gl, 2 * w * dim + gl + dim)
    return plan


def mg_depth(dim: int, size: int) -> int:
    """Coarse levels of the distributed multigrid (ldg_mg.cu mg_depth)."""
    if dim % size:
        return 0
    w, d, n = dim // size, dim, 0
    while d % 2 == 0 and d // 2 >= 2 and w % 2 == 0:
        d //= 2
        w //= 2
        n += 1
    return n


def weak_dim(base_dim: int, size: int) -> int:
    """Global FK dim for weak scaling: about base_dim^2 elements per rank,
    rounded so every rank owns a multiple-of-32 column count (multigrid depth)."""
    if size == 1:
        return base_dim
    unit = 32 * size
    return int(math.ceil(base_dim * math.sqrt(size) / unit)) * unit


def scaled_dim(base_dim: int, size: int, scaling: str = "weak", anchor: int = 1) -> int:
    """Global FK dim of a scaling run on `size` ranks.

    strong: the mesh is fixed (base_dim; every rank owns base_dim / size
    columns).  weak: about base_dim^2 / anchor elements per rank, i.e.
    dim = base_dim * sqrt(size / anchor) (config 5 is anchored
    at 8 GPUs, dim = 4096 sqrt(P/8) -> 1448, 2048, 2896, 4096), rounded up so
    every rank owns a multiple of 32 columns (multigrid depth)."""
    if scaling == "strong":
        if base_dim % size:
            raise ValueError(f"FK {base_dim} does not split into {size} equal strips")
        return base_dim
    if scaling != "weak":
        raise ValueError(f"unknown scaling {scaling!r}")
    if size == anchor:
        return base_dim
    unit = 32 * size
    return int(math.ceil(base_dim * math.sqrt(size / anchor) / unit - 1e-9)) * unit
