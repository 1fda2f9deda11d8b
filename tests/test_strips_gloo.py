"""The multi-rank path on CPU (world size 2 and 3, gloo): the strip plan of
paper_1408_3877_b200/strips.py, a halo exchange over torch.distributed and
a distributed block-SpMV + dot products with the CPU oracle's operator must
reproduce the global (W + dt A) x and x.y exactly as the library's NCCL path
is designed to."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1408_3877_b200 import strips


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _global_operator(dim: int, n_local: int, dt: float):
    from oracle import ldg_oracle as O

    m = O.domain_square(1.0 / dim)
    spec = O.ProblemSpec(d=(9, []), f=(10, []), c_d=(8, []), g_n=(11, []), c0=(8, []), eta=1.0,
                         boundary={1: "D", 2: "N", 3: "N", 4: "D"})
    s = O.LdgSystem(m, spec, O.build_ref_tensors(n_local))
    A, _ = s.build_blocks(0.3)
    return (A * dt + s.w_matrix()).tocsr(), m.num_t


def _worker(rank: int, size: int, port: int, dim: int, n_local: int, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        L, K = _global_operator(dim, n_local, 0.05)
        N = n_local
        rng = np.random.default_rng(7)
        x_glob = rng.uniform(-1, 1, L.shape[0])
        a, b = strips.strip_bounds(dim, size, rank)
        loc = strips.local_elements(dim, a, b)
        own = strips.owned_count(dim, a, b)
        plan = strips.halo_plan(dim, size, rank)
        # dof indices of local elements for the three unknown blocks (Z1, Z2, C)
        def dofs(elems):
            return np.concatenate([(u * K + elems)[:, None] * N + np.arange(N)[None, :] for u in range(3)]).ravel()

        own_dofs, loc_dofs = dofs(loc[:own]), dofs(loc)
        # ghost sufficiency: the owned rows have no entry outside the local columns
        rows = L[own_dofs]
        outside = np.setdiff1d(rows.indices, loc_dofs)
        assert outside.size == 0, f"rank {rank}: {outside.size} couplings outside owned+ghost"

        # local x: owned values known, ghosts exchanged with the neighbours
        x_loc = np.zeros((loc.size, 3, N))
        xg = x_glob.reshape(3, K, N)
        x_loc[:own] = xg[:, loc[:own], :].transpose(1, 0, 2)
        reqs, bufs = [], {}
        if "ghost_left" in plan:
            lo, hi = plan["own_left"]
            send = torch.from_numpy(np.ascontiguousarray(x_loc[lo:hi]))
            reqs.append(dist.isend(send, rank - 1))
            bufs["left"] = torch.zeros_like(send)
            reqs.append(dist.irecv(bufs["left"], rank - 1))
        if "ghost_right" in plan:
            lo, hi = plan["own_right"]
            send = torch.from_numpy(np.ascontiguousarray(x_loc[lo:hi]))
            reqs.append(dist.isend(send, rank + 1))
            bufs["right"] = torch.zeros_like(send)
            reqs.append(dist.irecv(bufs["right"], rank + 1))
        for r in reqs:
            r.wait()
        if "left" in bufs:
            lo, hi = plan["ghost_left"]
            x_loc[lo:hi] = bufs["left"].numpy()
        if "right" in bufs:
            lo, hi = plan["ghost_right"]
            x_loc[lo:hi] = bufs["right"].numpy()
        # halo-received values equal the global vector at the ghost elements
        np.testing.assert_array_equal(x_loc[own:], xg[:, loc[own:], :].transpose(1, 0, 2))

        # local matvec on owned rows with local columns
        x_vec = np.zeros(L.shape[0])  # only local (owned + ghost) entries are filled
        for u in range(3):
            idx = (u * K + loc)[:, None] * N + np.arange(N)[None, :]
            x_vec[idx.ravel()] = x_loc[:, u, :].ravel()
        y_own = L[own_dofs] @ x_vec
        y_ref = L[own_dofs] @ x_glob
        assert np.abs(y_own - y_ref).max() <= 1e-14 * max(1.0, np.abs(y_ref).max())

        # distributed dot product (owned entries only) with all_reduce
        part = torch.tensor([float(y_own @ x_glob[own_dofs])], dtype=torch.float64)
        dist.all_reduce(part)
        full = float((L @ x_glob) @ x_glob)
        assert abs(part.item() - full) <= 1e-12 * abs(full)
        q.put((rank, "ok", strips.mg_depth(dim, size)))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e), -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("size,dim,n_local", [(2, 8, 3), (3, 6, 6)])
def test_distributed_spmv_and_dots_gloo(size, dim, n_local):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, dim, n_local, q)) for r in range(size)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, depth in results:
        assert status == "ok", (rank, status)
    assert len({d for _, _, d in results}) == 1  # every rank builds the same multigrid depth


def test_strip_plan_covers_mesh():
    for dim, size in ((8, 2), (12, 3), (16, 4), (384, 2), (768, 8)):
        seen = np.zeros(2 * dim * dim, int)
        for r in range(size):
            a, b = strips.strip_bounds(dim, size, r)
            loc = strips.local_elements(dim, a, b)
            seen[loc[: strips.owned_count(dim, a, b)]] += 1
        assert np.all(seen == 1)
    assert strips.mg_depth(256, 1) == 7 and strips.mg_depth(32, 4) == 3 and strips.mg_depth(384, 2) == 6
    assert strips.weak_dim(256, 1) == 256 and strips.weak_dim(256, 2) == 384 and strips.weak_dim(256, 8) == 768


def test_scaling_dims():
    """bench.py's multi-GPU sizes: strong = the workload's
    mesh on every rank count; weak = its elements per GPU, C5 anchored at
    8 GPUs (dim = 4096 sqrt(P/8) -> 1448, 2048, 2896, 4096, rounded up to
    32-column strips so every rank keeps the multigrid depth)."""
    from paper_1408_3877_b200 import strips

    assert [strips.scaled_dim(4096, p, "strong") for p in (1, 2, 4, 8)] == [4096] * 4
    weak = [strips.scaled_dim(4096, p, "weak", anchor=8) for p in (1, 2, 4, 8)]
    assert weak == [1472, 2048, 2944, 4096]
    for p, d in zip((1, 2, 4, 8), weak):
        assert d % (32 * p) == 0 and abs(d * d / p - 4096 ** 2 / 8) / (4096 ** 2 / 8) < 0.1
        assert strips.mg_depth(d, p) >= 5
    assert [strips.scaled_dim(256, p) for p in (1, 2, 4, 8)] == [strips.weak_dim(256, p) for p in (1, 2, 4, 8)]
    import pytest

    with pytest.raises(ValueError):
        strips.scaled_dim(100, 3, "strong")
