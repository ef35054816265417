"""Host logic of the row-partitioned (multi-GPU) path, on CPU:
  * gse_dist_plan (C-ABI, host-only) against a direct set-based construction;
  * a world_size-2 gloo run: each rank plans its row block, the halo requests are exchanged
    over torch.distributed, x is exchanged through the plan, and the rank-local SpMV of the
    renumbered block (oracle) equals the global oracle SpMV rows bitwise (local renumbering
    keeps every row's storage order).
"""
import os

import numpy as np
import pytest

import gse_inputs as gi
import oracle as O


def plan_reference(col, row_begin, n_local, rank_rows):
    owned = (col >= row_begin) & (col < row_begin + n_local)
    halo = np.unique(col[~owned])
    local = np.where(owned, col - row_begin, 0).astype(np.int64)
    local[~owned] = n_local + np.searchsorted(halo, col[~owned])
    owner = np.searchsorted(rank_rows, halo, side="right") - 1
    recv = np.bincount(owner, minlength=rank_rows.size - 1)
    return local, halo, recv


def partition(n, P):
    return np.array([round(i * n / P) for i in range(P + 1)], dtype=np.int64)


@pytest.mark.parametrize("P", [1, 2, 3, 5])
@pytest.mark.parametrize("mk", [lambda: gi.poisson3d(9), lambda: gi.powerlaw_spd(3000, seed=2),
                                lambda: gi.convdiff3d(7)])
def test_plan_matches_reference(P, mk):
    import paper_2411_04686_b200 as g
    A = mk()
    rr = partition(A.rows, P)
    for r in range(P):
        a, b = rr[r], rr[r + 1]
        col = A.col[A.row_ptr[a]:A.row_ptr[b]]
        local, halo, recv = g.gse_dist_plan(col, int(a), int(b - a), rr)
        lr, hr, rc = plan_reference(col.astype(np.int64), a, b - a, rr)
        assert np.array_equal(local, lr) and np.array_equal(halo, hr)
        assert np.array_equal(recv, rc) and recv[r] == 0


def _rank_main(rank, world, port, out_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2411_04686_b200 as g
    A = gi.poisson3d(10, "varcoef")
    rr = partition(A.rows, world)
    a, b = int(rr[rank]), int(rr[rank + 1])
    rp = A.row_ptr[a:b + 1] - A.row_ptr[a]
    col = A.col[A.row_ptr[a]:A.row_ptr[b]]
    val = A.val[A.row_ptr[a]:A.row_ptr[b]]
    local, halo, recv = g.gse_dist_plan(col, a, b - a, rr)
    # halo requests per owner -> owners learn their send lists
    want, o = [], 0
    for p in range(world):
        want.append(halo[o:o + recv[p]])
        o += recv[p]
    gathered = [None] * world
    dist.all_gather_object(gathered, want)
    give = [gathered[p][rank] for p in range(world)]  # entries rank p needs from me
    x = gi.uniform_vec(A.rows, seed=3)
    x_mine = x[a:b].copy()
    # exchange through the plan: each rank ships x[give[p]] to p
    packets = [x_mine[np.asarray(give[p], dtype=np.int64) - a] for p in range(world)]
    allp = [None] * world
    dist.all_gather_object(allp, packets)
    x_ext = np.concatenate([x_mine] + [allp[p][rank] for p in range(world)])
    assert x_ext.size == (b - a) + halo.size
    F = O.fp64_csr(b - a, x_ext.size, rp, local, val)
    y_local = O.spmv_fp64(F, x_ext)
    y_ref = O.spmv_fp64(O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val), x)[a:b]
    out_q.put((rank, bool(np.array_equal(y_local.view(np.uint64), y_ref.view(np.uint64))),
               int(halo.size)))
    dist.destroy_process_group()


def test_two_rank_gloo_halo_exchange_spmv():
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    assert all(nh == 100 for _, _, nh in res)  # one 10x10 plane of halo per side
