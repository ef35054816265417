"""Row-partitioned path on one GPU via the thread backend (P host threads, one stream each):
the same distributed code (global table by histogram allreduce, local renumbering, halo
exchange, allreduced dots) as the NCCL backend, checked against the single-GPU path and the
oracle:
  * every rank's table equals the global table; head/tail planes of the row blocks
    concatenate to the global planes (bit-exact); EI bits equal;
  * P-rank SpMV within the SpMV tolerance of the oracle;
  * P-rank stepped CG: iterations within 2 of the single-GPU solve, true residual <= tol.
"""
import os
import threading
import time

import numpy as np
import pytest

import gse_inputs as gi
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def g():
    assert torch.cuda.is_available()
    import paper_2411_04686_b200 as lib
    return lib


def partition(n, P):
    return [round(i * n / P) for i in range(P + 1)]


def run_ranks(P, fn):
    """run fn(rank, dist_handle, stream) on P threads of one thread group"""
    import paper_2411_04686_b200 as g
    grp = g.gse_dist_thread_group_create(P)
    out, errs = [None] * P, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            D = g.gse_dist_create_thread(grp, r, 0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[r] = fn(r, D, st)
            st.synchronize()
            D.close()
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append((r, repr(e)))

    # daemon threads and a bounded wait: a rank that fails (or a collective that never
    # completes) fails the test instead of blocking the whole suite
    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    deadline = time.time() + 180
    for t in th:
        t.join(timeout=max(1.0, deadline - time.time()))
    alive = [r for r, t in enumerate(th) if t.is_alive()]
    assert not alive and not errs, (alive, errs)
    g.gse_dist_thread_group_free(grp)
    return out


def slab(A, a, b):
    rp = (A.row_ptr[a:b + 1] - A.row_ptr[a]).astype(np.int64)
    sl = slice(A.row_ptr[a], A.row_ptr[b])
    return rp, A.col[sl].copy(), A.val[sl].copy()


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("name", ["poisson", "powerlaw"])
def test_dist_encode_and_spmv(g, P, name):
    A = gi.poisson3d(16, "varcoef") if name == "poisson" else gi.powerlaw_spd(20000, seed=4)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    x = gi.uniform_vec(A.cols, seed=5)
    rr = partition(A.rows, P)

    def fn(r, D, st):
        a, b = rr[r], rr[r + 1]
        rp, col, val = slab(A, a, b)
        dev = lambda v: torch.from_numpy(v).cuda()
        M = g.gse_encode_dist(D, dev(rp), dev(col), dev(val), a, A.rows, stream=st.cuda_stream)
        ys = [g.gse_spmv(M, dev(x[a:b].copy()), segments=L, stream=st.cuda_stream)
              for L in (1, 2, 3)]
        st.synchronize()
        P_ = g.gse_matrix_copy_planes(M)  # host copies after the last collective
        res = (P_, [y.cpu().numpy() for y in ys], M.info)
        M.close()
        return res

    outs = run_ranks(P, fn)
    for r, (P_, ys, info) in enumerate(outs):
        assert list(P_["table"]) == list(R.table)
        a, b = rr[r], rr[r + 1]
        sl = slice(A.row_ptr[a], A.row_ptr[b])
        for k in ("head", "tail1", "tail2"):
            assert np.array_equal(P_[k], getattr(R, k)[sl]), k
        assert np.array_equal(P_["col_ei"] >> 29, R.col_ei[sl] >> 29)
        for L, y in zip((1, 2, 3), ys):
            yo = O.spmv_gse(R, x, L)[a:b]
            absR = O.GseCsr(R.rows, R.cols, R.nnz, R.row_ptr, R.col_ei, R.side_ei,
                            R.head & np.uint16(0x7FFF), R.tail1, R.tail2, R.table, R.ei_bits,
                            R.ei_in_column)
            bound = 1e-12 * O.spmv_gse(absR, np.abs(x), L)[a:b]
            assert np.all(np.abs(y - yo) <= bound), (r, L)


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("variant", ["const", "varcoef"])
def test_dist_cg(g, P, variant):
    A = gi.poisson3d(20, variant)
    b = gi.ones_rhs(A)
    M1 = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
    sched = lambda: g.gse_default_schedule("cg", l=30, t=10, m=10)
    _, r1 = g.gse_solve_cg(M1, b, tol=1e-10, sched=sched())
    rr = partition(A.rows, P)

    def fn(r, D, st):
        a, bb = rr[r], rr[r + 1]
        rp, col, val = slab(A, a, bb)
        dev = lambda v: torch.from_numpy(v).cuda()
        M = g.gse_encode_dist(D, dev(rp), dev(col), dev(val), a, A.rows, stream=st.cuda_stream)
        x, rep = g.gse_solve_cg(M, dev(b[a:bb].copy()), tol=1e-10, sched=sched(),
                                stream=st.cuda_stream)
        st.synchronize()
        M.close()
        return x.cpu().numpy(), rep

    outs = run_ranks(P, fn)
    reps = [rep for _, rep in outs]
    x = np.concatenate([xx for xx, _ in outs])
    for rep in reps:  # every rank took the same decisions
        assert rep["iterations"] == reps[0]["iterations"]
        assert rep["switch_iter"] == reps[0]["switch_iter"]
    rep = reps[0]
    assert rep["converged"] and abs(rep["iterations"] - r1["iterations"]) <= 2, (rep, r1)
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    res = np.linalg.norm(b - O.spmv_fp64(F, x)) / np.linalg.norm(b)
    assert res <= 1e-10 * 1.01


@pytest.mark.parametrize("P", [2, 3])
def test_dist_cg_vs_partitioned_oracle(g, P):
    """the row-partitioned GPU CG (R29-free scaled schedule; thread backend) against the
    oracle's partitioned mode with the same row blocks: iterations
    and switch points within 2, true residual <= tol"""
    A = gi.poisson3d(16, "varcoef")
    b = gi.ones_rhs(A)
    rr = partition(A.rows, P)
    kw = dict(l=30, t=10, m=10)

    def fn(r, D, st):
        a, bb = rr[r], rr[r + 1]
        rp, col, val = slab(A, a, bb)
        dev = lambda v: torch.from_numpy(v).cuda()
        M = g.gse_encode_dist(D, dev(rp), dev(col), dev(val), a, A.rows, stream=st.cuda_stream)
        x, rep = g.gse_solve_cg(M, dev(b[a:bb].copy()), tol=1e-10,
                                sched=g.gse_default_schedule("cg", **kw), stream=st.cuda_stream)
        st.synchronize()
        M.close()
        return x.cpu().numpy(), rep

    outs = run_ranks(P, fn)
    rep = outs[0][1]
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    _, ro = O.cg(R, b, tol=1e-10, sched=O.schedule("cg", **kw), parts=rr)
    assert rep["converged"] and abs(rep["iterations"] - ro.iterations) <= 2, (rep, ro)
    assert rep["n_switches"] == ro.n_switches
    for a_, b_ in zip(rep["switch_iter"], ro.switch_iter):
        assert abs(a_ - b_) <= 2
    x = np.concatenate([xx for xx, _ in outs])
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    assert np.linalg.norm(b - O.spmv_fp64(F, x)) / np.linalg.norm(b) <= 1e-10 * 1.01


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("mode", ["fp64", "stepped_scaled"])
def test_dist_gmres(g, P, mode):
    """row-partitioned GMRES(30) (halo per SpMV, one allreduce per MGS dot and norm): every
    rank takes the same decisions; iterations within 2 of the single-GPU solve and of the
    oracle; true residual <= tol"""
    A = gi.convdiff3d(12)
    b = gi.ones_rhs(A)
    if mode == "fp64":
        enc1 = lambda: g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols)
        sched, so = (lambda: None), None
        Ro = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    else:
        enc1 = lambda: g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
        sched = lambda: g.gse_default_schedule("gmres", l=30, t=10, m=10)
        so = O.schedule("gmres", l=30, t=10, m=10)
        Ro = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    _, r1 = g.gse_solve_gmres(enc1(), b, tol=1e-10, sched=sched())
    _, ro = O.gmres(Ro, b, tol=1e-10, sched=so)
    rr = partition(A.rows, P)

    def fn(r, D, st):
        a, bb = rr[r], rr[r + 1]
        rp, col, val = slab(A, a, bb)
        dev = lambda v: torch.from_numpy(v).cuda()
        M = g.gse_encode_dist(D, dev(rp), dev(col), dev(val), a, A.rows, stream=st.cuda_stream)
        s = sched()
        if s is None:  # fixed full precision on the GSE planes (the FP64 result, d <= 11)
            s = g.fixed_schedule(3)
        x, rep = g.gse_solve_gmres(M, dev(b[a:bb].copy()), tol=1e-10, sched=s,
                                   stream=st.cuda_stream)
        st.synchronize()
        M.close()
        return x.cpu().numpy(), rep

    outs = run_ranks(P, fn)
    reps = [rep for _, rep in outs]
    x = np.concatenate([xx for xx, _ in outs])
    for rep in reps:
        assert rep["iterations"] == reps[0]["iterations"]
        assert rep["switch_iter"] == reps[0]["switch_iter"]
    rep = reps[0]
    assert rep["converged"], rep
    assert abs(rep["iterations"] - r1["iterations"]) <= 2, (rep, r1)
    assert abs(rep["iterations"] - ro.iterations) <= 2, (rep, ro)
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    res = np.linalg.norm(b - O.spmv_fp64(F, x)) / np.linalg.norm(b)
    assert res <= 1e-10 * 1.01


@pytest.mark.parametrize("P", [2, 3])
def test_dist_per_shard_tables(g, P):
    """NEXT-3 per-shard ("group" = row block) tables: each rank's table, planes and EI bits
    equal the oracle's encoding of its row block alone; SpMV on the block within the SpMV
    tolerance of that encoding; a stepped CG over the shards converges with identical
    decisions on every rank"""
    A = gi.powerlaw_spd(20000, seed=6)
    # D A D with D = 2^3 on the second half of the rows: still SPD, and the row blocks'
    # exponent populations differ, so their tables must too
    sc = np.where(np.arange(A.rows) >= A.rows // 2, 2.0 ** 3, 1.0)
    rows_of = np.repeat(np.arange(A.rows), np.diff(A.row_ptr))
    A = gi.Csr(A.rows, A.cols, A.row_ptr, A.col, A.val * sc[rows_of] * sc[A.col], "scaled")
    x = gi.uniform_vec(A.cols, seed=2)
    rr = partition(A.rows, P)
    B = gi.poisson3d(20, "varcoef")
    sb = np.where(np.arange(B.rows) >= B.rows // 2, 2.0 ** 3, 1.0)
    rows_b = np.repeat(np.arange(B.rows), np.diff(B.row_ptr))
    B = gi.Csr(B.rows, B.cols, B.row_ptr, B.col, B.val * sb[rows_b] * sb[B.col], "scaled")
    bB = gi.ones_rhs(B)
    rc = partition(B.rows, P)

    def fn(r, D, st):
        a, b = rr[r], rr[r + 1]
        rp, col, val = slab(A, a, b)
        dev = lambda v: torch.from_numpy(v).cuda()
        M = g.gse_encode_dist(D, dev(rp), dev(col), dev(val), a, A.rows, stream=st.cuda_stream,
                              per_shard_table=True)
        ys = [g.gse_spmv(M, dev(x[a:b].copy()), segments=L, stream=st.cuda_stream)
              for L in (1, 2, 3)]
        # CG on a D B D-scaled 3D Poisson (the power-law system converges too slowly)
        c, d = rc[r], rc[r + 1]
        rp2, col2, val2 = slab(B, c, d)
        M2 = g.gse_encode_dist(D, dev(rp2), dev(col2), dev(val2), c, B.rows,
                               stream=st.cuda_stream, per_shard_table=True)
        _, rep = g.gse_solve_cg(M2, dev(bB[c:d].copy()), tol=1e-10, stream=st.cuda_stream,
                                sched=g.gse_default_schedule("cg", l=30, t=10, m=10))
        st.synchronize()
        # host copies only after this rank's last collective
        P_ = g.gse_matrix_copy_planes(M)
        ys = [y.cpu().numpy() for y in ys]
        M.close()
        M2.close()
        return P_, ys, rep

    outs = run_ranks(P, fn)
    tables = []
    for r, (P_, ys, rep) in enumerate(outs):
        a, b = rr[r], rr[r + 1]
        rp, col, val = slab(A, a, b)
        R = O.encode_csr(b - a, A.cols, rp, col, val)
        assert list(P_["table"]) == list(R.table)
        tables.append(tuple(R.table))
        for k in ("head", "tail1", "tail2"):
            assert np.array_equal(P_[k], getattr(R, k)), k
        assert np.array_equal(P_["col_ei"] >> 29, R.col_ei >> 29)
        absR = O.GseCsr(R.rows, R.cols, R.nnz, R.row_ptr, R.col_ei, R.side_ei,
                        R.head & np.uint16(0x7FFF), R.tail1, R.tail2, R.table, R.ei_bits,
                        R.ei_in_column)
        for L, y in zip((1, 2, 3), ys):
            assert np.all(np.abs(y - O.spmv_gse(R, x, L)) <= 1e-12 * O.spmv_gse(absR, np.abs(x), L))
        assert rep["converged"] and rep["rel_residual_true"] <= 1e-10
        assert rep["iterations"] == outs[0][2]["iterations"]
    assert len(set(tables)) > 1  # the shards really chose different tables


@pytest.mark.parametrize("P", [2, 3])
def test_dist_overlap_interior_rows(g, P):
    """slabs large enough for the halo / interior overlap (row-walk matrices: the interior
    rows' SpMV runs on a side stream during the exchange, the boundary rows after it, three
    partial dots summed in a fixed order): SpMV within the oracle's tolerance at every
    level, CG within 2 iterations of the single-GPU solve, GMRES converging"""
    A = gi.poisson3d(40, "varcoef")
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    x = gi.uniform_vec(A.cols, seed=9)
    b = gi.ones_rhs(A)
    M1 = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
    sched = lambda: g.gse_default_schedule("cg", l=30, t=10, m=10)
    _, r1 = g.gse_solve_cg(M1, b, tol=1e-10, sched=sched())
    rr = partition(A.rows, P)

    def fn(r, D, st):
        a, bb = rr[r], rr[r + 1]
        rp, col, val = slab(A, a, bb)
        dev = lambda v: torch.from_numpy(v).cuda()
        M = g.gse_encode_dist(D, dev(rp), dev(col), dev(val), a, A.rows, stream=st.cuda_stream)
        ys = [g.gse_spmv(M, dev(x[a:bb].copy()), segments=L, stream=st.cuda_stream)
              for L in (1, 2, 3)]
        xs, rep = g.gse_solve_cg(M, dev(b[a:bb].copy()), tol=1e-10, sched=sched(),
                                 stream=st.cuda_stream)
        xg, repg = g.gse_solve_gmres(M, dev(b[a:bb].copy()), tol=1e-10, stream=st.cuda_stream,
                                     sched=g.gse_default_schedule("gmres", l=30, t=10, m=10))
        st.synchronize()
        out = ([y.cpu().numpy() for y in ys], xs.cpu().numpy(), rep, repg, M.info["spmv_mode"])
        M.close()
        return out

    outs = run_ranks(P, fn)
    absR = O.GseCsr(R.rows, R.cols, R.nnz, R.row_ptr, R.col_ei, R.side_ei,
                    R.head & np.uint16(0x7FFF), R.tail1, R.tail2, R.table, R.ei_bits,
                    R.ei_in_column)
    for r, (ys, xs, rep, repg, mode) in enumerate(outs):
        assert mode == 1  # row walk: the overlap applies
        a, bb = rr[r], rr[r + 1]
        for L, y in zip((1, 2, 3), ys):
            yo = O.spmv_gse(R, x, L)[a:bb]
            assert np.all(np.abs(y - yo) <= 1e-12 * O.spmv_gse(absR, np.abs(x), L)[a:bb]), (r, L)
        assert rep["iterations"] == outs[0][2]["iterations"]
        assert abs(rep["iterations"] - r1["iterations"]) <= 2, (rep, r1)
        assert repg["converged"] and repg["iterations"] == outs[0][3]["iterations"]
    x_all = np.concatenate([o[1] for o in outs])
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    assert np.linalg.norm(b - O.spmv_fp64(F, x_all)) / np.linalg.norm(b) <= 1e-10 * 1.01


def test_nccl_backend_single_rank(g):
    """the NCCL backend on the one GPU this box has: a 1-rank communicator runs the real
    NCCL calls of the distributed path (unique id, init, allgather / alltoall of the plan,
    histogram and dot allreduces, grouped send/recv with no peers) through encode, SpMV,
    CG and GMRES; results equal the single-GPU matrix's"""
    A = gi.poisson3d(24, "varcoef")
    n = A.rows
    D = g.gse_dist_create(g.gse_nccl_unique_id(), 0, 1, 0)
    dev = lambda v: torch.from_numpy(v).cuda()
    M = g.gse_encode_dist(D, dev(A.row_ptr), dev(A.col), dev(A.val), 0, n)
    M1 = g.gse_encode(A.row_ptr, A.col, A.val, n, n)
    assert list(M.info["table"]) == list(M1.info["table"])
    x = gi.uniform_vec(n, seed=4)
    for L in (1, 2, 3):
        yd = g.gse_spmv(M, dev(x), segments=L).cpu().numpy()
        y1 = g.gse_spmv(M1, x, segments=L)
        assert np.array_equal(yd, y1), L  # same kernels, same order on one rank
    b = gi.ones_rhs(A)
    sched = lambda s: g.gse_default_schedule(s, l=30, t=10, m=10)
    _, rd = g.gse_solve_cg(M, dev(b), tol=1e-10, sched=sched("cg"))
    _, r1 = g.gse_solve_cg(M1, b, tol=1e-10, sched=sched("cg"))
    assert rd["converged"] and abs(rd["iterations"] - r1["iterations"]) <= 2
    _, rd = g.gse_solve_gmres(M, dev(b), tol=1e-10, sched=sched("gmres"))
    _, r1 = g.gse_solve_gmres(M1, b, tol=1e-10, sched=sched("gmres"))
    assert rd["converged"] and abs(rd["iterations"] - r1["iterations"]) <= 2
    M.close()
    D.close()


def _run_workers(world, prefix, env_extra=None, N=24, solver="cg"):
    import subprocess
    import sys
    env = dict(os.environ, **(env_extra or {}))
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dist_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), prefix, str(N), solver],
                              env=env)
             for r in range(world)]
    rcs = [p.wait(timeout=600) for p in procs]
    assert rcs == [0] * world
    import json
    out = [np.load(f"{prefix}_{r}.npz") for r in range(world)]
    return np.concatenate([o["x"] for o in out]), [json.loads(str(o["rep"])) for o in out]


def test_nccl_gmres_graph_capture_matches_host_driven(g, tmp_path):
    """the distributed GMRES(30) restart cycle captured as a CUDA graph per level (NCCL
    backend) gives bitwise the solution, inner iterations and switch points of the
    host-enqueued cycles (GSE_DIST_NO_GRAPH=1); stepped with level floors (two switches)"""
    xg, rg = _run_workers(1, str(tmp_path / "graph"), N=12, solver="gmres")
    xh, rh = _run_workers(1, str(tmp_path / "host"), {"GSE_DIST_NO_GRAPH": "1"}, N=12,
                          solver="gmres")
    assert rg[0]["converged"] and rg[0]["n_switches"] >= 1
    assert (rg[0]["iterations"], rg[0]["switch_iter"]) == (rh[0]["iterations"], rh[0]["switch_iter"])
    assert np.array_equal(xg.view(np.uint64), xh.view(np.uint64))


def test_nccl_cg_graph_capture_matches_host_driven(g, tmp_path):
    """the distributed CG batch captured as a CUDA graph (NCCL backend: halo send/recv, the
    two allreduces, the side-stream interior SpMV and the kernels) gives bitwise the solution,
    iterations and switch points of the host-driven batches (GSE_DIST_NO_GRAPH=1), with the
    scaled stepped schedule (two escalations)"""
    xg, rg = _run_workers(1, str(tmp_path / "graph"))
    xh, rh = _run_workers(1, str(tmp_path / "host"), {"GSE_DIST_NO_GRAPH": "1"})
    assert rg[0]["converged"] and rg[0]["n_switches"] >= 1
    assert (rg[0]["iterations"], rg[0]["switch_iter"]) == (rh[0]["iterations"], rh[0]["switch_iter"])
    assert np.array_equal(xg.view(np.uint64), xh.view(np.uint64))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="multi-rank NCCL needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2])
def test_nccl_multi_rank_cg(g, tmp_path, world):
    """P processes, one GPU each, NCCL over NVLink: the row-partitioned stepped CG matches the
    single-GPU solve (iterations +-2, switch points +-2) and every rank reports the same
    iterations and switch points (identical allreduced scalars)"""
    if torch.cuda.device_count() < world:
        pytest.skip("not enough GPUs")
    N = 24
    x, reps = _run_workers(world, str(tmp_path / "mr"), N=N)
    assert all(r["iterations"] == reps[0]["iterations"] for r in reps)
    assert all(r["switch_iter"] == reps[0]["switch_iter"] for r in reps)
    A = gi.poisson3d(N, "varcoef")
    M1 = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
    b = gi.ones_rhs(A)
    x1, r1 = g.gse_solve_cg(M1, b, tol=1e-10, sched=g.gse_default_schedule("cg", l=30, t=10, m=10))
    assert reps[0]["converged"] and abs(reps[0]["iterations"] - r1["iterations"]) <= 2
    for a_, b_ in zip(reps[0]["switch_iter"], r1["switch_iter"]):
        assert abs(a_ - b_) <= 2
    assert np.abs(x - x1).max() <= 1e-7


def test_dist_single_gpu_only_options_are_refused(g):
    """options defined for one GPU fail loudly on a distributed matrix (no silent fallback):
    gse_spmv_dot (its dot would need the solve's allreduce), the R29 trigger, the 16-bit
    Krylov basis; the plain solves on the same handle still work"""
    A = gi.poisson3d(12, "varcoef")
    b = gi.ones_rhs(A)

    def fn(r, D, st):
        rr = partition(A.rows, 2)
        a, bb = rr[r], rr[r + 1]
        rp, col, val = slab(A, a, bb)
        dev = lambda v: torch.from_numpy(v).cuda()
        M = g.gse_encode_dist(D, dev(rp), dev(col), dev(val), a, A.rows, stream=st.cuda_stream)
        x = dev(gi.uniform_vec(bb - a, seed=r))
        errs = []
        for call in (lambda: g.gse_spmv_dot(M, x, stream=st.cuda_stream),
                     lambda: g.gse_solve_cg(M, dev(b[a:bb].copy()), tol=1e-10, stream=st.cuda_stream,
                                            sched=g.gse_default_schedule("cg", perturb_c=0.1))):
            try:
                call()
                errs.append(None)
            except g.GseError as e:
                errs.append(e.status)
        k16 = g.gse_default_schedule("gmres")
        k16.krylov_gse16 = 1
        try:
            g.gse_solve_gmres(M, dev(b[a:bb].copy()), tol=1e-10, sched=k16, stream=st.cuda_stream)
            errs.append(None)
        except g.GseError as e:
            errs.append(e.status)
        try:  # R30 kept direction: single-GPU only too
            g.gse_solve_cg(M, dev(b[a:bb].copy()), tol=1e-10, stream=st.cuda_stream,
                           sched=g.gse_default_schedule("cg", cg_keep_direction=1))
            errs.append(None)
        except g.GseError as e:
            errs.append(e.status)
        _, rep = g.gse_solve_cg(M, dev(b[a:bb].copy()), tol=1e-10, stream=st.cuda_stream,
                                sched=g.gse_default_schedule("cg", l=30, t=10, m=10))
        st.synchronize()
        M.close()
        return errs, rep

    outs = run_ranks(2, fn)
    for errs, rep in outs:
        assert errs == [g.GSE_ERR_WRONG_FORMAT] * 4
        assert rep["converged"]
