"""A/B timing of the SpMV kernels (CUDA events, L2 flushed before each launch) on C2 and a
power-law matrix; prints one JSON line per (matrix, level).  Dev tool, not the bench."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gse_inputs as gi
import paper_2411_04686_b200 as g

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
tag = os.environ.get("TAG", "")

def timeit_steady(fn, reps=80):
    """back-to-back launches (as in the CG loop), average per launch"""
    fn()
    flush.fill_(0); flush.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


def timeit(fn, reps=30):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    fn()
    for i in range(reps):
        flush.fill_(i); flush.sum()  # write + read back: no dirty write-backs in the timing
        evs[i][0].record(); fn(); evs[i][1].record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in evs) * 1e-3

mats = {f"p3d_{N}": (lambda N=N: gi.poisson3d(N)) for N in [int(v) for v in os.environ.get("AB_NS", "128").split(",")]}
if os.environ.get("AB_POWERLAW", "1") == "1":
    mats["pl2m"] = lambda: gi.powerlaw_spd(int(os.environ.get("AB_PL_N", "2000000")))
src = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
dst = torch.empty_like(src)
tcopy = timeit(lambda: dst.copy_(src), 10)
print(json.dumps({"tag": tag, "copy_GBps": round(2 * src.numel() * 4 / tcopy / 1e9, 1)}), flush=True)
del src, dst
for name, mk in mats.items():
    A = mk()
    dev = lambda a: torch.from_numpy(a).cuda()
    rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
    M = g.gse_encode(rp, col, val, A.rows, A.cols)
    F = g.gse_fp64_matrix(rp, col, val, A.rows, A.cols)
    x = torch.rand(A.cols, dtype=torch.float64, device="cuda"); y = torch.empty(A.rows, dtype=torch.float64, device="cuda")
    x32 = x.float(); y32 = y.float()
    n, nnz = A.rows, A.nnz
    res = {}
    for L, s_l in ((1, 2), (2, 4), (3, 8)):
        t = timeit(lambda: g.gse_spmv(M, x, y, segments=L))
        b = nnz * (4 + s_l) + 4 * (n + 1) + 16 * n
        res[f"L{L}"] = round(b / t / 1e9, 1)
        t = timeit(lambda: g.gse_spmv_f32acc(M, x32, y32, segments=L))
        b = nnz * (4 + s_l) + 4 * (n + 1) + 8 * n
        res[f"L{L}f32"] = round(b / t / 1e9, 1)
    t = timeit(lambda: g.gse_spmv(F, x, y, segments=3))
    res["fp64"] = round((nnz * 12 + 4 * (n + 1) + 16 * n) / t / 1e9, 1)
    if os.environ.get("AB_STEADY", "1") == "1":
        for L, s_l in ((1, 2), (2, 4), (3, 8)):
            t = timeit_steady(lambda: g.gse_spmv(M, x, y, segments=L))
            res[f"L{L}_steady"] = round((nnz * (4 + s_l) + 4 * (n + 1) + 16 * n) / t / 1e9, 1)
    print(json.dumps({"tag": tag, "mat": name, "nnz": nnz, "GBps": res, "peak": peak}), flush=True)
