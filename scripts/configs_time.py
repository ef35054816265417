"""Time-to-solution on the other BASELINE.json configs, one JSON line per run (CUDA events on
the current stream around each solve, encode excluded, L2 flushed before each solve):
  * c2v: configs[1] shape with the varcoef values (head-lossy: the stepped driver switches);
  * c4:  configs[3] conv-diff 256^3, restarted GMRES(30) to 1e-10, stepped GSE (paper default
         and scaled schedules) vs FP64-CSR and the BF16 baseline;
  * c5:  configs[4] 3D Poisson 512^3 CG to 1e-10 on ONE GPU, stepped GSE vs FP64-CSR.
SECTIONS=c2v,c4,c5 selects."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gse_inputs as gi
import paper_2411_04686_b200 as g

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
dev = lambda a: torch.from_numpy(a).cuda()


def solve_time(fn, reps):
    ts, rep = [], None
    for i in range(reps):
        flush.fill_(i)
        flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        rep = fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts), rep


def summary(rep):
    return {k: rep[k] for k in ("status", "iterations", "iters_per_level", "switch_iter",
                                "rel_residual_true")}


def run(name, A, solver, runs, reps):
    t0 = time.time()
    rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
    b = dev(gi.ones_rhs(A))
    x = torch.zeros(A.rows, dtype=torch.float64, device="cuda")
    out = {"config": name, "n": int(A.rows), "nnz": int(A.nnz), "solver": solver, "tol": TOL}
    for label, kind, sched in runs:
        if kind == "gse":
            M = g.gse_encode(rp, col, val, A.rows, A.cols)
        elif kind == "fp64":
            M = g.gse_fp64_matrix(rp, col, val, A.rows, A.cols)
        else:
            M = g.gse_half_matrix(rp, col, val, A.rows, A.cols, kind=kind)

        def fn():
            x.zero_()
            if solver == "cg":
                return g.gse_solve_cg(M, b, x, tol=TOL, max_iters=20000, sched=sched)[1]
            return g.gse_solve_gmres(M, b, x, tol=TOL, max_iters=15000, sched=sched)[1]

        fn()
        ms, rep = solve_time(fn, reps)
        out[label] = {"ms": round(ms, 2), **summary(rep),
                      "us_per_iteration": round(1e3 * ms / max(rep["iterations"], 1), 2)}
        M.close()
        torch.cuda.synchronize()
    if "fp64" in out:
        for label, _, _ in runs:
            if label != "fp64" and out[label]["status"] == 0:
                out[label]["speedup_vs_fp64"] = round(out["fp64"]["ms"] / out[label]["ms"], 3)
    out["wall_s"] = round(time.time() - t0, 1)
    print(json.dumps(out), flush=True)


TOL = float(os.environ.get("TOL", "1e-10"))  # the paper's evaluation uses 1e-6


def k16(sched):
    sched.krylov_gse16 = 1
    return sched


secs = os.environ.get("SECTIONS", "c2v,c4,c5").split(",")
if "c2v" in secs:
    run("configs[1] shape, varcoef values (3D Poisson 128^3)", gi.poisson3d(128, "varcoef"), "cg",
        [("stepped_default", "gse", g.gse_default_schedule("cg")),
         ("stepped_scaled", "gse", g.gse_default_schedule("cg", l=30, t=10, m=10)),
         ("stepped_floors", "gse", g.gse_default_schedule("cg", level_floor=(1e-3, 1e-8))),
         ("fixed_L3", "gse", g.fixed_schedule(3)),
         ("fp64", "fp64", None), ("bf16", "bf16", None)], 3)
if "c4" in secs:
    N = int(os.environ.get("C4_N", "256"))
    run(f"configs[3] conv-diff {N}^3 GMRES(30)", gi.convdiff3d(N), "gmres",
        [("stepped_default", "gse", g.gse_default_schedule("gmres")),
         ("stepped_scaled", "gse", g.gse_default_schedule("gmres", l=300, t=100, m=100)),
         ("stepped_floors", "gse", g.gse_default_schedule("gmres", level_floor=(1e-3, 1e-8))),
         ("fp64", "fp64", None), ("bf16", "bf16", None),
         # NEXT-4: the Krylov basis as 16-bit GSE-SEM vectors
         ("fp64_krylov16", "fp64", k16(g.fixed_schedule(3))),
         ("stepped_floors_krylov16", "gse",
          k16(g.gse_default_schedule("gmres", level_floor=(1e-3, 1e-8))))], 2)
if "c5" in secs:
    N = int(os.environ.get("C5_N", "512"))
    run(f"configs[4] 3D Poisson {N}^3 CG, one GPU", gi.poisson3d(N), "cg",
        [("stepped_default", "gse", g.gse_default_schedule("cg")), ("fp64", "fp64", None)], 2)
