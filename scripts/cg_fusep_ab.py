"""A/B of the CG p update fused into the SpMV (GSE_CG_FUSEP=1) against the separate xpay
kernel: C2 stepped CG, FP64-CSR CG and a head-lossy varcoef matrix (escalations); time per
solve (CUDA events, median of 5), iterations, and x saved for a bitwise comparison."""
import os, sys, statistics, torch, numpy as np
import gse_inputs as gi
import paper_2411_04686_b200 as g

tag = sys.argv[1]
dev = torch.device("cuda")
s = torch.cuda.current_stream()
out = {}
for name, A in (("c2", gi.poisson3d(128)), ("var", gi.poisson3d(64, "varcoef"))):
    rp = torch.from_numpy(A.row_ptr.astype(np.int32)).to(dev)
    col = torch.from_numpy(A.col).to(dev); val = torch.from_numpy(A.val).to(dev)
    b = torch.from_numpy(gi.ones_rhs(A)).to(dev)
    for kind in ("gse", "fp64"):
        M = (g.gse_encode(rp, col, val, A.rows, A.cols, k_max=8) if kind == "gse"
             else g.gse_fp64_matrix(rp, col, val, A.rows, A.cols))
        sched = g.gse_default_schedule("cg") if kind == "gse" else None
        x = torch.zeros(A.rows, dtype=torch.float64, device=dev)
        ts = []
        for i in range(6):
            x.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _, rep = g.gse_solve_cg(M, b, x, tol=1e-10, max_iters=20000, sched=sched)
            e1.record(s); torch.cuda.synchronize()
            if i: ts.append(e0.elapsed_time(e1))
        np.save(f"gpurun_out/cgx_{tag}_{name}_{kind}.npy", x.cpu().numpy())
        print(tag, name, kind, "ms %.3f" % statistics.median(ts), "iters", rep["iterations"],
              rep["iters_per_level"], "res %.3e" % rep["rel_residual_true"],
              "us/iter %.2f" % (statistics.median(ts) * 1e3 / rep["iterations"]), flush=True)
        M.close()
