"""Time to a true relative residual of 1e-10 of the stepped solvers where they switch
levels: C2-shape varcoef CG and configs[3] conv-diff GMRES(30) (N from C4_N, default 256),
for the R29 trigger constants in R29_CS against FP64-CSR (bench.py's timing helpers).
One JSON line per config."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import gse_inputs as gi
import paper_2411_04686_b200 as g

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
cs = [float(c) for c in os.environ.get("R29_CS", "0.03,0.1,0.3,1").split(",")]
for solver, A in (("cg", gi.poisson3d(128, "varcoef")),
                  ("gmres", gi.convdiff3d(int(os.environ.get("C4_N", "256"))))):
    rp, col, val = bench._dev_csr(A, dev)
    b = torch.from_numpy(gi.ones_rhs(A)).to(dev)
    n = A.rows
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    M = g.gse_encode(rp, col, val, n, n)
    F = g.gse_fp64_matrix(rp, col, val, n, n)
    out = {"solver": solver, "n": n, "eta": g.gse_perturbation_bounds(M)}
    t64, r64 = bench._solve_ms(g, stream, flush, solver, F, b, x, None)
    out["fp64_csr"] = {"ms": round(t64, 2), "it": r64["iterations"]}
    for c in cs:
        t, r = bench._solve_ms(g, stream, flush, solver, M, b, x,
                               g.gse_default_schedule(solver, perturb_c=c))
        out[f"r29_c{c}"] = {"ms": round(t, 2), "it": r["iterations"], "per_level": r["iters_per_level"],
                            "switch": r["switch_iter"], "res": r["rel_residual_true"],
                            "x_fp64": round(t64 / t, 3)}
    print(json.dumps(out), flush=True)
    M.close()
    F.close()
