"""R30 A/B: stepped CG with the search direction kept at a level switch (GSE_CG_KEEP=1) vs
the R15 restart, on varcoef Poisson (N from KEEP_N), R29 trigger constants x start level,
against FP64-CSR.  One JSON line.  (Developer tool.)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import gse_inputs as gi
import paper_2411_04686_b200 as g

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
N = int(os.environ.get("KEEP_N", "128"))
A = gi.poisson3d(N, "varcoef")
rp, col, val = bench._dev_csr(A, dev)
b = torch.from_numpy(gi.ones_rhs(A)).to(dev)
n = A.rows
x = torch.zeros(n, dtype=torch.float64, device=dev)
M = g.gse_encode(rp, col, val, n, n)
F = g.gse_fp64_matrix(rp, col, val, n, n)
out = {"N": N, "keep": os.environ.get("GSE_CG_KEEP", "0"), "eta": g.gse_perturbation_bounds(M)}
t64, r64 = bench._solve_ms(g, stream, flush, "cg", F, b, x, None)
out["fp64_csr"] = {"ms": round(t64, 2), "it": r64["iterations"]}
for start in (1, 2):
    for c in [float(v) for v in os.environ.get("R29_CS", "0.1,1,3,10").split(",")]:
        t, r = bench._solve_ms(g, stream, flush, "cg", M, b, x,
                               g.gse_default_schedule("cg", perturb_c=c, start_level=start,
                                                     cg_keep_direction=int(os.environ.get("GSE_CG_KEEP", "0"))))
        out[f"s{start}_c{c}"] = {"ms": round(t, 2), "it": r["iterations"], "per_level": r["iters_per_level"],
                                 "switch": r["switch_iter"], "res": r["rel_residual_true"],
                                 "x_fp64": round(t64 / t, 3)}
print(json.dumps(out), flush=True)
