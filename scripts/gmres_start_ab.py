"""Stepped GMRES(30) on configs[3] conv-diff (C4_N, default 256): R29 trigger constants x
start level against FP64-CSR, time to 1e-10 (and to 1e-6).  One JSON line.  (Developer tool.)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import gse_inputs as gi
import paper_2411_04686_b200 as g

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
A = gi.convdiff3d(int(os.environ.get("C4_N", "256")))
rp, col, val = bench._dev_csr(A, dev)
b = torch.from_numpy(gi.ones_rhs(A)).to(dev)
n = A.rows
x = torch.zeros(n, dtype=torch.float64, device=dev)
M = g.gse_encode(rp, col, val, n, n)
F = g.gse_fp64_matrix(rp, col, val, n, n)
out = {"n": n}
t64, r64 = bench._solve_ms(g, stream, flush, "gmres", F, b, x, None)
out["fp64_csr"] = {"ms": round(t64, 1), "it": r64["iterations"]}
for start in (1, 2):
    for c in (0.1, 1.0, 10.0):
        t, r = bench._solve_ms(g, stream, flush, "gmres", M, b, x,
                               g.gse_default_schedule("gmres", perturb_c=c, start_level=start))
        out[f"s{start}_c{c}"] = {"ms": round(t, 1), "it": r["iterations"], "per_level": r["iters_per_level"],
                                 "res": r["rel_residual_true"], "x_fp64": round(t64 / t, 3)}
print(json.dumps(out), flush=True)
