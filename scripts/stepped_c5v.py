"""configs[4] shape (3D Poisson 512^3) with varcoef values: head-lossy, so the stepped CG
must switch levels.  Time to a true relative residual of 1e-10 for FP64-CSR and the stepped
schedules (paper defaults, floors, R29, and R29 starting at level 2).  One JSON line."""
import json, os, sys, time, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2411_04686_b200 as g

N = int(os.environ.get("C5V_N", "512"))
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
t0 = time.time()
rp, col, val, b = bench.device_poisson(types.SimpleNamespace(N=N, variant="varcoef"), 0, N ** 3, dev)
n = N ** 3
out = {"n": n, "generate_s": round(time.time() - t0, 1)}
x = torch.zeros(n, dtype=torch.float64, device=dev)
F = g.gse_fp64_matrix(rp, col, val, n, n)
t, r = bench._solve_ms(g, stream, flush, "cg", F, b, x, None)
out["fp64_csr"] = {"ms": round(t, 1), "it": r["iterations"], "res": r["rel_residual_true"]}
F.close()
torch.cuda.empty_cache()
M = g.gse_encode(rp, col, val, n, n)
out["eta"] = g.gse_perturbation_bounds(M)
for name, kw in (("stepped_default", {}), ("stepped_floors", {"level_floor": (1e-3, 1e-8)}),
                 ("stepped_r29", {"perturb_c": 0.1}),
                 ("stepped_r29_from_l2", {"perturb_c": 0.1, "start_level": 2})):
    t, r = bench._solve_ms(g, stream, flush, "cg", M, b, x, g.gse_default_schedule("cg", **kw))
    out[name] = {"ms": round(t, 1), "it": r["iterations"], "per_level": r["iters_per_level"],
                 "switch": r["switch_iter"], "res": r["rel_residual_true"],
                 "x_fp64": round(out["fp64_csr"]["ms"] / t, 3)}
    print(json.dumps({name: out[name]}), flush=True)
print(json.dumps(out), flush=True)
