"""configs[4] (512^3) row-walk SpMV A/B: levels 1-3 cold and the CG's fused SpMV + dot back
to back, for the library in GSE_LIB_PATH (prebuilt variants under ab/).  One JSON line."""
import json, os, statistics, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2411_04686_b200 as g

N = int(os.environ.get("PROF_N", "512"))
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
rp, col, val, b = bench.device_poisson(types.SimpleNamespace(N=N, variant="const"), 0, N ** 3, dev)
n, nnz = N ** 3, int(col.numel())
M = g.gse_encode(rp, col, val, n, n)
x = torch.rand(n, dtype=torch.float64, device=dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
d = torch.empty(1, dtype=torch.float64, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
peak = bench.peaks()[0]
out = {"lib": os.environ.get("GSE_LIB_PATH", "in-tree")}
for L, s_l in ((1, 2), (2, 4), (3, 8)):
    byt = nnz * (4 + s_l) + 4 * (n + 1) + 16 * n
    fn = lambda: g.gse_spmv(M, x, y, segments=L)
    fn()
    t = statistics.mean(bench.time_cuda(fn, 5, stream, flush)) * 1e3
    td = bench.time_b2b(lambda: g.gse_spmv_dot(M, x, y, segments=L, dot=d), 10, stream, flush) * 1e3
    out[f"L{L}"] = {"cold_us": round(t, 1), "cold_frac": round(byt / t / 1e3 / peak, 3),
                    "dot_b2b_us": round(td, 1), "dot_b2b_frac": round(byt / td / 1e3 / peak, 3)}
xs = torch.zeros(n, dtype=torch.float64, device=dev)
rep = g.gse_solve_cg(M, b, xs, tol=1e-10, sched=g.gse_default_schedule("cg"))[1]
out["cg_ms"] = round(statistics.median(bench.time_cuda(
    lambda: (xs.zero_(), g.gse_solve_cg(M, b, xs, tol=1e-10, sched=g.gse_default_schedule("cg"))),
    2, stream, flush)), 1)
out["cg_iters"] = rep["iterations"]
print(json.dumps(out), flush=True)
