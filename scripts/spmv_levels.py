"""SpMV time per level (cold, L2 flushed) and the fused SpMV + dot, on a chosen Poisson
variant (SPMV_N, SPMV_VARIANT) -- developer tool; JSON line with GB/s of algorithmic bytes."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import gse_inputs as gi
import paper_2411_04686_b200 as g

dev = torch.device("cuda", 0)
N = int(os.environ.get("SPMV_N", "256"))
var = os.environ.get("SPMV_VARIANT", "varcoef")
A = gi.poisson3d(N, var)
rp, col, val = bench._dev_csr(A, dev)
n, nnz = A.rows, A.nnz
M = g.gse_encode(rp, col, val, n, n)
F = g.gse_fp64_matrix(rp, col, val, n, n)
x = torch.rand(n, dtype=torch.float64, device=dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
def timeit(fn, reps=10):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    fn()
    for i in range(reps):
        flush.fill_(i); flush.sum()
        evs[i][0].record(); fn(); evs[i][1].record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in evs) * 1e-3
out = {"N": N, "variant": var, "info": {k: M.info[k] for k in ("spmv_mode",) if k in M.info}}
for L, sl in ((1, 2), (2, 4), (3, 8)):
    t = timeit(lambda: g.gse_spmv(M, x, y, segments=L))
    td = timeit(lambda: g.gse_spmv_dot(M, x, y, segments=L)) if hasattr(g, "gse_spmv_dot") else None
    b = nnz * (4 + sl) + 4 * (n + 1) + 16 * n
    out[f"L{L}"] = {"us": round(t * 1e6, 1), "GBps": round(b / t / 1e9), "dot_us": round(td * 1e6, 1) if td else None}
t = timeit(lambda: g.gse_spmv(F, x, y, segments=3))
out["fp64"] = {"us": round(t * 1e6, 1), "GBps": round((nnz * 12 + 20 * n) / t / 1e9)}
print(json.dumps(out))
