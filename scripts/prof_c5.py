"""Profiling driver for configs[4] (3D Poisson 512^3): the CG's fused level-1 SpMV + dot
(gse_spmv_dot, the dominant kernel of the bench step) and the level-2/3 SpMVs, for
`ncu --set full -k regex:k_spmv_rw`.  Not a benchmark (numbers under ncu are never reported)."""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2411_04686_b200 as g

N = int(os.environ.get("PROF_N", "512"))
args = types.SimpleNamespace(N=N, variant="const")
dev = torch.device("cuda", 0)
rp, col, val, b = bench.device_poisson(args, 0, N ** 3, dev)
n = N ** 3
M = g.gse_encode(rp, col, val, n, n)
x = torch.rand(n, dtype=torch.float64, device=dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
d = torch.empty(1, dtype=torch.float64, device=dev)
for L in (1, 1, 2, 3):
    g.gse_spmv_dot(M, x, y, segments=L, dot=d)
torch.cuda.synchronize()
print("done", float(d.item()))
