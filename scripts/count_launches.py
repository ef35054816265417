"""Kernels per bench step (encode + stepped CG on configs[1]), for checking bench.py's
gpu_launches estimate: run under ncu with STEPS=1 and STEPS=2 and take the difference."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gse_inputs as gi
import paper_2411_04686_b200 as g
import bench

A = gi.poisson3d(128)
dev = torch.device("cuda")
rp = torch.from_numpy(A.row_ptr.astype(np.int32)).to(dev)
col = torch.from_numpy(A.col).to(dev); val = torch.from_numpy(A.val).to(dev)
b = torch.from_numpy(gi.ones_rhs(A)).to(dev)
x = torch.zeros(A.rows, dtype=torch.float64, device=dev)
sched = g.gse_default_schedule("cg")
for _ in range(int(sys.argv[1])):
    M = g.gse_encode(rp, col, val, A.rows, A.cols, k_max=8)
    x.zero_()
    _, rep = g.gse_solve_cg(M, b, x, tol=1e-10, max_iters=20000, sched=sched)
    M.close()
torch.cuda.synchronize()
print("estimate per step", bench.estimate_launches(rep, 1), "iters", rep["iterations"])
