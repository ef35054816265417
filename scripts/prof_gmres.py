"""Profiling driver: one GMRES(30) restart cycle on conv-diff N^3 (per-step kernels at
N >= 160), for ncu -k regex:k_gm.  Not a benchmark."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gse_inputs as gi, paper_2411_04686_b200 as g
N = int(os.environ.get("GM_N", "256"))
A = gi.convdiff3d(N)
dev = lambda a: torch.from_numpy(a).cuda()
F = g.gse_fp64_matrix(dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val), A.rows, A.cols)
b = dev(gi.ones_rhs(A))
x = torch.zeros(A.rows, dtype=torch.float64, device="cuda")
g.gse_solve_gmres(F, b, x, tol=1e-10, max_iters=int(os.environ.get("GM_ITERS", "30")))
torch.cuda.synchronize()
print("done")
