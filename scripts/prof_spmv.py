"""Profiling driver: C2 (3D Poisson 128^3) SpMV at each level + a short stepped CG solve,
for ncu (`ncu --set full -k regex:k_spmv ...`).  Not a benchmark (numbers under ncu are
never reported)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gse_inputs as gi
import paper_2411_04686_b200 as g

N = int(os.environ.get("PROF_N", "128"))
variant = os.environ.get("PROF_VARIANT", "const")
A = gi.poisson3d(N, variant) if os.environ.get("PROF_MAT", "poisson") == "poisson" else gi.powerlaw_spd(N)
dev = lambda a: torch.from_numpy(a).cuda()
rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
M = g.gse_encode(rp, col, val, A.rows, A.cols)
F = g.gse_fp64_matrix(rp, col, val, A.rows, A.cols)
x = torch.rand(A.cols, dtype=torch.float64, device="cuda")
y = torch.empty(A.rows, dtype=torch.float64, device="cuda")
for rep in range(2):
    for L in (1, 2, 3):
        g.gse_spmv(M, x, y, segments=L)
    g.gse_spmv(F, x, y, segments=3)
b = dev(gi.ones_rhs(A))
g.gse_solve_cg(M, b, tol=1e-10, max_iters=int(os.environ.get("PROF_CG_ITERS", "20")),
               sched=g.gse_default_schedule("cg"))
torch.cuda.synchronize()
print("done")
