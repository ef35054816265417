"""Time stepped GMRES(30) (GSE) vs FP64-CSR GMRES on conv-diff N^3 (configs[3] shape)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gse_inputs as gi, paper_2411_04686_b200 as g
N = int(os.environ.get("GM_N", "64"))
A = gi.convdiff3d(N)
dev = lambda a: torch.from_numpy(a).cuda()
rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
b = dev(gi.ones_rhs(A))
M = g.gse_encode(rp, col, val, A.rows, A.cols)
F = g.gse_fp64_matrix(rp, col, val, A.rows, A.cols)
x = torch.zeros(A.rows, dtype=torch.float64, device="cuda")
for name, Mx, sch in (("gse-stepped", M, g.gse_default_schedule("gmres")),
                      ("gse-scaled", M, g.gse_default_schedule("gmres", l=300, t=100, m=100)),
                      ("fp64", F, None)):
    for rep_i in range(2):
        x.zero_(); torch.cuda.synchronize(); t0 = time.perf_counter()
        _, rep = g.gse_solve_gmres(Mx, b, x, tol=1e-10, sched=sch)
        torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"N={N} {name}: {t*1e3:.1f} ms wall, device {rep['seconds']*1e3:.1f} ms, iters {rep['iterations']}, "
          f"levels {rep['iters_per_level']}, switches {rep['switch_iter']}, true {rep['rel_residual_true']:.2e}, "
          f"us/inner {1e6*rep['seconds']/max(rep['iterations'],1):.1f}", flush=True)
