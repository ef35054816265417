"""Time the CG solve (no encode) on C2 for A/B experiments; prints ms and iterations."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gse_inputs as gi, paper_2411_04686_b200 as g
N = int(os.environ.get("CG_N", "128"))
A = gi.poisson3d(N, os.environ.get("CG_VARIANT", "const"))
dev = lambda a: torch.from_numpy(a).cuda()
rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
b = dev(gi.ones_rhs(A))
M = g.gse_encode(rp, col, val, A.rows, A.cols)
F = g.gse_fp64_matrix(rp, col, val, A.rows, A.cols)
x = torch.zeros(A.rows, dtype=torch.float64, device="cuda")
for name, Mx, sch in (("gse", M, g.gse_default_schedule("cg")), ("fp64", F, None)):
    ts = []
    for i in range(4):
        x.zero_(); torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); _, rep = g.gse_solve_cg(Mx, b, x, tol=1e-10, sched=sch); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"{os.environ.get('TAG','')} {name}: {statistics.median(ts[1:]):.2f} ms, iters {rep['iterations']}, "
          f"us/iter {1000*statistics.median(ts[1:])/rep['iterations']:.1f}", flush=True)
