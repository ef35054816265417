"""Where the bench step's time goes beyond encode + cached solve: first solve on a freshly
encoded matrix (workspace + graph build) vs a second solve on the same matrix."""
import time, statistics, torch, numpy as np
import gse_inputs as gi
import paper_2411_04686_b200 as g

A = gi.poisson3d(128)
dev = torch.device("cuda")
rp = torch.from_numpy(A.row_ptr.astype(np.int32)).to(dev)
col = torch.from_numpy(A.col).to(dev); val = torch.from_numpy(A.val).to(dev)
b = torch.from_numpy(gi.ones_rhs(A)).to(dev)
x = torch.zeros(A.rows, dtype=torch.float64, device=dev)
sched = g.gse_default_schedule("cg")
s = torch.cuda.current_stream()

def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(s); return e

rows = []
for it in range(8):
    torch.cuda.synchronize()
    h0 = time.perf_counter(); e0 = ev()
    M = g.gse_encode(rp, col, val, A.rows, A.cols, k_max=8)
    e1 = ev(); h1 = time.perf_counter()
    x.zero_(); g.gse_solve_cg(M, b, x, tol=1e-10, sched=sched)
    e2 = ev(); h2 = time.perf_counter()
    x.zero_(); g.gse_solve_cg(M, b, x, tol=1e-10, sched=sched)
    e3 = ev(); h3 = time.perf_counter()
    M.close()
    e4 = ev(); torch.cuda.synchronize(); h4 = time.perf_counter()
    rows.append([e0.elapsed_time(e1), e1.elapsed_time(e2), e2.elapsed_time(e3), e3.elapsed_time(e4),
                 (h1 - h0) * 1e3, (h2 - h1) * 1e3, (h3 - h2) * 1e3, (h4 - h3) * 1e3])
r = np.median(np.array(rows[3:]), axis=0)
print("gpu ms: encode %.3f first_solve %.3f second_solve %.3f close %.3f" % tuple(r[:4]))
print("host ms: encode %.3f first_solve %.3f second_solve %.3f close %.3f" % tuple(r[4:]))
