"""e2e step breakdown on configs[1]: pinned H2D of the CSR + b + x0 alone, D2H of x alone,
host x.zero_(), and the full C-ABI step with host buffers (as bench.py's e2e)."""
import time, statistics, torch, numpy as np
import gse_inputs as gi
import paper_2411_04686_b200 as g

A = gi.poisson3d(128)
dev = torch.device("cuda")
h = [torch.from_numpy(A.row_ptr.astype(np.int32)).pin_memory(), torch.from_numpy(A.col).pin_memory(),
     torch.from_numpy(A.val).pin_memory(), torch.from_numpy(gi.ones_rhs(A)).pin_memory(),
     torch.zeros(A.rows, dtype=torch.float64).pin_memory()]
d = [t.to(dev) for t in h]
nbytes = sum(t.numel() * t.element_size() for t in h)

def tm(fn, k=5):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3

def h2d():
    for a, b in zip(d, h):
        a.copy_(b, non_blocking=True)
t = tm(h2d); print("H2D %.1f MB: %.3f ms = %.1f GB/s" % (nbytes / 1e6, t, nbytes / t / 1e6))
t = tm(lambda: h[4].copy_(d[4], non_blocking=True)); print("D2H x 16.8 MB: %.3f ms" % t)
t = tm(lambda: h[4].zero_()); print("host x.zero_: %.3f ms" % t)
sched = g.gse_default_schedule("cg")
def step():
    M = g.gse_encode(h[0], h[1], h[2], A.rows, A.cols, k_max=8)
    h[4].zero_()
    g.gse_solve_cg(M, h[3], h[4], tol=1e-10, max_iters=20000, sched=sched)
    M.close()
step()
t = tm(step); print("e2e step: %.3f ms = %.2f solves/s" % (t, 1e3 / t))
def dstep():
    M = g.gse_encode(d[0], d[1], d[2], A.rows, A.cols, k_max=8)
    d[4].zero_()
    g.gse_solve_cg(M, d[3], d[4], tol=1e-10, max_iters=20000, sched=sched)
    M.close()
dstep()
t = tm(dstep); print("device step (host clock): %.3f ms" % t)
