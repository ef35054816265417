"""Host-side cost of the C-ABI calls on C2 (enqueue time without sync, and wall time with
sync) next to their device time -- finds launch-path overheads that CUDA-event timing of
a step would absorb.  Dev tool."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gse_inputs as gi, paper_2411_04686_b200 as g

A = gi.poisson3d(int(os.environ.get("HO_N", "128")))
dev = lambda a: torch.from_numpy(a).cuda()
rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
b = dev(gi.ones_rhs(A))
M = g.gse_encode(rp, col, val, A.rows, A.cols)
x = torch.rand(A.cols, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
x32, y32 = x.float(), torch.empty(A.rows, dtype=torch.float32, device="cuda")


def host(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t_enq, t_wall = [], []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); t1 = time.perf_counter(); torch.cuda.synchronize()
        t2 = time.perf_counter()
        t_enq.append((t1 - t0) * 1e6); t_wall.append((t2 - t0) * 1e6)
    return statistics.median(t_enq), statistics.median(t_wall)


for name, fn in [
        ("spmv L1", lambda: g.gse_spmv(M, x, y, segments=1)),
        ("spmv L2", lambda: g.gse_spmv(M, x, y, segments=2)),
        ("spmv_f32 L1", lambda: g.gse_spmv_f32acc(M, x32, y32, segments=1)),
        ("spmv_f32 L2", lambda: g.gse_spmv_f32acc(M, x32, y32, segments=2)),
        ("encode+close", lambda: g.gse_encode(rp, col, val, A.rows, A.cols).close()),
        ("solve_cg (same M)", lambda: g.gse_solve_cg(M, b, torch.zeros_like(b), tol=1e-10,
                                                     sched=g.gse_default_schedule("cg"))),
]:
    e, w = host(fn, 5 if "solve" in name or "encode" in name else 20)
    print(f"{name:22s} enqueue {e:9.1f} us   wall {w:9.1f} us", flush=True)


def step():
    m = g.gse_encode(rp, col, val, A.rows, A.cols)
    xs = torch.zeros_like(b)
    g.gse_solve_cg(m, b, xs, tol=1e-10, sched=g.gse_default_schedule("cg"))
    m.close()


e, w = host(step, 5)
print(f"{'bench step':22s} enqueue {e:9.1f} us   wall {w:9.1f} us", flush=True)
