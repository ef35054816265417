"""Per-kernel device time of one CG solve on C2 under torch.profiler (CUPTI activity
records: real concurrent timing, not ncu's serialised replay).  Prints per-kernel count,
mean duration, share, and the idle gaps between consecutive kernels.  Dev tool."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gse_inputs as gi, paper_2411_04686_b200 as g

N = int(os.environ.get("CG_N", "128"))
A = gi.poisson3d(N, os.environ.get("CG_VARIANT", "const"))
dev = lambda a: torch.from_numpy(a).cuda()
rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
b = dev(gi.ones_rhs(A))
M = g.gse_encode(rp, col, val, A.rows, A.cols)
x = torch.zeros(A.rows, dtype=torch.float64, device="cuda")
sch = g.gse_default_schedule("cg")
g.gse_solve_cg(M, b, x, tol=1e-10, sched=sch)  # warm-up (graphs built)
x.zero_(); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g.gse_solve_cg(M, b, x, tol=1e-10, sched=sch)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
kern = [e for e in evs if "Memcpy" not in e.name and "Memset" not in e.name]
tot = collections.defaultdict(float); cnt = collections.Counter()
gap = collections.defaultdict(float)
for i, e in enumerate(kern):
    d = e.time_range.end - e.time_range.start
    tot[e.name] += d; cnt[e.name] += 1
    if i:
        gp = e.time_range.start - kern[i - 1].time_range.end
        gap[e.name] += gp
span = kern[-1].time_range.end - kern[0].time_range.start
busy = sum(tot.values())
print(f"{os.environ.get('TAG','')} span {span/1000:.2f} ms, kernels busy {busy/1000:.2f} ms, "
      f"{len(kern)} launches")
for k in sorted(tot, key=lambda k: -tot[k])[:12]:
    print(f"  {k[:60]:60s} n={cnt[k]:5d} avg={tot[k]/cnt[k]:7.2f}us share={tot[k]/span*100:5.1f}% "
          f"gap_before_avg={gap[k]/cnt[k]:6.2f}us")
