"""Measure L2-resident streaming bandwidth (copy / axpy of 16-64 MB vectors, no flush)."""
import torch, statistics, json
def t(fn, reps=50):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3
for mb in (8, 16, 32, 64, 512):
    n = mb * 1024 * 1024 // 8
    a = torch.rand(n, dtype=torch.float64, device="cuda"); b = torch.rand_like(a); c = torch.empty_like(a)
    tc = t(lambda: c.copy_(a))
    ta = t(lambda: torch.add(a, b, alpha=0.5, out=c))
    print(json.dumps({"MB_per_vec": mb, "copy_GBps": round(2*n*8/tc/1e9), "axpy_GBps": round(3*n*8/ta/1e9)}))
