import json, os, sys, statistics
sys.path.insert(0, '/root/repo')
import torch, bench, gse_inputs as gi, paper_2411_04686_b200 as g
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
A = gi.poisson3d(128, "varcoef"); rp, col, val = bench._dev_csr(A, dev)
b = torch.from_numpy(gi.ones_rhs(A)).to(dev); n = A.rows
x = torch.zeros(n, dtype=torch.float64, device=dev)
M = g.gse_encode(rp, col, val, n, n); F = g.gse_fp64_matrix(rp, col, val, n, n)
out = {}
for name, MM, s in (("fp64", F, None), ("keep_l2", M, g.gse_default_schedule("cg", perturb_c=3.0, start_level=2, cg_keep_direction=1)),
                    ("restart_l2", M, g.gse_default_schedule("cg", perturb_c=3.0, start_level=2)),
                    ("fixed_l2", M, g.fixed_schedule(2))):
    ts = [bench._solve_ms(g, stream, flush, "cg", MM, b, x, s)[0] for _ in range(8)]
    out[name] = [round(t, 2) for t in ts]
print(json.dumps(out))
