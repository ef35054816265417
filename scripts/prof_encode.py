"""Encode of configs[1] (3D Poisson 128^3) a few times: for the ncu launch list and for
event timing of the whole gse_encode call."""
import sys, torch, numpy as np
import gse_inputs as gi
import paper_2411_04686_b200 as g

A = gi.poisson3d(128)
dev = torch.device("cuda")
rp = torch.from_numpy(A.row_ptr.astype(np.int32)).to(dev)
col = torch.from_numpy(A.col).to(dev); val = torch.from_numpy(A.val).to(dev)
s = torch.cuda.current_stream()
ts = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    M = g.gse_encode(rp, col, val, A.rows, A.cols, k_max=8)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    M.close()
print("encode ms", ["%.3f" % t for t in ts], "median %.3f" % float(np.median(ts[2:])))
