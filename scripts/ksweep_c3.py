"""the paper's k-sweep (section 4.2; Figs. 4-5 are stripped
from PAPER.md, only "k = 8 is best on average" survives): encode configs[2] (the
power-law SPD, 10M rows, ~200M nnz) with k_max in {1, 2, 4, 8, 16, 32, 64} shared
exponents and report, per k, the GSE SpMV time / GB/s at 1, 2, 3 segments and the error of
the result against the FP64-CSR SpMV (max abs and max relative-to-row-scale), with
x = 1 as in the paper.  The "exact" column is the fraction of rows whose level-L
result equals the FP64 result bit for bit (the paper's "identical to FP64" count).
One JSON line.  CUDA events, L2 flushed before each launch."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gse_inputs as gi
import paper_2411_04686_b200 as g

n = int(os.environ.get("C3_N", "10000000"))
ks = [int(k) for k in os.environ.get("KS", "1,2,4,8,16,32,64").split(",")]
t0 = time.time()
A = gi.powerlaw_spd(n, seed=42)
tgen = time.time() - t0
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pp = os.path.join(root, "MEASURED_PEAKS.json")
peak = json.load(open(pp))["hbm_gbs"] if os.path.exists(pp) else 6650.0
dev = lambda a: torch.from_numpy(a).cuda()
rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
x = torch.ones(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def timeit(fn, reps=10):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    fn()
    for i in range(reps):
        flush.fill_(i)
        flush.sum()
        evs[i][0].record()
        fn()
        evs[i][1].record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in evs) * 1e-3


F = g.gse_fp64_matrix(rp, col, val, A.rows, A.cols)
g.gse_spmv(F, x, y, segments=3)
y64 = y.clone()
absval = torch.from_numpy(np.abs(A.val)).cuda()
Fa = g.gse_fp64_matrix(rp, col, absval, A.rows, A.cols)
scale = g.gse_spmv(Fa, x, torch.empty_like(y), segments=3)  # sum_j |a_ij| x_j
del Fa
t = timeit(lambda: g.gse_spmv(F, x, y, segments=3))
res = {"fp64_csr": {"us": round(t * 1e6, 1),
                    "GBps": round((A.nnz * 12 + 4 * (n + 1) + 16 * n) / t / 1e9, 1)}}
F.close()
for k in ks:
    M = g.gse_encode(rp, col, val, A.rows, A.cols, k_max=k)
    info = M.info
    r = {"table_len": info["table_len"], "ei_in_column": info["ei_in_column"],
         "n_zero_values": info["n_zero_values"]}
    for L, s_l in ((1, 2), (2, 4), (3, 8)):
        t = timeit(lambda: g.gse_spmv(M, x, y, segments=L))
        side = 0 if info["ei_in_column"] else 1
        b = A.nnz * (4 + s_l + side) + 4 * (n + 1) + 16 * n
        g.gse_spmv(M, x, y, segments=L)
        err = (y - y64).abs()
        r[f"L{L}"] = {"us": round(t * 1e6, 1), "GBps": round(b / t / 1e9, 1),
                      "frac_hbm": round(b / t / 1e9 / peak, 3),
                      "max_abs_err": float(err.max()),
                      "max_rel_err": float((err / scale.clamp_min(1e-300)).max()),
                      "rows_exact": float((y == y64).double().mean())}
    res[f"k{k}"] = r
    M.close()
    torch.cuda.synchronize()
print(json.dumps({"config": "configs[2] power-law SPD k-sweep (P:372-402)", "n": n,
                  "nnz": int(A.nnz), "gen_s": round(tgen, 1), "x": "ones (P:299)",
                  "peak_GBps": peak, "sweep": res}))
