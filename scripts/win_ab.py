"""A/B of the SpMV kernels on configs[2] (power-law SPD, 10M rows, ~200M nnz): the window
kernel (spmv_win.cu, default for irregular rows) against the strided-products kernel
(GSE_SPMV_MODE=sp).  One JSON line: per level / accumulation us, GB/s, fraction of the
measured HBM peak (algorithmic bytes, L2 flushed before every launch) plus back-to-back
times, and a sampled parity check of the window kernel against the oracle."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gse_inputs as gi, oracle as O, paper_2411_04686_b200 as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(os.environ.get("C3_N", "10000000"))
modes = os.environ.get("MODES", "win,sp").split(",")
t0 = time.time()
A = gi.powerlaw_spd(n, seed=42)
tgen = time.time() - t0
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
dev = lambda a: torch.from_numpy(a).cuda()
rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
x = torch.from_numpy(gi.uniform_vec(n, seed=7)).cuda()
y = torch.empty(n, dtype=torch.float64, device="cuda")
x32, y32 = x.float(), torch.empty(n, dtype=torch.float32, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
nnz = A.nnz


def timeit(fn, reps=10, cold=True):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    fn()
    for i in range(reps):
        if cold:
            flush.fill_(i)
            flush.sum()
        evs[i][0].record(); fn(); evs[i][1].record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in evs) * 1e-3


out = {"n": n, "nnz": nnz, "gen_s": round(tgen, 1), "peak_GBps": peak}
Ms = {}
for mode in modes:
    if mode == "sp":
        os.environ["GSE_SPMV_MODE"] = "sp"
    else:
        os.environ.pop("GSE_SPMV_MODE", None)
    te = time.time()
    M = g.gse_encode(rp, col, val, A.rows, A.cols)
    torch.cuda.synchronize()
    F = g.gse_fp64_matrix(rp, col, val, A.rows, A.cols)
    res = {"spmv_mode": M.info["spmv_mode"], "encode_s": round(time.time() - te, 3)}
    for L, s_l in ((1, 2), (2, 4), (3, 8)):
        for acc in ("f64", "f32"):
            if acc == "f64":
                fn = lambda: g.gse_spmv(M, x, y, segments=L); vb = 16 * n
            else:
                fn = lambda: g.gse_spmv_f32acc(M, x32, y32, segments=L); vb = 8 * n
            b = nnz * (4 + s_l) + 4 * (n + 1) + vb
            t = timeit(fn)
            tw = timeit(fn, reps=20, cold=False)
            res[f"L{L}_{acc}"] = {"us": round(t * 1e6, 1), "frac": round(b / t / 1e9 / peak, 3),
                                  "us_b2b": round(tw * 1e6, 1), "frac_b2b": round(b / tw / 1e9 / peak, 3)}
    b = nnz * 12 + 4 * (n + 1) + 16 * n
    t = timeit(lambda: g.gse_spmv(F, x, y, segments=3))
    res["fp64_csr"] = {"us": round(t * 1e6, 1), "frac": round(b / t / 1e9 / peak, 3)}
    out[mode] = res
    Ms[mode] = M
    print(json.dumps({mode: res}), flush=True)

# sampled parity of every mode against the oracle
rng = np.random.default_rng(0)
rows = np.unique(rng.integers(0, n, 3000))
sel = np.concatenate([np.arange(A.row_ptr[r], A.row_ptr[r + 1]) for r in rows])
rps = np.zeros(rows.size + 1, np.int64); np.cumsum(A.row_ptr[rows + 1] - A.row_ptr[rows], out=rps[1:])
R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
xh = x.cpu().numpy()
for mode, M in Ms.items():
    ok = True
    for L in (1, 2, 3):
        yg = g.gse_spmv(M, x, y, segments=L).cpu().numpy()[rows]
        subp = O.GseCsr(rows.size, n, sel.size, rps, R.col_ei[sel].copy(), None, R.head[sel].copy(),
                        R.tail1[sel].copy(), R.tail2[sel].copy(), R.table, 3, True)
        yo = O.spmv_gse(subp, xh, L)
        absP = O.GseCsr(rows.size, n, sel.size, rps, subp.col_ei, None, subp.head & np.uint16(0x7FFF),
                        subp.tail1, subp.tail2, subp.table, 3, True)
        ok &= bool(np.all(np.abs(yg - yo) <= 1e-12 * O.spmv_gse(absP, np.abs(xh), L)))
    out[mode]["sampled_parity_ok"] = ok
print(json.dumps(out))
