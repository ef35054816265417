"""configs[2]: SuiteSparse-shaped power-law SPD (10M rows, ~200M nnz) SpMV segment sweep.
Prints one JSON line: GB/s / GFLOP/s / fraction of the measured HBM peak per segment count
(FP64 and FP32 accumulation) and the FP64-CSR comparator, plus a sampled parity check of
2000 rows against the oracle (same seeded inputs).  CUDA events, L2 flushed per launch."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gse_inputs as gi, oracle as O, paper_2411_04686_b200 as g

n = int(os.environ.get("C3_N", "10000000"))
t0 = time.time()
A = gi.powerlaw_spd(n, seed=42)
tgen = time.time() - t0
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
dev = lambda a: torch.from_numpy(a).cuda()
rp, col, val = dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val)
M = g.gse_encode(rp, col, val, A.rows, A.cols)
F = g.gse_fp64_matrix(rp, col, val, A.rows, A.cols)
x = torch.from_numpy(gi.uniform_vec(n, seed=7)).cuda()
y = torch.empty(n, dtype=torch.float64, device="cuda")
x32, y32 = x.float(), torch.empty(n, dtype=torch.float32, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
nnz = A.nnz

def timeit(fn, reps=10):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    fn()
    for i in range(reps):
        flush.fill_(i); evs[i][0].record(); fn(); evs[i][1].record()
    torch.cuda.synchronize()
    return statistics.mean(s.elapsed_time(e) for s, e in evs) * 1e-3

res = {}
for L, s_l in ((1, 2), (2, 4), (3, 8)):
    for acc in ("f64", "f32"):
        if acc == "f64":
            t = timeit(lambda: g.gse_spmv(M, x, y, segments=L)); vb = 16 * n
        else:
            t = timeit(lambda: g.gse_spmv_f32acc(M, x32, y32, segments=L)); vb = 8 * n
        b = nnz * (4 + s_l) + 4 * (n + 1) + vb
        res[f"L{L}_{acc}"] = {"us": round(t * 1e6, 1), "GBps": round(b / t / 1e9, 1),
                              "GFLOPs": round(2 * nnz / t / 1e9, 1), "frac_hbm": round(b / t / 1e9 / peak, 3)}
t = timeit(lambda: g.gse_spmv(F, x, y, segments=3)); b = nnz * 12 + 4 * (n + 1) + 16 * n
res["fp64_csr"] = {"us": round(t * 1e6, 1), "GBps": round(b / t / 1e9, 1), "GFLOPs": round(2 * nnz / t / 1e9, 1),
                   "frac_hbm": round(b / t / 1e9 / peak, 3)}
# sampled parity vs the oracle (rows re-encoded by the oracle with the full-matrix table)
rng = np.random.default_rng(0)
rows = np.unique(rng.integers(0, n, 2000))
P = g.gse_matrix_copy_planes(M)
sel = np.concatenate([np.arange(A.row_ptr[r], A.row_ptr[r + 1]) for r in rows])
rps = np.zeros(rows.size + 1, np.int64); np.cumsum(A.row_ptr[rows + 1] - A.row_ptr[rows], out=rps[1:])
R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)  # oracle, full matrix
ok = list(R.table) == list(P["table"])
for k in ("col_ei", "head", "tail1", "tail2"):
    ok &= bool(np.array_equal(P[k][sel], getattr(R, k)[sel]))
xh = x.cpu().numpy()
for L in (1, 2, 3):
    yg = g.gse_spmv(M, x, y, segments=L).cpu().numpy()[rows]
    subp = O.GseCsr(rows.size, n, sel.size, rps, R.col_ei[sel].copy(), None, R.head[sel].copy(),
                    R.tail1[sel].copy(), R.tail2[sel].copy(), R.table, 3, True)
    yo = O.spmv_gse(subp, xh, L)
    absP = O.GseCsr(rows.size, n, sel.size, rps, subp.col_ei, None, subp.head & np.uint16(0x7FFF),
                    subp.tail1, subp.tail2, subp.table, 3, True)
    ok &= bool(np.all(np.abs(yg - yo) <= 1e-12 * O.spmv_gse(absP, np.abs(xh), L)))
print(json.dumps({"config": "configs[2] power-law SPD", "n": n, "nnz": nnz, "gen_s": round(tgen, 1),
                  "mode": "SP" if M.info["n_blocks"] else "?", "sampled_parity_ok": ok, "sweep": res,
                  "peak_GBps": peak}))
