"""debug: per-shard table encode + CG on the thread backend (P from argv), daemon threads,
report per-rank exceptions after a timeout instead of hanging."""
import os, sys, threading, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gse_inputs as gi, paper_2411_04686_b200 as g
P = int(sys.argv[1]) if len(sys.argv) > 1 else 3
phase = sys.argv[2] if len(sys.argv) > 2 else "both"
def partition(n, P): return [round(i * n / P) for i in range(P + 1)]
def slab(A, a, b):
    rp = (A.row_ptr[a:b + 1] - A.row_ptr[a]).astype(np.int64); sl = slice(A.row_ptr[a], A.row_ptr[b])
    return rp, A.col[sl].copy(), A.val[sl].copy()
A = gi.powerlaw_spd(20000, seed=6)
sc = np.where(np.arange(A.rows) >= A.rows // 2, 2.0 ** 3, 1.0)
rows_of = np.repeat(np.arange(A.rows), np.diff(A.row_ptr))
A = gi.Csr(A.rows, A.cols, A.row_ptr, A.col, A.val * sc[rows_of] * sc[A.col], "scaled")
B = gi.poisson3d(20, "varcoef")
sb = np.where(np.arange(B.rows) >= B.rows // 2, 2.0 ** 3, 1.0)
rows_b = np.repeat(np.arange(B.rows), np.diff(B.row_ptr))
B = gi.Csr(B.rows, B.cols, B.row_ptr, B.col, B.val * sb[rows_b] * sb[B.col], "scaled")
bB = gi.ones_rhs(B)
rr, rc = partition(A.rows, P), partition(B.rows, P)
x = gi.uniform_vec(A.cols, seed=2)
grp = g.gse_dist_thread_group_create(P)
log = []
def body(r):
    try:
        torch.cuda.set_device(0)
        D = g.gse_dist_create_thread(grp, r, 0)
        st = torch.cuda.Stream()
        dev = lambda v: torch.from_numpy(v).cuda()
        with torch.cuda.stream(st):
            if phase in ("both", "a"):
                a, b = rr[r], rr[r + 1]
                rp, col, val = slab(A, a, b)
                M = g.gse_encode_dist(D, dev(rp), dev(col), dev(val), a, A.rows, stream=st.cuda_stream, per_shard_table=True)
                log.append((r, "encA", M.info["table"]))
                for L in (1, 2, 3):
                    g.gse_spmv(M, dev(x[a:b].copy()), segments=L, stream=st.cuda_stream)
                log.append((r, "spmvA"))
                M.close()
                log.append((r, "closeA"))
            if phase in ("both", "b"):
                c, d = rc[r], rc[r + 1]
                rp2, col2, val2 = slab(B, c, d)
                M2 = g.gse_encode_dist(D, dev(rp2), dev(col2), dev(val2), c, B.rows, stream=st.cuda_stream, per_shard_table=True)
                log.append((r, "encB", M2.info["table"]))
                _, rep = g.gse_solve_cg(M2, dev(bB[c:d].copy()), tol=1e-10, stream=st.cuda_stream,
                                        sched=g.gse_default_schedule("cg", l=30, t=10, m=10))
                log.append((r, "cg", rep))
                M2.close()
        st.synchronize()
        D.close()
        log.append((r, "done"))
    except Exception:
        log.append((r, "EXC", traceback.format_exc()))
th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(P)]
for t in th: t.start()
t0 = time.time()
while time.time() - t0 < 90 and any(t.is_alive() for t in th): time.sleep(1)
for e in log: print(e, flush=True)
print("alive:", [t.is_alive() for t in th], flush=True)
os._exit(0)
