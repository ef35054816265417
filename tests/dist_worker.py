"""Worker for the NCCL-backend tests (tests/test_gpu_dist.py): rank RANK of WORLD solves the
row-partitioned 3D Poisson varcoef CG (scaled stepped schedule) with the NCCL backend and
writes its x slice and report to OUT_rank.npz.  The unique id travels through a file.
usage: python dist_worker.py RANK WORLD OUT_PREFIX [N] [cg|gmres]  (gmres: conv-diff N^3)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gse_inputs as gi
import paper_2411_04686_b200 as g

rank, world, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 24
solver = sys.argv[5] if len(sys.argv) > 5 else "cg"
torch.cuda.set_device(rank % torch.cuda.device_count())
uid_path = out + "_uid.bin"
if rank == 0:
    with open(uid_path + ".tmp", "wb") as f:
        f.write(g.gse_nccl_unique_id())
    os.replace(uid_path + ".tmp", uid_path)
t0 = time.time()
while not os.path.exists(uid_path):
    if time.time() - t0 > 60:
        raise SystemExit("no unique id")
    time.sleep(0.05)
uid = open(uid_path, "rb").read()
D = g.gse_dist_create(uid, rank, world, rank % torch.cuda.device_count())
n = N ** 3
planes = [round(i * N / world) * N * N for i in range(world + 1)]
r0, r1 = planes[rank], planes[rank + 1]
A = (gi.poisson3d(N, "varcoef", row_begin=r0, row_end=r1) if solver == "cg"
     else gi.convdiff3d(N, row_begin=r0, row_end=r1))
dev = lambda v: torch.from_numpy(v).cuda()
M = g.gse_encode_dist(D, dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val), r0, n)
b = gi.ones_rhs(A)
if solver == "cg":
    x, rep = g.gse_solve_cg(M, dev(b), tol=1e-10, sched=g.gse_default_schedule("cg", l=30, t=10, m=10))
else:
    x, rep = g.gse_solve_gmres(M, dev(b), tol=1e-10,
                               sched=g.gse_default_schedule("gmres", level_floor=(1e-3, 1e-8)))
np.savez(f"{out}_{rank}.npz", x=x.cpu().numpy(), rep=json.dumps(rep, default=list))
M.close()
D.close()
