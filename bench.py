#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the GSE-SEM hot path on B200.

Workload (default, every N): BASELINE.json configs[4], 3D Poisson 7-point 512^3
(n = 134,217,728, nnz = 937,951,232; 11.3 GB of GSE planes, far larger than the 126 MB L2),
b = A*1, x0 = 0.  It is the largest single-GPU configuration in BASELINE.json and the
scaling config.  One STEP = the whole hot path on it: gse_encode (histogram, table,
encode into head/tail1/tail2 planes, row-walk partition) then the stepped mixed-precision
CG solve to a TRUE relative residual <= 1e-10 (paper-default schedule + verify_at_full,
R16).  value = solves / s.  Every timed step must report converged with a true residual
<= tol, else the bench fails.

N > 1 (torchrun, one process per GPU): the same 512^3 problem is row-partitioned over the
N GPUs by z-slabs (gse_encode_dist: global table by histogram allreduce, local column
renumbering; CG with the NCCL halo exchange overlapped with the interior rows and
allreduced dots) -> "scaling": "strong".

Also in the line (N = 1, rank 0): the C5 SpMV segment sweep (GB/s, GFLOP/s, fraction of
the measured HBM peak per segment count, FP64 / FP32 accumulation, the CG's fused SpMV+dot
kernel back to back as in the CG loop, FP64-CSR comparator), the FP64-CSR CG on the same
GPU, the roofline of the dominant kernel, the end-to-end number through the C-ABI from
pinned host buffers, the oracle CPU baseline, SM clocks; and compact sub-objects for
configs[1] (C2 128^3 const: step, SpMV sweep), C2-shape varcoef stepped CG (where the
solver switches levels), configs[2] (power-law 10M rows SpMV segment sweep) and configs[3]
(conv-diff 256^3 GMRES(30)).  `--quick` skips the sub-objects.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gse|reference]
                  [--workload c5|c2] [--quick]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("GSE SpMV GB/s & GFLOP/s (frac of HBM peak) per segment count; "
          "CG time-to-1e-10")
WORKLOADS = {"c5": (512, "configs[4]"), "c2": (128, "configs[1]")}
TOL = 1e-10
R29_C = 0.1  # the R29 trigger constant of the stepped_r29 sub-results (R29)
R30_C = 3.0  # R29 constant of the kept-direction (R30) sub-result


def unit_for(N):
    return f"CG solves to 1e-10 per s (encode + stepped CG, 3D Poisson {N}^3)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gse", choices=["gse", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="const", choices=["const", "varcoef"])
    ap.add_argument("--quick", action="store_true",
                    help="skip the configs[1]/[2]/[3] sub-objects")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--dist1", action="store_true",
                    help="diagnostic: the distributed (NCCL) path even at N = 1 (1-rank communicator)")
    a = ap.parse_args()
    a.N, a.cfg = WORKLOADS[a.workload]
    return a


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def r3(v):
    """3 significant digits (keeps the JSON line short enough for the driver's tail)"""
    if v is None or not isinstance(v, float) or v == 0 or not np.isfinite(v):
        return v
    return float(f"{v:.3g}") if abs(v) < 1000 else round(v, 1) if abs(v) < 1e5 else round(v)


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.path = index, None, None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # nvidia-smi's start-up (NVML init, driver locks) can stall CUDA calls for tens of
        # ms: wait for its first sample so that happens before the timed region
        t0 = time.time()
        while self.proc and time.time() - t0 < 10.0:
            if self.proc.poll() is not None or os.path.getsize(self.path) > 0:
                break
            time.sleep(0.05)
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nme, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nme)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------ distributed plumbing
def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "reference":
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    return world, rank, local, pg


def max_over_ranks(v: float, pg, device=None):
    if pg is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


def slab_partition(N, P):
    """z-slab row partition: rank i owns planes [round(iN/P), round((i+1)N/P))"""
    return [round(i * N / P) * N * N for i in range(P + 1)]


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _config(args, n, nnz, world):
    return {"workload": f"{args.cfg} 3D Poisson 7-point {args.N}^3 ({args.variant}): gse_encode + "
                        f"stepped GSE CG to a true relative residual of 1e-10",
            "n": int(n), "nnz": int(nnz), "k_max": 8, "tol": TOL,
            "schedule": "paper default CG (l=3000,t=250,m=500) + verify_at_full (R16)",
            "inputs": "CSR resident in HBM before the timed region",
            "l2": ("inputs larger than L2 (planes 11.3 GB); L2 also flushed before every timed step"
                   if args.N >= 256 else "flushed before every timed step (256 MiB write + read)"),
            "parallelism": (f"row-partitioned x{world} z-slabs (NCCL halo + allreduce)"
                            if world > 1 else "single GPU")}


def l2_flush(buf, i):
    """Evict L2: write a 256 MiB buffer (2x the 126 MB L2), then read it back once, so the
    write-backs of the dirty lines happen here and not inside the next timed region."""
    buf.fill_(float(i))
    buf.sum()


def time_cuda(fn, reps, stream, flush):
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for i in range(reps):
        if flush is not None:
            l2_flush(flush, i)
        evs[i][0].record(stream)
        fn()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in evs]


def time_b2b(fn, reps, stream, flush):
    """mean per call of `reps` back-to-back calls (after one flush), CUDA events"""
    import torch
    fn()
    l2_flush(flush, 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


# ------------------------------------------------------------------ inputs on the device
def device_poisson(args, r0, r1, dev, keep_host=False):
    """rows [r0, r1) of the Poisson matrix (gse_inputs recipe, generated in chunks by a
    thread pool) -> device CSR (row_ptr int32 local, col int32, val f64) and b = A*1."""
    import torch
    import gse_inputs as gi
    rps, cols, vals, bs = [], [], [], []
    base = 0
    for _, A in gi.poisson3d_chunks(args.N, args.variant, r0, r1):
        rps.append(torch.from_numpy((A.row_ptr[:-1] + base).astype(np.int32)).to(dev))
        cols.append(torch.from_numpy(A.col).to(dev))
        vals.append(torch.from_numpy(A.val).to(dev))
        bs.append(torch.from_numpy(gi.ones_rhs(A)).to(dev))
        base += A.nnz
    rp = torch.cat(rps + [torch.tensor([base], dtype=torch.int32, device=dev)])
    del rps
    col, val, b = torch.cat(cols), torch.cat(vals), torch.cat(bs)
    return rp, col, val, b


# ------------------------------------------------------------------ reference arm (oracle)
def oracle_iters(O, R, b, iters):
    """`iters` level-1 CG iterations of the oracle (the level the stepped solve runs at on
    this head-exact workload); returns seconds per iteration"""
    s = O.schedule("cg", verify_at_full=0)
    t0 = time.perf_counter()
    _, rep = O.cg(R, b, tol=1e-300, max_iters=iters, sched=s)
    return (time.perf_counter() - t0) / max(rep.iterations, 1)


def oracle_count_c2(O, gi, variant):
    """The oracle's own iteration count for the workload: the FP64 CG count at 128^3 (a full
    oracle solve, seconds) scaled linearly with N (3D Poisson CG iterations grow ~ N: 2.85 N
    measured N = 16..64)."""
    A = gi.poisson3d(128, variant)
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    return O.cg(F, gi.ones_rhs(A), tol=TOL)[1].iterations


def host_poisson(args):
    import gse_inputs as gi
    parts = list(gi.poisson3d_chunks(args.N, args.variant))
    nnz = sum(A.nnz for _, A in parts)
    rp = np.zeros(args.N ** 3 + 1, np.int64)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    b = np.empty(args.N ** 3)
    o = 0
    for r0, A in parts:
        rp[r0:r0 + A.rows] = A.row_ptr[:-1] + o
        col[o:o + A.nnz] = A.col
        val[o:o + A.nnz] = A.val
        b[r0:r0 + A.rows] = gi.ones_rhs(A)
        o += A.nnz
    rp[-1] = o
    return gi.Csr(args.N ** 3, args.N ** 3, rp, col, val, "poisson"), b


def run_reference(args, world, rank, pg):
    """The oracle (plain C, OpenMP rows) on the host cores of rank 0 (other ranks exit).
    Step = a bounded sample of the workload: k level-1 oracle CG iterations.  value = 1 /
    (oracle encode + t_iteration x the oracle's iteration count for the workload);
    ms_per_step = the measured sample time per step (what the timed region really ran)."""
    if rank != 0:
        return
    import gse_inputs as gi
    import oracle as O
    # all host cores (torchrun exports OMP_NUM_THREADS=1 to every rank; only rank 0 runs here)
    cores = O.set_threads(len(os.sched_getaffinity(0)))
    t0 = time.perf_counter()
    if args.N == 128:
        A = gi.poisson3d(128, args.variant)
        b = gi.ones_rhs(A)
    else:
        A, b = host_poisson(args)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    t_enc = time.perf_counter() - t0
    n128 = oracle_count_c2(O, gi, args.variant)
    iters_full = int(round(n128 * args.N / 128))
    t1 = oracle_iters(O, R, b, 1 if args.N > 256 else 8)
    times = []
    # (GSE_REF_FULL_S: the budget for running full solves instead of sampled iterations)
    if t_enc + t1 * iters_full < float(os.environ.get("GSE_REF_FULL_S", "30")):
        # a full oracle solve costs seconds: each step IS the workload (oracle encode +
        # stepped CG to a true relative residual of 1e-10), nothing extrapolated
        its = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            Ri = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
            _, rep = O.cg(Ri, b, tol=TOL, sched=O.schedule("cg"))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
                its.append(rep.iterations)
        value = 1.0 / statistics.mean(times)
        sample = (f"each step a full oracle solve: encode + stepped CG (paper defaults) to a true "
                  f"relative residual of 1e-10 ({its[-1]} iterations)")
    else:
        # iterations per step: the whole (W + K)-step run takes ~2 minutes of CG work
        k = max(1, min(50, int(120.0 / max(t1, 1e-6) / (args.warmup + args.steps))))
        per_it = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            ti = oracle_iters(O, R, b, k)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
                per_it.append(ti)
        t_it = statistics.mean(per_it)
        value = 1.0 / (t_enc + t_it * iters_full)
        sample = (f"per step {k} level-1 oracle CG iterations ({t_it * 1e3:.0f} ms each; "
                  f"{k * args.steps} timed in all); value = 1 / (oracle encode {t_enc:.1f} s + "
                  f"{iters_full} iterations), {iters_full} = the oracle's FP64 CG count at 128^3 "
                  f"({n128}) x N/128")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": unit_for(args.N),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(times) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {**_config(args, A.rows, A.nnz, world), "inputs": "host memory",
                       "parallelism": f"the plain CPU oracle on rank 0's host cores ({cores} threads)"},
            "cpu_baseline": {"value": value, "unit": unit_for(args.N), "cores": cores,
                             "kind": "oracle", "cpu": cpu_model(), "sample": sample,
                             "generate_s": round(t_gen, 1)},
            "e2e": {"value": value, "unit": unit_for(args.N), "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GSE arm
def check_rep(rep, where):
    if not (rep["converged"] and rep["rel_residual_true"] <= TOL * (1 + 1e-12)):
        raise SystemExit(f"bench: {where} did not converge to {TOL}: {rep}")


def run_gse(args, world, rank, local, pg):
    import torch
    import paper_2411_04686_b200 as g

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    hbm_peak, peak_src = peaks()
    n_glob = args.N ** 3
    nnz_glob = 7 * args.N ** 3 - 6 * args.N ** 2
    part = slab_partition(args.N, world)
    r0, r1 = part[rank], part[rank + 1]
    rp, col, val, b = device_poisson(args, r0, r1, dev)
    n_loc = r1 - r0
    x = torch.zeros(n_loc, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    sched = g.gse_default_schedule("cg")

    D = None
    if world > 1:
        import torch.distributed as tdist
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(g.gse_nccl_unique_id()), dtype=torch.uint8))
        tdist.broadcast(uid, 0)
        D = g.gse_dist_create(bytes(uid.cpu().numpy()), rank, world, local)
    elif args.dist1:
        D = g.gse_dist_create(g.gse_nccl_unique_id(), 0, 1, local)

    def encode(rp_, col_, val_, **kw):
        if D is None:
            return g.gse_encode(rp_, col_, val_, n_loc, n_glob, k_max=8, **kw)
        return g.gse_encode_dist(D, rp_, col_, val_, r0, n_glob, **kw)

    def step():
        M = encode(rp, col, val)
        x.zero_()
        _, rep = g.gse_solve_cg(M, b, x, tol=TOL, max_iters=20000, sched=sched)
        M.close()
        return rep

    for _ in range(args.warmup):
        check_rep(step(), "warm-up step")
    torch.cuda.synchronize()
    barrier(pg)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    reps = []
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        barrier(pg)
        for i in range(args.steps):
            l2_flush(flush, i)
            ev[i][0].record(stream)
            reps.append(step())
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    clocks = clk.summary()
    for i, rep in enumerate(reps):  # every timed solve must have converged (true residual)
        check_rep(rep, f"timed step {i}")
    step_ms = [s.elapsed_time(e) for s, e in ev]
    total_ms = max_over_ranks(sum(step_ms), pg, dev)
    barrier(pg)
    rep = reps[-1]
    value = args.steps / (total_ms * 1e-3)  # one (row-partitioned) problem per step

    line = {
        "metric": METRIC, "value": value, "unit": unit_for(args.N), "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gse_inputs recipe, DESIGN.md 4)",
        "config": _config(args, n_glob, nnz_glob, world)}
    sub = {}
    if args.dist1:
        line["config"]["parallelism"] = "distributed path, 1-rank NCCL communicator (diagnostic)"
    extra = None
    if world == 1 and not args.no_sweep and not args.dist1:
        # right after the timed steps, in the same thermal / power state
        extra = main_sweep(args, rp, col, val, b, n_loc, dev, stream, flush, hbm_peak)
    if world == 1 and rank == 0 and not args.quick and not args.no_sweep and not args.dist1:
        sub = sub_workloads(dev, stream, flush, hbm_peak)
    e2e = None if args.no_e2e else e2e_measure(args, rp, col, val, b, dev, stream, encode)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        del flush
        cpu = cpu_baseline(args, rp, col, val, b, rep["iterations"])
    launches = estimate_launches(rep, world) * args.steps
    if D is not None:
        barrier(pg)
        D.close()
    if rank != 0:
        return
    line.update(sub)
    line["solve"] = {"iterations": rep["iterations"], "iters_per_level": rep["iters_per_level"],
                     "switch_iter": rep["switch_iter"],
                     "rel_residual_true": r3(rep["rel_residual_true"]),
                     "step_ms_each": [round(t, 1) for t in step_ms]}
    if extra is not None:
        line["solve"]["fp64_csr_iterations"] = extra["cg_fp64_iters"]
        line["time_to_1e-10_ms"] = {
            "stepped_gse_step": r3(statistics.median(step_ms)),
            "stepped_gse_solve_only": r3(extra["cg_gse_ms"]), "encode": r3(extra["encode_ms"]),
            "fp64_csr_cg": r3(extra["cg_fp64_ms"]),
            "speedup_vs_fp64_csr": r3(extra["cg_fp64_ms"] / extra["cg_gse_ms"])}
        line["spmv_sweep"] = extra["spmv"]
        dot = extra["dot_l1"]
        line["roofline"] = {
            "bound": "hbm", "achieved": r3(dot["GBps"]), "peak": hbm_peak, "unit": "GB/s",
            "frac": r3(dot["GBps"] / hbm_peak), "traffic": _profiled_traffic(),
            "kernel": "k_spmv_rw<L=1,DOT>: the CG's fused level-1 SpMV + p.q",
            "algorithmic_bytes_per_launch": dot["bytes"], "avg_launch_us": r3(dot["us"]),
            "peak_source": peak_src,
            "timing": "gse_spmv_dot back to back right after the timed steps, CUDA events on "
                      "its stream, mean per launch"}
    line["e2e"] = e2e
    line["cpu_baseline"] = cpu
    line["gpu_launches"] = launches
    line["clocks"] = clocks
    print(json.dumps(line, separators=(",", ":")), flush=True)


def estimate_launches(rep, world):
    """Kernels of this library launched per step (ncu launch list, profiles/launches_c5_r02h.txt):
    gse_encode 17 (row_ptr, histogram, table, encode, group statistics, block / tile flags,
    2 x 3 compaction kernels, 2 descriptor fills, row bitmap, chunk rows), CG setup 3 (||b||,
    SpMV, residual), 3 per iteration (SpMV + dot, update, xpay), 2 per level switch or
    verification (SpMV + residual) and 2 for the final true residual.  The single-GPU graph
    body holds 8 iterations (GSE_CG_UNROLL): the kernels of the pass that sees the event still
    launch (and return at once), so each level's count rounds up to a multiple of 8.  The
    distributed path adds the plan (7) and per iteration the halo pack and the event kernel."""
    if world == 1:
        u = int(os.environ.get("GSE_CG_UNROLL", "8"))
        u = min(max(u, 1), 32)
        its = sum(-(-i // u) * u for i in rep["iters_per_level"] if i > 0)
        return 17 + 3 + 2 * rep["n_switches"] + 3 * its + 2
    its = -(-rep["iterations"] // 16) * 16  # captured batches of 16
    return 17 + 7 + 3 + 6 * its + 2 * rep["n_switches"] + 2


def _profiled_traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    summary (profiles/ncu_summary_c5_*.json), or None"""
    import glob
    found = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_c5_r*.json")))
    if found:
        try:
            return json.load(open(found[-1])).get("k_spmv_dot_L1", {}).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def spmv_entry(byt, nnz, us, peak):
    t = us * 1e-6
    return {"us": r3(us), "GBps": r3(byt / t / 1e9), "GFLOPs": r3(2 * nnz / t / 1e9),
            "frac": r3(byt / t / 1e9 / peak)}


def main_sweep(args, rp, col, val, b, n, dev, stream, flush, hbm_peak):
    """C5 (or C2) on one GPU: SpMV per segment count (cold: one launch after an L2 flush),
    FP32 accumulation, the CG's fused SpMV+dot back to back, FP64-CSR; CG solve-only times."""
    import torch
    import paper_2411_04686_b200 as g
    nnz = int(col.numel())
    M = g.gse_encode(rp, col, val, n, n)
    x = torch.rand(n, dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    x32, y32 = x.float(), torch.empty(n, dtype=torch.float32, device=dev)
    dd = torch.empty(1, dtype=torch.float64, device=dev)
    out = {}
    rows_b = 4 * (n + 1)
    reps = 5 if n > 2 ** 24 else 20

    def cold(fn):
        fn()
        return statistics.mean(time_cuda(fn, reps, stream, flush))

    for L, s_l in ((1, 2), (2, 4), (3, 8)):
        byt = nnz * (4 + s_l) + rows_b + 16 * n
        out[f"L{L}"] = spmv_entry(byt, nnz, 1e3 * cold(lambda: g.gse_spmv(M, x, y, segments=L)), hbm_peak)
    for L, s_l in ((1, 2), (2, 4), (3, 8)):
        byt = nnz * (4 + s_l) + rows_b + 8 * n
        out[f"L{L}_f32acc"] = spmv_entry(
            byt, nnz, 1e3 * cold(lambda: g.gse_spmv_f32acc(M, x32, y32, segments=L)), hbm_peak)
    b1 = nnz * 6 + rows_b + 16 * n
    us_dot = 1e3 * time_b2b(lambda: g.gse_spmv_dot(M, x, y, segments=1, dot=dd), 4 * reps,
                            stream, flush)
    out["L1_dot_cg_loop"] = spmv_entry(b1, nnz, us_dot, hbm_peak)
    dot = {"bytes": b1, "us": us_dot, "GBps": b1 / (us_dot * 1e-6) / 1e9}
    del x32, y32
    # the paper's FP16 / BF16 storage baselines: 6 B/nnz, FP64 products and sums
    for kind in ("fp16", "bf16"):
        H = g.gse_half_matrix(rp, col, val, n, n, kind=kind)
        out[kind] = spmv_entry(nnz * 6 + rows_b + 16 * n, nnz,
                               1e3 * cold(lambda: g.gse_spmv(H, x, y, segments=3)), hbm_peak)
        H.close()
    F = g.gse_fp64_matrix(rp, col, val, n, n)
    out["fp64_csr"] = spmv_entry(nnz * 12 + rows_b + 16 * n, nnz,
                                 1e3 * cold(lambda: g.gse_spmv(F, x, y, segments=3)), hbm_peak)
    del x, y
    xs = torch.zeros(n, dtype=torch.float64, device=dev)
    sched = g.gse_default_schedule("cg")

    def solve(A, s):
        xs.zero_()
        rep = g.gse_solve_cg(A, b, xs, tol=TOL, max_iters=20000, sched=s)[1]
        check_rep(rep, "sweep solve")
        return rep

    solve(M, sched)
    t_gse = statistics.median(time_cuda(lambda: solve(M, sched), 2, stream, flush))
    rf = solve(F, None)
    t_f64 = statistics.median(time_cuda(lambda: solve(F, None), 2, stream, flush))
    M.close()
    F.close()

    def enc():
        g.gse_encode(rp, col, val, n, n).close()

    t_enc = statistics.median(time_cuda(enc, 3, stream, flush))
    torch.cuda.empty_cache()
    return {"spmv": out, "dot_l1": dot, "cg_gse_ms": t_gse, "cg_fp64_ms": t_f64,
            "cg_fp64_iters": rf["iterations"], "encode_ms": t_enc}


# ------------------------------------------------------------------ sub-workloads (N = 1)
def _dev_csr(A, dev):
    import torch
    return (torch.from_numpy(A.row_ptr.astype(np.int32)).to(dev), torch.from_numpy(A.col).to(dev),
            torch.from_numpy(A.val).to(dev))


def _solve_ms(g, stream, flush, solver, M, b, x, sched, tol=TOL):
    """one warm solve (graphs built), then one timed solve after an L2 flush"""
    import torch
    fn = g.gse_solve_cg if solver == "cg" else g.gse_solve_gmres
    x.zero_()
    fn(M, b, x, tol=tol, sched=sched)
    x.zero_()
    l2_flush(flush, 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rep = fn(M, b, x, tol=tol, sched=sched)[1]
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), rep


def sub_workloads(dev, stream, flush, peak):
    """the auxiliary sub-objects; a failure in one is recorded in the line, never fatal to
    the headline"""
    import torch
    out = {}
    for key, fn in (("c2", lambda: sub_c2(dev, stream, flush, peak)),
                    ("c2_varcoef_cg", lambda: sub_c2_varcoef(dev, stream, flush)),
                    ("c3_spmv", lambda: sub_c3(dev, stream, flush, peak)),
                    ("c4_gmres", lambda: sub_c4(dev, stream, flush))):
        try:
            out[key] = fn()
        except Exception as e:  # noqa: BLE001 -- reported, not hidden
            out[key] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
        torch.cuda.empty_cache()
    return out


def sub_c2(dev, stream, flush, peak):
    """configs[1] (3D Poisson 128^3 const): step (encode + stepped CG) and SpMV sweep"""
    import torch
    import gse_inputs as gi
    import paper_2411_04686_b200 as g
    A = gi.poisson3d(128)
    rp, col, val = _dev_csr(A, dev)
    b = torch.from_numpy(gi.ones_rhs(A)).to(dev)
    n, nnz = A.rows, A.nnz
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    sched = g.gse_default_schedule("cg")

    def step():
        M = g.gse_encode(rp, col, val, n, n)
        x.zero_()
        rep = g.gse_solve_cg(M, b, x, tol=TOL, sched=sched)[1]
        M.close()
        return rep

    step()
    t = statistics.median(time_cuda(step, 5, stream, flush))
    M = g.gse_encode(rp, col, val, n, n)
    F = g.gse_fp64_matrix(rp, col, val, n, n)
    t64, r64 = _solve_ms(g, stream, flush, "cg", F, b, x, None)
    tg, rg = _solve_ms(g, stream, flush, "cg", M, b, x, sched)
    xv = torch.rand(n, dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    dd = torch.empty(1, dtype=torch.float64, device=dev)
    sw = {}
    for L, s_l in ((1, 2), (2, 4), (3, 8)):
        byt = nnz * (4 + s_l) + 4 * (n + 1) + 16 * n
        fn = lambda: g.gse_spmv(M, xv, y, segments=L)
        fn()
        sw[f"L{L}"] = spmv_entry(byt, nnz, 1e3 * statistics.mean(time_cuda(fn, 20, stream, flush)), peak)
    b1 = nnz * 6 + 4 * (n + 1) + 16 * n
    sw["L1_dot_cg_loop"] = spmv_entry(b1, nnz, 1e3 * time_b2b(
        lambda: g.gse_spmv_dot(M, xv, y, segments=1, dot=dd), 80, stream, flush), peak)
    fn = lambda: g.gse_spmv(F, xv, y, segments=3)
    fn()
    sw["fp64_csr"] = spmv_entry(nnz * 12 + 4 * (n + 1) + 16 * n, nnz,
                                1e3 * statistics.mean(time_cuda(fn, 20, stream, flush)), peak)
    # the paper's 16-bit storage baselines and its GSE-SEM* projection (Eq. 7,
    # the FP16 solver's time per iteration x the GSE iteration count)
    half = {}
    for kind in ("fp16", "bf16"):
        H = g.gse_half_matrix(rp, col, val, n, n, kind=kind)
        th, rh = _solve_ms(g, stream, flush, "cg", H, b, x, None)
        half[kind] = {"ms": r3(th), "it": rh["iterations"],
                      "res_vs_rounded_matrix": r3(rh["rel_residual_true"])}
        H.close()
    eq7 = half["fp16"]["ms"] / max(half["fp16"]["it"], 1) * rg["iterations"]
    M.close()
    F.close()
    return {"solves_per_s": r3(1e3 / t), "step_ms": r3(t), "cg_ms": r3(tg), "iters": rg["iterations"],
            "fp64_csr_cg_ms": r3(t64), "fp64_iters": r64["iterations"],
            "speedup_vs_fp64_csr": r3(t64 / tg), "half_storage_cg": half,
            "gse_sem_star_eq7_ms": r3(eq7), "gse_sem_star_x_fp64": r3(t64 / eq7), "spmv": sw}


def sub_c2_varcoef(dev, stream, flush):
    """C2 shape with varcoef values (head-lossy: the stepped solver switches levels): time
    to 1e-10 for the paper-default schedule, the level floors (R17), the R29 perturbation
    trigger and FP64-CSR"""
    import torch
    import gse_inputs as gi
    import paper_2411_04686_b200 as g
    A = gi.poisson3d(128, "varcoef")
    rp, col, val = _dev_csr(A, dev)
    b = torch.from_numpy(gi.ones_rhs(A)).to(dev)
    n = A.rows
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    M = g.gse_encode(rp, col, val, n, n)
    F = g.gse_fp64_matrix(rp, col, val, n, n)
    out = {}
    t64, r64 = _solve_ms(g, stream, flush, "cg", F, b, x, None)
    out["fp64_csr"] = {"ms": r3(t64), "it": r64["iterations"]}
    for name, s in (("stepped_default", g.gse_default_schedule("cg")),
                    ("stepped_floors", g.gse_default_schedule("cg", level_floor=(1e-3, 1e-8))),
                    ("stepped_r29", g.gse_default_schedule("cg", perturb_c=R29_C)),
                    # R29 trigger from level 2 with the R30 kept direction (R30)
                    ("stepped_r29_keep_l2", g.gse_default_schedule(
                        "cg", perturb_c=R30_C, start_level=2, cg_keep_direction=1))):
        t, r = _solve_ms(g, stream, flush, "cg", M, b, x, s)
        out[name] = {"ms": r3(t), "it": r["iterations"], "per_level": r["iters_per_level"],
                     "res": r3(r["rel_residual_true"]), "x_fp64": r3(t64 / t)}
    M.close()
    F.close()
    return out


def sub_c3(dev, stream, flush, peak):
    """configs[2]: power-law SPD (10M rows, ~200M nnz; DESIGN.md recipe) SpMV segment sweep
    (window kernel), FP64 and FP32 accumulation, FP64-CSR; cold launches"""
    import torch
    import gse_inputs as gi
    import paper_2411_04686_b200 as g
    A = gi.powerlaw_spd(10_000_000, seed=42)
    n, nnz = A.rows, A.nnz
    rp, col, val = _dev_csr(A, dev)
    del A
    x = torch.from_numpy(gi.uniform_vec(n, seed=7)).to(dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    x32, y32 = x.float(), torch.empty(n, dtype=torch.float32, device=dev)
    out = {"n": n, "nnz": nnz}

    def rec(key, fn, byt):
        fn()
        out[key] = spmv_entry(byt, nnz, 1e3 * statistics.mean(time_cuda(fn, 10, stream, flush)), peak)

    M = g.gse_encode(rp, col, val, n, n)
    rows_b = 4 * (n + 1)
    for L, s_l in ((1, 2), (2, 4), (3, 8)):
        rec(f"L{L}", lambda: g.gse_spmv(M, x, y, segments=L), nnz * (4 + s_l) + rows_b + 16 * n)
    for L, s_l in ((1, 2), (2, 4), (3, 8)):
        rec(f"L{L}_f32acc", lambda: g.gse_spmv_f32acc(M, x32, y32, segments=L),
            nnz * (4 + s_l) + rows_b + 8 * n)
    M.close()
    F = g.gse_fp64_matrix(rp, col, val, n, n)
    rec("fp64_csr", lambda: g.gse_spmv(F, x, y, segments=3), nnz * 12 + rows_b + 16 * n)
    F.close()
    return out


def sub_c4(dev, stream, flush):
    """configs[3]: conv-diff 256^3 restarted GMRES(30) to a true relative residual of 1e-10
    (and the paper's 1e-6): FP64-CSR vs stepped GSE (paper defaults, level floors, R29, R29
    from level 2)"""
    import torch
    import gse_inputs as gi
    import paper_2411_04686_b200 as g
    A = gi.convdiff3d(256)
    n = A.rows
    rp, col, val = _dev_csr(A, dev)
    b = torch.from_numpy(gi.ones_rhs(A)).to(dev)
    del A
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    M = g.gse_encode(rp, col, val, n, n)
    F = g.gse_fp64_matrix(rp, col, val, n, n)
    out = {}
    for tol, tag in ((1e-10, ""), (1e-6, "_tol1e-6")):
        t64, r64 = _solve_ms(g, stream, flush, "gmres", F, b, x, None, tol)
        out["fp64_csr" + tag] = {"ms": r3(t64), "it": r64["iterations"]}
        runs = [("stepped_default", g.gse_default_schedule("gmres"))]
        if tol == 1e-10:
            runs.append(("stepped_floors", g.gse_default_schedule("gmres", level_floor=(1e-3, 1e-8))))
            runs.append(("stepped_r29", g.gse_default_schedule("gmres", perturb_c=R29_C)))
            # the R29 trigger from level 2 (head + tail1): one switch, near the end
            runs.append(("stepped_r29_l2", g.gse_default_schedule("gmres", perturb_c=R29_C,
                                                                  start_level=2)))
        for name, s in runs:
            t, r = _solve_ms(g, stream, flush, "gmres", M, b, x, s, tol)
            out[name + tag] = {"ms": r3(t), "it": r["iterations"], "per_level": r["iters_per_level"],
                               "x_fp64": r3(t64 / t)}
    M.close()
    F.close()
    return out


# ------------------------------------------------------------------ end to end, CPU baseline
def e2e_measure(args, rp, col, val, b, dev, stream, encode):
    """The same step through the C-ABI with HOST (pinned) buffers: H2D of the CSR, b and x0
    inside the calls, D2H of x at the end (host wall clock around the synchronous calls)."""
    import torch
    import paper_2411_04686_b200 as g
    hp = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)
    rp_h, col_h, val_h, b_h = hp(rp), hp(col), hp(val), hp(b)
    x = torch.zeros(b_h.numel(), dtype=torch.float64).pin_memory()
    sched = g.gse_default_schedule("cg")
    s = stream.cuda_stream

    def step():
        M = encode(rp_h, col_h, val_h, stream=s)
        x.zero_()
        rep = g.gse_solve_cg(M, b_h, x, tol=TOL, max_iters=20000, sched=sched, stream=s)[1]
        M.close()
        check_rep(rep, "e2e step")

    step()
    ts = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    h2d = rp_h.numel() * 4 + col_h.numel() * 4 + val_h.numel() * 8 + b_h.numel() * 8 + x.numel() * 8
    return {"value": 1.0 / t, "unit": unit_for(args.N), "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(x.numel() * 8), "ms_per_step": r3(t * 1e3),
            "timer": "host wall clock around the synchronous C-ABI calls (rank 0)"}


def cpu_baseline(args, rp, col, val, b, iters_gpu):
    """The oracle as it stands on the host cores: oracle encode of the whole matrix + a
    bounded number of level-1 CG iterations (~20 s), extrapolated to the GPU solve's
    iteration count; plus the single-thread time per iteration."""
    import torch
    import gse_inputs as gi
    import oracle as O
    del torch
    A = gi.Csr(int(b.numel()), int(b.numel()), rp.cpu().numpy().astype(np.int64),
               col.cpu().numpy(), val.cpu().numpy())
    bh = b.cpu().numpy()
    cores = O.set_threads(len(os.sched_getaffinity(0)))
    t0 = time.perf_counter()
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    te = time.perf_counter() - t0
    t1 = oracle_iters(O, R, bh, 1)
    k = max(2, min(200, int(20.0 / max(t1, 1e-6))))
    ti = oracle_iters(O, R, bh, k)
    O.set_threads(1)
    t_single = oracle_iters(O, R, bh, 1 if t1 * cores > 2.0 else 3)
    O.set_threads(cores)
    t = te + ti * iters_gpu
    return {"value": 1.0 / t, "unit": unit_for(args.N), "cores": cores, "kind": "oracle",
            "cpu": cpu_model(),
            "sample": f"oracle encode of the whole matrix ({te:.1f} s) + {k} level-1 CG iterations "
                      f"({ti * 1e3:.0f} ms each), extrapolated to the GPU solve's {iters_gpu} "
                      f"iterations; OpenMP rows in SpMV/encode, sequential dots",
            "single_thread_ms_per_iteration": r3(t_single * 1e3)}


def main():
    args = parse()
    world, rank, local, pg = dist_init(args)
    args.gpus = world if world > 1 else args.gpus
    if args.impl == "reference":
        run_reference(args, world, rank, pg)
    else:
        run_gse(args, world, rank, local, pg)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
