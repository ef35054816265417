"""Pins of the oracle SpMV, residual monitor and CG / GMRES(30) drivers against what the
paper and the mathematics fix:
  * SPEC worked examples (golden file), brute-force dense matvec, exactness of integer /
    dyadic data, level-3 == FP64 bitwise for d <= 11, head-exact Poisson;
  * Eq. 3-6 / Conditions 1-3 on hand windows; section 4.4.1 defaults;
  * CG/GMRES solutions against dense direct solves (numpy.linalg.solve), iteration counts
    against an independent implementation (scipy.sparse.linalg.cg), Krylov exactness
    (diagonal matrices), <= n-step convergence on SPD systems.
"""
import json
import math
import os

import numpy as np
import pytest

import gse_inputs as gi
import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def enc(A, k=8):
    return O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, k)


def f64(A):
    return O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)


def bitseq(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


# ------------------------------------------------------------------ SpMV
@pytest.mark.parametrize("ex", GOLD["spmv"], ids=lambda e: e["cite"])
def test_spmv_examples(ex):
    A = gi.from_dense(np.array(ex["dense"]))
    x = np.array(ex["x"])
    if "level" not in ex:
        assert list(O.spmv_fp64(f64(A), x)) == ex["y"]
    for L in ([ex["level"]] if "level" in ex else [1, 2, 3]):
        assert list(O.spmv_gse(enc(A), x, L)) == ex["y"]


@pytest.mark.parametrize("kind", ["classes", "wide", "mixed"])
def test_spmv_brute_force_dense(kind):
    """y = D_L x where D_L is the dense matrix of per-element decoded values."""
    A = gi.random_csr(40, 37, 6, seed=11, value_kind=kind, empty_rows=0.1)
    G = enc(A)
    x = gi.uniform_vec(A.cols, seed=7)
    for L in (1, 2, 3):
        dv = O.decode_all(G, L)
        D = np.zeros((A.rows, A.cols))
        r = np.repeat(np.arange(A.rows), np.diff(A.row_ptr))
        D[r, A.col] = dv
        y = O.spmv_gse(G, x, L)
        ref = D @ x
        scale = np.abs(D) @ np.abs(x)
        assert np.all(np.abs(y - ref) <= 1e-14 * scale + 0.0)
        assert np.all(y[np.diff(A.row_ptr) == 0] == 0.0)


def test_spmv_fp64_brute_force_and_integer_exact():
    A = gi.random_csr(60, 50, 8, seed=12)
    x = gi.uniform_vec(A.cols)
    y = O.spmv_fp64(f64(A), x)
    scale = np.abs(A.dense()) @ np.abs(x)
    assert np.all(np.abs(y - A.dense() @ x) <= 1e-14 * scale)
    B = gi.Csr(A.rows, A.cols, A.row_ptr, A.col, np.round(A.val * 8))
    xi = np.arange(B.cols, dtype=float) - 20
    assert np.array_equal(O.spmv_fp64(f64(B), xi), B.dense() @ xi)  # integers: exact


@pytest.mark.parametrize("seed", range(10))
def test_spmv_level3_bitwise_equals_fp64_when_d_le_11(seed):
    """S:296 / S:468: every d <= 11 -> level 3 decode is lossless and the accumulation order
    is identical, so spmv_gse(3) == spmv_fp64 bitwise."""
    A = gi.random_csr(100, 100, 7, seed=seed, exps=[1013, 1018, 1022, 1023])
    G = enc(A)
    assert max(G.table) - 1013 <= 11
    x = gi.uniform_vec(A.cols, seed=seed)
    assert bitseq(O.spmv_gse(G, x, 3), O.spmv_fp64(f64(A), x))


@pytest.mark.parametrize("mk", [lambda: gi.poisson2d(32), lambda: gi.poisson3d(12)])
def test_constant_poisson_exact_in_head(mk):
    """4/-1 and 6/-1 have <= 2 significant bits at d = 1: all levels bitwise equal FP64."""
    A = mk()
    G = enc(A)
    x = gi.uniform_vec(A.cols)
    ref = O.spmv_fp64(f64(A), x)
    for L in (1, 2, 3):
        assert bitseq(O.spmv_gse(G, x, L), ref)


def test_spmv_1x1_head_error_equals_codec_error():
    """on a 1x1 matrix the head-only SpMV error equals the codec truncation error."""
    rng = np.random.default_rng(8)
    for v in rng.uniform(-3, 3, 200):
        A = gi.from_dense(np.array([[v]]))
        G = enc(A)
        w, ei = O.encode_value(v, G.table)
        h, _, _ = O.segment(w)
        dec1 = O.decode(O.assemble(h, 0, 0, 1), ei, G.table)
        assert O.spmv_gse(G, np.array([1.0]), 1)[0] == dec1


def test_spmv_level_monotone_error_ones():
    """with x = 1, max abs error vs FP64 is non-increasing in the level."""
    A = gi.poisson2d(32, "varcoef")
    G = enc(A)
    x = np.ones(A.cols)
    ref = O.spmv_fp64(f64(A), x)
    errs = [np.abs(O.spmv_gse(G, x, L) - ref).max() for L in (1, 2, 3)]
    assert errs[0] >= errs[1] >= errs[2] and errs[0] > 0


# ------------------------------------------------------------------ monitor
def test_monitor_examples():
    for ex in GOLD["monitor"]["rsd"]:
        assert O.rsd(ex["window"]) == pytest.approx(ex["value"], abs=1e-15)
    for ex in GOLD["monitor"]["n_dec"]:
        assert O.n_dec(ex["window"]) == ex["value"]
    for ex in GOLD["monitor"]["rel_dec"]:
        assert O.rel_dec(ex["window"], ex["t"]) == pytest.approx(ex["value"], abs=1e-15)


def test_monitor_properties():
    w = np.array([4.0, 1.0, 3.0, 2.0, 5.0, 0.5])
    t = w.size - 1
    # Eq. 3 evaluated from its definition: population std / mean of resid[j-t..j-1]
    head = w[:t]
    assert O.rsd(w, t) == pytest.approx(math.sqrt(((head - head.mean()) ** 2).mean()) / head.mean())
    assert O.rsd(7.5 * w, t) == pytest.approx(O.rsd(w, t))  # scale invariance
    assert O.n_dec(np.linspace(1, 0.1, 11)) == 10  # strictly decreasing window -> t
    assert O.n_dec(np.full(11, 0.3)) == 0  # ties score 0 (Eq. 5)
    assert O.rsd(np.zeros(5)) == 0.0  # avg < 1e-300 guard


def test_conditions():
    t = 10
    const = np.full(t + 1, 0.2)
    assert O.should_escalate(const, 0.5, 5, 0.45)  # C3: nDec = 0
    halving = 0.5 ** np.arange(t + 1)
    assert not O.should_escalate(halving, 0.5, 5, 0.45)
    osc = np.array([1.0, 0.05, 1.0, 0.05, 1.0, 0.05, 1.0, 0.05, 1.0, 0.05, 1.0])
    assert O.rsd(osc, t) > 0.9 and O.n_dec(osc) == 5
    assert O.should_escalate(osc, 0.5, 6, 0.45)  # C1: RSD > lim and nDec < nDec_lim
    assert not O.should_escalate(osc, 0.95, 6, -10.0)
    slow = np.linspace(1.0, 0.9, t + 1)  # nDec = t, relDec = 0.09
    assert O.should_escalate(slow, 10.0, 5, 0.45)  # C2
    assert not O.should_escalate(slow, 10.0, 5, 0.05)
    assert not O.should_escalate(np.zeros(t + 1), 0.5, 5, 0.45)  # zero leading residual


def test_defaults_equal_section_4_4_1():
    d = GOLD["defaults"]
    for solver in ("cg", "gmres"):
        s = O.default_schedule(solver)
        for k in ("l", "t", "m", "ndec_limit"):
            assert getattr(s, k) == d[solver][k]
        for k in ("rsd_limit", "reldec_limit"):
            assert getattr(s, k) == d[solver][k]
        assert s.enabled == 1 and s.start_level == 1 and s.max_level == 3


# ------------------------------------------------------------------ CG
@pytest.mark.parametrize("ex", GOLD["cg"], ids=lambda e: e["cite"])
def test_cg_examples(ex):
    A = gi.from_dense(np.array(ex["dense"]))
    x, rep = O.cg(f64(A), np.array(ex["b"]), tol=1e-12, max_iters=100)
    assert rep.converged
    if "x_num" in ex:
        want = np.array(ex["x_num"]) / ex["x_den"]
        assert np.abs(x - want).max() <= 1e-10 and rep.iterations <= ex["max_iters_allowed"]
    else:
        assert rep.iterations == ex["iterations"] and np.allclose(x, ex["b"])


@pytest.mark.parametrize("n", [5, 17, 40, 64])
def test_cg_spd_converges_within_3n_and_matches_direct(n):
    A = gi.spd_small(n, seed=n)
    b = gi.uniform_vec(n, seed=n)
    x, rep = O.cg(f64(A), b, tol=1e-12, max_iters=3 * n)
    assert rep.converged and rep.iterations <= 3 * n
    xd = np.linalg.solve(A.dense(), b)
    assert np.abs(x - xd).max() <= 1e-9 * np.abs(xd).max()


@pytest.mark.parametrize("N", [8, 16])
def test_cg_iterations_match_independent_scipy(N):
    """Iteration count of the oracle's plain CG equals scipy.sparse.linalg.cg (independent
    implementation, same criterion ||r_k|| <= tol ||b||) within +-1 on 3D Poisson."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    A = gi.poisson3d(N)
    b = gi.ones_rhs(A)
    x, rep = O.cg(f64(A), b, tol=1e-10, max_iters=5000)
    S = sp.csr_matrix((A.val, A.col, A.row_ptr), shape=(A.rows, A.cols))
    its = []
    xs, info = spla.cg(S, b, rtol=1e-10, atol=0.0, maxiter=5000, callback=lambda xk: its.append(1))
    assert info == 0 and abs(len(its) - rep.iterations) <= 1
    assert np.abs(x - 1.0).max() < 1e-7  # b = A 1 -> x = 1


def test_cg_breakdown_on_indefinite():
    A = gi.from_dense(np.array([[1.0, 0.0], [0.0, -1.0]]))
    _, rep = O.cg(f64(A), np.array([1.0, 1.0]), tol=1e-10)
    assert rep.status == O.NUMERICAL_ABORT


def test_cg_zero_rhs():
    A = gi.poisson2d(4)
    x, rep = O.cg(f64(A), np.zeros(16), x0=np.ones(16))
    assert rep.converged and rep.iterations == 0 and np.all(x == 0)


# ------------------------------------------------------------------ GMRES
@pytest.mark.parametrize("ex", GOLD["gmres"], ids=lambda e: e["cite"])
def test_gmres_examples(ex):
    A = gi.from_dense(np.array(ex["dense"]))
    x, rep = O.gmres(f64(A), np.array(ex["b"]), tol=1e-12)
    assert rep.converged and rep.iterations == ex["iterations"] and np.allclose(x, ex["x"])


@pytest.mark.parametrize("k", [1, 3, 7])
def test_gmres_diagonal_krylov_exactness(k):
    """diagonal A with k distinct eigenvalues -> converges within k inner steps."""
    n = 50
    rng = np.random.default_rng(k)
    eig = rng.uniform(1, 10, k)[rng.integers(0, k, n)]
    A = gi.from_dense(np.diag(eig))
    x, rep = O.gmres(f64(A), rng.uniform(-1, 1, n), tol=1e-12)
    assert rep.converged and rep.iterations <= k


@pytest.mark.parametrize("N", [6, 10])
def test_gmres_matches_direct_solve(N):
    A = gi.convdiff3d(N)
    b = gi.uniform_vec(A.rows, seed=N)
    x, rep = O.gmres(f64(A), b, tol=1e-11, restart=30)
    assert rep.converged and rep.rel_residual_true <= 1e-11 * 1.01
    xd = np.linalg.solve(A.dense(), b)
    assert np.abs(x - xd).max() <= 1e-8 * np.abs(xd).max()


def test_gmres_full_equals_fp64_when_d_le_11():
    """identical inner-iteration count and bitwise-identical iterate."""
    A = gi.random_csr(80, 80, 5, seed=3, exps=[1020, 1022, 1023])
    A = gi.Csr(A.rows, A.cols, A.row_ptr, A.col, A.val)  # add a strong diagonal
    d = A.dense() + 12 * np.eye(80)
    A = gi.from_dense(d)
    b = gi.uniform_vec(80)
    x1, r1 = O.gmres(f64(A), b, tol=1e-12)
    x2, r2 = O.gmres(enc(A), b, tol=1e-12, sched=O.fixed_schedule(3))
    assert r1.iterations == r2.iterations and bitseq(x1, x2)


# ------------------------------------------------------------------ stepped driver
def test_stepped_cg_no_switch_when_head_exact():
    """Constant Poisson is exact in the head: the stepped solve runs at level 1 only and
    the level-3 verification (R16) accepts it; iterations equal FP64 CG."""
    A = gi.poisson3d(10)
    b = gi.ones_rhs(A)
    _, r64 = O.cg(f64(A), b, tol=1e-10)
    x, rep = O.cg(enc(A), b, tol=1e-10, sched=O.schedule("cg"))
    assert rep.converged and rep.n_switches == 0 and rep.iters_per_level == (r64.iterations, 0, 0)
    assert rep.rel_residual_true <= 1e-10


@pytest.mark.parametrize("solver", ["cg", "gmres"])
def test_stepped_stall_escalates_and_converges(solver):
    """head-only truncation stalls above tol -> >= 1 switch, monotone tag, true
    residual <= tol (scaled schedule l=30, t=10, m=10)."""
    A = gi.poisson2d(32, "varcoef") if solver == "cg" else gi.convdiff3d(10)
    b = gi.ones_rhs(A)
    G = enc(A)
    s = O.schedule(solver, l=30, t=10, m=10)
    run = O.cg if solver == "cg" else O.gmres
    x, rep = run(G, b, tol=1e-10, sched=s)
    assert rep.converged and rep.n_switches >= 1 and rep.rel_residual_true <= 1e-10
    assert list(rep.switch_to_level) == sorted(rep.switch_to_level)
    assert list(rep.switch_iter) == sorted(rep.switch_iter)
    # without verification the head-only run "converges" on A_1 but not on A (R16)
    s0 = O.schedule(solver, verify_at_full=0)
    _, rep0 = run(G, b, tol=1e-10, sched=s0)
    assert rep0.converged and rep0.n_switches == 0 and rep0.rel_residual_true > 1e-8


def test_stepped_forced_escalation_reaches_full():
    """l=0, m=1, nDec_limit=t+1 -> level 3 within 2 checks."""
    A = gi.poisson2d(16, "varcoef")
    b = gi.ones_rhs(A)
    t = 5
    s = O.schedule("cg", l=0, t=t, m=1, ndec_limit=t + 1, rsd_limit=-1.0)
    _, rep = O.cg(enc(A), b, tol=1e-10, sched=s)
    assert rep.n_switches == 2 and rep.switch_to_level == (2, 3)
    assert rep.switch_iter == (t + 1, t + 2)


@pytest.mark.parametrize("solver", ["cg", "gmres"])
def test_level_floors(solver):
    """R17 level floors (build heuristic, off by default): a floor above every residual
    escalates after the first iteration at each level (switches at iterations 1 and 2, then
    the full-precision solve converges); a floor below every residual never fires (the same
    solve as without floors); floors between act before the monitor's first check at l."""
    A = gi.poisson2d(24, "varcoef") if solver == "cg" else gi.convdiff3d(8)
    b = gi.ones_rhs(A)
    G = enc(A)
    run = O.cg if solver == "cg" else O.gmres
    _, rep = run(G, b, tol=1e-10, sched=O.schedule(solver, level_floor=(1e300, 1e300)))
    assert rep.switch_iter == (1, 2) and rep.switch_to_level == (2, 3)
    assert rep.converged and rep.rel_residual_true <= 1e-10
    _, r0 = run(G, b, tol=1e-10, sched=O.schedule(solver))
    _, r1 = run(G, b, tol=1e-10, sched=O.schedule(solver, level_floor=(1e-300, 1e-300)))
    assert (r1.iterations, r1.switch_iter) == (r0.iterations, r0.switch_iter)
    _, rf = run(G, b, tol=1e-10, sched=O.schedule(solver, level_floor=(1e-3, 1e-8)))
    assert rf.converged and rf.n_switches == 2 and rf.rel_residual_true <= 1e-10
    assert rf.switch_iter[0] < r0.switch_iter[0]  # before the head-only solve "converges"


# ------------------------------------------------------------------ R29 perturbation trigger
def _two_bit_rows_matrix(seed=4):
    """rows holding a_i values +-(1 + 2^-20) and b_i values +-(1 + 2^-40): with the table
    {1024} (d = 1) the head keeps 15 fraction bits and tail1 16 more, so per value
    |dec_3 - dec_1| = 2^-20 (first kind) or 2^-40 (second), |dec_3 - dec_2| = 0 or 2^-40."""
    rng = np.random.default_rng(seed)
    rows = 40
    a = rng.integers(0, 9, rows)
    bb = rng.integers(0, 9, rows)
    lens = a + bb
    rp = np.zeros(rows + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    cols, vals = [], []
    for i in range(rows):
        c = np.sort(rng.choice(60, lens[i], replace=False))
        v = np.concatenate([np.full(a[i], 1 + 2.0 ** -20), np.full(bb[i], 1 + 2.0 ** -40)])
        v = rng.permutation(v) * rng.choice([-1.0, 1.0], lens[i])
        cols.append(c)
        vals.append(v)
    A = gi.Csr(rows, 60, rp, np.concatenate(cols).astype(np.int32), np.concatenate(vals))
    return A, a, bb


def test_perturbation_bounds_closed_form():
    """R29 eta_L = max_i sum_j |dec_3 - dec_L|: closed form on a matrix whose truncation
    errors are known exactly per value; 0 on the head-exact Poisson stencil."""
    A, a, bb = _two_bit_rows_matrix()
    G = enc(A)
    assert list(G.table) == [1024]
    e1, e2 = O.perturbation_bounds(G)
    assert e1 == max(a * 2.0 ** -20 + bb * 2.0 ** -40)
    assert e2 == max(bb * 2.0 ** -40)
    assert O.perturbation_bounds(enc(gi.poisson3d(6))) == (0.0, 0.0)


def test_perturbation_bound_is_the_row_sum_of_the_level_gap():
    """eta_L >= |(A_3 - A_L) s|_inf for every sign vector s (with equality for the row's own
    signs), checked with the decoded values (dense) on a lossy matrix"""
    A = gi.poisson2d(12, "varcoef")
    G = enc(A)
    eta = O.perturbation_bounds(G)
    d3 = gi.Csr(A.rows, A.cols, A.row_ptr, A.col, O.decode_all(G, 3)).dense()
    for L in (1, 2):
        dL = gi.Csr(A.rows, A.cols, A.row_ptr, A.col, O.decode_all(G, L)).dense()
        E = d3 - dL
        assert np.all(E * np.sign(d3) >= 0)  # truncation toward zero
        assert abs(np.abs(E).sum(axis=1).max() - eta[L - 1]) <= 1e-15 * eta[L - 1]
        assert eta[L - 1] > 0


@pytest.mark.parametrize("solver", ["cg", "gmres"])
def test_perturbation_trigger_behaviour(solver):
    """R29: c = 0 is the default solve; a huge c escalates at the first check where ||x|| > 0
    (CG: iteration 2, then 3; GMRES: the first inner step of the second cycle, then the
    next); c = 0.1 switches before the head-only solve 'converges' and still reaches 1e-10"""
    A = gi.poisson3d(12, "varcoef") if solver == "cg" else gi.convdiff3d(10)
    b = gi.ones_rhs(A)
    G = enc(A)
    run = O.cg if solver == "cg" else O.gmres
    _, r0 = run(G, b, tol=1e-10, sched=O.schedule(solver))
    _, rz = run(G, b, tol=1e-10, sched=O.schedule(solver, perturb_c=0.0))
    assert (rz.iterations, rz.switch_iter) == (r0.iterations, r0.switch_iter)
    _, rb = run(G, b, tol=1e-10, sched=O.schedule(solver, perturb_c=1e300))
    first = 2 if solver == "cg" else 31
    assert rb.switch_iter == (first, first + 1) and rb.switch_to_level == (2, 3)
    assert rb.converged and rb.rel_residual_true <= 1e-10
    _, rc = run(G, b, tol=1e-10, sched=O.schedule(solver, perturb_c=0.1))
    assert rc.converged and rc.n_switches == 2 and rc.rel_residual_true <= 1e-10
    assert rc.switch_iter[0] < r0.switch_iter[0]
    assert rc.iterations < r0.iterations


@pytest.mark.parametrize("keep,c", [(0, 0.1), (1, 0.1), (1, 3.0)])
def test_perturbation_trigger_matches_independent_numpy_cg(keep, c):
    """The oracle's R29 switch points against a plain numpy CG on the decoded level
    matrices (scipy CSR products, BLAS dots) with the same rule: escalate when
    ||r||/||b|| <= c eta_L ||x_{j-1}|| / ||b||; at a switch r = b - A_new x and either the
    R15 restart p = r or the R30 kept direction p = r + (r.r / rr_{j-1}) p."""
    import scipy.sparse as sp
    A = gi.poisson3d(10, "varcoef")
    G = enc(A)
    b = gi.ones_rhs(A)
    tol = 1e-10
    eta = O.perturbation_bounds(G)
    mats = {L: sp.csr_matrix((O.decode_all(G, L), A.col, A.row_ptr), shape=(A.rows, A.cols))
            for L in (1, 2, 3)}
    nb = np.linalg.norm(b)
    x = np.zeros(A.rows)
    L, r = 1, b.copy()
    p, rr, sw, j = r.copy(), r @ r, [], 0
    while j < 2000:
        j += 1
        q = mats[L] @ p
        xx = x @ x
        al = rr / (p @ q)
        x = x + al * p
        r = r - al * q
        rn = r @ r
        res = np.sqrt(rn) / nb
        if res <= tol:
            if L == 3 or np.linalg.norm(b - mats[3] @ x) / nb <= tol:
                break
            esc = True
        else:
            esc = L < 3 and xx > 0 and res <= c * eta[L - 1] * np.sqrt(xx) / nb
        if esc:
            L += 1
            sw.append(j)
            r = b - mats[L] @ x
            if keep:
                rn = r @ r
                p = r + (rn / rr) * p
                rr = rn
            else:
                p, rr = r.copy(), r @ r
            continue
        p = r + (rn / rr) * p
        rr = rn
    _, rep = O.cg(G, b, tol=tol, sched=O.schedule("cg", perturb_c=c, cg_keep_direction=keep))
    assert rep.converged and rep.rel_residual_true <= tol
    assert len(sw) == rep.n_switches == 2
    assert all(abs(a_ - b_) <= 1 for a_, b_ in zip(sw, rep.switch_iter))
    assert abs(j - rep.iterations) <= 2


def test_kept_direction_is_a_pure_residual_replacement_on_exact_levels():
    """R30 on a head-exact matrix (Poisson const: A_1 = A_2 = A_3), switches forced by the
    level floors (R17): r = b - A_new x equals the recurrence residual up to rounding, so
    keeping p continues the same Krylov process -- the iteration count is the fixed-level
    CG's (within 1) -- while the R15 restart p = r discards the search directions and needs
    more iterations (both take the first switch at the same iteration, the restarted solve
    reaches the second floor later)."""
    A = gi.poisson3d(14)
    G = enc(A)
    b = gi.ones_rhs(A)
    _, r3 = O.cg(G, b, tol=1e-10, sched=O.fixed_schedule(3))
    kw = dict(level_floor=(1e-2, 1e-5))
    _, rk = O.cg(G, b, tol=1e-10, sched=O.schedule("cg", cg_keep_direction=1, **kw))
    _, rr_ = O.cg(G, b, tol=1e-10, sched=O.schedule("cg", **kw))
    assert rk.n_switches == rr_.n_switches == 2
    assert rk.switch_iter[0] == rr_.switch_iter[0] and rk.switch_iter[1] < rr_.switch_iter[1]
    assert abs(rk.iterations - r3.iterations) <= 1
    assert rr_.iterations >= r3.iterations + 5
    assert rk.converged and rk.rel_residual_true <= 1e-10


def test_kept_direction_schedule_validation():
    """cg_keep_direction is 0 or 1 (anything else: invalid argument)"""
    A = gi.poisson3d(4)
    with pytest.raises(O.OracleError):
        O.cg(enc(A), gi.ones_rhs(A), sched=O.schedule("cg", cg_keep_direction=2))


# ------------------------------------------------------------------ c.1 step 10: partitioned mode
def _parts(n, P):
    return [round(i * n / P) for i in range(P + 1)]


def _seq_dot(a, b):
    """sequential left-to-right sum of the rounded products (np.cumsum accumulates in order)"""
    return float(np.cumsum(a * b)[-1]) if len(a) else 0.0


@pytest.mark.parametrize("P", [2, 3])
def test_partitioned_cg_matches_independent_rank_loop(P):
    """the oracle's partitioned CG (R29-stepped, so the switching
    logic runs on the rank-summed dots) against an independent numpy CG in which every dot
    is a per-rank sequential sum added in rank order and each rank's SpMV rows come from the
    decoded level matrices (scipy CSR): same iteration count and switch points, same x to
    1e-13 relative"""
    import scipy.sparse as sp
    A = gi.poisson3d(10, "varcoef")
    G = enc(A)
    b = gi.ones_rhs(A)
    parts = _parts(A.rows, P)
    c, tol = 0.1, 1e-10
    eta = O.perturbation_bounds(G)
    mats = {L: sp.csr_matrix((O.decode_all(G, L), A.col, A.row_ptr), shape=(A.rows, A.cols))
            for L in (1, 2, 3)}

    def dot(u, v):
        s = 0.0
        for r in range(P):
            s = s + _seq_dot(u[parts[r]:parts[r + 1]], v[parts[r]:parts[r + 1]])
        return s

    nb = np.sqrt(dot(b, b))
    x = np.zeros(A.rows)
    L, r = 1, b - mats[1] @ x
    p, rr, sw, j = r.copy(), dot(r, r), [], 0
    while j < 2000:
        j += 1
        q = mats[L] @ p
        pq = dot(p, q)
        xx = dot(x, x)
        al = rr / pq
        x = x + al * p
        r = r - al * q
        rn = dot(r, r)
        res = np.sqrt(rn) / nb
        if res <= tol:
            if L == 3 or np.sqrt(dot(b - mats[3] @ x, b - mats[3] @ x)) / nb <= tol:
                break
            esc = True
        else:
            esc = L < 3 and xx > 0 and res <= c * eta[L - 1] * np.sqrt(xx) / nb
        if esc:
            L += 1
            sw.append(j)
            r = b - mats[L] @ x
            p, rr = r.copy(), dot(r, r)
            continue
        p = r + (rn / rr) * p
        rr = rn
    xo, rep = O.cg(G, b, tol=tol, sched=O.schedule("cg", perturb_c=c), parts=parts)
    assert tuple(sw) == rep.switch_iter and j == rep.iterations
    assert np.abs(xo - x).max() <= 1e-13 * np.abs(x).max()


@pytest.mark.parametrize("solver", ["cg", "gmres"])
def test_partitioned_mode_properties(solver):
    """P = 1 is the unpartitioned solver bit for bit; P = 2, 3, 7 (uneven blocks, an empty
    block) change only the dot order: iterations within 2, the same switches, true residual
    <= tol; malformed bounds are rejected"""
    A = gi.poisson3d(12, "varcoef") if solver == "cg" else gi.convdiff3d(10)
    G = enc(A)
    b = gi.ones_rhs(A)
    run = O.cg if solver == "cg" else O.gmres
    sch = lambda: O.schedule(solver, perturb_c=0.1)
    x0, r0 = run(G, b, tol=1e-10, sched=sch())
    x1, r1 = run(G, b, tol=1e-10, sched=sch(), parts=[0, A.rows])
    assert np.array_equal(x0, x1) and r1.iterations == r0.iterations
    n = A.rows
    for parts in (_parts(n, 2), _parts(n, 3), [0, 5, 5, n // 3, n // 2, n - 1, n - 1, n]):
        x, r = run(G, b, tol=1e-10, sched=sch(), parts=parts)
        assert r.converged and r.rel_residual_true <= 1e-10
        assert abs(r.iterations - r0.iterations) <= 2 and r.n_switches == r0.n_switches
    for bad in ([0, n + 1], [1, n], [0, n // 2, n // 3, n]):
        with pytest.raises(O.OracleError):
            run(G, b, tol=1e-10, sched=sch(), parts=bad)


# ------------------------------------------------------------------ independent iteration gauges
@pytest.mark.parametrize("N,gauge", [(16, 46), (32, 93)])
def test_cg_iteration_gauges(N, gauge):
    """3D Poisson, b = A 1, tol 1e-10 -> 46 / 93 CG iterations at N = 16 / 32
    (scratch gauge, unchanged under dot orders); scipy's CG agrees within 1."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    A = gi.poisson3d(N)
    b = gi.ones_rhs(A)
    _, rep = O.cg(f64(A), b, tol=1e-10)
    assert rep.iterations == gauge
    its = []
    S = sp.csr_matrix((A.val, A.col, A.row_ptr), shape=(A.rows, A.cols))
    spla.cg(S, b, rtol=1e-10, atol=0.0, maxiter=5000, callback=lambda xk: its.append(1))
    assert abs(len(its) - rep.iterations) <= 1


@pytest.mark.parametrize("N,gauge", [(16, 135), (32, 363)])
def test_gmres30_iteration_gauges(N, gauge):
    """SURVEY 8(c.3) / S:381-383: conv-diff (beta = 64, 128, 192), b = A 1, GMRES(30) to
    1e-10 takes 135 / 363 inner iterations at N = 16 / 32 (scipy gauge); scipy's
    gmres(restart=30) counted here independently agrees within 3."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    A = gi.convdiff3d(N)
    b = gi.ones_rhs(A)
    x, rep = O.gmres(f64(A), b, tol=1e-10, restart=30)
    assert rep.converged and abs(rep.iterations - gauge) <= 3
    S = sp.csr_matrix((A.val, A.col, A.row_ptr), shape=(A.rows, A.cols))
    its = []
    spla.gmres(S, b, rtol=1e-10, atol=0.0, restart=30, maxiter=1000,
               callback=lambda pr: its.append(1), callback_type="pr_norm")
    assert abs(len(its) - rep.iterations) <= 3


@pytest.mark.parametrize("solver", ["cg", "gmres"])
def test_verify_respects_max_level(solver):
    """R16 within max_level (advisor finding): a schedule capped at level 2 on a head-lossy
    matrix never runs at level 3; when the level-2 recurrence converges but A_3's residual
    does not, the solve reports NOT_CONVERGED (it may not escalate) -- unless level 2 alone
    reaches tol against A_3."""
    A = gi.poisson2d(16, "varcoef") if solver == "cg" else gi.convdiff3d(8)
    b = gi.ones_rhs(A)
    G = enc(A)
    run = O.cg if solver == "cg" else O.gmres
    _, r1 = run(G, b, tol=1e-10, sched=O.schedule(solver, max_level=1))
    assert r1.status == O.NOT_CONVERGED and r1.n_switches == 0 and r1.iters_per_level[1:] == (0, 0)
    assert r1.rel_residual_true > 1e-10
    _, r2 = run(G, b, tol=1e-13, sched=O.schedule(solver, max_level=2))
    assert r2.iters_per_level[2] == 0 and max(r2.switch_to_level, default=1) <= 2
    assert r2.status == (O.OK if r2.rel_residual_true <= 1e-13 else O.NOT_CONVERGED)


def _numpy_stepped_gmres(mats, b, tol, m, floors=None, c=None, eta=None, max_iters=3000):
    """An independent stepped GMRES(m) (numpy, decoded level matrices): MGS Arnoldi, Givens
    rotations in the R18 form, the estimate |g_{j+1}|/||b|| monitored after every inner
    step; a switch (floor R17 or R29 bound with ||x|| at the cycle start) ends the cycle
    (x += V y) and restarts at the next level (R15); an explicit-residual convergence at
    L < 3 is verified with A_3 (R16)."""
    n = b.size
    nb = np.linalg.norm(b)
    x = np.zeros(n)
    L, jg, sw = 1, 0, []
    while jg < max_iters:
        r = b - mats[L] @ x
        beta = np.linalg.norm(r)
        if beta / nb <= tol:
            if L < 3 and np.linalg.norm(b - mats[3] @ x) / nb > tol:
                L += 1
                sw.append(jg)
                continue
            break
        xx = x @ x
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        V[0] = r / beta
        g[0] = beta
        k, esc = 0, False
        for j in range(m):
            jg += 1
            w = mats[L] @ V[j]
            for i in range(j + 1):
                H[i, j] = w @ V[i]
                w = w - H[i, j] * V[i]
            hn = np.linalg.norm(w)
            H[j + 1, j] = hn
            for i in range(j):
                h1, h2 = H[i, j], H[i + 1, j]
                H[i, j], H[i + 1, j] = cs[i] * h1 + sn[i] * h2, cs[i] * h2 - sn[i] * h1
            h1, h2 = H[j, j], H[j + 1, j]
            if h2 == 0:
                cc, ss = 1.0, 0.0
            elif abs(h2) > abs(h1):
                tau = h1 / h2
                ss = 1 / np.sqrt(1 + tau * tau)
                cc = ss * tau
            else:
                tau = h2 / h1
                cc = 1 / np.sqrt(1 + tau * tau)
                ss = cc * tau
            cs[j], sn[j] = cc, ss
            H[j, j], H[j + 1, j] = cc * h1 + ss * h2, 0.0
            g[j + 1], g[j] = -ss * g[j], cc * g[j]
            res = abs(g[j + 1]) / nb
            k = j + 1
            if res <= tol or hn == 0.0:
                break
            if L < 3 and ((floors and res < floors[L - 1]) or
                          (c and xx > 0 and res <= c * eta[L - 1] * np.sqrt(xx) / nb)):
                esc = True
                break
            V[j + 1] = w / hn
        y = np.linalg.solve(np.triu(H[:k, :k]), g[:k])
        x = x + V[:k].T @ y
        if esc:
            L += 1
            sw.append(jg)
    return jg, sw, np.linalg.norm(b - mats[3] @ x) / nb


@pytest.mark.parametrize("mode", ["floors", "r29"])
def test_stepped_gmres_matches_independent_numpy(mode):
    """The oracle's stepped GMRES(30) switch points and inner-iteration count against the
    independent numpy implementation above (floors R17 and the R29 trigger), conv-diff 10^3"""
    import scipy.sparse as sp
    A = gi.convdiff3d(10)
    G = enc(A)
    b = gi.ones_rhs(A)
    mats = {L: sp.csr_matrix((O.decode_all(G, L), A.col, A.row_ptr), shape=(A.rows, A.cols))
            for L in (1, 2, 3)}
    if mode == "floors":
        kw, args = {"level_floor": (1e-3, 1e-8)}, {"floors": (1e-3, 1e-8)}
    else:
        kw, args = {"perturb_c": 0.1}, {"c": 0.1, "eta": O.perturbation_bounds(G)}
    its, sw, res = _numpy_stepped_gmres(mats, b, 1e-10, 30, **args)
    _, rep = O.gmres(G, b, tol=1e-10, restart=30, sched=O.schedule("gmres", **kw))
    assert rep.converged and res <= 1e-10
    assert len(sw) == rep.n_switches >= 1
    assert all(abs(a_ - b_) <= 2 for a_, b_ in zip(sw, rep.switch_iter)), (sw, rep.switch_iter)
    assert abs(its - rep.iterations) <= 2, (its, rep.iterations)
