"""Pins of the oracle's FP16 / BF16 storage baselines (P:406 [4.3]; R26):
round-to-nearest-even conversion FP64 -> 16 bit, exact conversion back, FP64-accumulated
SpMV, and the solvers on the baseline matrices.  The pins are independent of the oracle's
arithmetic: numpy's binary16 conversion, a brute-force nearest-value search over all 65536
codes, round trips, and dense row sums written out in Python."""
import math

import numpy as np
import pytest

import gse_inputs as gi
import oracle as O


def _finite_table(kind):
    codes = np.arange(65536, dtype=np.uint16)
    vals = O.half_values(codes, kind)
    ok = np.isfinite(vals)
    return codes[ok], vals[ok]


def _brute_round(v, kind):
    """Nearest representable value, ties to the even code; beyond the largest finite value
    by at least half its spacing -> Inf (IEEE 754 overflow under RNE)."""
    codes, vals = _finite_table(kind)
    pos = vals >= 0
    pc, pv = codes[pos], vals[pos]
    order = np.argsort(pv, kind="stable")
    pc, pv = pc[order], pv[order]
    # drop -0/+0 duplicates: keep +0 (code 0)
    keep = np.ones(pv.size, bool)
    keep[1:] = pv[1:] != pv[:-1]
    pc, pv = pc[keep], pv[keep]
    inf_code = 0x7C00 if kind == "fp16" else 0x7F80
    out = []
    for x in v:
        s = 0x8000 if math.copysign(1.0, x) < 0 else 0
        a = abs(x)
        top, spacing = pv[-1], pv[-1] - pv[-2]
        if a >= top + spacing / 2:
            out.append(s | inf_code)
            continue
        i = np.searchsorted(pv, a)
        if i == pv.size:  # between the largest finite value and the overflow threshold
            out.append(s | int(pc[-1]))
            continue
        if pv[i] == a:
            out.append(s | int(pc[i]))
            continue
        lo, hi = pv[i - 1], pv[i]
        dl, dh = a - lo, hi - a
        if dl < dh:
            c = pc[i - 1]
        elif dh < dl:
            c = pc[i]
        else:
            c = pc[i - 1] if int(pc[i - 1]) % 2 == 0 else pc[i]
        out.append(s | int(c))
    return np.array(out, dtype=np.uint16)


def _samples(kind, n=4000, seed=0):
    rng = np.random.default_rng(seed)
    lo, hi = (-30, 17) if kind == "fp16" else (-140, 129)
    mag = rng.uniform(0.5, 2.0, n) * np.ldexp(1.0, rng.integers(lo, hi, n))
    sgn = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    v = list(mag * sgn)
    # exact midpoints between neighbours (ties) and the overflow boundary
    codes, vals = _finite_table(kind)
    pv = np.unique(vals[vals > 0])
    idx = rng.integers(0, pv.size - 1, 300)
    v += list((pv[idx] + pv[idx + 1]) / 2)
    top, sp = pv[-1], pv[-1] - pv[-2]
    v += [top, top + sp / 4, top + sp / 2, -(top + sp / 2), top + sp, 0.0, -0.0]
    return np.array(v)


@pytest.mark.parametrize("kind", ["fp16", "bf16"])
def test_round_half_brute_force_nearest(kind):
    v = _samples(kind)
    got = O.round_half(v, kind)
    want = _brute_round(v, kind)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [(v[i], hex(got[i]), hex(want[i])) for i in bad[:5]]


def test_round_fp16_matches_numpy():
    """numpy's float64 -> float16 cast is RNE directly from the double."""
    rng = np.random.default_rng(3)
    v = np.concatenate([rng.standard_normal(20000) * np.ldexp(1.0, rng.integers(-28, 18, 20000)),
                        _samples("fp16", 2000, seed=5)])
    with np.errstate(over="ignore"):
        want = v.astype(np.float16).view(np.uint16)
    assert np.array_equal(O.round_half(v, "fp16"), want)


@pytest.mark.parametrize("kind", ["fp16", "bf16"])
def test_half_values_round_trip(kind):
    codes = np.arange(65536, dtype=np.uint16)
    vals = O.half_values(codes, kind)
    fin = np.isfinite(vals)
    assert np.array_equal(O.round_half(vals[fin], kind), codes[fin])
    nan_codes = codes[np.isnan(vals)]
    assert nan_codes.size == (2046 if kind == "fp16" else 254)
    inf_code = 0x7C00 if kind == "fp16" else 0x7F80
    assert vals[inf_code] == np.inf and vals[inf_code | 0x8000] == -np.inf


def test_half_spec_examples():
    """1.0 exact in BF16; 70000 -> +Inf in FP16 (max finite 65504); 1 + 2^-9
    rounds to 1.0 in BF16 (a tie, to even)."""
    assert O.half_values(O.round_half([1.0], "bf16"), "bf16")[0] == 1.0
    assert O.round_half([70000.0], "fp16")[0] == 0x7C00
    assert O.half_values(O.round_half([65504.0], "fp16"), "fp16")[0] == 65504.0
    assert O.half_values(O.round_half([1 + 2.0 ** -9], "bf16"), "bf16")[0] == 1.0
    assert O.half_values(O.round_half([1 + 3 * 2.0 ** -9], "bf16"), "bf16")[0] == 1 + 2.0 ** -7


@pytest.mark.parametrize("kind", ["fp16", "bf16"])
def test_spmv_half_equals_written_out_row_sums(kind):
    A = gi.random_csr(60, 50, 6, seed=4, value_kind="mixed", empty_rows=0.1)
    H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, kind)
    x = gi.uniform_vec(A.cols, seed=2)
    vals = O.half_values(H.half, kind)
    want = np.zeros(A.rows)
    for i in range(A.rows):
        s = 0.0
        for j in range(A.row_ptr[i], A.row_ptr[i + 1]):
            s = s + vals[j] * x[A.col[j]]
        want[i] = s
    got = O.spmv_half(H, x)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_spmv_fp16_overflow_nonfinite_gse_finite():
    """a matrix containing 70000.0 gives a non-finite FP16-baseline SpMV result and
    a finite GSE head-only result (the '/' entries of the paper's Tables IV-V)."""
    A = gi.from_dense(np.array([[4.0, 70000.0], [1.0, 3.0]]))
    H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, "fp16")
    x = np.ones(2)
    y = O.spmv_half(H, x)
    assert not np.isfinite(y[0]) and y[1] == 4.0
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, 8)
    assert np.all(np.isfinite(O.spmv_gse(R, x, 1)))


@pytest.mark.parametrize("kind", ["fp16", "bf16"])
def test_cg_on_half_baseline(kind):
    """CG on the rounded matrix: converges to the solution of the ROUNDED system (checked
    with a dense solve of the rounded matrix); BF16's 8-bit significand perturbs the
    varcoef Poisson matrix enough that the FP64 system's residual stalls far above 1e-10."""
    A = gi.poisson2d(12, "varcoef")
    b = gi.ones_rhs(A)
    H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, kind)
    x, rep = O.cg(H, b, tol=1e-10, max_iters=2000)
    assert rep.converged
    dense = np.zeros((A.rows, A.cols))
    for i in range(A.rows):
        for j in range(A.row_ptr[i], A.row_ptr[i + 1]):
            dense[i, A.col[j]] = O.half_values(H.half[j:j + 1], kind)[0]
    xd = np.linalg.solve(dense, b)
    assert np.max(np.abs(x - xd)) <= 1e-8 * np.max(np.abs(xd))
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    true_res = np.linalg.norm(b - O.spmv_fp64(F, x)) / np.linalg.norm(b)
    assert true_res > 1e-6  # the rounded system is not the FP64 one


def test_gmres_on_half_baseline():
    A = gi.convdiff3d(8)
    b = gi.ones_rhs(A)
    H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, "bf16")
    x, rep = O.gmres(H, b, tol=1e-10, max_iters=3000)
    assert rep.converged
    r = b - O.spmv_half(H, x)
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-9
