"""GPU parity of the FP16 / BF16 storage baselines (P:406 [4.3]; R26)
against the oracle on the same seeded inputs, through the C-ABI:
  * 16-bit codes: bit-exact (round to nearest even straight from the double, overflow to Inf);
  * SpMV: |y_gpu - y_orc| <= 1e-12 * sum_j |v_ij x_j| (FP64 products and sums);
  * CG / GMRES on the rounded matrix: iterations within 2, true residual ratio in [0.1, 10].
"""
import numpy as np
import pytest

import gse_inputs as gi
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KINDS = ["fp16", "bf16"]


@pytest.fixture(scope="module")
def g():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2411_04686_b200 as lib
    return lib


def special_values(kind, n=20000, seed=0):
    """random magnitudes across (and beyond) the format's range, exact ties between
    neighbouring codes, the overflow boundary, signed zeros and FP64 subnormals"""
    rng = np.random.default_rng(seed)
    lo, hi = (-40, 20) if kind == "fp16" else (-150, 131)
    v = rng.uniform(0.5, 2.0, n) * np.ldexp(1.0, rng.integers(lo, hi, n))
    v *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
    codes = np.arange(65536, dtype=np.uint16)
    vals = O.half_values(codes, kind)
    pv = np.unique(vals[np.isfinite(vals) & (vals > 0)])
    i = rng.integers(0, pv.size - 1, 2000)
    ties = (pv[i] + pv[i + 1]) / 2
    top, sp = pv[-1], pv[-1] - pv[-2]
    extra = [top, top + sp / 4, top + sp / 2, -(top + sp / 2), top + sp, 1e300, -1e300,
             0.0, -0.0, 5e-324, -2.2e-308, pv[0], pv[0] / 2, pv[0] * 0.75, pv[0] / 4]
    return np.concatenate([v, ties, -ties, np.array(extra)])


def as_matrix(v, cols=97):
    """values laid out as a CSR matrix (rows of <= 7 entries, distinct sorted columns)"""
    rp = np.arange(0, v.size + 7, 7)
    rp[-1] = v.size
    rp = np.unique(rp)
    col = np.concatenate([np.arange(rp[i + 1] - rp[i]) * 13 % cols for i in range(rp.size - 1)])
    col = np.concatenate([np.sort(col[rp[i]:rp[i + 1]]) for i in range(rp.size - 1)]).astype(np.int32)
    return gi.Csr(rp.size - 1, cols, rp.astype(np.int64), col, v.astype(np.float64), "values")


@pytest.mark.parametrize("kind", KINDS)
def test_half_codes_bit_exact(g, kind):
    A = as_matrix(special_values(kind))
    M = g.gse_half_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols, kind=kind)
    P = g.gse_matrix_copy_planes(M)
    want = O.round_half(A.val, kind)
    bad = np.nonzero(P["half"] != want)[0]
    assert bad.size == 0, [(A.val[i], hex(P["half"][i]), hex(want[i])) for i in bad[:5]]
    assert np.array_equal(P["col"], A.col.astype(np.uint32))
    info = M.info
    assert info["kind"] == (g.GSE_KIND_FP16 if kind == "fp16" else g.GSE_KIND_BF16)
    assert info["plane_bytes"][:2] == [4 * A.nnz, 2 * A.nnz]


MATS = {
    "poisson3d_40": lambda: gi.poisson3d(40, "varcoef"),
    "powerlaw_30k": lambda: gi.powerlaw_spd(30000, seed=5),
    "random_mixed": lambda: gi.random_csr(2000, 2000, 7, seed=3, value_kind="mixed",
                                          empty_rows=0.2),
    "convdiff_20": lambda: gi.convdiff3d(20),
}


@pytest.mark.parametrize("name", sorted(MATS))
@pytest.mark.parametrize("kind", KINDS)
def test_spmv_half_parity(g, name, kind):
    A = MATS[name]()
    M = g.gse_half_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols, kind=kind)
    H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, kind)
    x = gi.uniform_vec(A.cols, seed=3)
    yg = g.gse_spmv(M, x, segments=3)
    yo = O.spmv_half(H, x)
    Ha = O.HalfCsr(H.rows, H.cols, H.row_ptr, H.col, H.half & np.uint16(0x7FFF), H.kind)
    bound = 1e-12 * O.spmv_half(Ha, np.abs(x))
    fin = np.isfinite(yo)
    assert np.all(np.abs(yg[fin] - yo[fin]) <= bound[fin])
    assert np.array_equal(np.isfinite(yg), fin)
    assert np.all(yg[bound == 0] == 0)


def test_spmv_half_device_inputs_and_segments(g):
    A = gi.poisson3d(24, "varcoef")
    dev = lambda a: torch.from_numpy(a).cuda()
    M = g.gse_half_matrix(dev(A.row_ptr), dev(A.col), dev(A.val), A.rows, A.cols, kind="bf16")
    H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, "bf16")
    x = gi.uniform_vec(A.cols, seed=8)
    yg = g.gse_spmv(M, dev(x), segments=3).cpu().numpy()
    assert np.max(np.abs(yg - O.spmv_half(H, x))) <= 1e-12 * np.max(np.abs(yg)) * 10
    with pytest.raises(g.GseError):
        g.gse_spmv(M, x, segments=1)  # a 16-bit matrix has one precision
    with pytest.raises(g.GseError):
        g.gse_spmv_f32acc(M, x.astype(np.float32), segments=3)
    with pytest.raises(g.GseError):
        g.gse_decode(M, 3)


def test_fp16_overflow_row(g):
    """S:470 / Tables IV-V '/': 70000 overflows FP16 -> the row's SpMV is non-finite; BF16
    and the GSE head stay finite."""
    A = gi.from_dense(np.array([[4.0, 70000.0], [1.0, 3.0]]))
    x = np.ones(2)
    M16 = g.gse_half_matrix(A.row_ptr, A.col, A.val, 2, 2, kind="fp16")
    y = g.gse_spmv(M16, x, segments=3)
    assert not np.isfinite(y[0]) and y[1] == 4.0
    Mb = g.gse_half_matrix(A.row_ptr, A.col, A.val, 2, 2, kind="bf16")
    assert np.all(np.isfinite(g.gse_spmv(Mb, x, segments=3)))


def _cmp(rg, ro):
    assert rg["status"] == ro.status, (rg, ro)
    assert abs(rg["iterations"] - ro.iterations) <= 2, (rg, ro)
    if ro.rel_residual_true > 0 and np.isfinite(ro.rel_residual_true):
        ratio = rg["rel_residual_true"] / ro.rel_residual_true
        assert 0.1 <= ratio <= 10, (rg, ro)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("variant", ["const", "varcoef"])
def test_cg_half_parity(g, kind, variant):
    A = gi.poisson2d(32, variant)
    b = gi.ones_rhs(A)
    M = g.gse_half_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols, kind=kind)
    H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, kind)
    # a stepped schedule is accepted and never steps on a one-precision matrix
    xg, rg = g.gse_solve_cg(M, b, tol=1e-10, max_iters=5000, sched=g.gse_default_schedule("cg"))
    xo, ro = O.cg(H, b, tol=1e-10, max_iters=5000)
    _cmp(rg, ro)
    assert rg["n_switches"] == 0


def test_cg_fp16_overflow_aborts(g):
    """an FP16 overflow makes the CG residual non-finite: numerical abort (the paper's '/')"""
    A = gi.poisson2d(8, "const")
    val = A.val * 2e4  # diagonal 8e4 > 65504
    M = g.gse_half_matrix(A.row_ptr, A.col, val, A.rows, A.cols, kind="fp16")
    H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, val, "fp16")
    b = np.ones(A.rows)
    _, rg = g.gse_solve_cg(M, b, tol=1e-10)
    _, ro = O.cg(H, b, tol=1e-10)
    assert rg["status"] == ro.status == g.GSE_NUMERICAL_ABORT


@pytest.mark.parametrize("kind", KINDS)
def test_gmres_half_parity(g, kind):
    A = gi.convdiff3d(12)
    b = gi.ones_rhs(A)
    M = g.gse_half_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols, kind=kind)
    H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, kind)
    xg, rg = g.gse_solve_gmres(M, b, tol=1e-10, max_iters=3000)
    xo, ro = O.gmres(H, b, tol=1e-10, max_iters=3000)
    _cmp(rg, ro)


def test_spmv_half_full_size_c2(g):
    """configs[1] 128^3 varcoef at full size, BF16 (lossy) and FP16: every row vs the oracle."""
    A = gi.poisson3d(128, "varcoef")
    dev = lambda a: torch.from_numpy(a).cuda()
    x = gi.uniform_vec(A.cols, seed=7)
    O.set_threads(0)
    for kind in KINDS:
        M = g.gse_half_matrix(dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val), A.rows,
                              A.cols, kind=kind)
        H = O.half_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, kind)
        assert np.array_equal(g.gse_matrix_copy_planes(M)["half"], H.half[:A.nnz])
        yg = g.gse_spmv(M, dev(x), segments=3).cpu().numpy()
        Ha = O.HalfCsr(H.rows, H.cols, H.row_ptr, H.col, H.half & np.uint16(0x7FFF), H.kind)
        assert np.all(np.abs(yg - O.spmv_half(H, x)) <= 1e-12 * O.spmv_half(Ha, np.abs(x)))
