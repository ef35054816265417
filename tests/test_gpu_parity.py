"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same seeded
inputs.  Bars (BASELINE.json north_star):
  * encode / decode: bit-exact (table, col_ei, head, tail1, tail2, side array, decoded FP64);
  * SpMV: |y_gpu - y_orc| <= 1e-12 * sum_j |dec_L(a_ij) x_j| (FP64 accumulate), 1e-5 (FP32);
    rows whose sum is 0 must be exactly 0;
  * solvers: |iters_gpu - iters_orc| <= 2, final true relative residual ratio in [0.1, 10].
"""
import numpy as np
import pytest

import gse_inputs as gi
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def g():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2411_04686_b200 as lib  # fails loudly when the extension is missing
    return lib


def enc_both(g, A, k=8, device_inputs=False):
    if device_inputs:
        M = g.gse_encode(torch.from_numpy(A.row_ptr).cuda(), torch.from_numpy(A.col).cuda(),
                         torch.from_numpy(A.val).cuda(), A.rows, A.cols, k_max=k)
    else:
        M = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols, k_max=k)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, k)
    return M, R


def spmv_bound(R, x, level, tol):
    """tol * sum_j |dec_L(a_ij) x_j| per row, via the oracle's SpMV of |A_L| |x|."""
    absR = O.GseCsr(R.rows, R.cols, R.nnz, R.row_ptr, R.col_ei, R.side_ei,
                    R.head & np.uint16(0x7FFF), R.tail1, R.tail2, R.table, R.ei_bits,
                    R.ei_in_column)
    return tol * O.spmv_gse(absR, np.abs(x), level)


MATS = {
    "poisson2d_const": lambda: gi.poisson2d(32),
    "poisson2d_varcoef": lambda: gi.poisson2d(32, "varcoef"),
    "poisson3d_40": lambda: gi.poisson3d(40, "varcoef"),
    "random_classes": lambda: gi.random_csr(3000, 2500, 9, seed=1, empty_rows=0.05),
    "random_wide": lambda: gi.random_csr(2000, 3000, 5, seed=2, value_kind="wide"),
    "random_mixed": lambda: gi.random_csr(2000, 2000, 7, seed=3, value_kind="mixed",
                                          empty_rows=0.2),
    "powerlaw_30k": lambda: gi.powerlaw_spd(30000, seed=5),
    "convdiff_20": lambda: gi.convdiff3d(20),
}


def long_rows_matrix():
    """rows of length 0, 1, LMAX-1, LMAX, LMAX+1, 2047, 2048, 2049, 5000 (DESIGN.md partition
    boundaries) interleaved with short rows."""
    rng = np.random.default_rng(9)
    lens = [3, 0, 1, 63, 64, 65, 191, 192, 193, 255, 256, 257, 7, 2047, 2048, 2049, 0, 5000, 2, 6]
    lens = lens * 3
    cols = 6000
    rp = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    col = np.concatenate([np.sort(rng.choice(cols, L, replace=False)) for L in lens]).astype(np.int32)
    val = rng.uniform(-2, 2, rp[-1]) * np.ldexp(1.0, rng.integers(-8, 8, rp[-1]))
    return gi.Csr(len(lens), cols, rp, col, val, "long_rows")


MATS["long_rows"] = long_rows_matrix


# ------------------------------------------------------------------ encode / decode
@pytest.mark.parametrize("name", sorted(MATS))
def test_encode_bit_exact(g, name):
    A = MATS[name]()
    M, R = enc_both(g, A, device_inputs=(name.startswith("poisson")))
    P = g.gse_matrix_copy_planes(M)
    assert list(P["table"]) == list(R.table)
    assert M.info["ei_bits"] == R.ei_bits and M.info["ei_in_column"] == R.ei_in_column
    for k in ("col_ei", "head", "tail1", "tail2"):
        assert np.array_equal(P[k], getattr(R, k)), k


@pytest.mark.parametrize("k", [1, 2, 4, 16, 64])
def test_encode_k_sweep_bit_exact(g, k):
    A = gi.powerlaw_spd(5000, seed=k)
    M, R = enc_both(g, A, k)
    P = g.gse_matrix_copy_planes(M)
    assert list(P["table"]) == list(R.table)
    for key in ("col_ei", "head", "tail1", "tail2"):
        assert np.array_equal(P[key], getattr(R, key)), key


@pytest.mark.parametrize("offset", [0, 1])
def test_encode_alignment_and_tail(g, offset):
    """k_hist / k_encode take four nonzeros per thread when every array is 16-byte aligned
    and one otherwise; nnz % 4 != 0 leaves a scalar tail.  offset 1: val / col are views one
    element into their buffers (8 / 4 bytes: the one-element path).  Planes bit-exact, and
    the FIRST bad element is the one reported (in the quad body and in the tail)."""
    A = gi.random_csr(3001, 2900, 7, seed=14, value_kind="mixed", empty_rows=0.1)
    assert A.nnz % 4 != 0
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, 8)

    def views(val, col):
        vb = torch.zeros(A.nnz + offset, dtype=torch.float64, device="cuda")
        cb = torch.zeros(A.nnz + offset, dtype=torch.int32, device="cuda")
        vb[offset:] = torch.from_numpy(val).cuda()
        cb[offset:] = torch.from_numpy(col).cuda()
        return vb[offset:], cb[offset:]

    rp = torch.from_numpy(A.row_ptr).cuda()
    v, c = views(A.val, A.col)
    assert (v.data_ptr() % 16 == 0) == (offset == 0)
    M = g.gse_encode(rp, c, v, A.rows, A.cols, k_max=8)
    P = g.gse_matrix_copy_planes(M)
    assert list(P["table"]) == list(R.table)
    for k in ("col_ei", "head", "tail1", "tail2"):
        assert np.array_equal(P[k], getattr(R, k)), k
    M.close()
    for first, second in ((A.nnz - 2, A.nnz - 1), (9, A.nnz - 1), (6, 7)):
        val = A.val.copy()
        val[second] = np.nan
        val[first] = np.inf
        v, c = views(val, A.col)
        with pytest.raises(g.GseError) as e:
            g.gse_encode(rp, c, v, A.rows, A.cols)
        assert e.value.status == g.GSE_ERR_NONFINITE
        assert f"(element {first})" in e.value.detail, e.value.detail
        col = A.col.copy()
        col[second] = -1
        col[first] = A.cols
        v, c = views(A.val, col)
        with pytest.raises(g.GseError) as e:
            g.gse_encode(rp, c, v, A.rows, A.cols)
        assert e.value.status == g.GSE_ERR_INVALID_ARG
        assert f"element {first}" in e.value.detail, e.value.detail


def test_encode_side_array(g):
    """cols >= 2^(32 - ei_bits): EI in a side array."""
    rng = np.random.default_rng(4)
    rows, cols = 300, (1 << 29) + 1000
    lens = rng.integers(0, 12, rows)
    rp = np.zeros(rows + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    col = np.concatenate([np.sort(rng.choice(cols, L, replace=False)) for L in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1]) * np.ldexp(1.0, rng.integers(-20, 20, rp[-1]))
    A = gi.Csr(rows, cols, rp, col, val)
    M, R = enc_both(g, A)
    P = g.gse_matrix_copy_planes(M)
    assert not R.ei_in_column and not M.info["ei_in_column"]
    for key in ("col_ei", "head", "tail1", "tail2", "side_ei"):
        assert np.array_equal(P[key], getattr(R, key)), key
    x = gi.uniform_vec(cols, seed=1)
    for L in (1, 2, 3):
        yg = g.gse_spmv(M, x, segments=L)
        yo = O.spmv_gse(R, x, L)
        assert np.all(np.abs(yg - yo) <= spmv_bound(R, x, L, 1e-12))


@pytest.mark.parametrize("name", ["random_wide", "random_mixed", "poisson2d_varcoef"])
def test_decode_bit_exact(g, name):
    A = MATS[name]()
    M, R = enc_both(g, A)
    for L in (1, 2, 3):
        got = g.gse_decode(M, L)
        want = O.decode_all(R, L)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), L


# ------------------------------------------------------------------ SpMV
@pytest.mark.parametrize("name", sorted(MATS))
def test_spmv_levels_parity(g, name):
    A = MATS[name]()
    M, R = enc_both(g, A)
    x = gi.uniform_vec(A.cols, seed=7)
    xt = torch.from_numpy(x).cuda()
    for L in (1, 2, 3):
        yg = g.gse_spmv(M, xt, segments=L).cpu().numpy()
        yo = O.spmv_gse(R, x, L)
        bound = spmv_bound(R, x, L, 1e-12)
        bad = np.abs(yg - yo) > bound
        assert not bad.any(), (L, np.nonzero(bad)[0][:5])
        assert np.all(yg[bound == 0] == 0.0)


@pytest.mark.parametrize("name", ["poisson2d_varcoef", "poisson3d_40", "powerlaw_30k", "convdiff_20"])
def test_spmv_dot_parity(g, name):
    """gse_spmv_dot (the CG's fused SpMV + p.q kernel, row walk or window): y within the SpMV
    bound, the dot within sum_i |x_i| bound_i + 1e-13 sum_i |x_i y_i|, repeat bit-identical;
    the FP64-CSR matrix the same way"""
    A = MATS[name]()
    M, R = enc_both(g, A)
    x = gi.uniform_vec(A.cols, seed=13)
    xt = torch.from_numpy(x).cuda()
    for L in (1, 2, 3):
        yt, dt = g.gse_spmv_dot(M, xt, segments=L)
        yg, dg = yt.cpu().numpy(), float(dt.item())
        yo = O.spmv_gse(R, x, L)
        bound = spmv_bound(R, x, L, 1e-12)
        assert np.all(np.abs(yg - yo) <= bound), L
        do = float(np.dot(x, yo))
        assert abs(dg - do) <= float(np.abs(x) @ bound) + 1e-13 * float(np.abs(x) @ np.abs(yo)), L
        _, d2 = g.gse_spmv_dot(M, xt, segments=L)
        assert float(d2.item()) == dg
    F = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols)
    hd = np.zeros(1)
    yf, _ = g.gse_spmv_dot(F, x, segments=3, dot=hd)  # host x, y and dot
    yo = O.spmv_fp64(O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val), x)
    Fa = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, np.abs(A.val))
    bound = 1e-12 * O.spmv_fp64(Fa, np.abs(x))
    assert np.all(np.abs(yf - yo) <= bound)
    assert abs(hd[0] - x @ yo) <= float(np.abs(x) @ bound) + 1e-13 * float(np.abs(x) @ np.abs(yo))


@pytest.mark.parametrize("k", [1, 2, 8, 16, 64])
def test_spmv_k_sweep_parity(g, k):
    """window kernel (power-law rows): scale tables of 1..64 entries (1-6 EI bits) at all
    levels, FP64 and FP32 accumulation"""
    A = gi.powerlaw_spd(20000, seed=11 + k)
    M, R = enc_both(g, A, k)
    assert M.info["spmv_mode"] == 2
    x = gi.uniform_vec(A.cols, seed=5)
    for L in (1, 2, 3):
        yg = g.gse_spmv(M, x, segments=L)
        yo = O.spmv_gse(R, x, L)
        assert np.all(np.abs(yg - yo) <= spmv_bound(R, x, L, 1e-12)), L
        yf = g.gse_spmv_f32acc(M, x.astype(np.float32), segments=L).astype(np.float64)
        yo32 = O.spmv_gse(R, x.astype(np.float32).astype(np.float64), L)
        bound = spmv_bound(R, x.astype(np.float32).astype(np.float64), L, 1e-5)
        assert np.all(np.abs(yf - yo32) <= bound), L


def short_rows_matrix():
    """blocks of > 32 rows (rows of 0-3 entries) next to ordinary ones: the strided kernel's
    lane-per-row fallback and the segmented path in one matrix"""
    rng = np.random.default_rng(21)
    lens = np.concatenate([rng.integers(0, 4, 3000), rng.integers(5, 40, 2000),
                           rng.integers(1, 3, 2000), rng.integers(20, 64, 500)])
    rows = lens.size
    cols = 5000
    rp = np.zeros(rows + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    col = np.concatenate([np.sort(rng.choice(cols, L, replace=False)) for L in lens]).astype(np.int32)
    val = rng.uniform(-2, 2, rp[-1]) * np.ldexp(1.0, rng.integers(-6, 6, rp[-1]))
    return gi.Csr(rows, cols, rp, col, val, "short_rows")


@pytest.mark.parametrize("mode", ["sp", "win", "auto"])
def test_spmv_short_rows_and_sp_cg(g, mode, monkeypatch):
    A = short_rows_matrix()
    M, R = enc_both(g, A)
    x = gi.uniform_vec(A.cols, seed=2)
    for L in (1, 2, 3):
        yg = g.gse_spmv(M, x, segments=L)
        yo = O.spmv_gse(R, x, L)
        bound = spmv_bound(R, x, L, 1e-12)
        assert np.all(np.abs(yg - yo) <= bound), L
        assert np.all(yg[bound == 0] == 0.0)
    # CG through the strided kernel's fused dot (DOT variant) on an SPD stencil
    if mode != "auto":
        monkeypatch.setenv("GSE_SPMV_MODE", mode)
    B = gi.poisson3d(20, "varcoef")
    Mb, Rb = enc_both(g, B)
    assert Mb.info["spmv_mode"] == {"sp": 0, "win": 2, "auto": 1}[mode]
    b = gi.ones_rhs(B)
    _, rg = g.gse_solve_cg(Mb, b, tol=1e-10, sched=g.gse_default_schedule("cg", l=30, t=10, m=10))
    _, ro = O.cg(Rb, b, tol=1e-10, sched=O.schedule("cg", l=30, t=10, m=10))
    _cmp_reports(rg, ro)


@pytest.mark.parametrize("name", ["poisson3d_40", "powerlaw_30k", "long_rows", "random_mixed"])
def test_spmv_fp64_comparator_parity(g, name):
    A = MATS[name]()
    M = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols)
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    x = gi.uniform_vec(A.cols, seed=3)
    yg = g.gse_spmv(M, x, segments=3)
    yo = O.spmv_fp64(F, x)
    Fa = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, np.abs(A.val))
    assert np.all(np.abs(yg - yo) <= 1e-12 * O.spmv_fp64(Fa, np.abs(x)))


@pytest.mark.parametrize("name", ["poisson3d_40", "powerlaw_30k", "long_rows", "random_classes"])
def test_spmv_f32acc_parity(g, name):
    A = MATS[name]()
    M, R = enc_both(g, A)
    x = gi.uniform_vec(A.cols, seed=4)
    x32 = x.astype(np.float32)
    for L in (1, 2, 3):
        y32 = g.gse_spmv_f32acc(M, x32, segments=L)
        yo = O.spmv_gse(R, x32.astype(np.float64), L)
        assert np.all(np.abs(y32.astype(np.float64) - yo) <= spmv_bound(R, x32.astype(np.float64), L, 1e-5))


@pytest.mark.parametrize("rpl", ["1", "2"])
@pytest.mark.parametrize("name", ["poisson3d_40", "poisson2d_varcoef", "convdiff_20"])
def test_spmv_row_walk_rows_per_lane(g, name, rpl, monkeypatch):
    """Both row-walk variants (32-row groups, lane = row; 64-row groups, two rows per lane)
    at every level and both accumulations, forced with GSE_RW_RPL (read per launch)."""
    A = MATS[name]()
    M, R = enc_both(g, A)
    assert M.info["spmv_mode"] == 1, "row-walk matrix expected"
    monkeypatch.setenv("GSE_RW_RPL", rpl)
    x = gi.uniform_vec(A.cols, seed=11)
    for L in (1, 2, 3):
        yg = g.gse_spmv(M, x, segments=L)
        yo = O.spmv_gse(R, x, L)
        assert np.all(np.abs(yg - yo) <= spmv_bound(R, x, L, 1e-12)), L
        y32 = g.gse_spmv_f32acc(M, x.astype(np.float32), segments=L)
        x64 = x.astype(np.float32).astype(np.float64)
        assert np.all(np.abs(y32.astype(np.float64) - O.spmv_gse(R, x64, L))
                      <= spmv_bound(R, x64, L, 1e-5)), L
    F = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols)
    yf = g.gse_spmv(F, x, segments=3)
    Fo = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    Fa = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, np.abs(A.val))
    assert np.all(np.abs(yf - O.spmv_fp64(Fo, x)) <= 1e-12 * O.spmv_fp64(Fa, np.abs(x)))


def window_edge_matrix(kind):
    """window-kernel edges (spmv_win.cu): 'huge' -- one row of 70000 non-zeros (longer than a
    tile, spans every warp of its CTA) among 1-entry rows (tiles capped at WIN_RMAX = 2048
    rows); 'banded_empty' -- partners within the x window plus 10 % empty rows (row lookup
    path); 'wide' -- 3000 rows x 400000 columns (window clipped, mostly global gathers)"""
    rng = np.random.default_rng({"huge": 31, "banded_empty": 32, "wide": 33}[kind])
    if kind == "huge":
        lens = np.concatenate([np.ones(5000, np.int64), [70000], np.ones(3000, np.int64),
                               rng.integers(1, 40, 3000)])
        rows, cols = lens.size, 80000
        col = [np.sort(rng.choice(cols, L, replace=False)) for L in lens]
    elif kind == "banded_empty":
        rows = cols = 60000
        lens = rng.integers(1, 30, rows)
        lens[rng.random(rows) < 0.1] = 0
        col = []
        for r, L in enumerate(lens):
            c = np.unique(np.clip(r + rng.integers(-600, 600, L), 0, cols - 1))
            col.append(c)
        lens = np.array([c.size for c in col])
    else:
        rows, cols = 3000, 400000
        lens = rng.integers(0, 60, rows)
        col = [np.sort(rng.choice(cols, L, replace=False)) for L in lens]
    rp = np.zeros(rows + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    colv = np.concatenate(col).astype(np.int32)
    val = rng.uniform(-2, 2, rp[-1]) * np.ldexp(1.0, rng.integers(-8, 8, rp[-1]))
    return gi.Csr(rows, cols, rp, colv, val, kind)


@pytest.mark.parametrize("kind", ["huge", "banded_empty", "wide"])
def test_spmv_window_edges(g, kind):
    """window kernel against the oracle at every level, FP64 / FP32 accumulation, the
    FP64-CSR comparator and an x that is not 16-byte aligned (window staging off)"""
    A = window_edge_matrix(kind)
    M, R = enc_both(g, A)
    assert M.info["spmv_mode"] == 2
    x = gi.uniform_vec(A.cols, seed=4)
    buf = torch.empty(A.cols + 1, dtype=torch.float64, device="cuda")
    xu = buf[1:]
    xu.copy_(torch.from_numpy(x))
    for L in (1, 2, 3):
        yo = O.spmv_gse(R, x, L)
        bound = spmv_bound(R, x, L, 1e-12)
        for xin in (torch.from_numpy(x).cuda(), xu):
            yg = g.gse_spmv(M, xin, segments=L).cpu().numpy()
            bad = np.abs(yg - yo) > bound
            assert not bad.any(), (kind, L, np.nonzero(bad)[0][:5])
            assert np.all(yg[bound == 0] == 0.0)
        yf = g.gse_spmv_f32acc(M, x.astype(np.float32), segments=L).astype(np.float64)
        x32 = x.astype(np.float32).astype(np.float64)
        assert np.all(np.abs(yf - O.spmv_gse(R, x32, L)) <= spmv_bound(R, x32, L, 1e-5)), L
    F = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols)
    yF = g.gse_spmv(F, x, segments=3)
    yo = O.spmv_fp64(O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val), x)
    absF = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, np.abs(A.val))
    assert np.all(np.abs(yF - yo) <= 1e-12 * O.spmv_fp64(absF, np.abs(x)))


def test_spmv_window_nan_isolation(g):
    """a non-finite x entry reaches only the rows that reference its column (masked lanes
    and slots never multiply it), in both irregular- and regular-row kernels"""
    for A in (gi.powerlaw_spd(20000, seed=3), gi.poisson3d(24, "varcoef")):
        M, R = enc_both(g, A)
        x = gi.uniform_vec(A.cols, seed=9)
        bad_col = A.cols // 2
        x[bad_col] = np.nan
        touched = np.zeros(A.rows, bool)
        rr = np.repeat(np.arange(A.rows), np.diff(A.row_ptr))
        touched[rr[A.col == bad_col]] = True
        for L in (1, 3):
            y = g.gse_spmv(M, x, segments=L)
            assert np.all(np.isnan(y[touched])), L
            assert np.all(np.isfinite(y[~touched])), (L, np.nonzero(~np.isfinite(y) & ~touched)[0][:5])


def test_spmv_head_exact_poisson_bitwise(g):
    """Constant Poisson is exact in the head: levels 1/2/3 and FP64 agree bitwise, and
    short rows are summed in storage order like the oracle."""
    A = gi.poisson3d(24)
    M, R = enc_both(g, A)
    x = gi.uniform_vec(A.cols, seed=5)
    yo = O.spmv_fp64(O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val), x)
    for L in (1, 2, 3):
        assert np.array_equal(g.gse_spmv(M, x, segments=L).view(np.uint64), yo.view(np.uint64))


def test_spmv_edge_cases(g):
    # one row, one column
    A = gi.from_dense(np.array([[2.5]]))
    M, _ = enc_both(g, A)
    assert g.gse_spmv(M, np.array([2.0]), segments=1)[0] == 5.0
    # all rows empty but one
    A = gi.random_csr(500, 40, 0.01, seed=2)
    A.val[:] = 3.0
    if A.nnz == 0:
        A = gi.from_dense(np.pad(np.array([[3.0]]), ((0, 499), (0, 39))))
    M, R = enc_both(g, A)
    x = np.ones(40)
    assert np.array_equal(g.gse_spmv(M, x, segments=2), O.spmv_gse(R, x, 2))
    # zero-size matrix
    Z = g.gse_fp64_matrix(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0), 0, 0)
    assert Z.info["rows"] == 0


def test_errors(g):
    A = gi.poisson2d(8)
    val = A.val.copy()
    val[17] = np.nan
    with pytest.raises(g.GseError) as e:
        g.gse_encode(A.row_ptr, A.col, val, A.rows, A.cols)
    assert e.value.status == g.GSE_ERR_NONFINITE and "row" in e.value.detail
    col = A.col.copy()
    col[3] = A.cols + 5
    with pytest.raises(g.GseError) as e:
        g.gse_encode(A.row_ptr, col, A.val, A.rows, A.cols)
    assert e.value.status == g.GSE_ERR_INVALID_ARG
    with pytest.raises(g.GseError) as e:
        g.gse_encode(A.row_ptr, A.col, np.zeros_like(A.val), A.rows, A.cols)
    assert e.value.status == g.GSE_ERR_NO_VALUES
    M = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
    with pytest.raises(g.GseError):
        g.gse_spmv(M, np.ones(A.cols), segments=4)
    big = A.val * 2.0 ** 300
    Mb = g.gse_encode(A.row_ptr, A.col, big, A.rows, A.cols)
    with pytest.raises(g.GseError) as e:
        g.gse_spmv_f32acc(Mb, np.ones(A.cols, np.float32), segments=1)
    assert e.value.status == g.GSE_ERR_FP32_RANGE


# ------------------------------------------------------------------ full-size sampled SpMV
def test_spmv_full_size_c2_sampled(g):
    """C2 (3D Poisson 128^3, varcoef) at full size, in bench.py's launch configuration:
    sampled rows against the oracle computed on just those rows."""
    A = gi.poisson3d(128, "varcoef")
    M = g.gse_encode(torch.from_numpy(A.row_ptr).cuda(), torch.from_numpy(A.col).cuda(),
                     torch.from_numpy(A.val).cuda(), A.rows, A.cols)
    P = g.gse_matrix_copy_planes(M)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([rng.integers(0, A.rows, 3000), [0, A.rows - 1]]))
    x = gi.uniform_vec(A.cols, seed=11)
    xt = torch.from_numpy(x).cuda()
    # oracle on the sampled rows: build the sub-CSR of those rows with the GPU-independent
    # oracle encoding of the same values (table from the full matrix)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    assert list(P["table"]) == list(R.table)
    sel = np.concatenate([np.arange(A.row_ptr[r], A.row_ptr[r + 1]) for r in rows])
    rp = np.zeros(rows.size + 1, np.int64)
    np.cumsum(A.row_ptr[rows + 1] - A.row_ptr[rows], out=rp[1:])
    sub = O.GseCsr(rows.size, A.cols, sel.size, rp, R.col_ei[sel].copy(), None,
                   R.head[sel].copy(), R.tail1[sel].copy(), R.tail2[sel].copy(), R.table,
                   R.ei_bits, R.ei_in_column)
    for L in (1, 2, 3):
        yg = g.gse_spmv(M, xt, segments=L).cpu().numpy()[rows]
        yo = O.spmv_gse(sub, x, L)
        assert np.all(np.abs(yg - yo) <= spmv_bound(sub, x, L, 1e-12))
    # the full planes are bit-exact too
    for k in ("col_ei", "head", "tail1", "tail2"):
        assert np.array_equal(P[k], getattr(R, k)), k


# ------------------------------------------------------------------ solvers
def _cmp_reports(rg, ro, iters_tol=2):
    assert rg["status"] == ro.status
    assert abs(rg["iterations"] - ro.iterations) <= iters_tol, (rg, ro)
    if ro.rel_residual_true > 0:
        ratio = rg["rel_residual_true"] / ro.rel_residual_true
        assert 0.1 <= ratio <= 10, (rg, ro)


@pytest.mark.parametrize("variant", ["const", "varcoef"])
@pytest.mark.parametrize("mode", ["fp64", "fixed3", "stepped", "stepped_scaled"])
def test_cg_parity_c1(g, variant, mode):
    A = gi.poisson2d(32, variant)
    b = gi.ones_rhs(A)
    if mode == "fp64":
        M = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols)
        Rm = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
        sg, so = None, None
    else:
        M, Rm = enc_both(g, A)
        if mode == "fixed3":
            sg, so = g.fixed_schedule(3), O.fixed_schedule(3)
        elif mode == "stepped":
            sg, so = g.gse_default_schedule("cg"), O.schedule("cg")
        else:
            sg = g.gse_default_schedule("cg", l=30, t=10, m=10)
            so = O.schedule("cg", l=30, t=10, m=10)
    xg, rg = g.gse_solve_cg(M, b, tol=1e-10, max_iters=5000, sched=sg)
    xo, ro = O.cg(Rm, b, tol=1e-10, max_iters=5000, sched=so)
    _cmp_reports(rg, ro)
    assert rg["n_switches"] == ro.n_switches
    for a, c in zip(rg["switch_iter"], ro.switch_iter):
        assert abs(a - c) <= 2
    assert rg["converged"] and rg["rel_residual_true"] <= 1e-10


@pytest.mark.parametrize("solver", ["cg", "gmres"])
@pytest.mark.parametrize("max_level", [1, 2])
def test_verify_respects_max_level(g, solver, max_level):
    """R16 capped by max_level: the GPU reports what the oracle reports (status, levels used,
    iterations +-2)"""
    A = gi.poisson2d(16, "varcoef") if solver == "cg" else gi.convdiff3d(8)
    b = gi.ones_rhs(A)
    M, R = enc_both(g, A)
    run_g = g.gse_solve_cg if solver == "cg" else g.gse_solve_gmres
    run_o = O.cg if solver == "cg" else O.gmres
    tol = 1e-10 if max_level == 1 else 1e-13
    _, rg = run_g(M, b, tol=tol, sched=g.gse_default_schedule(solver, max_level=max_level))
    _, ro = run_o(R, b, tol=tol, sched=O.schedule(solver, max_level=max_level))
    assert rg["status"] == ro.status and abs(rg["iterations"] - ro.iterations) <= 2
    assert all(v == 0 for v in rg["iters_per_level"][max_level:])


@pytest.mark.parametrize("name", ["poisson2d_varcoef", "powerlaw_30k", "random_mixed", "random_wide"])
def test_perturbation_bounds_bit_exact(g, name):
    """R29 eta_L = ||A_3 - A_L||_inf: bit-identical to the oracle (row sums in storage order)"""
    A = MATS[name]()
    M, R = enc_both(g, A)
    assert g.gse_perturbation_bounds(M) == O.perturbation_bounds(R)
    assert g.gse_perturbation_bounds(enc_both(g, gi.poisson3d(12))[0]) == (0.0, 0.0)


@pytest.mark.parametrize("solver", ["cg", "gmres"])
@pytest.mark.parametrize("c", [0.1, 1.0, 1e300])
def test_perturbation_trigger_parity(g, solver, c):
    """R29 trigger on the GPU (||x||^2 from the CG's xpay kernel / at the GMRES cycle start)
    against the oracle: iterations +-2, switch points +-2, residual ratio; the same handle
    then solves without the trigger exactly as before (graphs rebuilt)"""
    A = gi.poisson3d(16, "varcoef") if solver == "cg" else gi.convdiff3d(12)
    b = gi.ones_rhs(A)
    M, R = enc_both(g, A)
    run_g = g.gse_solve_cg if solver == "cg" else g.gse_solve_gmres
    run_o = O.cg if solver == "cg" else O.gmres
    _, r_plain = run_g(M, b, tol=1e-10, sched=g.gse_default_schedule(solver))
    _, rg = run_g(M, b, tol=1e-10, sched=g.gse_default_schedule(solver, perturb_c=c))
    _, ro = run_o(R, b, tol=1e-10, sched=O.schedule(solver, perturb_c=c))
    _cmp_reports(rg, ro)
    assert rg["n_switches"] == ro.n_switches == 2
    if c == 1e300:
        assert rg["switch_iter"] == ro.switch_iter
    for a_, b_ in zip(rg["switch_iter"], ro.switch_iter):
        assert abs(a_ - b_) <= 2
    assert rg["converged"] and rg["rel_residual_true"] <= 1e-10
    _, r_again = run_g(M, b, tol=1e-10, sched=g.gse_default_schedule(solver))
    assert (r_again["iterations"], r_again["switch_iter"]) == (r_plain["iterations"],
                                                               r_plain["switch_iter"])


@pytest.mark.parametrize("start,c", [(1, 0.1), (1, 1.0), (2, 3.0), (1, 1e300)])
def test_kept_direction_parity(g, start, c):
    """R30 (CG switch keeps p: r = b - A_new x, p = r + (r.r / rr_{j-1}) p) on the GPU
    against the oracle: iterations +-2, switch points +-2, residual ratio"""
    A = gi.poisson3d(16, "varcoef")
    b = gi.ones_rhs(A)
    M, R = enc_both(g, A)
    kw = dict(perturb_c=c, start_level=start, cg_keep_direction=1)
    _, rg = g.gse_solve_cg(M, b, tol=1e-10, sched=g.gse_default_schedule("cg", **kw))
    _, ro = O.cg(R, b, tol=1e-10, sched=O.schedule("cg", **kw))
    _cmp_reports(rg, ro)
    assert rg["n_switches"] == ro.n_switches == 3 - start
    for a_, b_ in zip(rg["switch_iter"], ro.switch_iter):
        assert abs(a_ - b_) <= 2
    assert rg["converged"] and rg["rel_residual_true"] <= 1e-10


def test_kept_direction_exact_levels_gpu(g):
    """R30 on a head-exact matrix with floor-forced switches: the GPU's kept-direction solve
    takes the fixed-level iteration count (within 1), the R15 restart more -- as the
    oracle's pin (tests/test_oracle_spmv_solvers.py)"""
    A = gi.poisson3d(14)
    b = gi.ones_rhs(A)
    M, _ = enc_both(g, A)
    kw = dict(level_floor=(1e-2, 1e-5))
    _, r3 = g.gse_solve_cg(M, b, tol=1e-10, sched=g.fixed_schedule(3))
    _, rk = g.gse_solve_cg(M, b, tol=1e-10, sched=g.gse_default_schedule("cg", cg_keep_direction=1, **kw))
    _, rr_ = g.gse_solve_cg(M, b, tol=1e-10, sched=g.gse_default_schedule("cg", **kw))
    assert rk["n_switches"] == rr_["n_switches"] == 2
    assert abs(rk["iterations"] - r3["iterations"]) <= 1
    assert rr_["iterations"] >= r3["iterations"] + 5


def test_kept_direction_rejects_bad_value(g):
    A = gi.poisson3d(4)
    M, _ = enc_both(g, A)
    with pytest.raises(g.GseError) as e:
        g.gse_solve_cg(M, gi.ones_rhs(A), sched=g.gse_default_schedule("cg", cg_keep_direction=2))
    assert e.value.status == g.GSE_ERR_INVALID_ARG


@pytest.mark.parametrize("mode", ["stepped_scaled", "stepped", "fp64"])
def test_cg_graph_unroll_invariant(g, mode, monkeypatch):
    """the CG graph's while body holds GSE_CG_UNROLL iterations; the kernels after an event
    are no-ops, so 1, 3 (odd: events mid-body) and 8 iterations per body give bitwise the
    same solution, iteration counts and switch points, escalations included"""
    A = gi.poisson3d(24, "varcoef")
    b = gi.ones_rhs(A)
    res = []
    for u in ("1", "3", "8"):
        monkeypatch.setenv("GSE_CG_UNROLL", u)
        if mode == "fp64":
            M, sg = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols), None
        else:
            M = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
            sg = (g.gse_default_schedule("cg", l=30, t=10, m=10) if mode == "stepped_scaled"
                  else g.gse_default_schedule("cg"))
        x, r = g.gse_solve_cg(M, b, tol=1e-10, max_iters=5000, sched=sg)
        res.append((x, r))
        M.close()
    x1, r1 = res[0]
    assert r1["converged"]
    if mode == "stepped_scaled":
        assert r1["n_switches"] >= 1
    for x, r in res[1:]:
        assert r["iterations"] == r1["iterations"]
        assert r["iters_per_level"] == r1["iters_per_level"]
        assert r["switch_iter"] == r1["switch_iter"]
        assert np.array_equal(x.view(np.uint64), x1.view(np.uint64))


def test_cg_parity_c2_full_size(g):
    """configs[1]: 3D Poisson 128^3 stepped CG to 1e-10 on one B200 vs the oracle."""
    A = gi.poisson3d(128)
    b = gi.ones_rhs(A)
    M, R = enc_both(g, A, device_inputs=True)
    bt = torch.from_numpy(b).cuda()
    xg, rg = g.gse_solve_cg(M, bt, tol=1e-10, sched=g.gse_default_schedule("cg"))
    O.set_threads(0)
    xo, ro = O.cg(R, b, tol=1e-10, sched=O.schedule("cg"))
    _cmp_reports(rg, ro)
    assert rg["iters_per_level"][0] == rg["iterations"]  # head-exact: level 1 only
    # independent property: true residual of the GPU solution with the oracle FP64 SpMV
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    res = np.linalg.norm(b - O.spmv_fp64(F, xg.cpu().numpy())) / np.linalg.norm(b)
    assert res <= 1e-10 * 1.001


@pytest.mark.parametrize("sched", ["default", "floors", "r29", "r29_keep_l2"])
def test_cg_parity_c2_varcoef_full_size_switching(g, sched):
    """configs[1] shape with varcoef values (head-lossy): full-size stepped CG that SWITCHES
    levels -- paper defaults (verify-at-full escalations, R16), level floors (R17) and the R29
    trigger -- against the oracle: iterations +-2, both switch points +-2, residual ratio in
    [0.1, 10]"""
    A = gi.poisson3d(128, "varcoef")
    b = gi.ones_rhs(A)
    M, R = enc_both(g, A, device_inputs=True)
    kw = {"default": {}, "floors": {"level_floor": (1e-3, 1e-8)}, "r29": {"perturb_c": 0.1},
          "r29_keep_l2": {"perturb_c": 3.0, "start_level": 2, "cg_keep_direction": 1}}[sched]
    _, rg = g.gse_solve_cg(M, torch.from_numpy(b).cuda(), tol=1e-10,
                           sched=g.gse_default_schedule("cg", **kw))
    O.set_threads(0)
    _, ro = O.cg(R, b, tol=1e-10, sched=O.schedule("cg", **kw))
    _cmp_reports(rg, ro)
    assert rg["n_switches"] == ro.n_switches == (1 if sched == "r29_keep_l2" else 2)
    for a_, b_ in zip(rg["switch_iter"], ro.switch_iter):
        assert abs(a_ - b_) <= 2, (rg, ro)
    assert rg["converged"] and rg["rel_residual_true"] <= 1e-10


@pytest.mark.parametrize("sched", ["floors", "r29", "r29_l2"])
def test_gmres_parity_convdiff64_switching(g, sched):
    """C4-shaped conv-diff at 64^3: stepped GMRES(30) that switches levels against the
    oracle (iterations +-2, switch points +-2, residual ratio)"""
    A = gi.convdiff3d(64)
    b = gi.ones_rhs(A)
    M, R = enc_both(g, A, device_inputs=True)
    kw = {"floors": {"level_floor": (1e-3, 1e-8)}, "r29": {"perturb_c": 0.1},
          "r29_l2": {"perturb_c": 0.1, "start_level": 2}}[sched]
    _, rg = g.gse_solve_gmres(M, torch.from_numpy(b).cuda(), tol=1e-10,
                              sched=g.gse_default_schedule("gmres", **kw))
    O.set_threads(0)
    _, ro = O.gmres(R, b, tol=1e-10, sched=O.schedule("gmres", **kw))
    _cmp_reports(rg, ro)
    assert rg["n_switches"] == ro.n_switches and rg["n_switches"] >= 1
    for a_, b_ in zip(rg["switch_iter"], ro.switch_iter):
        assert abs(a_ - b_) <= 2, (rg, ro)
    assert rg["converged"] and rg["rel_residual_true"] <= 1e-10


def test_cg_breakdown_abort(g):
    A = gi.from_dense(np.array([[1.0, 0.0], [0.0, -1.0]]))
    M = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, 2, 2)
    x, r = g.gse_solve_cg(M, np.array([1.0, 1.0]), tol=1e-10)
    assert r["status"] == g.GSE_NUMERICAL_ABORT


@pytest.mark.parametrize("coop", ["1", "0", "g"])
@pytest.mark.parametrize("mode", ["fp64", "stepped", "stepped_scaled"])
def test_gmres_parity(g, mode, coop, monkeypatch):
    """coop 1: one cooperative Arnoldi kernel per inner step (w in shared memory); g: the
    same with w in global memory (long vectors); 0: the per-MGS-step kernels."""
    monkeypatch.setenv("GSE_GM_COOP", coop)
    A = gi.convdiff3d(16)
    b = gi.ones_rhs(A)
    if mode == "fp64":
        M = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols)
        Rm = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
        sg, so = None, None
    else:
        M, Rm = enc_both(g, A)
        if mode == "stepped":
            sg, so = g.gse_default_schedule("gmres"), O.schedule("gmres")
        else:
            sg = g.gse_default_schedule("gmres", l=30, t=10, m=10)
            so = O.schedule("gmres", l=30, t=10, m=10)
    xg, rg = g.gse_solve_gmres(M, b, tol=1e-10, sched=sg)
    xo, ro = O.gmres(Rm, b, tol=1e-10, sched=so)
    _cmp_reports(rg, ro)
    assert rg["n_switches"] == ro.n_switches
    assert rg["converged"] and rg["rel_residual_true"] <= 1e-10


def test_gmres_small_exact(g):
    A = gi.from_dense(np.array([[2.0]]))
    M = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, 1, 1)
    x, r = g.gse_solve_gmres(M, np.array([4.0]), tol=1e-12)
    assert r["converged"] and r["iterations"] == 1 and abs(x[0] - 2.0) < 1e-15


def test_solver_x0_and_host_device_paths(g):
    A = gi.poisson2d(16, "varcoef")
    b = gi.ones_rhs(A)
    M, R = enc_both(g, A)
    x0 = gi.uniform_vec(A.rows, seed=3)
    xh, rh = g.gse_solve_cg(M, b, x=x0.copy(), tol=1e-10, sched=g.fixed_schedule(3))
    xd, rd = g.gse_solve_cg(M, torch.from_numpy(b).cuda(), x=torch.from_numpy(x0.copy()).cuda(),
                            tol=1e-10, sched=g.fixed_schedule(3))
    assert rh["iterations"] == rd["iterations"]
    assert np.array_equal(xh, xd.cpu().numpy())  # deterministic reductions
    xo, ro = O.cg(R, b, x0=x0, tol=1e-10, sched=O.fixed_schedule(3))
    _cmp_reports(rh, ro)


# ------------------------------------------------------------------ NEXT-3 sampled tables
@pytest.mark.parametrize("B,seed,k", [(1, 0, 8), (16, 42, 8), (64, 7, 4), (1000, 3, 16),
                                      (100000, 9, 8)])
def test_encode_sampled_bit_exact(g, B, seed, k):
    """P:116 / S:63-71: one SplitMix64-chosen row per block of B rows (R27) -> the same table
    and planes as the oracle, bit for bit (B = 1 equals the full table; B >= rows samples
    one row for the whole matrix)"""
    A = gi.powerlaw_spd(30000, seed=B % 97)
    M = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols, k_max=k, sample_block_rows=B,
                     seed=seed)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, k, sample_block_rows=B, seed=seed)
    P = g.gse_matrix_copy_planes(M)
    assert list(P["table"]) == list(R.table)
    for key in ("col_ei", "head", "tail1", "tail2"):
        assert np.array_equal(P[key], getattr(R, key)), key
    if B == 1:
        assert list(P["table"]) == list(O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, k).table)
    x = gi.uniform_vec(A.cols, seed=1)
    for L in (1, 3):
        yg = g.gse_spmv(M, x, segments=L)
        assert np.all(np.abs(yg - O.spmv_gse(R, x, L)) <= spmv_bound(R, x, L, 1e-12))


def test_encode_sampled_unsampled_max_and_errors(g):
    n = 64
    rng = np.random.default_rng(4)
    d = np.diag(rng.uniform(1, 2, n))
    r_s = O.sample_row(n, n, 11, 0)
    d[(r_s + 5) % n, (r_s + 6) % n] = 2.0 ** 40  # never sampled
    A = gi.from_dense(d)
    M = g.gse_encode(A.row_ptr, A.col, A.val, n, n, k_max=2, sample_block_rows=n, seed=11)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, 2, sample_block_rows=n, seed=11)
    assert list(M.info["table"]) == list(R.table) and max(R.table) == 1023 + 40 + 1
    assert len(R.table) == 2  # R27b: the sampled class keeps its entry, e_max takes the free slot
    assert np.array_equal(g.gse_decode(M, 3), O.decode_all(R, 3))
    with pytest.raises(g.GseError):
        g.gse_encode(A.row_ptr, A.col, A.val, n, n, sample_block_rows=-1)


def _sampled_rows_parity(g, A, x, n_rows=3000, seed=0, fp32=False, fp64_too=False):
    """GPU SpMV at every level vs the oracle on sampled rows (sub-CSR of those rows, encoded
    by the oracle with the full matrix's table); planes bit-exact in full"""
    dev = lambda a: torch.from_numpy(a).cuda()
    M = g.gse_encode(dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val), A.rows, A.cols)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    P = g.gse_matrix_copy_planes(M)
    assert list(P["table"]) == list(R.table)
    for k in ("col_ei", "head", "tail1", "tail2"):
        assert np.array_equal(P[k], getattr(R, k)), k
    del P
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([rng.integers(0, A.rows, n_rows), [0, A.rows - 1]]))
    sel = np.concatenate([np.arange(A.row_ptr[r], A.row_ptr[r + 1]) for r in rows])
    rp = np.zeros(rows.size + 1, np.int64)
    np.cumsum(A.row_ptr[rows + 1] - A.row_ptr[rows], out=rp[1:])
    sub = O.GseCsr(rows.size, A.cols, sel.size, rp, R.col_ei[sel].copy(), None,
                   R.head[sel].copy(), R.tail1[sel].copy(), R.tail2[sel].copy(), R.table,
                   R.ei_bits, R.ei_in_column)
    xt = dev(x)
    for L in (1, 2, 3):
        yg = g.gse_spmv(M, xt, segments=L).cpu().numpy()[rows]
        assert np.all(np.abs(yg - O.spmv_gse(sub, x, L)) <= spmv_bound(sub, x, L, 1e-12)), L
        if fp32:
            x32 = x.astype(np.float32)
            yf = g.gse_spmv_f32acc(M, dev(x32), segments=L).cpu().numpy()[rows].astype(np.float64)
            x64 = x32.astype(np.float64)
            assert np.all(np.abs(yf - O.spmv_gse(sub, x64, L)) <= spmv_bound(sub, x64, L, 1e-5)), L
    if fp64_too:
        F = g.gse_fp64_matrix(dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val), A.rows, A.cols)
        yg = g.gse_spmv(F, xt, segments=3).cpu().numpy()[rows]
        Fs = O.fp64_csr(rows.size, A.cols, rp, A.col[sel], A.val[sel])
        Fa = O.fp64_csr(rows.size, A.cols, rp, A.col[sel], np.abs(A.val[sel]))
        assert np.all(np.abs(yg - O.spmv_fp64(Fs, x)) <= 1e-12 * O.spmv_fp64(Fa, np.abs(x)))
    return M


def test_spmv_full_size_c3_sampled(g):
    """configs[2] (power-law SPD, 10M rows, ~200M nnz) at full size through the strided-
    products kernel bench.py times: planes bit-exact, sampled rows at every level, FP32
    accumulation and the FP64-CSR comparator"""
    O.set_threads(0)
    A = gi.powerlaw_spd(10_000_000, seed=42)
    M = _sampled_rows_parity(g, A, gi.uniform_vec(A.cols, seed=7), fp32=True, fp64_too=True)
    assert M.info["spmv_mode"] == 2


def test_spmv_full_size_c4_sampled_and_gmres(g):
    """configs[3] (conv-diff 256^3, 16.8M rows) at full size: sampled-row SpMV parity, then a
    stepped GMRES(30) solve to 1e-10 whose true residual is checked with the oracle's FP64
    SpMV (the oracle GMRES itself is out of reach at this size)"""
    O.set_threads(0)
    A = gi.convdiff3d(256)
    M = _sampled_rows_parity(g, A, gi.uniform_vec(A.cols, seed=3))
    assert M.info["spmv_mode"] == 1
    b = gi.ones_rhs(A)
    x, rep = g.gse_solve_gmres(M, torch.from_numpy(b).cuda(), tol=1e-10,
                               sched=g.gse_default_schedule("gmres", l=300, t=100, m=100))
    assert rep["converged"] and rep["n_switches"] >= 1
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    res = np.linalg.norm(b - O.spmv_fp64(F, x.cpu().numpy())) / np.linalg.norm(b)
    assert res <= 1e-10 * 1.01 and abs(res - rep["rel_residual_true"]) <= 1e-3 * res


@pytest.mark.parametrize("solver", ["cg", "gmres"])
@pytest.mark.parametrize("floors", [(1e300, 1e300), (1e-3, 1e-8)])
def test_level_floors_parity(g, solver, floors):
    """R17 level floors: the GPU escalates at the same iterations as the oracle (+-2)"""
    A = gi.poisson2d(32, "varcoef") if solver == "cg" else gi.convdiff3d(12)
    b = gi.ones_rhs(A)
    M, R = enc_both(g, A)
    run_g = g.gse_solve_cg if solver == "cg" else g.gse_solve_gmres
    run_o = O.cg if solver == "cg" else O.gmres
    _, rg = run_g(M, b, tol=1e-10, sched=g.gse_default_schedule(solver, level_floor=floors))
    _, ro = run_o(R, b, tol=1e-10, sched=O.schedule(solver, level_floor=floors))
    _cmp_reports(rg, ro)
    assert rg["n_switches"] == ro.n_switches == 2
    for a, c in zip(rg["switch_iter"], ro.switch_iter):
        assert abs(a - c) <= 2


def test_full_size_c5_sampled_and_cg(g):
    """configs[4] (3D Poisson 512^3: 134M rows, 938M nnz) at full size on one GPU: planes of
    sampled row slabs bit-exact against the oracle's encoding of those slabs (the table is
    the global one), sampled-row SpMV at every level, and the stepped CG to 1e-10 whose
    true residual is checked with the oracle's FP64 SpMV"""
    O.set_threads(0)
    N = 512
    A = gi.poisson3d(N)
    n = A.rows
    dev = lambda a: torch.from_numpy(a).cuda()
    M = g.gse_encode(dev(A.row_ptr.astype(np.int32)), dev(A.col), dev(A.val), n, n)
    info = M.info
    # the whole-matrix table from the oracle's encoding of a slab with every stencil value
    nnz = A.nnz
    planes = {k: torch.empty(nnz, dtype=dt, device="cuda") for k, dt in
              (("col_ei", torch.int32), ("head", torch.int16), ("tail1", torch.int16),
               ("tail2", torch.int32))}
    st = g._lib.gse_matrix_copy_planes(M.handle, planes["col_ei"].data_ptr(), None,
                                       planes["head"].data_ptr(), planes["tail1"].data_ptr(),
                                       planes["tail2"].data_ptr(), None, None)
    assert st == 0
    rng = np.random.default_rng(1)
    slabs = [0, n // 2, n - N * N] + list(rng.integers(0, n - N * N, 3))
    x = gi.uniform_vec(n, seed=5)
    xt = dev(x)
    ys = {L: g.gse_spmv(M, xt, segments=L).cpu().numpy() for L in (1, 2, 3)}
    for r0 in slabs:
        r1 = r0 + N * N
        sl = slice(A.row_ptr[r0], A.row_ptr[r1])
        rp = (A.row_ptr[r0:r1 + 1] - A.row_ptr[r0]).astype(np.int64)
        R = O.encode_csr(r1 - r0, n, rp, A.col[sl], A.val[sl])
        assert list(R.table) == list(info["table"])  # const Poisson: the slab has every value
        for k in ("col_ei", "head", "tail1", "tail2"):
            got = planes[k][sl.start:sl.stop].cpu().numpy().view(getattr(R, k).dtype)
            assert np.array_equal(got, getattr(R, k)), (k, r0)
        for L in (1, 2, 3):
            yo = O.spmv_gse(R, x, L)
            assert np.all(np.abs(ys[L][r0:r1] - yo) <= spmv_bound(R, x, L, 1e-12)), (L, r0)
    del planes
    b = gi.ones_rhs(A)
    xs, rep = g.gse_solve_cg(M, dev(b), tol=1e-10, max_iters=20000,
                             sched=g.gse_default_schedule("cg"))
    assert rep["converged"] and rep["iters_per_level"][0] == rep["iterations"]
    F = O.fp64_csr(n, n, A.row_ptr, A.col, A.val)
    res = np.linalg.norm(b - O.spmv_fp64(F, xs.cpu().numpy())) / np.linalg.norm(b)
    assert res <= 1e-10 * 1.01


def test_concurrent_spmv_threads(g):
    """include/gse.h: concurrent gse_spmv on different streams is safe -- here from host
    threads on matrices whose row-walk stages differ in size (the per-function dynamic
    shared-memory attribute must never drop below a concurrent launch's need)"""
    import threading
    mats = [gi.poisson3d(40, "varcoef"), gi.convdiff3d(24), gi.poisson2d(64, "varcoef"),
            gi.powerlaw_spd(20000, seed=3)]
    Ms = [g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols) for A in mats]
    xs = [torch.from_numpy(gi.uniform_vec(A.cols, seed=i)).cuda() for i, A in enumerate(mats)]
    ref = {(i, L): g.gse_spmv(Ms[i], xs[i], segments=L).cpu().numpy()
           for i in range(len(mats)) for L in (1, 2, 3)}
    errs = []

    def body(t):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for it in range(30):
                    i = (t + it) % len(mats)
                    L = 1 + (it % 3)
                    y = g.gse_spmv(Ms[i], xs[i], segments=L)
                    st.synchronize()
                    if not np.array_equal(y.cpu().numpy(), ref[(i, L)]):
                        errs.append((t, it, i, L))
        except Exception as e:  # pragma: no cover
            errs.append((t, repr(e)))

    th = [threading.Thread(target=body, args=(t,), daemon=True) for t in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th) and not errs, errs


# ------------------------------------------------------------------ allocator hook
def test_set_allocator_torch_and_alignment(g):
    """gse_set_allocator: every device allocation of an encode + SpMV + CG goes through the
    caller's allocator (torch's caching allocator here: torch sees the planes), results are
    bitwise those of the default pool; a misaligned allocator is refused with a detail message
    and its block handed back; NULL restores the default"""
    A = gi.poisson3d(20, "varcoef")
    b = gi.ones_rhs(A)
    x = gi.uniform_vec(A.cols, seed=3)
    sched = g.gse_default_schedule("cg", l=30, t=10, m=10)
    M0 = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
    y0 = g.gse_spmv(M0, x, segments=1)
    x0, r0 = g.gse_solve_cg(M0, b, tol=1e-10, sched=sched)
    M0.close()
    calls = {"alloc": 0, "free": 0}
    ta, tf = g.torch_allocator()

    def alloc(n, s):
        calls["alloc"] += 1
        return ta(n, s)

    def free(p, s):
        calls["free"] += 1
        tf(p, s)

    try:
        g.gse_set_allocator(alloc, free)
        torch.cuda.synchronize()
        before = torch.cuda.memory_allocated()
        M1 = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
        assert torch.cuda.memory_allocated() - before >= 12 * A.nnz  # the planes live in torch
        y1 = g.gse_spmv(M1, x, segments=1)
        x1, r1 = g.gse_solve_cg(M1, b, tol=1e-10, sched=sched)
        M1.close()
        assert calls["alloc"] > 0 and calls["free"] == calls["alloc"]
        assert np.array_equal(y0, y1) and np.array_equal(x0, x1)
        assert (r0["iterations"], r0["switch_iter"]) == (r1["iterations"], r1["switch_iter"])
        held = {}

        def bad_alloc(n, s):  # 16 bytes off a 256-byte boundary
            p = ta(n + 256, s)
            held[p + 16] = p
            return p + 16

        def bad_free(p, s):
            tf(held.pop(p), s)

        g.gse_set_allocator(bad_alloc, bad_free)
        with pytest.raises(g.GseError) as ei:
            g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
        assert "aligned" in str(ei.value) and not held
    finally:
        g.gse_set_allocator(None, None)
    M2 = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
    assert np.array_equal(g.gse_spmv(M2, x, segments=1), y0)
