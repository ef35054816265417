"""GPU parity of the 16-bit GSE-SEM vectors (Alg. 1 P:128-160 in its
16-bit layout; R28) against the oracle, through the C-ABI:
  * gse_encode_vector16 / gse_decode_vector16: table, words and decoded values bit-exact;
  * GMRES(30) with the Krylov basis in 16-bit form: iterations within 2 and true residual
    ratio within [0.1, 10] of the oracle's compressed-basis GMRES.
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
    import paper_2411_04686_b200 as lib
    return lib


def vectors():
    rng = np.random.default_rng(3)
    v1 = rng.standard_normal(100003)
    v1 /= np.linalg.norm(v1)  # a Krylov-like unit vector, ragged length
    v2 = rng.uniform(-1, 1, 5000) * np.ldexp(1.0, rng.integers(-40, 40, 5000))  # wide: d > mbits
    v2[::31] = 0.0
    v2[1::37] = -0.0
    v2[2::41] = 5e-324  # subnormal
    v3 = np.zeros(257)
    v4 = np.array([1.0, -1.0, 0.5, 1.5, 2.0 ** -1022, -3.0 * 2.0 ** 40, 1 + 2.0 ** -52])
    return {"unit": v1, "wide": v2, "zeros": v3, "small": v4}


@pytest.mark.parametrize("k", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("name", ["unit", "wide", "zeros", "small"])
def test_vector16_bit_exact(g, name, k):
    v = vectors()[name]
    eb = int(np.log2(k))
    wo, to = O.encode_vector16(v, k)
    wg, tg = g.gse_encode_vector16(v, k)
    assert list(tg) == list(to)
    assert np.array_equal(wg, wo)
    dg = g.gse_decode_vector16(wg, tg, eb)
    do = O.decode_vector16(wo, to, eb)
    assert np.array_equal(dg.view(np.uint64), do.view(np.uint64))
    # device inputs give the same words
    wd, td = g.gse_encode_vector16(torch.from_numpy(v).cuda(), k)
    assert list(td) == list(to)
    assert np.array_equal(wd.cpu().numpy().view(np.uint16), wo)
    dd = g.gse_decode_vector16(wd, td, eb)
    assert np.array_equal(dd.cpu().numpy().view(np.uint64), do.view(np.uint64))


def test_vector16_errors(g):
    with pytest.raises(g.GseError):
        g.gse_encode_vector16(np.ones(4), 3)
    with pytest.raises(g.GseError):
        g.gse_encode_vector16(np.ones(4), 32)
    with pytest.raises(g.GseError):
        g.gse_decode_vector16(np.zeros(4, np.uint16), np.array([1024, 1025, 1026], np.uint16), 1)


def _cmp(rg, ro):
    assert rg["status"] == ro.status, (rg, ro)
    assert abs(rg["iterations"] - ro.iterations) <= 2, (rg, ro)
    ratio = rg["rel_residual_true"] / ro.rel_residual_true
    assert 0.1 <= ratio <= 10, (rg, ro)


@pytest.mark.parametrize("coop", ["1", "s"])
@pytest.mark.parametrize("mode", ["fp64_matrix", "fixed3", "stepped_scaled"])
def test_gmres_krylov16_parity(g, mode, coop, monkeypatch):
    """coop 1: one cooperative kernel per Arnoldi step (MGS, norm, histogram, table, encode);
    s: the per-step kernels"""
    monkeypatch.setenv("GSE_GM_COOP", coop)
    A = gi.convdiff3d(16)
    b = gi.ones_rhs(A)
    if mode == "fp64_matrix":
        M = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols)
        R = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
        sg, so = g.fixed_schedule(3), O.fixed_schedule(3)
    else:
        M = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
        R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
        if mode == "fixed3":
            sg, so = g.fixed_schedule(3), O.fixed_schedule(3)
        else:
            sg = g.gse_default_schedule("gmres", l=30, t=10, m=10)
            so = O.schedule("gmres", l=30, t=10, m=10)
    sg.krylov_gse16 = 1
    so.krylov_gse16 = 1
    xg, rg = g.gse_solve_gmres(M, b, tol=1e-10, sched=sg)
    xo, ro = O.gmres(R, b, tol=1e-10, sched=so)
    _cmp(rg, ro)
    assert rg["converged"] and rg["rel_residual_true"] <= 1e-10
    # the FP64-basis solve on the same matrix is a different trajectory (sanity: the flag acts)
    sg.krylov_gse16 = 0
    _, r64 = g.gse_solve_gmres(M, b, tol=1e-10, sched=sg)
    assert r64["converged"]


def test_gmres_krylov16_c1_and_switching_back(g):
    """varcoef 2D Poisson (SPD, head-lossy) with the 16-bit basis, then the same matrix
    handle solved with the FP64 basis again (graphs rebuilt for the format)"""
    A = gi.poisson2d(32, "varcoef")
    b = gi.ones_rhs(A)
    M = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    sg, so = g.fixed_schedule(3), O.fixed_schedule(3)
    sg.krylov_gse16 = so.krylov_gse16 = 1
    _, rg = g.gse_solve_gmres(M, b, tol=1e-10, sched=sg)
    _, ro = O.gmres(R, b, tol=1e-10, sched=so)
    _cmp(rg, ro)
    sg.krylov_gse16 = so.krylov_gse16 = 0
    _, rg = g.gse_solve_gmres(M, b, tol=1e-10, sched=sg)
    _, ro = O.gmres(R, b, tol=1e-10, sched=so)
    _cmp(rg, ro)
