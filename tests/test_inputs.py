"""Input recipes: sizes of SURVEY.md section 8(a) configs,
structural properties, and the power-law calibration to P:105's top-k coverage."""
import numpy as np
import pytest

import gse_inputs as gi


@pytest.mark.parametrize("N", [4, 32])
def test_poisson2d_shape(N):
    A = gi.poisson2d(N)
    assert A.rows == N * N and A.nnz == 5 * N * N - 4 * N
    d = A.dense()
    assert np.array_equal(d, d.T) and np.all(np.diag(d) == 4)


def test_c1_exact_size():
    assert gi.poisson2d(32).nnz == 4992


@pytest.mark.parametrize("N", [3, 7])
def test_poisson3d_shape_and_row_range(N):
    A = gi.poisson3d(N)
    assert A.rows == N ** 3 and A.nnz == 7 * N ** 3 - 6 * N * N
    assert np.all(np.diff(A.row_ptr) > 0)
    for r in range(A.rows):  # sorted, duplicate-free rows
        c = A.col[A.row_ptr[r]:A.row_ptr[r + 1]]
        assert np.all(np.diff(c) > 0)
    part = gi.poisson3d(N, row_begin=5, row_end=20)
    assert np.array_equal(part.col, A.col[A.row_ptr[5]:A.row_ptr[20]])


@pytest.mark.parametrize("variant", ["const", "varcoef"])
def test_poisson3d_chunks_concatenate_to_the_matrix(variant):
    """bench.py's chunked C5 generation yields exactly poisson3d's rows"""
    N = 9
    A = gi.poisson3d(N, variant)
    r0, r1 = 2 * N * N + 5, A.rows - 7
    parts = list(gi.poisson3d_chunks(N, variant, r0, r1, planes=2, workers=3))
    assert [p[0] for p in parts] == sorted(p[0] for p in parts) and parts[0][0] == r0
    assert sum(p[1].rows for p in parts) == r1 - r0
    col = np.concatenate([p[1].col for p in parts])
    val = np.concatenate([p[1].val for p in parts])
    s, e = A.row_ptr[r0], A.row_ptr[r1]
    assert np.array_equal(col, A.col[s:e]) and np.array_equal(val, A.val[s:e])
    lens = np.concatenate([np.diff(p[1].row_ptr) for p in parts])
    assert np.array_equal(lens, np.diff(A.row_ptr)[r0:r1])


def test_c2_c5_sizes_by_formula():
    # 7-point stencil nnz = 7 N^3 - 6 N^2 (14,581,760 and 937,951,232)
    assert 7 * 128 ** 3 - 6 * 128 ** 2 == 14581760
    assert 7 * 512 ** 3 - 6 * 512 ** 2 == 937951232
    assert 7 * 256 ** 3 - 6 * 256 ** 2 == 117047296


def test_varcoef_spd():
    A = gi.poisson3d(5, "varcoef")
    d = A.dense()
    assert np.allclose(d, d.T) and np.all(np.linalg.eigvalsh(d) > 0)


def test_convdiff_m_matrix_nonsymmetric():
    A = gi.convdiff3d(5)
    d = A.dense()
    assert not np.allclose(d, d.T)
    off = d - np.diag(np.diag(d))
    assert np.all(off <= 0) and np.all(np.diag(d) >= -off.sum(axis=1))


def test_powerlaw_calibration():
    A = gi.powerlaw_spd(100000)
    lens = np.diff(A.row_ptr)
    assert 19.0 < A.nnz / A.rows < 22.0  # -> ~200M nnz at 10M rows (C3)
    d = A.dense() if A.rows < 3000 else None
    off = A.val[A.val < 0]
    e = (off.view(np.uint64) >> 52) & 0x7FF
    c = np.sort(np.bincount(e))[::-1]
    cov = np.cumsum(c[c > 0]) / c.sum()
    # average top-k coverage 64.7/73.1/82.4/90.9/96.5/98.9/99.8 %
    want = [64.7, 73.1, 82.4, 90.9, 96.5, 98.9, 99.8]
    got = [cov[k - 1] * 100 for k in (1, 2, 4, 8, 16, 32, 64)]
    assert np.allclose(got, want, atol=0.6)
    # symmetric pattern and values; strictly diagonally dominant
    r = np.repeat(np.arange(A.rows), lens)
    key = r * A.rows + A.col
    keyT = A.col.astype(np.int64) * A.rows + r
    o1, o2 = np.argsort(key), np.argsort(keyT)
    assert np.array_equal(key[o1], keyT[o2]) and np.array_equal(A.val[o1], A.val[o2])
    diag = A.val[r == A.col]
    offsum = np.bincount(r[r != A.col], weights=np.abs(A.val[r != A.col]), minlength=A.rows)
    assert np.all(diag > offsum)
