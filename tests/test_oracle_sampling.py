"""Pins of the oracle's sampled table extraction ("the shared
exponents can be calculated using sampling techniques ... the exponents' distribution in a
random row is calculated for each row block"; reading R27 for the generator).
Independent of the oracle's arithmetic: a Python SplitMix64 checked against the published
first output for seed 0, exponents taken with math.frexp, SPEC's worked examples, brute
force over table subsets, and representability of every value."""
import itertools
import math

import numpy as np
import pytest

import gse_inputs as gi
import oracle as O

M64 = (1 << 64) - 1


def splitmix64(seed: int, b: int) -> int:
    """SplitMix64 (Steele, Lea, Flood 2014), output for counter b + 1 from `seed`"""
    z = (seed + (b + 1) * 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def biased_exponent(v: float) -> int:
    """IEEE biased exponent via frexp (0 for zero / subnormal)"""
    if v == 0.0:
        return 0
    m, e = math.frexp(abs(v))  # |v| = m 2^e, m in [0.5, 1)
    be = e - 1 + 1023
    return be if be >= 1 else 0


def test_splitmix64_reference_values():
    # the first output of SplitMix64 seeded with 0 (the generator's published test value)
    assert splitmix64(0, 0) == 0xE220A8397B1DCDAF
    assert O.sample_z(0, 0) == 0xE220A8397B1DCDAF
    rng = np.random.default_rng(1)
    for _ in range(200):
        seed = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        b = int(rng.integers(0, 10**9))
        assert O.sample_z(seed, b) == splitmix64(seed, b)


@pytest.mark.parametrize("rows,B", [(100, 7), (10, 10), (1, 1), (1000, 1), (37, 64)])
def test_sample_rows_in_their_block(rows, B):
    nb = (rows + B - 1) // B
    for seed in (0, 42, 2**63 + 5):
        for b in range(nb):
            r = O.sample_row(rows, B, seed, b)
            assert b * B <= r < min((b + 1) * B, rows)
            assert r == b * B + splitmix64(seed, b) % min(B, rows - b * B)


def test_sample_rows_roughly_uniform():
    B, nb = 8, 40000
    pos = np.array([O.sample_row(B * nb, B, 7, b) - b * B for b in range(nb)])
    counts = np.bincount(pos, minlength=B)
    assert np.all(np.abs(counts - nb / B) < 5 * math.sqrt(nb / B))


def _full_table(A, k):
    return O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, k).table


def test_spec_one_sampled_row_diagonal():
    """block_rows = rows (one sampled row), diagonal of all 1.0 -> entries {1024}"""
    A = gi.from_dense(np.eye(50))
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, 8, sample_block_rows=50, seed=3)
    assert list(R.table) == [1024]


@pytest.mark.parametrize("k", [1, 2, 8, 64])
@pytest.mark.parametrize("name", ["powerlaw", "random_wide", "varcoef"])
def test_spec_block_rows_one_equals_full(name, k):
    """block_rows = 1 samples every row -> the full-scan table, bit for bit"""
    A = {"powerlaw": lambda: gi.powerlaw_spd(3000, seed=2),
         "random_wide": lambda: gi.random_csr(500, 400, 6, seed=5, value_kind="wide"),
         "varcoef": lambda: gi.poisson2d(16, "varcoef")}[name]()
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, k, sample_block_rows=1, seed=99)
    assert np.array_equal(R.table, _full_table(A, k))


def test_spec_parity_classes():
    """100x100, two exponent classes by row parity, block_rows = 2 (every block holds
    one row of each class): the sampled table has the full-scan table's entries"""
    d = np.zeros((100, 100))
    for i in range(100):
        d[i, i] = 1.5 if i % 2 == 0 else 3.0 * 2.0 ** -20
        d[i, (i + 1) % 100] = 1.25 if i % 2 == 0 else 2.0 ** -20
    A = gi.from_dense(d)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, 8, sample_block_rows=2, seed=42)
    assert sorted(R.table) == sorted(_full_table(A, 8))


@pytest.mark.parametrize("seed", [0, 1, 42])
@pytest.mark.parametrize("B", [1, 3, 16, 1000])
def test_sampled_histogram_is_the_sampled_rows(seed, B):
    A = gi.random_csr(400, 300, 5, seed=seed + 10, value_kind="mixed", empty_rows=0.1)
    h = O.sampled_histogram(A.rows, A.row_ptr, A.val, B, seed)
    want = np.zeros(2048, np.uint64)
    for b in range((A.rows + B - 1) // B):
        r = b * B + splitmix64(seed, b) % min(B, A.rows - b * B)
        for j in range(A.row_ptr[r], A.row_ptr[r + 1]):
            e = biased_exponent(A.val[j])
            if e:
                want[e] += 1
    assert np.array_equal(h, want)


@pytest.mark.parametrize("seed", range(30))
def test_table_emax_brute_force(seed):
    """selection on a sample with the TRUE e_max forced: maximal sample coverage among
    subsets containing e_max_true of size min(k, #distinct sampled), or one more when e_max
    was not sampled and a slot is free (R27b)"""
    rng = np.random.default_rng(seed)
    nd = int(rng.integers(1, 7))
    exps = rng.choice(np.arange(1, 2000), nd, replace=False)
    counts = rng.integers(1, 6, nd)
    hist = np.zeros(2048, np.uint64)
    for e, c in zip(exps, counts):
        hist[int(e)] = int(c)
    e_true = int(max(exps)) + int(rng.integers(0, 3))  # may exceed every sampled exponent
    k = int(rng.choice([1, 2, 4]))
    table = [int(t) for t in O.build_table_emax(hist, k, e_true)]
    sel = [t - 1 for t in table]
    sampled_max = e_true in set(int(e) for e in exps)
    size = min(k, nd) if (sampled_max or nd >= k) else nd + 1
    assert e_true in sel and len(set(sel)) == len(sel) == size
    pool = sorted(set(int(e) for e in exps) | {e_true})
    best = max(sum(int(hist[e]) for e in c) for c in itertools.combinations(pool, len(sel))
               if e_true in c)
    assert sum(int(hist[e]) for e in sel) == best


def test_free_slot_takes_the_true_max():
    """R27b (advisor finding): a sample {1023} with the true e_max 1030 and k = 8 keeps the
    sampled class and appends 1031 instead of overwriting it"""
    hist = np.zeros(2048, np.uint64)
    hist[1023] = 5
    assert list(O.build_table_emax(hist, 8, 1030)) == [1024, 1031]
    assert list(O.build_table_emax(hist, 1, 1030)) == [1031]


def test_empty_sample_gives_forced_entry_only():
    hist = np.zeros(2048, np.uint64)
    assert list(O.build_table_emax(hist, 8, 1030)) == [1031]


def test_unsampled_max_exponent_stays_representable():
    """the largest value sits in a row the sampler skips: the table still ends at e_max + 1,
    every value encodes, and level 3 round-trips every value with d <= 11"""
    rng = np.random.default_rng(4)
    n = 64
    d = np.diag(rng.uniform(1, 2, n))
    seed, B = 11, n  # one sampled row for the whole matrix
    r_s = O.sample_row(n, B, seed, 0)
    r_big = (r_s + 5) % n
    d[r_big, (r_big + 1) % n] = 2.0 ** 40
    A = gi.from_dense(d)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, 2, sample_block_rows=B, seed=seed)
    assert max(R.table) == biased_exponent(2.0 ** 40) + 1
    back = O.decode_all(R, 3)
    for v, w, t in zip(A.val, back, range(A.nnz)):
        e = biased_exponent(v)
        dd = min(E - e for E in R.table if E - e >= 1)
        if dd <= 11:
            assert v == w
