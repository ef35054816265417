"""Pins of the oracle codec (histogram, table, encode, segment, decode) against what the
paper and the mathematics fix -- never against the oracle itself:
  * worked examples printed in SPEC.md (tests/golden/spec_examples.json, cited per entry);
  * brute force over all k-subsets of tiny histograms (P:116 + P:123);
  * the closed form |v| = trunc53(D_L) * 2^(E-1086), evaluated with Python integers;
  * literal transcriptions of Alg. 1 and Alg. 2;
  * invariants of S:107-113 (round trip for d <= 11, truncation monotonicity, tight
    head-only bound 2^-(15-d) -- reading R23).
"""
import itertools
import json
import math
import os
import struct

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def flt(u: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", u))[0]


# ------------------------------------------------------------------ golden examples
@pytest.mark.parametrize("ex", GOLD["build_table"], ids=lambda e: e["cite"])
def test_table_examples(ex):
    hist = {int(k): v for k, v in ex["hist"].items()}
    assert list(O.build_table(hist, ex["k_max"])) == ex["entries"]


@pytest.mark.parametrize("ex", GOLD["exponent_histogram"], ids=lambda e: e["cite"])
def test_histogram_examples(ex):
    st, hist, nz, bad = O.exponent_histogram(np.array(ex["values"]))
    assert st == O.OK and bad == -1 and nz == 0
    got = {int(e): int(hist[e]) for e in np.nonzero(hist)[0]}
    assert got == {int(k): v for k, v in ex["hist"].items()}


def test_histogram_zero_subnormal_nonfinite():
    st, hist, nz, bad = O.exponent_histogram(np.array([0.0, -0.0, 5e-324, 1.0]))
    assert st == O.OK and nz == 3 and hist.sum() == 1
    st, _, _, bad = O.exponent_histogram(np.array([1.0, 2.0, np.inf, np.nan]))
    assert st == O.ERR_NONFINITE and bad == 2


def test_table_errors():
    with pytest.raises(O.OracleError) as e:
        O.build_table({}, 8)
    assert e.value.status == O.ERR_NO_VALUES
    with pytest.raises(O.OracleError):
        O.build_table({1023: 1}, 3)  # k_max must be a power of two


@pytest.mark.parametrize("ex", GOLD["encode"], ids=lambda e: e["cite"])
def test_encode_examples(ex):
    w, ei = O.encode_value(ex["x"], ex["table"])
    assert w == int(ex["word"], 16) and ei == ex["ei"]
    assert O.segment(w)[0] == int(ex["head"], 16)


@pytest.mark.parametrize("ex", GOLD["decode"], ids=lambda e: e["cite"])
def test_decode_examples(ex):
    w = O.assemble(int(ex["head"], 16), 0, 0, ex["level"])
    v = O.decode(w, ex["ei"], ex["table"])
    assert v == ex["value"] and math.copysign(1, v) == math.copysign(1, ex["value"])


@pytest.mark.parametrize("ex", GOLD["round_trip"], ids=lambda e: e["cite"])
def test_round_trip_example(ex):
    x = flt(int(ex["x_hex"], 16))
    w, ei = O.encode_value(x, ex["table"])
    assert bits(O.decode(w, ei, ex["table"])) == bits(x)


@pytest.mark.parametrize("ex", GOLD["head16"], ids=lambda e: e["cite"])
def test_head16_examples(ex):
    assert O.encode_head16_with_ei(ex["x"], ex["table"], ex["ei_bits"]) == int(ex["word"], 16)


@pytest.mark.parametrize("ex", GOLD["segment"], ids=lambda e: e["cite"])
def test_segment_examples(ex):
    w = int(ex["word"], 16)
    if "head" in ex:
        assert O.segment(w) == (int(ex["head"], 16), int(ex["tail1"], 16), int(ex["tail2"], 16))
    else:
        h, t1, t2 = O.segment(w)
        assert O.assemble(h, t1, t2, ex["level"]) == int(ex["assembled"], 16)


def test_segment_round_trip_random():
    rng = np.random.default_rng(1)
    for w in rng.integers(0, 2**63, 20000, dtype=np.uint64).tolist() + [2**64 - 1, 0]:
        h, t1, t2 = O.segment(w)
        assert O.assemble(h, t1, t2, 3) == w
        assert O.assemble(h, t1, t2, 1) == (w >> 48) << 48


# ------------------------------------------------------------------ table: brute force
def _coverage(hist, exps):
    return sum(hist[e] for e in exps)


@pytest.mark.parametrize("seed", range(40))
def test_table_brute_force(seed):
    """P:116 (top-k by count) + P:123 (e_max+1 mandatory): among all subsets of size
    min(k, #distinct) that contain e_max, the oracle's table reaches the maximal coverage;
    entries are e+1, distinct, max(entries)-1 = e_max."""
    rng = np.random.default_rng(seed)
    nd = int(rng.integers(1, 8))
    exps = rng.choice(np.arange(1, 2047), nd, replace=False)
    counts = rng.integers(1, 6, nd)  # small counts -> many ties
    hist = {int(e): int(c) for e, c in zip(exps, counts)}
    k = int(rng.choice([1, 2, 4]))
    table = [int(t) for t in O.build_table(hist, k)]
    sel = [t - 1 for t in table]
    e_max = max(hist)
    take = min(k, nd)
    assert len(sel) == take == len(set(sel)) and max(sel) == e_max
    best = max(_coverage(hist, s) for s in itertools.combinations(hist, take) if e_max in s)
    assert _coverage(hist, sel) == best
    # order: (count desc, e desc) except the forced e_max slot, which is last
    core = sel if e_max in sel[:-1] or len(sel) == 1 else sel[:-1]
    keys = [(-hist[e], -e) for e in core]
    assert keys == sorted(keys)


# ------------------------------------------------------------------ encode/decode laws
def _closed_form(word: int, E: int) -> float:
    """|v| = trunc53(D_L) * 2^(E-1086) with flush when the true exponent <= 0 (S:84,
    R11): evaluated with Python integers and math.ldexp (exact for normal results)."""
    s = word >> 63
    D = word & (2**63 - 1)
    if D == 0:
        return -0.0 if s else 0.0
    pos = D.bit_length() - 1
    if E - (63 - pos) <= 0:
        return -0.0 if s else 0.0
    if pos > 52:
        D = (D >> (pos - 52)) << (pos - 52)
    v = math.ldexp(float(D), E - 1086)
    return -v if s else v


def test_decode_closed_form_random_words():
    rng = np.random.default_rng(2)
    table = [1, 2, 40, 1023, 1024, 1100, 2046, 2047]
    for _ in range(30000):
        w = int(rng.integers(0, 2**64, dtype=np.uint64))
        if rng.random() < 0.5:  # few significant bits, exercise small D and flushes
            w &= ~((1 << int(rng.integers(0, 63))) - 1)
            w &= (1 << 63) | ((1 << int(rng.integers(1, 64))) - 1)
        ei = int(rng.integers(0, len(table)))
        for level in (1, 2, 3):
            h, t1, t2 = O.segment(w)
            wl = O.assemble(h, t1, t2, level)
            got, want = O.decode(wl, ei, table), _closed_form(wl, table[ei])
            assert bits(got) == bits(want), (hex(w), ei, level)


def test_decode_invalid_index():
    with pytest.raises(O.OracleError) as e:
        O.decode(1 << 62, 1, [1024])
    assert e.value.status == O.ERR_INVALID_EXP_INDEX


def _rand_values(rng, n, exps):
    f = rng.integers(0, 1 << 52, n, dtype=np.int64)
    e = np.asarray(exps)[rng.integers(0, len(exps), n)]
    s = rng.integers(0, 2, n)
    return [flt((int(si) << 63) | (int(ei) << 52) | int(fi)) for si, ei, fi in zip(s, e, f)]


def test_round_trip_bit_exact_for_d_le_11():
    """decode(Full, encode(x)) == x bitwise whenever d <= 11."""
    rng = np.random.default_rng(3)
    exps = [1013, 1016, 1020, 1022, 1023]
    table = list(O.build_table({1023: 10, 1016: 3}, 2))  # [1024, 1017]
    n_checked = 0
    for x in _rand_values(rng, 20000, exps):
        w, ei = O.encode_value(x, table)
        d = table[ei] - ((bits(x) >> 52) & 0x7FF)
        if d <= 11:
            n_checked += 1
            assert bits(O.decode(w, ei, table)) == bits(x)
    assert n_checked > 15000


def test_truncation_monotone_and_tight_head_bound():
    """S:109-110 with the tight bound of R23: |x - dec_1| / |x| < 2^-(15-d) for d <= 14;
    |dec_1| <= |dec_2| <= |dec_3| <= |x|, errors non-increasing in the level."""
    rng = np.random.default_rng(4)
    table = [1024, 1020, 1010]
    worst = {}
    for x in _rand_values(rng, 20000, list(range(1000, 1024))):
        w, ei = O.encode_value(x, table)
        h, t1, t2 = O.segment(w)
        dec = [O.decode(O.assemble(h, t1, t2, L), ei, table) for L in (1, 2, 3)]
        mags = [abs(v) for v in dec]
        assert mags[0] <= mags[1] <= mags[2] <= abs(x)
        errs = [abs(x - v) for v in dec]
        assert errs[0] >= errs[1] >= errs[2]
        for v in dec:
            assert v == 0 or math.copysign(1, v) == math.copysign(1, x)
        d = table[ei] - ((bits(x) >> 52) & 0x7FF)
        if d <= 14:
            rel = errs[0] / abs(x)
            assert rel < 2.0 ** -(15 - d)
            worst[d] = max(worst.get(d, 0.0), rel)
    assert worst[1] > 2.0 ** -15  # the bound is tight: 15-d fraction bits, not 14-d


def test_encode_zero_subnormal_flush_nonfinite():
    assert O.encode_value(-0.0, [1024]) == (1 << 63, 0)
    assert O.encode_value(5e-324, [1024]) == (0, 0)  # subnormal -> signed zero (R2)
    w, ei = O.encode_value(2.0 ** -100, [1024, 1030])  # d > 63 -> flush, EI kept (R3)
    assert w == 0 and ei == 0
    for bad in (np.inf, -np.inf, np.nan):
        with pytest.raises(O.OracleError) as e:
            O.encode_value(bad, [1024])
        assert e.value.status == O.ERR_NONFINITE
    with pytest.raises(O.OracleError) as e:
        O.encode_value(4.0, [1024])  # no entry > e (caller table) -> unrepresentable
    assert e.value.status == O.ERR_UNREPRESENTABLE


def test_encode_explicit_one_position():
    """the highest set bit of D is at 63-d (d = E - e >= 1, nearest entry above)."""
    rng = np.random.default_rng(5)
    table = [1030, 1024, 1000, 1015]
    for x in _rand_values(rng, 5000, list(range(980, 1030))):
        e = (bits(x) >> 52) & 0x7FF
        w, ei = O.encode_value(x, table)
        cands = [t - e for t in table if t - e >= 1]
        d = min(cands)
        assert table[ei] - e == d
        D = w & (2**63 - 1)
        if d <= 63:
            assert D.bit_length() - 1 == 63 - d


# ------------------------------------------------------------------ literal Alg. 1 / Alg. 2
MAX_52 = (1 << 52) - 1


def alg1_literal(valD: int, SEM, EI_bit: int) -> int:
    """Line-by-line transcription of Alg. 1 for one element."""
    sign = (valD >> 48) & 0x8000
    exp = (valD >> 52) & 0x7FF
    minDiff = 0xFFFFFFFF
    numExp = len(SEM)
    expIdx = 0
    k = 0
    while k < numExp:
        if exp + 1 == SEM[k]:
            expIdx = k
            minDiff = 1
            break
        k += 1
    if k == numExp:
        for jj in range(numExp):
            diff = SEM[jj] - exp
            if diff > 0 and diff < minDiff:
                minDiff = diff
                expIdx = jj
    expIdx = expIdx << (15 - EI_bit)
    valD = (valD & MAX_52) >> minDiff
    valD = valD >> (37 + EI_bit)
    valD = valD | (0x1 << (15 - EI_bit - minDiff))
    return (sign | expIdx | valD) & 0xFFFF


@pytest.mark.parametrize("k", [2, 4, 8])
def test_head16_equals_literal_alg1(k):
    """encode_head16_with_ei == literal Alg. 1 on random normal inputs whose
    d keeps the explicit one inside the word (the only case Alg. 1 defines, R3)."""
    rng = np.random.default_rng(10 + k)
    eib = int(math.log2(k))
    table = sorted(rng.choice(np.arange(1000, 1040), k, replace=False).tolist(), reverse=True)
    n = 0
    for x in _rand_values(rng, 30000, list(range(995, max(table)))):
        e = (bits(x) >> 52) & 0x7FF
        d = min(t - e for t in table if t - e >= 1)
        if d > 15 - eib:
            continue
        n += 1
        assert O.encode_head16_with_ei(x, table, eib) == alg1_literal(bits(x), table, eib)
    assert n > 10000


def alg2_head_literal(val: int, E: int) -> float:
    """Transcription of Alg. 2 l.6-17 for one head (R7, R8)."""
    val_FP64 = (val & 0x8000) << 48
    pos = None
    for b in range(14, -1, -1):  # __fns(val, 14, -1): first set bit at or below bit 14
        if (val >> b) & 1:
            pos = b
            break
    if pos is not None:
        val_FP64 |= (E - (15 - pos)) << 52
        temp = (val & 0x7FFF) << 36
        temp = (temp << (16 - pos)) & MAX_52
        val_FP64 |= temp
    else:
        val_FP64 = 0
    return flt(val_FP64)


def test_decode_head_equals_literal_alg2():
    """Alg. 2 equals the oracle's level-1 decode on every nonzero head (R10: only the sign
    of a zero head differs)."""
    for E in (30, 1024, 2047):
        for head in range(1 << 16):
            if head & 0x7FFF == 0:
                continue
            assert bits(O.decode(head << 48, 0, [E])) == bits(alg2_head_literal(head, E))


# ------------------------------------------------------------------ CSR conversion
@pytest.mark.parametrize("ex", GOLD["convert"], ids=lambda e: e["cite"])
def test_convert_examples(ex):
    import gse_inputs as gi
    A = gi.from_dense(np.array(ex["dense"]))
    G = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, ex["k_max"])
    assert [hex(h) for h in G.head] == [hex(int(h, 16)) for h in ex["heads"]]
    if "table" in ex:
        assert list(G.table) == ex["table"]
        assert list(G.tail1) == ex["tail1"] and list(G.tail2) == ex["tail2"]
        assert list(G.col_ei >> 29) == ex["ei"]


def test_convert_embedding_and_side_array():
    """P:168 / Alg. 2 l.3-5: EI in the top log2(k) bits of the column index; side array
    iff cols >= 2^(32-ei_bits)."""
    import gse_inputs as gi
    A = gi.random_csr(50, 60, 5, seed=3, exps=[1010, 1023, 1030, 1040])
    G = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val, 8)
    assert G.ei_bits == 3 and G.ei_in_column
    assert np.array_equal(G.col_ei & ((1 << 29) - 1), A.col.astype(np.uint32))
    for i in range(A.nnz):
        w, ei = O.encode_value(A.val[i], G.table)
        assert int(G.col_ei[i]) >> 29 == ei
        assert O.assemble(int(G.head[i]), int(G.tail1[i]), int(G.tail2[i]), 3) == w
    # capacity rule: cols = 2^30 with ei_bits 3 -> side array
    rp = np.array([0, 2], np.int64)
    G2 = O.encode_csr(1, 1 << 30, rp, np.array([5, (1 << 30) - 1], np.int32),
                      np.array([1.0, 3.0]), 8)
    assert not G2.ei_in_column and G2.side_ei is not None
    assert list(G2.col_ei) == [5, (1 << 30) - 1] and list(G2.side_ei) == [1, 0]


def test_convert_errors():
    rp = np.array([0, 2], np.int64)
    with pytest.raises(O.OracleError) as e:
        O.encode_csr(1, 4, rp, np.array([0, 3], np.int32), np.array([1.0, np.nan]))
    assert e.value.status == O.ERR_NONFINITE and e.value.bad_index == 1
    with pytest.raises(O.OracleError) as e:
        O.encode_csr(1, 4, rp, np.array([0, 3], np.int32), np.array([0.0, 0.0]))
    assert e.value.status == O.ERR_NO_VALUES
    with pytest.raises(O.OracleError) as e:
        O.encode_csr(1, 3, rp, np.array([0, 3], np.int32), np.array([1.0, 1.0]))
    assert e.value.status == O.ERR_INVALID_ARG
