"""ORACLE -- plain CPU reference of the GSE-SEM method (arXiv 2411.04686).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2411_04686_b200``) never imports it; the two share no code.

This module is a ctypes wrapper over ``gse_oracle.c`` (plain C99, fp64, no fast-math).
Every numerical step lives in the C file, each function citing the PAPER.md/SPEC.md
passage it follows; this file only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gse_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
# ORACLE_SANITIZE=1: an ASan + UBSan build (scripts/oracle_sanitize.sh; run with libasan
# preloaded) in a separate file, so the normal build is untouched
_SANITIZE = os.environ.get("ORACLE_SANITIZE") == "1"
if _SANITIZE:
    _LIB_PATH = os.path.join(_HERE, "liboracle_san.so")

OK, NOT_CONVERGED, NUMERICAL_ABORT = 0, 2, 3
ERR_INVALID_ARG, ERR_DIM, ERR_NONFINITE, ERR_NO_VALUES = 10, 11, 12, 13
ERR_UNREPRESENTABLE, ERR_INVALID_EXP_INDEX = 14, 15


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, -ffp-contract=off so a*b+c is never fused)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "gse_oracle.h"))
    ):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        san = ["-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
               "-fno-omit-frame-pointer", "-g"] if _SANITIZE else []
        subprocess.check_call(
            ["gcc", "-std=c99", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
             "-fopenmp", *san, "-shared", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


def _p(t):
    return C.POINTER(t)


class OrcMatrix(C.Structure):
    _fields_ = [
        ("rows", C.c_int64), ("cols", C.c_int64),
        ("row_ptr", _p(C.c_int64)), ("col", _p(C.c_int32)), ("val", _p(C.c_double)),
        ("col_ei", _p(C.c_uint32)), ("side_ei", _p(C.c_uint8)),
        ("ei_bits", C.c_int), ("ei_in_column", C.c_int),
        ("head", _p(C.c_uint16)), ("tail1", _p(C.c_uint16)), ("tail2", _p(C.c_uint32)),
        ("table", _p(C.c_uint16)), ("table_len", C.c_int),
        ("half_kind", C.c_int), ("half", _p(C.c_uint16)),
    ]


class OrcSchedule(C.Structure):
    _fields_ = [
        ("enabled", C.c_int), ("start_level", C.c_int), ("max_level", C.c_int),
        ("l", C.c_int64), ("t", C.c_int64), ("m", C.c_int64),
        ("rsd_limit", C.c_double), ("ndec_limit", C.c_int64), ("reldec_limit", C.c_double),
        ("verify_at_full", C.c_int), ("level_floor", C.c_double * 2),
        ("krylov_gse16", C.c_int), ("perturb_c", C.c_double),
        ("cg_keep_direction", C.c_int),
    ]


class OrcReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64), ("iters_per_level", C.c_int64 * 3),
        ("converged", C.c_int), ("n_switches", C.c_int),
        ("switch_iter", C.c_int64 * 2), ("switch_to_level", C.c_int * 2),
        ("rel_residual_recurrence", C.c_double), ("rel_residual_true", C.c_double),
        ("spmv_count", C.c_int64 * 3),
    ]


def _declare(L):
    i64, i32, dbl = C.c_int64, C.c_int, C.c_double
    L.orc_exponent_histogram.argtypes = [i64, _p(dbl), _p(C.c_uint64), _p(i64), _p(i64)]
    L.orc_build_table.argtypes = [_p(C.c_uint64), i32, _p(C.c_uint16), _p(i32)]
    L.orc_encode_value.argtypes = [dbl, _p(C.c_uint16), i32, _p(C.c_uint64), _p(i32)]
    L.orc_segment.argtypes = [C.c_uint64, _p(C.c_uint16), _p(C.c_uint16), _p(C.c_uint32)]
    L.orc_segment.restype = None
    L.orc_assemble.argtypes = [C.c_uint16, C.c_uint16, C.c_uint32, i32]
    L.orc_assemble.restype = C.c_uint64
    L.orc_decode.argtypes = [C.c_uint64, i32, _p(C.c_uint16), i32, _p(dbl)]
    L.orc_encode_head16_with_ei.argtypes = [dbl, _p(C.c_uint16), i32, i32, _p(C.c_uint16)]
    L.orc_decode_head16_with_ei.argtypes = [C.c_uint16, _p(C.c_uint16), i32, i32, _p(dbl)]
    L.orc_encode_vector16.argtypes = [i64, _p(dbl), i32, _p(C.c_uint16), _p(C.c_uint16), _p(i32)]
    L.orc_decode_vector16.argtypes = [i64, _p(C.c_uint16), _p(C.c_uint16), i32, i32, _p(dbl)]
    L.orc_encode_csr.argtypes = [i64, i64, i64, _p(i64), _p(C.c_int32), _p(dbl), i32,
                                 _p(C.c_uint16), _p(i32), _p(i32), _p(i32), _p(C.c_uint32),
                                 _p(C.c_uint8), _p(C.c_uint16), _p(C.c_uint16),
                                 _p(C.c_uint32), _p(i64)]
    L.orc_encode_csr_sampled.argtypes = [i64, i64, i64, _p(i64), _p(C.c_int32), _p(dbl), i32,
                                         i64, C.c_uint64, _p(C.c_uint16), _p(i32), _p(i32),
                                         _p(i32), _p(C.c_uint32), _p(C.c_uint8),
                                         _p(C.c_uint16), _p(C.c_uint16), _p(C.c_uint32), _p(i64)]
    L.orc_build_table_emax.argtypes = [_p(C.c_uint64), i32, i32, _p(C.c_uint16), _p(i32)]
    L.orc_sample_z.argtypes = [C.c_uint64, i64]
    L.orc_sample_z.restype = C.c_uint64
    L.orc_sample_row.argtypes = [i64, i64, C.c_uint64, i64]
    L.orc_sample_row.restype = i64
    L.orc_sampled_histogram.argtypes = [i64, _p(i64), _p(dbl), i64, C.c_uint64, _p(C.c_uint64)]
    L.orc_spmv_fp64.argtypes = [i64, _p(i64), _p(C.c_int32), _p(dbl), _p(dbl), _p(dbl)]
    L.orc_spmv_gse.argtypes = [_p(OrcMatrix), i32, _p(dbl), _p(dbl)]
    L.orc_rsd.argtypes = [_p(dbl), i64]
    L.orc_rsd.restype = dbl
    L.orc_ndec.argtypes = [_p(dbl), i64]
    L.orc_ndec.restype = i64
    L.orc_reldec.argtypes = [_p(dbl), i64]
    L.orc_reldec.restype = dbl
    L.orc_should_escalate.argtypes = [_p(dbl), i64, dbl, i64, dbl]
    L.orc_perturbation_bounds.argtypes = [C.c_void_p, _p(dbl)]
    L.orc_default_schedule.argtypes = [i32, _p(OrcSchedule)]
    L.orc_default_schedule.restype = None
    L.orc_cg.argtypes = [_p(OrcMatrix), _p(dbl), _p(dbl), dbl, i64, _p(OrcSchedule),
                         _p(OrcReport)]
    L.orc_cg_part.argtypes = [_p(OrcMatrix), _p(dbl), _p(dbl), dbl, i64, _p(OrcSchedule), i32,
                              _p(i64), _p(OrcReport)]
    L.orc_gmres_part.argtypes = [_p(OrcMatrix), _p(dbl), _p(dbl), dbl, i32, i64, _p(OrcSchedule),
                                 i32, _p(i64), _p(OrcReport)]
    L.orc_gmres.argtypes = [_p(OrcMatrix), _p(dbl), _p(dbl), dbl, i32, i64, _p(OrcSchedule),
                            _p(OrcReport)]
    L.orc_set_threads.argtypes = [i32]
    L.orc_round_half.argtypes = [dbl, i32]
    L.orc_round_half.restype = C.c_uint16
    L.orc_half_value.argtypes = [C.c_uint16, i32]
    L.orc_half_value.restype = dbl
    L.orc_round_half_array.argtypes = [i64, _p(dbl), _p(C.c_uint16), i32]
    L.orc_round_half_array.restype = None
    L.orc_half_value_array.argtypes = [i64, _p(C.c_uint16), _p(dbl), i32]
    L.orc_half_value_array.restype = None
    L.orc_spmv_half.argtypes = [_p(OrcMatrix), _p(dbl), _p(dbl)]


def _ptr(a: np.ndarray, ct):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ct))


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what}: status {status}")
        self.status = status


def set_threads(n: int = 0) -> int:
    """GSE_THREADS knob. n <= 0 keeps the OpenMP default. Returns threads used."""
    return lib().orc_set_threads(n)


# ------------------------------------------------------------------ codec
def exponent_histogram(values: np.ndarray):
    v = np.ascontiguousarray(values, dtype=np.float64)
    hist = np.zeros(2048, dtype=np.uint64)
    nz, bad = C.c_int64(), C.c_int64()
    st = lib().orc_exponent_histogram(v.size, _ptr(v, C.c_double), _ptr(hist, C.c_uint64),
                                      C.byref(nz), C.byref(bad))
    return st, hist, nz.value, bad.value


def build_table(hist, k_max: int = 8):
    h = np.zeros(2048, dtype=np.uint64)
    if isinstance(hist, dict):
        for e, c in hist.items():
            h[e] = c
    else:
        h[:] = hist
    table = np.zeros(64, dtype=np.uint16)
    n = C.c_int()
    st = lib().orc_build_table(_ptr(h, C.c_uint64), k_max, _ptr(table, C.c_uint16), C.byref(n))
    if st != OK:
        raise OracleError(st, "build_table")
    return table[: n.value].copy()


def decode_head16_with_ei(word: int, table, ei_bits: int) -> float:
    t = np.ascontiguousarray(table, dtype=np.uint16)
    out = C.c_double()
    st = lib().orc_decode_head16_with_ei(word, _ptr(t, C.c_uint16), t.size, ei_bits, C.byref(out))
    if st != OK:
        raise OracleError(st, "decode_head16_with_ei")
    return out.value


def encode_vector16(v, k_max: int = 8):
    """NEXT-4: a vector in 16-bit GSE-SEM form (Alg. 1): (words uint16[n], table)."""
    x = np.ascontiguousarray(v, dtype=np.float64)
    words = np.zeros(max(x.size, 1), np.uint16)
    table = np.zeros(64, np.uint16)
    tl = C.c_int()
    st = lib().orc_encode_vector16(x.size, _ptr(x, C.c_double), k_max, _ptr(words, C.c_uint16),
                                   _ptr(table, C.c_uint16), C.byref(tl))
    if st != OK:
        raise OracleError(st, "encode_vector16")
    return words[:x.size].copy(), table[:tl.value].copy()


def decode_vector16(words, table, ei_bits: int = 3):
    w = np.ascontiguousarray(words, dtype=np.uint16)
    t = np.ascontiguousarray(table, dtype=np.uint16)
    tt = t if t.size else np.zeros(1, np.uint16)
    out = np.zeros(max(w.size, 1), np.float64)
    st = lib().orc_decode_vector16(w.size, _ptr(w, C.c_uint16), _ptr(tt, C.c_uint16), t.size,
                                   ei_bits, _ptr(out, C.c_double))
    if st != OK:
        raise OracleError(st, "decode_vector16")
    return out[:w.size]


def sample_row(rows: int, block_rows: int, seed: int, b: int) -> int:
    """NEXT-3 (R27): the random row of row block b."""
    return lib().orc_sample_row(rows, block_rows, seed, b)


def sample_z(seed: int, b: int) -> int:
    return lib().orc_sample_z(seed, b)


def sampled_histogram(rows, row_ptr, val, block_rows: int, seed: int):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    v = np.ascontiguousarray(val, dtype=np.float64)
    hist = np.zeros(2048, dtype=np.uint64)
    st = lib().orc_sampled_histogram(rows, _ptr(rp, C.c_int64), _ptr(v, C.c_double), block_rows,
                                     seed, _ptr(hist, C.c_uint64))
    if st != OK:
        raise OracleError(st, "sampled_histogram")
    return hist


def build_table_emax(hist, k_max: int, e_max_true: int):
    h = np.ascontiguousarray(hist, dtype=np.uint64)
    table = np.zeros(64, dtype=np.uint16)
    n = C.c_int()
    st = lib().orc_build_table_emax(_ptr(h, C.c_uint64), k_max, e_max_true,
                                    _ptr(table, C.c_uint16), C.byref(n))
    if st != OK:
        raise OracleError(st, "build_table_emax")
    return table[: n.value].copy()


def encode_value(x: float, table):
    t = np.ascontiguousarray(table, dtype=np.uint16)
    w, ei = C.c_uint64(), C.c_int()
    st = lib().orc_encode_value(float(x), _ptr(t, C.c_uint16), t.size, C.byref(w), C.byref(ei))
    if st != OK:
        raise OracleError(st, "encode_value")
    return w.value, ei.value


def segment(word: int):
    h, t1, t2 = C.c_uint16(), C.c_uint16(), C.c_uint32()
    lib().orc_segment(C.c_uint64(word), C.byref(h), C.byref(t1), C.byref(t2))
    return h.value, t1.value, t2.value


def assemble(head: int, tail1: int, tail2: int, level: int) -> int:
    return lib().orc_assemble(head, tail1, tail2, level)


def decode(word: int, ei: int, table) -> float:
    t = np.ascontiguousarray(table, dtype=np.uint16)
    out = C.c_double()
    st = lib().orc_decode(C.c_uint64(word), ei, _ptr(t, C.c_uint16), t.size, C.byref(out))
    if st != OK:
        raise OracleError(st, "decode")
    return out.value


def encode_head16_with_ei(x: float, table, ei_bits: int) -> int:
    t = np.ascontiguousarray(table, dtype=np.uint16)
    out = C.c_uint16()
    st = lib().orc_encode_head16_with_ei(float(x), _ptr(t, C.c_uint16), t.size, ei_bits,
                                         C.byref(out))
    if st != OK:
        raise OracleError(st, "encode_head16_with_ei")
    return out.value


# ------------------------------------------------------------------ matrices
@dataclass
class GseCsr:
    """Encoded matrix as produced by the oracle (numpy arrays, host)."""
    rows: int
    cols: int
    nnz: int
    row_ptr: np.ndarray  # int64
    col_ei: np.ndarray  # uint32
    side_ei: np.ndarray | None  # uint8 or None
    head: np.ndarray  # uint16
    tail1: np.ndarray  # uint16
    tail2: np.ndarray  # uint32
    table: np.ndarray  # uint16
    ei_bits: int
    ei_in_column: bool
    _keep: list = field(default_factory=list, repr=False)

    def orc(self) -> OrcMatrix:
        m = OrcMatrix()
        m.rows, m.cols = self.rows, self.cols
        m.row_ptr = _ptr(self.row_ptr, C.c_int64)
        m.col_ei = _ptr(self.col_ei, C.c_uint32)
        side = self.side_ei if self.side_ei is not None else np.zeros(1, np.uint8)
        self._keep = [side]
        m.side_ei = _ptr(side, C.c_uint8)
        m.ei_bits, m.ei_in_column = self.ei_bits, int(self.ei_in_column)
        m.head = _ptr(self.head, C.c_uint16)
        m.tail1 = _ptr(self.tail1, C.c_uint16)
        m.tail2 = _ptr(self.tail2, C.c_uint32)
        m.table = _ptr(self.table, C.c_uint16)
        m.table_len = self.table.size
        return m


@dataclass
class Fp64Csr:
    rows: int
    cols: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    def orc(self) -> OrcMatrix:
        m = OrcMatrix()
        m.rows, m.cols = self.rows, self.cols
        m.row_ptr = _ptr(self.row_ptr, C.c_int64)
        m.col = _ptr(self.col, C.c_int32)
        m.val = _ptr(self.val, C.c_double)
        return m


def _csr_arrays(row_ptr, col, val):
    return (np.ascontiguousarray(row_ptr, dtype=np.int64),
            np.ascontiguousarray(col, dtype=np.int32),
            np.ascontiguousarray(val, dtype=np.float64))


FP16, BF16 = 1, 2  # orc_round_half kinds (P:406 baselines)


def _half_kind(kind) -> int:
    return {"fp16": FP16, "bf16": BF16, FP16: FP16, BF16: BF16}[kind]


def round_half(values, kind) -> np.ndarray:
    """FP64 -> FP16 / BF16 bit patterns, round-to-nearest-even (R26), overflow -> +-Inf."""
    v = np.ascontiguousarray(values, dtype=np.float64).ravel()
    out = np.zeros(max(v.size, 1), np.uint16)
    lib().orc_round_half_array(v.size, _ptr(v, C.c_double), _ptr(out, C.c_uint16),
                               _half_kind(kind))
    return out[:v.size]


def half_values(bits, kind) -> np.ndarray:
    """FP16 / BF16 bit patterns -> their exact FP64 values."""
    h = np.ascontiguousarray(bits, dtype=np.uint16).ravel()
    out = np.zeros(max(h.size, 1), np.float64)
    lib().orc_half_value_array(h.size, _ptr(h, C.c_uint16), _ptr(out, C.c_double),
                               _half_kind(kind))
    return out[:h.size]


@dataclass
class HalfCsr:
    """The FP16 / BF16 storage baseline: CSR with 16-bit stored values."""
    rows: int
    cols: int
    row_ptr: np.ndarray
    col: np.ndarray
    half: np.ndarray  # uint16 bit patterns
    kind: int

    def orc(self) -> OrcMatrix:
        m = OrcMatrix()
        m.rows, m.cols = self.rows, self.cols
        m.row_ptr = _ptr(self.row_ptr, C.c_int64)
        m.col = _ptr(self.col, C.c_int32)
        m.half_kind = self.kind
        m.half = _ptr(self.half, C.c_uint16)
        return m


def half_csr(rows, cols, row_ptr, col, val, kind) -> HalfCsr:
    rp, c, v = _csr_arrays(row_ptr, col, val)
    h = round_half(v, kind)
    if h.size == 0:
        h = np.zeros(1, np.uint16)
    return HalfCsr(rows, cols, rp, c, np.ascontiguousarray(h), _half_kind(kind))


def spmv_half(A: HalfCsr, x) -> np.ndarray:
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(A.rows, np.float64)
    m = A.orc()
    st = lib().orc_spmv_half(C.byref(m), _ptr(xx, C.c_double), _ptr(y, C.c_double))
    if st != OK:
        raise OracleError(st, "spmv_half")
    return y


def fp64_csr(rows, cols, row_ptr, col, val) -> Fp64Csr:
    rp, c, v = _csr_arrays(row_ptr, col, val)
    return Fp64Csr(rows, cols, rp, c, v)


def encode_csr(rows: int, cols: int, row_ptr, col, val, k_max: int = 8,
               sample_block_rows: int = 0, seed: int = 0) -> GseCsr:
    rp, c, v = _csr_arrays(row_ptr, col, val)
    nnz = v.size
    table = np.zeros(64, dtype=np.uint16)
    tl, eb, inc = C.c_int(), C.c_int(), C.c_int()
    col_ei = np.zeros(max(nnz, 1), np.uint32)
    side = np.zeros(max(nnz, 1), np.uint8)
    head = np.zeros(max(nnz, 1), np.uint16)
    t1 = np.zeros(max(nnz, 1), np.uint16)
    t2 = np.zeros(max(nnz, 1), np.uint32)
    bad = C.c_int64()
    st = lib().orc_encode_csr_sampled(rows, cols, nnz, _ptr(rp, C.c_int64), _ptr(c, C.c_int32),
                              _ptr(v, C.c_double), k_max, sample_block_rows, seed,
                              _ptr(table, C.c_uint16),
                              C.byref(tl), C.byref(eb), C.byref(inc), _ptr(col_ei, C.c_uint32),
                              _ptr(side, C.c_uint8), _ptr(head, C.c_uint16),
                              _ptr(t1, C.c_uint16), _ptr(t2, C.c_uint32), C.byref(bad))
    if st != OK:
        err = OracleError(st, "encode_csr")
        err.bad_index = bad.value
        raise err
    return GseCsr(rows, cols, nnz, rp, col_ei[:nnz].copy(),
                  None if inc.value else side[:nnz].copy(), head[:nnz].copy(),
                  t1[:nnz].copy(), t2[:nnz].copy(), table[: tl.value].copy(), eb.value,
                  bool(inc.value))


def spmv_fp64(A: Fp64Csr, x) -> np.ndarray:
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(A.rows, np.float64)
    lib().orc_spmv_fp64(A.rows, _ptr(A.row_ptr, C.c_int64), _ptr(A.col, C.c_int32),
                        _ptr(A.val, C.c_double), _ptr(xx, C.c_double), _ptr(y, C.c_double))
    return y


def spmv_gse(A: GseCsr, x, level: int) -> np.ndarray:
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(A.rows, np.float64)
    m = A.orc()
    st = lib().orc_spmv_gse(C.byref(m), level, _ptr(xx, C.c_double), _ptr(y, C.c_double))
    if st != OK:
        raise OracleError(st, "spmv_gse")
    return y


def perturbation_bounds(A: GseCsr) -> tuple:
    """R29: (eta_1, eta_2), eta_L = max_i sum_j |dec_3(a_ij) - dec_L(a_ij)|."""
    m = A.orc()
    eta = np.zeros(2)
    st = lib().orc_perturbation_bounds(C.byref(m), _ptr(eta, C.c_double))
    if st != 0:
        raise OracleError(st, "perturbation_bounds")
    return float(eta[0]), float(eta[1])


def decode_all(A: GseCsr, level: int) -> np.ndarray:
    """Decoded values of every stored element (per-element orc_decode)."""
    out = np.empty(A.nnz, np.float64)
    sh = 32 - A.ei_bits
    for i in range(A.nnz):
        c = int(A.col_ei[i])
        ei = (c >> sh if A.ei_bits else 0) if A.ei_in_column else int(A.side_ei[i])
        w = assemble(int(A.head[i]), int(A.tail1[i]), int(A.tail2[i]), level)
        out[i] = decode(w, ei, A.table)
    return out


# ------------------------------------------------------------------ monitor
def _arr(w):
    return np.ascontiguousarray(w, dtype=np.float64)


def rsd(window, t: int | None = None) -> float:
    w = _arr(window)
    return lib().orc_rsd(_ptr(w, C.c_double), len(w) if t is None else t)


def n_dec(window) -> int:
    w = _arr(window)
    return lib().orc_ndec(_ptr(w, C.c_double), len(w) - 1)


def rel_dec(window, t: int | None = None) -> float:
    w = _arr(window)
    return lib().orc_reldec(_ptr(w, C.c_double), len(w) if t is None else t)


def should_escalate(window, rsd_limit, ndec_limit, reldec_limit) -> bool:
    w = _arr(window)
    return bool(lib().orc_should_escalate(_ptr(w, C.c_double), len(w) - 1, rsd_limit,
                                          ndec_limit, reldec_limit))


# ------------------------------------------------------------------ solvers
def default_schedule(solver: str) -> OrcSchedule:
    s = OrcSchedule()
    lib().orc_default_schedule(0 if solver == "cg" else 1, C.byref(s))
    return s


def schedule(solver: str = "cg", **kw) -> OrcSchedule:
    s = default_schedule(solver)
    for k, v in kw.items():
        if k == "level_floor":
            s.level_floor[0], s.level_floor[1] = v
        else:
            setattr(s, k, v)
    return s


def fixed_schedule(level: int = 3) -> OrcSchedule:
    s = default_schedule("cg")
    s.enabled = 0
    s.start_level = level
    return s


@dataclass
class Report:
    status: int
    iterations: int
    iters_per_level: tuple
    converged: bool
    n_switches: int
    switch_iter: tuple
    switch_to_level: tuple
    rel_residual_recurrence: float
    rel_residual_true: float
    spmv_count: tuple


def _report(st, r: OrcReport) -> Report:
    ns = min(r.n_switches, 2)
    return Report(st, r.iterations, tuple(r.iters_per_level), bool(r.converged), r.n_switches,
                  tuple(r.switch_iter[:ns]), tuple(r.switch_to_level[:ns]),
                  r.rel_residual_recurrence, r.rel_residual_true, tuple(r.spmv_count))


def _bounds(parts):
    bd = np.ascontiguousarray(parts, dtype=np.int64)
    return len(bd) - 1, bd


def cg(A, b, x0=None, tol=1e-10, max_iters=5000, sched: OrcSchedule | None = None, parts=None):
    """parts: row-block bounds [0, ..., rows] -> c.1 step 10 partitioned mode"""
    m = A.orc()
    bb = _arr(b)
    x = np.zeros(A.rows, np.float64) if x0 is None else _arr(x0).copy()
    s = sched if sched is not None else fixed_schedule(3)
    rep = OrcReport()
    if parts is None:
        st = lib().orc_cg(C.byref(m), _ptr(bb, C.c_double), _ptr(x, C.c_double), tol, max_iters,
                          C.byref(s), C.byref(rep))
    else:
        P, bd = _bounds(parts)
        st = lib().orc_cg_part(C.byref(m), _ptr(bb, C.c_double), _ptr(x, C.c_double), tol,
                               max_iters, C.byref(s), P, _ptr(bd, C.c_int64), C.byref(rep))
    if st >= 10:
        raise OracleError(st, "cg")
    return x, _report(st, rep)


def gmres(A, b, x0=None, tol=1e-10, restart=30, max_iters=15000,
          sched: OrcSchedule | None = None, parts=None):
    m = A.orc()
    bb = _arr(b)
    x = np.zeros(A.rows, np.float64) if x0 is None else _arr(x0).copy()
    s = sched if sched is not None else fixed_schedule(3)
    rep = OrcReport()
    if parts is None:
        st = lib().orc_gmres(C.byref(m), _ptr(bb, C.c_double), _ptr(x, C.c_double), tol, restart,
                             max_iters, C.byref(s), C.byref(rep))
    else:
        P, bd = _bounds(parts)
        st = lib().orc_gmres_part(C.byref(m), _ptr(bb, C.c_double), _ptr(x, C.c_double), tol,
                                  restart, max_iters, C.byref(s), P, _ptr(bd, C.c_int64),
                                  C.byref(rep))
    if st >= 10:
        raise OracleError(st, "gmres")
    return x, _report(st, rep)
