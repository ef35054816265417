"""paper_2411_04686_b200 -- thin Python binding of the B200-native GSE-SEM library.

The product is the C-ABI shared library ``libgse_b200.so`` (include/gse.h), built from
``csrc/*.cu`` for sm_100a.  This module only marshals arguments (torch tensors or numpy
arrays -> raw pointers, the current CUDA stream) and raises on error statuses; every step of
the method runs in the library's kernels.  There is no CPU fallback: if the library cannot
be loaded, importing this package fails.

Function names follow the C-ABI: gse_encode, gse_fp64_matrix, gse_half_matrix, gse_spmv, gse_spmv_f32acc,
gse_decode, gse_matrix_copy_planes, gse_matrix_get_info, gse_solve_cg, gse_solve_gmres,
gse_default_schedule, gse_matrix_free.
"""
from __future__ import annotations

import ctypes as C
import os
import shutil

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
# GSE_LIB_PATH: developer A/B override (a prebuilt variant of the same library)
LIB_PATH = os.environ.get("GSE_LIB_PATH") or _build.LIB

# ---------------------------------------------------------------------------- status codes
GSE_OK, GSE_NOT_CONVERGED, GSE_NUMERICAL_ABORT = 0, 2, 3
GSE_ERR_INVALID_ARG, GSE_ERR_DIM_MISMATCH, GSE_ERR_NONFINITE, GSE_ERR_NO_VALUES = 10, 11, 12, 13
GSE_ERR_UNREPRESENTABLE, GSE_ERR_INVALID_EXP_INDEX, GSE_ERR_FP32_RANGE = 14, 15, 16
GSE_ERR_WRONG_FORMAT, GSE_ERR_CUDA, GSE_ERR_NCCL, GSE_ERR_OOM = 17, 20, 21, 22
GSE_KIND_GSE, GSE_KIND_FP64, GSE_KIND_FP16, GSE_KIND_BF16 = 0, 1, 2, 3

ABI_SYMBOLS = (
    "gse_encode", "gse_fp64_matrix", "gse_half_matrix", "gse_matrix_get_info", "gse_matrix_copy_planes",
    "gse_decode", "gse_spmv", "gse_spmv_f32acc", "gse_spmv_dot", "gse_perturbation_bounds", "gse_default_schedule", "gse_solve_cg",
    "gse_solve_gmres", "gse_matrix_free", "gse_status_string", "gse_last_error_detail",
    "gse_set_allocator", "gse_nccl_unique_id", "gse_dist_create", "gse_encode_dist",
    "gse_dist_free", "gse_dist_thread_group_create", "gse_dist_thread_group_free",
    "gse_dist_create_thread", "gse_dist_plan", "gse_encode_vector16", "gse_decode_vector16",
)


def _load():
    # torch (when installed) goes first: the library needs libnccl.so.2, and torch's bundled
    # NCCL must be the copy the process loads (a system NCCL loaded first shadows it and
    # torch's CUDA library then fails to resolve its symbols)
    try:
        import torch  # noqa: F401
    except ImportError:
        pass
    if LIB_PATH == _build.LIB and _build.stale():
        if shutil.which(_build.NVCC) or os.path.exists(_build.NVCC):
            _build.build()
        elif not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing and nvcc is unavailable: run "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
    return C.CDLL(LIB_PATH)


_lib = _load()


# ---------------------------------------------------------------------------- ctypes structs
class CsrF64(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("row_ptr_64", C.c_int),
                ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class EncodeOpts(C.Structure):
    _fields_ = [("k_max", C.c_int), ("device", C.c_int), ("sample_block_rows", C.c_int64),
                ("seed", C.c_uint64), ("per_shard_table", C.c_int)]


class MatrixInfo(C.Structure):
    _fields_ = [("kind", C.c_int), ("k_max", C.c_int), ("ei_bits", C.c_int),
                ("ei_in_column", C.c_int), ("table_len", C.c_int), ("table", C.c_uint16 * 64),
                ("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("n_blocks", C.c_int64), ("n_zero_values", C.c_int64), ("device", C.c_int),
                ("plane_bytes", C.c_size_t * 5),
                ("spmv_mode", C.c_int)]


class StepSchedule(C.Structure):
    _fields_ = [("enabled", C.c_int), ("start_level", C.c_int), ("max_level", C.c_int),
                ("l", C.c_int64), ("t", C.c_int64), ("m", C.c_int64),
                ("rsd_limit", C.c_double), ("ndec_limit", C.c_int64),
                ("reldec_limit", C.c_double), ("verify_at_full", C.c_int),
                ("level_floor", C.c_double * 2), ("krylov_gse16", C.c_int),
                ("perturb_c", C.c_double), ("cg_keep_direction", C.c_int)]


class SolveReport(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("iters_per_level", C.c_int64 * 3),
                ("converged", C.c_int), ("n_switches", C.c_int),
                ("switch_iter", C.c_int64 * 2), ("switch_to_level", C.c_int * 2),
                ("rel_residual_recurrence", C.c_double), ("rel_residual_true", C.c_double),
                ("seconds", C.c_double), ("spmv_count", C.c_int64 * 3)]


def _declare(L):
    vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
    L.gse_encode.argtypes = [C.POINTER(CsrF64), C.POINTER(EncodeOpts), C.POINTER(vp), vp]
    L.gse_fp64_matrix.argtypes = [C.POINTER(CsrF64), i32, C.POINTER(vp), vp]
    L.gse_half_matrix.argtypes = [C.POINTER(CsrF64), i32, i32, C.POINTER(vp), vp]
    L.gse_matrix_get_info.argtypes = [vp, C.POINTER(MatrixInfo)]
    L.gse_matrix_copy_planes.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
    L.gse_decode.argtypes = [vp, i32, vp, vp]
    L.gse_spmv.argtypes = [vp, vp, vp, i32, vp]
    L.gse_spmv_f32acc.argtypes = [vp, vp, vp, i32, vp]
    L.gse_spmv_dot.argtypes = [vp, vp, vp, i32, vp, vp]
    L.gse_perturbation_bounds.argtypes = [vp, vp, vp]
    L.gse_default_schedule.argtypes = [i32, C.POINTER(StepSchedule)]
    L.gse_default_schedule.restype = None
    L.gse_solve_cg.argtypes = [vp, vp, vp, dbl, i64, C.POINTER(StepSchedule),
                               C.POINTER(SolveReport), vp]
    L.gse_solve_gmres.argtypes = [vp, vp, vp, dbl, i32, i64, C.POINTER(StepSchedule),
                                  C.POINTER(SolveReport), vp]
    L.gse_matrix_free.argtypes = [vp]
    L.gse_matrix_free.restype = None
    L.gse_status_string.argtypes = [i32]
    L.gse_status_string.restype = C.c_char_p
    L.gse_last_error_detail.argtypes = []
    L.gse_last_error_detail.restype = C.c_char_p
    L.gse_nccl_unique_id.argtypes = [vp]
    L.gse_set_allocator.argtypes = [vp, vp, vp]
    L.gse_dist_create.argtypes = [vp, i32, i32, i32, C.POINTER(vp)]
    L.gse_dist_thread_group_create.argtypes = [i32, C.POINTER(vp)]
    L.gse_dist_thread_group_free.argtypes = [vp]
    L.gse_dist_thread_group_free.restype = None
    L.gse_dist_create_thread.argtypes = [vp, i32, i32, C.POINTER(vp)]
    L.gse_encode_dist.argtypes = [vp, C.POINTER(CsrF64), i64, i64, C.POINTER(EncodeOpts),
                                  C.POINTER(vp), vp]
    L.gse_dist_free.argtypes = [vp]
    L.gse_dist_free.restype = None
    L.gse_dist_plan.argtypes = [i64, vp, i64, i64, i32, vp, vp, C.POINTER(i64), vp, vp]
    L.gse_encode_vector16.argtypes = [vp, i64, i32, vp, vp, C.POINTER(i32), vp]
    L.gse_decode_vector16.argtypes = [vp, i64, vp, i32, i32, vp, vp]


_declare(_lib)


class GseError(RuntimeError):
    def __init__(self, status: int, where: str):
        detail = _lib.gse_last_error_detail().decode(errors="replace")
        msg = _lib.gse_status_string(status).decode()
        super().__init__(f"{where}: {msg} (status {status}){': ' + detail if detail else ''}")
        self.status = status
        self.detail = detail


def _check(status: int, where: str, ok=(GSE_OK,)):
    if status not in ok:
        raise GseError(status, where)
    return status


# ---------------------------------------------------------------------------- marshalling
def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _addr(a):
    """Raw address of a contiguous torch tensor or numpy array (None -> NULL)."""
    if a is None:
        return None
    if _is_torch(a):
        assert a.is_contiguous(), "tensor must be contiguous"
        return a.data_ptr()
    assert isinstance(a, np.ndarray) and a.flags["C_CONTIGUOUS"], "array must be contiguous"
    return a.ctypes.data


def _stream(*arrays, stream=None):
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    for a in arrays:
        if a is not None and _is_torch(a) and a.is_cuda:
            import torch
            return torch.cuda.current_stream(a.device).cuda_stream
    return None


def _device_of(*arrays):
    for a in arrays:
        if a is not None and _is_torch(a) and a.is_cuda:
            return a.device.index
    return -1


def _dtype_ok(a, np_dtype):
    if _is_torch(a):
        import torch
        want = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32,
                np.int64: torch.int64}[np_dtype]
        return a.dtype == want
    return a.dtype == np_dtype


class Matrix:
    """Owning handle of a gse_matrix (freed on close / garbage collection)."""

    def __init__(self, handle: int):
        self.handle = C.c_void_p(handle)
        self._info = None

    @property
    def info(self) -> dict:
        if self._info is None:
            self._info = gse_matrix_get_info(self)
        return self._info

    def close(self):
        if self.handle and self.handle.value:
            _lib.gse_matrix_free(self.handle)
            self.handle = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _csr(rows, cols, row_ptr, col_idx, values):
    assert _dtype_ok(col_idx, np.int32) and _dtype_ok(values, np.float64)
    rp64 = 1 if _dtype_ok(row_ptr, np.int64) else 0
    assert rp64 or _dtype_ok(row_ptr, np.int32), "row_ptr must be int32 or int64"
    nnz = int(values.numel() if _is_torch(values) else values.size)
    return CsrF64(rows, cols, nnz, _addr(row_ptr), rp64, _addr(col_idx), _addr(values))


def gse_encode(row_ptr, col_idx, values, rows: int, cols: int, k_max: int = 8,
               device: int | None = None, stream=None, sample_block_rows: int = 0,
               seed: int = 0) -> Matrix:
    """a1-a3: build the GSE-SEM matrix (host or device CSR input; see include/gse.h).
    sample_block_rows > 0: table from one random row per row block (NEXT-3)."""
    A = _csr(rows, cols, row_ptr, col_idx, values)
    dev = _device_of(values, col_idx, row_ptr) if device is None else device
    if dev < 0:
        dev = _current_device()
    opts = EncodeOpts(k_max, dev, sample_block_rows, seed, 0)
    out = C.c_void_p()
    _check(_lib.gse_encode(C.byref(A), C.byref(opts), C.byref(out),
                           _stream(values, col_idx, row_ptr, stream=stream)), "gse_encode")
    return Matrix(out.value)


def gse_fp64_matrix(row_ptr, col_idx, values, rows: int, cols: int, device: int | None = None,
                    stream=None) -> Matrix:
    """The FP64-CSR comparator matrix (paper's FP64-SpMV baseline)."""
    A = _csr(rows, cols, row_ptr, col_idx, values)
    dev = _device_of(values, col_idx, row_ptr) if device is None else device
    if dev < 0:
        dev = _current_device()
    out = C.c_void_p()
    _check(_lib.gse_fp64_matrix(C.byref(A), dev, C.byref(out),
                                _stream(values, col_idx, row_ptr, stream=stream)),
           "gse_fp64_matrix")
    return Matrix(out.value)


def gse_half_matrix(row_ptr, col_idx, values, rows: int, cols: int, kind: str = "fp16",
                    device: int | None = None, stream=None) -> Matrix:
    """The FP16 / BF16 storage baselines: values rounded to nearest-even 16-bit codes
    on the device, read with FP64 products and sums (gse_spmv segments = 3)."""
    k = {"fp16": GSE_KIND_FP16, "bf16": GSE_KIND_BF16}[kind]
    A = _csr(rows, cols, row_ptr, col_idx, values)
    dev = _device_of(values, col_idx, row_ptr) if device is None else device
    if dev < 0:
        dev = _current_device()
    out = C.c_void_p()
    _check(_lib.gse_half_matrix(C.byref(A), k, dev, C.byref(out),
                                _stream(values, col_idx, row_ptr, stream=stream)),
           "gse_half_matrix")
    return Matrix(out.value)


def _current_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0


def gse_matrix_get_info(A: Matrix) -> dict:
    info = MatrixInfo()
    _check(_lib.gse_matrix_get_info(A.handle, C.byref(info)), "gse_matrix_get_info")
    return {
        "kind": info.kind, "k_max": info.k_max, "ei_bits": info.ei_bits,
        "ei_in_column": bool(info.ei_in_column), "table_len": info.table_len,
        "table": [info.table[i] for i in range(info.table_len)], "rows": info.rows,
        "cols": info.cols, "nnz": info.nnz, "n_blocks": info.n_blocks,
        "n_zero_values": info.n_zero_values, "device": info.device,
        "plane_bytes": [info.plane_bytes[i] for i in range(5)],
        "spmv_mode": info.spmv_mode,
    }


def _current_stream():
    """torch's current stream on the current device (None without CUDA): host copies of the
    library's planes are ordered on it instead of the legacy default stream, which would
    wait for every other thread's blocking work (multi-rank thread backend)"""
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
    except Exception:
        pass
    return None


def gse_matrix_copy_planes(A: Matrix, stream=None) -> dict:
    """Copy the encoded planes to host numpy arrays (for bit-exact parity checks)."""
    stream = _current_stream() if stream is None else _stream(stream=stream)
    inf = A.info
    n = inf["nnz"]
    out = {"col_ei": np.zeros(max(n, 1), np.uint32), "head": np.zeros(max(n, 1), np.uint16),
           "tail1": np.zeros(max(n, 1), np.uint16), "tail2": np.zeros(max(n, 1), np.uint32),
           "table": np.zeros(64, np.uint16)}
    side = None if inf["ei_in_column"] else np.zeros(max(n, 1), np.uint8)
    if inf["kind"] != GSE_KIND_GSE:  # FP64: columns; FP16 / BF16: columns + 16-bit codes
        head = out["head"] if inf["kind"] in (GSE_KIND_FP16, GSE_KIND_BF16) else None
        _check(_lib.gse_matrix_copy_planes(A.handle, _addr(out["col_ei"]), None, _addr(head),
                                           None, None, None, stream), "gse_matrix_copy_planes")
        return {"col": out["col_ei"][:n], "half": None if head is None else head[:n]}
    _check(_lib.gse_matrix_copy_planes(A.handle, _addr(out["col_ei"]), _addr(side),
                                       _addr(out["head"]), _addr(out["tail1"]),
                                       _addr(out["tail2"]), _addr(out["table"]), stream),
           "gse_matrix_copy_planes")
    res = {k: v[:n] for k, v in out.items() if k != "table"}
    res["table"] = out["table"][: inf["table_len"]]
    res["side_ei"] = None if side is None else side[:n]
    return res


def _like(x, n, np_dtype):
    if _is_torch(x):
        import torch
        dt = torch.float64 if np_dtype == np.float64 else torch.float32
        return torch.empty(n, dtype=dt, device=x.device)
    return np.empty(n, dtype=np_dtype)


def gse_decode(A: Matrix, segments: int, out=None, like=None):
    """a4: every stored value decoded at `segments` to FP64."""
    n = A.info["nnz"]
    if out is None:
        out = _like(like, n, np.float64) if like is not None else np.empty(n, np.float64)
    _check(_lib.gse_decode(A.handle, segments, _addr(out), _stream(out)), "gse_decode")
    return out


def gse_spmv(A: Matrix, x, y=None, segments: int = 3, stream=None):
    """a5/a6: y = A_L x, FP64 accumulation."""
    if y is None:
        y = _like(x, A.info["rows"], np.float64)
    assert _dtype_ok(x, np.float64) and _dtype_ok(y, np.float64)
    _check(_lib.gse_spmv(A.handle, _addr(x), _addr(y), segments, _stream(x, y, stream=stream)),
           "gse_spmv")
    return y


def gse_spmv_dot(A: Matrix, x, y=None, segments: int = 3, dot=None, stream=None):
    """a7's fused kernel: y = A_L x and x . y in one launch.  `dot` (one float64, host numpy
    or device tensor) receives the dot; returns (y, dot)."""
    if y is None:
        y = _like(x, A.info["rows"], np.float64)
    if dot is None:
        dot = _like(x, 1, np.float64)
    assert _dtype_ok(x, np.float64) and _dtype_ok(y, np.float64) and _dtype_ok(dot, np.float64)
    _check(_lib.gse_spmv_dot(A.handle, _addr(x), _addr(y), segments, _addr(dot),
                             _stream(x, y, stream=stream)), "gse_spmv_dot")
    return y, dot


def gse_spmv_f32acc(A: Matrix, x, y=None, segments: int = 3, stream=None):
    """y = A_L x with FP32 accumulation (R20)."""
    if y is None:
        y = _like(x, A.info["rows"], np.float32)
    assert _dtype_ok(x, np.float32) and _dtype_ok(y, np.float32)
    _check(_lib.gse_spmv_f32acc(A.handle, _addr(x), _addr(y), segments,
                                _stream(x, y, stream=stream)), "gse_spmv_f32acc")
    return y


def gse_perturbation_bounds(A: Matrix, stream=None) -> tuple:
    """R29: (eta_1, eta_2), eta_L = ||A_3 - A_L||_inf."""
    eta = np.zeros(2)
    _check(_lib.gse_perturbation_bounds(A.handle, eta.ctypes.data,
                                        _stream(stream=stream)), "gse_perturbation_bounds")
    return float(eta[0]), float(eta[1])


def gse_default_schedule(solver: str = "cg", **overrides) -> StepSchedule:
    s = StepSchedule()
    _lib.gse_default_schedule(0 if solver == "cg" else 1, C.byref(s))
    for k, v in overrides.items():
        if k == "level_floor":
            s.level_floor[0], s.level_floor[1] = v
        else:
            setattr(s, k, v)
    return s


def fixed_schedule(level: int = 3) -> StepSchedule:
    s = gse_default_schedule("cg")
    s.enabled = 0
    s.start_level = level
    return s


def _report(r: SolveReport, status: int) -> dict:
    ns = min(r.n_switches, 2)
    return {"status": status, "iterations": r.iterations,
            "iters_per_level": tuple(r.iters_per_level), "converged": bool(r.converged),
            "n_switches": r.n_switches, "switch_iter": tuple(r.switch_iter[:ns]),
            "switch_to_level": tuple(r.switch_to_level[:ns]),
            "rel_residual_recurrence": r.rel_residual_recurrence,
            "rel_residual_true": r.rel_residual_true, "seconds": r.seconds,
            "spmv_count": tuple(r.spmv_count)}


_SOLVE_OK = (GSE_OK, GSE_NOT_CONVERGED, GSE_NUMERICAL_ABORT)


def gse_solve_cg(A: Matrix, b, x=None, tol: float = 1e-10, max_iters: int = 5000,
                 sched: StepSchedule | None = None, stream=None):
    """Stepped CG (a7, a9, a10).  x (in: x0, out: solution) is overwritten.  Returns
    (x, report)."""
    if x is None:
        x = _like(b, A.info["rows"], np.float64)
        x[:] = 0
    rep = SolveReport()
    st = _lib.gse_solve_cg(A.handle, _addr(b), _addr(x), tol, max_iters,
                           None if sched is None else C.byref(sched), C.byref(rep),
                           _stream(b, x, stream=stream))
    _check(st, "gse_solve_cg", _SOLVE_OK)
    return x, _report(rep, st)


def gse_solve_gmres(A: Matrix, b, x=None, tol: float = 1e-10, restart: int = 30,
                    max_iters: int = 15000, sched: StepSchedule | None = None, stream=None):
    """Stepped restarted GMRES(restart) (a8, a9, a10).  Returns (x, report)."""
    if x is None:
        x = _like(b, A.info["rows"], np.float64)
        x[:] = 0
    rep = SolveReport()
    st = _lib.gse_solve_gmres(A.handle, _addr(b), _addr(x), tol, restart, max_iters,
                              None if sched is None else C.byref(sched), C.byref(rep),
                              _stream(b, x, stream=stream))
    _check(st, "gse_solve_gmres", _SOLVE_OK)
    return x, _report(rep, st)


def gse_encode_vector16(v, k_max: int = 8, stream=None):
    """NEXT-4 / Alg. 1: a vector in 16-bit GSE-SEM form.  Returns (words, table): words a
    uint16 array like v (torch tensor on v's device, or numpy), table a numpy uint16 array."""
    n = v.numel() if _is_torch(v) else np.asarray(v).size
    if _is_torch(v):
        import torch
        words = torch.empty(n, dtype=torch.int16, device=v.device)
    else:
        v = np.ascontiguousarray(v, dtype=np.float64)
        words = np.empty(n, np.uint16)
    table = np.zeros(16, np.uint16)
    tl = C.c_int()
    _check(_lib.gse_encode_vector16(_addr(v), n, k_max, _addr(words), _addr(table), C.byref(tl),
                                    _stream(v, stream=stream)), "gse_encode_vector16")
    return words, table[: tl.value].copy()


def gse_decode_vector16(words, table, ei_bits: int = 3, stream=None):
    n = words.numel() if _is_torch(words) else np.asarray(words).size
    t = np.ascontiguousarray(table, dtype=np.uint16)
    if _is_torch(words):
        import torch
        out = torch.empty(n, dtype=torch.float64, device=words.device)
    else:
        words = np.ascontiguousarray(words, dtype=np.uint16)
        out = np.empty(n, np.float64)
    _check(_lib.gse_decode_vector16(_addr(words), n, _addr(t) if t.size else None, t.size,
                                    ei_bits, _addr(out), _stream(words, stream=stream)),
           "gse_decode_vector16")
    return out


_ALLOC_T = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_T = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)
_alloc_keep = None  # the installed ctypes callbacks must outlive every allocation


def gse_set_allocator(alloc=None, free=None):
    """Route the library's device allocations through Python callables alloc(bytes,
    stream) -> int pointer and free(ptr, stream) (both None: back to cudaMallocAsync)."""
    global _alloc_keep
    if (alloc is None) != (free is None):
        raise ValueError("alloc and free must both be set or both be None")
    if alloc is None:
        _check(_lib.gse_set_allocator(None, None, None), "gse_set_allocator")
        _alloc_keep = None
        return
    a = _ALLOC_T(lambda nbytes, stream, ctx: alloc(int(nbytes), stream) or None)
    f = _FREE_T(lambda ptr, stream, ctx: free(int(ptr), stream))
    _check(_lib.gse_set_allocator(C.cast(a, C.c_void_p), C.cast(f, C.c_void_p), None),
           "gse_set_allocator")
    _alloc_keep = (a, f)


def torch_allocator():
    """(alloc, free) callables over torch's caching allocator, for gse_set_allocator."""
    import torch

    def alloc(nbytes, stream):
        return torch.cuda.caching_allocator_alloc(nbytes, stream=stream or 0)

    def free(ptr, stream):
        torch.cuda.caching_allocator_delete(ptr)

    return alloc, free


def gse_matrix_free(A: Matrix):
    A.close()


# ---------------------------------------------------------------------------- multi-GPU
class Dist:
    """Owning handle of a gse_dist (one rank's communicator)."""

    def __init__(self, handle: int):
        self.handle = C.c_void_p(handle)

    def close(self):
        if self.handle and self.handle.value:
            _lib.gse_dist_free(self.handle)
            self.handle = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gse_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.gse_nccl_unique_id(buf), "gse_nccl_unique_id")
    return buf.raw


def gse_dist_create(unique_id: bytes, rank: int, nranks: int, device: int) -> Dist:
    """NCCL backend (one process per GPU)."""
    buf = C.create_string_buffer(bytes(unique_id), 128)
    out = C.c_void_p()
    _check(_lib.gse_dist_create(buf, rank, nranks, device, C.byref(out)), "gse_dist_create")
    return Dist(out.value)


def gse_dist_thread_group_create(nranks: int) -> int:
    out = C.c_void_p()
    _check(_lib.gse_dist_thread_group_create(nranks, C.byref(out)),
           "gse_dist_thread_group_create")
    return out.value


def gse_dist_thread_group_free(group: int):
    _lib.gse_dist_thread_group_free(C.c_void_p(group))


def gse_dist_create_thread(group: int, rank: int, device: int = 0) -> Dist:
    """Thread backend: `rank` of a thread group in this process."""
    out = C.c_void_p()
    _check(_lib.gse_dist_create_thread(C.c_void_p(group), rank, device, C.byref(out)),
           "gse_dist_create_thread")
    return Dist(out.value)


def gse_encode_dist(D: Dist, row_ptr, col_idx, values, row_begin: int, global_rows: int,
                    k_max: int = 8, stream=None, per_shard_table: bool = False) -> Matrix:
    """Collective: encode this rank's row block (global column ids).  per_shard_table: the
    rank's own table instead of the global one (no histogram allreduce)."""
    rows = int((row_ptr.numel() if _is_torch(row_ptr) else row_ptr.size) - 1)
    A = _csr(rows, global_rows, row_ptr, col_idx, values)
    opts = EncodeOpts(k_max, -1, 0, 0, 1 if per_shard_table else 0)
    out = C.c_void_p()
    _check(_lib.gse_encode_dist(D.handle, C.byref(A), row_begin, global_rows, C.byref(opts),
                                C.byref(out), _stream(values, col_idx, row_ptr, stream=stream)),
           "gse_encode_dist")
    return Matrix(out.value)


def gse_dist_plan(col, row_begin: int, n_local: int, rank_rows):
    """Host-only local renumbering / halo plan (no GPU): returns (local_col, halo_cols,
    recv_count) as numpy arrays."""
    col = np.ascontiguousarray(col, dtype=np.int32)
    rr = np.ascontiguousarray(rank_rows, dtype=np.int64)
    nranks = rr.size - 1
    local = np.empty(max(col.size, 1), np.int32)
    halo = np.empty(max(col.size, 1), np.int64)
    recv = np.zeros(nranks, np.int64)
    nh = C.c_int64()
    _check(_lib.gse_dist_plan(col.size, col.ctypes.data, row_begin, n_local, nranks,
                              rr.ctypes.data, local.ctypes.data, C.byref(nh), halo.ctypes.data,
                              recv.ctypes.data), "gse_dist_plan")
    return local[: col.size].copy(), halo[: nh.value].copy(), recv


def lib():
    return _lib
