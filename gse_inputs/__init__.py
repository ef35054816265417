"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no exponent table, no encoding, no
decoding, no SpMV, no solver step): it only builds plain FP64 CSR matrices and vectors
with the shapes and value structure of the paper's workloads, as recipes stated in
DESIGN.md section "Input recipes".

All matrices are returned as ``Csr(rows, cols, row_ptr:int64, col:int32, val:float64)``
with sorted, duplicate-free rows.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Csr:
    rows: int
    cols: int
    row_ptr: np.ndarray  # int64[rows+1]
    col: np.ndarray  # int32[nnz]
    val: np.ndarray  # float64[nnz]
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.val.size)

    def dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols))
        r = np.repeat(np.arange(self.rows), np.diff(self.row_ptr))
        d[r, self.col] = self.val
        return d


def from_dense(d: np.ndarray, name: str = "") -> Csr:
    d = np.asarray(d, dtype=np.float64)
    rows, cols = d.shape
    r, c = np.nonzero(d)
    rp = np.zeros(rows + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return Csr(rows, cols, np.cumsum(rp), c.astype(np.int32), d[r, c].copy(), name)


def ones_rhs(A: Csr) -> np.ndarray:
    """b = A * 1 (R19): row sums of the stored values (input recipe only)."""
    b = np.zeros(A.rows)
    lens = np.diff(A.row_ptr)
    nz = lens > 0
    if A.nnz:
        sums = np.add.reduceat(A.val, A.row_ptr[:-1][nz])
        b[nz] = sums
    return b


def uniform_vec(n: int, seed: int = 7, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    return np.random.default_rng(seed).uniform(lo, hi, n)


# ------------------------------------------------------------------ stencils
def _stencil(dims, offsets, coef_fn, row_begin=0, row_end=None, name=""):
    """Generic lexicographic (x fastest) stencil on an interior grid, Dirichlet boundary
    eliminated.  ``offsets`` = list of (dx,dy,dz) in ascending column order;
    ``coef_fn(idx, k, valid)`` returns the values of stencil entry k for rows ``idx``."""
    nx, ny, nz = dims
    n = nx * ny * nz
    row_end = n if row_end is None else row_end
    rows = row_end - row_begin
    idx = np.arange(row_begin, row_end, dtype=np.int64)
    ix, iy, iz = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    K = len(offsets)
    cols = np.empty((rows, K), np.int64)
    valid = np.empty((rows, K), bool)
    vals = np.empty((rows, K), np.float64)
    for k, (dx, dy, dz) in enumerate(offsets):
        jx, jy, jz = ix + dx, iy + dy, iz + dz
        ok = (jx >= 0) & (jx < nx) & (jy >= 0) & (jy < ny) & (jz >= 0) & (jz < nz)
        valid[:, k] = ok
        cols[:, k] = idx + dx + dy * nx + dz * nx * ny
        vals[:, k] = coef_fn(idx, k, ok)
    cnt = valid.sum(axis=1)
    rp = np.zeros(rows + 1, np.int64)
    np.cumsum(cnt, out=rp[1:])
    return Csr(rows, n, rp, cols[valid].astype(np.int32), vals[valid], name)


_OFF2 = [(0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0)]
_OFF3 = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]


def _kappa(n, seed):
    # node coefficient kappa = exp(U(0, ln 10))  (DESIGN.md recipe C1/C2 varcoef)
    return np.exp(np.random.default_rng(seed).uniform(0.0, np.log(10.0), n))


def _varcoef_fn(dims, offsets, kappa):
    nx, ny, _ = dims
    diag_k = [k for k, o in enumerate(offsets) if o == (0, 0, 0)][0]

    def face(idx, k, ok):
        dx, dy, dz = offsets[k]
        j = np.where(ok, idx + dx + dy * nx + dz * nx * ny, idx)
        ki, kj = kappa[idx], kappa[j]
        hm = 2.0 * ki * kj / (ki + kj)  # harmonic mean; boundary faces -> kappa_i
        return np.where(ok, hm, ki)

    def fn(idx, k, ok):
        if k == diag_k:
            s = np.zeros(idx.size)
            for kk in range(len(offsets)):
                if kk != diag_k:
                    s = s + face(idx, kk, np.ones(idx.size, bool) & _inside(idx, offsets[kk], dims))
            return s
        return -face(idx, k, ok)

    return fn


def _inside(idx, off, dims):
    nx, ny, nz = dims
    ix, iy, iz = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    dx, dy, dz = off
    return ((ix + dx >= 0) & (ix + dx < nx) & (iy + dy >= 0) & (iy + dy < ny)
            & (iz + dz >= 0) & (iz + dz < nz))


def poisson2d(N: int, variant: str = "const", seed: int = 42) -> Csr:
    """C1 (N=32): 5-point Laplacian on an N x N interior grid.  const: 4 / -1 (exact in the
    head); varcoef: harmonic-mean face coefficients of kappa = exp(U(0, ln 10))."""
    dims = (N, N, 1)
    if variant == "const":
        fn = lambda idx, k, ok: np.full(idx.size, 4.0 if k == 2 else -1.0)
    else:
        fn = _varcoef_fn(dims, _OFF2, _kappa(N * N, seed))
    return _stencil(dims, _OFF2, fn, name=f"poisson2d_{N}_{variant}")


def poisson3d(N: int, variant: str = "const", seed: int = 42, row_begin: int = 0,
              row_end: int | None = None) -> Csr:
    """C2 (N=128) / C5 (N=512): 7-point Laplacian, const 6 / -1 or varcoef.  A row range
    may be requested (row-partitioned generation for multi-GPU runs)."""
    dims = (N, N, N)
    if variant == "const":
        fn = lambda idx, k, ok: np.full(idx.size, 6.0 if k == 3 else -1.0)
    else:
        fn = _varcoef_fn(dims, _OFF3, _kappa(N ** 3, seed))
    return _stencil(dims, _OFF3, fn, row_begin, row_end, name=f"poisson3d_{N}_{variant}")


def poisson3d_chunks(N: int, variant: str = "const", row_begin: int = 0,
                     row_end: int | None = None, planes: int = 8, workers: int | None = None):
    """poisson3d's rows [row_begin, row_end) as consecutive row chunks of <= `planes` x-y
    planes each, generated by a thread pool and yielded in row order as (r0, Csr): the same
    matrix, without one 938M-non-zero temporary for C5 (bench.py streams the chunks to the
    GPU).  Each chunk's row_ptr starts at 0."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    n = N ** 3
    row_end = n if row_end is None else row_end
    step = planes * N * N
    bounds = [(a, min(a + step, row_end)) for a in range(row_begin, row_end, step)]
    kappa = None if variant == "const" else _kappa(n, 42)
    dims = (N, N, N)
    if variant == "const":
        fn = lambda idx, k, ok: np.full(idx.size, 6.0 if k == 3 else -1.0)
    else:
        fn = _varcoef_fn(dims, _OFF3, kappa)
    work = lambda ab: (ab[0], _stencil(dims, _OFF3, fn, ab[0], ab[1], name=f"poisson3d_{N}_{variant}"))
    workers = workers or min(16, os.cpu_count() or 1)
    with ThreadPoolExecutor(workers) as ex:
        # bounded look-ahead: at most 2 x workers chunks in host memory
        pending = [ex.submit(work, ab) for ab in bounds[:2 * workers]]
        nxt = len(pending)
        while pending:
            yield pending.pop(0).result()
            if nxt < len(bounds):
                pending.append(ex.submit(work, bounds[nxt]))
                nxt += 1


def convdiff3d(N: int, beta=(64.0, 128.0, 192.0), row_begin: int = 0,
               row_end: int | None = None) -> Csr:
    """C4 (N=256): first-order upwind convection-diffusion, per dimension the unscaled
    stencil (-1 - beta_k h, 2 + beta_k h, -1) with h = 1/(N+1), summed over x, y, z.
    Nonsymmetric M-matrix with non-dyadic values (head-lossy)."""
    h = 1.0 / (N + 1)
    bx, by, bz = (b * h for b in beta)
    # ascending column order: z-1, y-1, x-1, diag, x+1, y+1, z+1
    coef = [-1.0 - bz, -1.0 - by, -1.0 - bx, 6.0 + bx + by + bz, -1.0, -1.0, -1.0]
    fn = lambda idx, k, ok: np.full(idx.size, coef[k])
    return _stencil((N, N, N), _OFF3, fn, row_begin, row_end, name=f"convdiff3d_{N}")


# ------------------------------------------------------------------ power-law SPD (C3)
# rank profile of exponent offsets: (first rank, last rank, probability of the band)
_RANK_BANDS = [(1, 1, 0.647), (2, 2, 0.084), (3, 4, 0.093), (5, 8, 0.085), (9, 16, 0.056),
               (17, 32, 0.024), (33, 64, 0.009), (65, 128, 0.002)]


def _rank_to_offset(seed):
    offs = np.arange(-64, 64)
    perm = np.random.default_rng(seed + 1).permutation(offs[offs != 0])
    return np.concatenate([[0], perm])  # rank 1 -> offset 0


def powerlaw_spd(n: int, seed: int = 42, xm: float = 4.3, max_half: int = 20000,
                 p_local: float = 0.85, mean_local: float = 64.0) -> Csr:
    """C3 (n = 10M): SuiteSparse-shaped SPD matrix (recipe in DESIGN.md):
    half-degree h_i = min(max_half, floor(xm * U^(-1/1.5))); partner j = i + delta with
    delta ~ Geometric(1/mean_local) w.p. p_local else Uniform[1, n); drop j >= n, dedupe,
    mirror.  Off-diagonal value -(1 + f) 2^o, o drawn by the exponent rank profile that
    reproduces P:105's top-k coverage; diagonal = sum |a_ij| (1 + 2^-8 U) + 2^-20
    (strict diagonal dominance => SPD)."""
    rng = np.random.default_rng(seed)
    u = rng.random(n)
    h = np.minimum(max_half, np.floor(xm * u ** (-1.0 / 1.5))).astype(np.int64)
    total = int(h.sum())
    src = np.repeat(np.arange(n, dtype=np.int64), h)
    local = rng.random(total) < p_local
    delta = np.where(local, rng.geometric(1.0 / mean_local, total),
                     rng.integers(1, max(n, 2), total))
    dst = src + delta
    keep = dst < n
    src, dst = src[keep], dst[keep]
    key = np.sort(src * n + dst)  # sorted unique (np.unique's hash path is ~6x slower here)
    key = key[np.concatenate(([True], key[1:] != key[:-1]))]
    src, dst = key // n, key % n
    del key
    m = src.size
    # exponent offsets by rank profile
    band = rng.choice(len(_RANK_BANDS), size=m, p=[b[2] for b in _RANK_BANDS])
    lo = np.array([b[0] for b in _RANK_BANDS])[band]
    hi = np.array([b[1] for b in _RANK_BANDS])[band]
    rank = lo + (rng.random(m) * (hi - lo + 1)).astype(np.int64)
    o = _rank_to_offset(seed)[rank - 1]
    f = rng.integers(0, 1 << 52, m, dtype=np.int64).astype(np.float64) / float(1 << 52)
    v = -(1.0 + f) * np.ldexp(1.0, o)
    # mirror + diagonal
    diag = np.zeros(n)
    np.add.at(diag, src, np.abs(v))
    np.add.at(diag, dst, np.abs(v))
    diag = diag * (1.0 + rng.random(n) / 256.0) + 2.0 ** -20
    rows = np.concatenate([src, dst, np.arange(n, dtype=np.int64)])
    cols = np.concatenate([dst, src, np.arange(n, dtype=np.int64)])
    vals = np.concatenate([v, v, diag])
    del src, dst, v
    order = np.argsort(rows * n + cols, kind="stable")
    rows, cols, vals = rows[order], cols[order], vals[order]
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    return Csr(n, n, rp, cols.astype(np.int32), vals, name=f"powerlaw_{n}")


# ------------------------------------------------------------------ small random matrices
def random_csr(rows: int, cols: int, nnz_per_row: float, seed: int = 0, exps=None,
               empty_rows: float = 0.0, value_kind: str = "classes") -> Csr:
    """Random sparse matrix for parity tests.  value_kind:
    'classes' -> (1+f) 2^e with e drawn from ``exps`` (biased exponents), full 52-bit f;
    'wide'    -> exponents spread over [-60, 60] (exercises d > 1 and flushes);
    'mixed'   -> 'classes' plus zeros and subnormals."""
    rng = np.random.default_rng(seed)
    lens = rng.poisson(nnz_per_row, rows).clip(0, cols)
    if empty_rows > 0:
        lens[rng.random(rows) < empty_rows] = 0
    rp = np.zeros(rows + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    nnz = int(rp[-1])
    col = np.empty(nnz, np.int32)
    for r in range(rows):
        col[rp[r]:rp[r + 1]] = np.sort(rng.choice(cols, lens[r], replace=False))
    f = rng.integers(0, 1 << 52, nnz, dtype=np.int64).astype(np.float64) / float(1 << 52)
    sign = np.where(rng.random(nnz) < 0.5, -1.0, 1.0)
    if value_kind == "wide":
        e = rng.integers(-60, 61, nnz)
    else:
        ex = np.array(exps if exps is not None else [1023, 1022, 1025], dtype=np.int64)
        e = ex[rng.integers(0, ex.size, nnz)] - 1023
    val = sign * (1.0 + f) * np.ldexp(1.0, e)
    if value_kind == "mixed" and nnz:
        z = rng.random(nnz)
        val[z < 0.05] = 0.0
        val[(z >= 0.05) & (z < 0.08)] = np.ldexp(1.0, -1060) * sign[(z >= 0.05) & (z < 0.08)]
    return Csr(rows, cols, rp, col, val, name=f"random_{rows}x{cols}_{seed}")


def spd_small(n: int, seed: int = 0) -> Csr:
    """Dense-ish small SPD matrix M M^T + n I (for CG <= n-step checks)."""
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    return from_dense(M @ M.T + n * np.eye(n), name=f"spd_{n}_{seed}")
