// encode.cu -- GSE-SEM format conversion on the GPU and the
// SpMV row-block partition.
//
//   a1 k_hist     : histogram of biased exponents (P:116 [3.2.1]); zero/subnormal counted
//                   apart; first NaN/Inf index.  Warp-aggregated smem atomics.
//   a2 k_select   : one CTA: top-k_max exponents by (count desc, e desc), e_max forced into
//                   the last slot, entries e+1 (R4, R5); then the 2048-entry
//                   LUT e -> (EI, d = min{E - e >= 1}) used by a3 (Alg. formatConvert
//                   l.6-21, precomputed once per exponent instead of per value).
//   a3 k_encode   : per value Alg. formatConvert l.22-26 generalised to the 64-bit SEM:
//                   D = 1<<(63-d) | f<<(11-d) (or f>>(d-11)), truncation (R1); zero ->
//                   signed zero (R2); d > 63 -> signed zero (R3); split head/tail1/tail2
//                   (P:163); EI into the column index or the side array.
#include <cstdlib>
#include <cstring>

#include "decode.cuh"
#include "gse_internal.cuh"
#include "scan.cuh"

namespace gse {

struct EncodeStatus {
  unsigned long long hist[2048];
  unsigned long long n_zero;
  unsigned long long first_nonfinite;  // ~0ull if none
  unsigned long long first_bad_col;    // ~0ull if none
  unsigned int bad_structure;          // row_ptr not monotone / wrong ends
  int table_len;
  int n_distinct;
  int e_max;
  unsigned short table[64];
  unsigned int lut[2048];  // ei | d << 8 ; 0xFFFFFFFF = no entry above e
  unsigned long long shist[2048];  // sampled histogram (NEXT-3), selection input if sampled
};

// ------------------------------------------------------------------ a1 histogram
// one value into the block histogram: warp-aggregated increment (one smem atomic per
// distinct exponent in the warp); zeros/subnormals counted, first non-finite index kept
__device__ __forceinline__ void hist_one(double v, int64_t i, unsigned* h, unsigned& zc,
                                         unsigned long long& first) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  unsigned e = (unsigned)(u >> 52) & 0x7FFu;
  if (e == 0x7FFu) {
    first = min(first, (unsigned long long)i);
    e = 0xFFFFFFFFu;
  } else if (e == 0u) {
    ++zc;
    e = 0xFFFFFFFFu;
  }
  const unsigned peers = __match_any_sync(__activemask(), e);
  if (e != 0xFFFFFFFFu && (int)(threadIdx.x & 31) == __ffs(peers) - 1)
    atomicAdd(&h[e], (unsigned)__popc(peers));
}

// Four values per thread per iteration (two 16-byte streaming loads) when val is 16-byte
// aligned: one 8-byte load per iteration kept too few bytes in flight (1.9 TB/s on C2)
__global__ void __launch_bounds__(512) k_hist(const double* __restrict__ val, int64_t nnz,
                                              EncodeStatus* __restrict__ st) {
  __shared__ unsigned int h[2048];
  __shared__ unsigned long long s_first;
  __shared__ unsigned int s_zero;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) h[i] = 0;
  if (threadIdx.x == 0) {
    s_first = ~0ull;
    s_zero = 0;
  }
  __syncthreads();
  unsigned int zc = 0;
  unsigned long long first = ~0ull;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (((uintptr_t)val & 15u) == 0) {
    const int64_t nq = nnz >> 2;
    const double2* v2 = reinterpret_cast<const double2*>(val);
    for (int64_t q = tid; q < nq; q += stride) {
      const double2 a = __ldcs(v2 + 2 * q), b = __ldcs(v2 + 2 * q + 1);
      hist_one(a.x, 4 * q, h, zc, first);
      hist_one(a.y, 4 * q + 1, h, zc, first);
      hist_one(b.x, 4 * q + 2, h, zc, first);
      hist_one(b.y, 4 * q + 3, h, zc, first);
    }
    done = nq << 2;
  }
  for (int64_t i = done + tid; i < nnz; i += stride) hist_one(__ldcs(val + i), i, h, zc, first);
  if (first != ~0ull) atomicMin(&s_first, first);
  if (zc) atomicAdd(&s_zero, zc);
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (h[i]) atomicAdd(&st->hist[i], (unsigned long long)h[i]);
  if (threadIdx.x == 0) {
    if (s_zero) atomicAdd(&st->n_zero, (unsigned long long)s_zero);
    if (s_first != ~0ull) atomicMin(&st->first_nonfinite, s_first);
  }
}

// ------------------------------------------------------------------ NEXT-3 sampled histogram
// P:116 "a sparse matrix is divided into several row blocks, and the exponents'
// distribution in a random row is calculated for each row block".  Block b =
// rows [b B, min((b+1) B, rows)); its row = b B + z mod len, z = SplitMix64 output for
// counter b + 1 from the seed (R27).  One thread per block; the max-exponent rule keeps
// the TRUE e_max from the full histogram (k_select), so every value stays representable.
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long seed, long long b) {
  unsigned long long z = seed + (unsigned long long)(b + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_hist_sampled(const uint32_t* __restrict__ rp, const double* __restrict__ val,
                               int64_t rows, int64_t nnz, int64_t B, unsigned long long seed,
                               EncodeStatus* __restrict__ st) {
  const int64_t nb = (rows + B - 1) / B;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
    const int64_t r0 = b * B, len = rows - r0 < B ? rows - r0 : B;
    const int64_t r = r0 + (int64_t)(splitmix64(seed, b) % (unsigned long long)len);
    const uint32_t j1 = (int64_t)rp[r + 1] < nnz ? rp[r + 1] : (uint32_t)nnz;  // (bad structure
    for (uint32_t j = rp[r]; j < j1; ++j) {                                      //  is reported later)
      const unsigned e = (unsigned)((unsigned long long)__double_as_longlong(val[j]) >> 52) & 0x7FFu;
      if (e >= 1u && e <= 2046u) atomicAdd(&st->shist[e], 1ull);
    }
  }
}

// ------------------------------------------------------------------ a2 table + LUT
__device__ unsigned long long block_max_u64(unsigned long long v, unsigned long long* red) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < (int)(blockDim.x >> 5)) ? red[l] : 0ull;
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    if (l == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}

// sampled: the selection counts come from st->shist (NEXT-3); e_max always from the full
// histogram st->hist
__global__ void __launch_bounds__(1024) k_select(EncodeStatus* __restrict__ st, int k_max,
                                                 int sampled) {
  __shared__ unsigned long long key[2048];
  __shared__ unsigned long long red[33];
  __shared__ int sel[64];
  unsigned long long mloc = 0, nd = 0;
  for (int e = threadIdx.x; e < 2048; e += blockDim.x) {
    const bool ok = e >= 1 && e <= 2046;
    unsigned long long c = ok ? (sampled ? st->shist[e] : st->hist[e]) : 0ull;
    // key orders by count desc, then exponent desc (R4); unique because e is in the key
    key[e] = c ? ((c << 11) | (unsigned long long)e) : 0ull;
    if (c) ++nd;
    if (ok && st->hist[e]) mloc = max(mloc, (unsigned long long)e);
  }
  const unsigned long long e_max = block_max_u64(mloc, red);
  // count distinct exponents (sum via max-reduction of per-thread prefix is overkill:
  // use an atomic into shared)
  __shared__ unsigned int s_nd;
  if (threadIdx.x == 0) s_nd = 0;
  __syncthreads();
  if (nd) atomicAdd(&s_nd, (unsigned)nd);
  __syncthreads();
  const int n_distinct = (int)s_nd;
  int take = n_distinct < k_max ? n_distinct : k_max;
  if (take == 0 && e_max > 0) {  // a sample without normal values: the forced entry alone
    take = 1;
    if (threadIdx.x == 0) sel[0] = (int)e_max;
    __syncthreads();
  }
  for (int k = 0; k < (n_distinct < take ? n_distinct : take); ++k) {
    unsigned long long loc = 0;
    for (int e = threadIdx.x; e < 2048; e += blockDim.x) loc = max(loc, key[e]);
    unsigned long long best = block_max_u64(loc, red);
    if (threadIdx.x == 0) {
      sel[k] = (int)(best & 0x7FFull);
      key[best & 0x7FFull] = 0ull;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && take > 0) {
    bool have = false;
    for (int k = 0; k < take; ++k) have |= (sel[k] == (int)e_max);
    if (!have) {  // P:123 forced e_max + 1: a free slot (R27b), else the last one (R5)
      if (take < k_max)
        sel[take++] = (int)e_max;
      else
        sel[take - 1] = (int)e_max;
    }
    for (int k = 0; k < take; ++k) st->table[k] = (unsigned short)(sel[k] + 1);
    st->table_len = take;
    st->n_distinct = n_distinct;
    st->e_max = (int)e_max;
  }
  if (threadIdx.x == 0 && take == 0) {
    st->table_len = 0;
    st->n_distinct = 0;
  }
  __shared__ int s_take;  // thread 0 may have appended e_max (R27b)
  if (threadIdx.x == 0) s_take = take;
  __syncthreads();
  take = s_take;
  // LUT: nearest larger shared exponent per biased exponent (Alg. formatConvert l.6-21)
  for (int e = threadIdx.x; e < 2048; e += blockDim.x) {
    int best = -1, dbest = 1 << 30;
    for (int k = 0; k < take; ++k) {
      int d = (sel[k] + 1) - e;
      if (d >= 1 && d < dbest) {
        dbest = d;
        best = k;
      }
    }
    st->lut[e] = best < 0 ? 0xFFFFFFFFu : ((unsigned)best | ((unsigned)dbest << 8));
  }
}

// ------------------------------------------------------------------ a3 encode
// one value -> (64-bit SEM word, table index), Alg. 1 with the per-exponent lut
__device__ __forceinline__ unsigned long long encode_word(double v, const unsigned* lut,
                                                          unsigned& ei) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const unsigned e = (unsigned)(u >> 52) & 0x7FFu;
  const unsigned long long f = u & ((1ull << 52) - 1);
  unsigned long long w = (u >> 63) << 63;
  ei = 0;
  if (e != 0u && e != 0x7FFu) {
    const unsigned lu = lut[e];
    ei = lu & 0xFFu;
    const unsigned d = lu >> 8;
    if (d <= 63u) {
      unsigned long long D = 1ull << (63 - d);
      D |= (d <= 11u) ? (f << (11 - d)) : (f >> (d - 11));
      w |= D;
    }
  }
  return w;
}

// Four nonzeros per thread per iteration with 16-byte loads and stores when every array
// is 16-byte aligned (the pool's planes are; a custom allocator's may not be): ~2.6x the bytes in flight of the one-element
// loop (C2: 87.6 us at 0.61 of HBM before)
template <bool IN_COL>
__global__ void __launch_bounds__(256) k_encode(const double* __restrict__ val,
                                                const int32_t* __restrict__ col, int64_t nnz,
                                                int64_t cols, const EncodeStatus* __restrict__ st,
                                                int ei_bits, uint32_t* __restrict__ col_ei,
                                                uint8_t* __restrict__ side,
                                                uint16_t* __restrict__ head,
                                                uint16_t* __restrict__ tail1,
                                                uint32_t* __restrict__ tail2,
                                                unsigned long long* __restrict__ bad_col) {
  __shared__ unsigned int lut[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) lut[i] = st->lut[i];
  __syncthreads();
  const int sh = 32 - ei_bits;
  unsigned long long bad = ~0ull;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  const uintptr_t al = (uintptr_t)val | (uintptr_t)col | (uintptr_t)col_ei | (uintptr_t)head |
                       (uintptr_t)tail1 | (uintptr_t)tail2 | (IN_COL ? 0 : (uintptr_t)side);
  if ((al & 15u) == 0) {
    const int64_t nq = nnz >> 2;
    for (int64_t q = tid; q < nq; q += stride) {
      const double2 a = __ldcs(reinterpret_cast<const double2*>(val) + 2 * q);
      const double2 b = __ldcs(reinterpret_cast<const double2*>(val) + 2 * q + 1);
      const int4 c = __ldcs(reinterpret_cast<const int4*>(col) + q);
      const double v[4] = {a.x, a.y, b.x, b.y};
      const int32_t cc[4] = {c.x, c.y, c.z, c.w};
      uint32_t ce[4], t2[4];
      uint16_t hd[4], t1[4];
      uint8_t sd[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (cc[j] < 0 || (int64_t)cc[j] >= cols) bad = min(bad, (unsigned long long)(4 * q + j));
        unsigned ei;
        const unsigned long long w = encode_word(v[j], lut, ei);
        hd[j] = (uint16_t)(w >> 48);
        t1[j] = (uint16_t)(w >> 32);
        t2[j] = (uint32_t)w;
        ce[j] = IN_COL ? ((uint32_t)cc[j] | (ei_bits ? (ei << sh) : 0u)) : (uint32_t)cc[j];
        sd[j] = (uint8_t)ei;
      }
      reinterpret_cast<uint2*>(head)[q] =
          make_uint2(hd[0] | ((uint32_t)hd[1] << 16), hd[2] | ((uint32_t)hd[3] << 16));
      reinterpret_cast<uint2*>(tail1)[q] =
          make_uint2(t1[0] | ((uint32_t)t1[1] << 16), t1[2] | ((uint32_t)t1[3] << 16));
      reinterpret_cast<uint4*>(tail2)[q] = make_uint4(t2[0], t2[1], t2[2], t2[3]);
      reinterpret_cast<uint4*>(col_ei)[q] = make_uint4(ce[0], ce[1], ce[2], ce[3]);
      if (!IN_COL)
        reinterpret_cast<uint32_t*>(side)[q] =
            sd[0] | ((uint32_t)sd[1] << 8) | ((uint32_t)sd[2] << 16) | ((uint32_t)sd[3] << 24);
    }
    done = nq << 2;
  }
  for (int64_t i = done + tid; i < nnz; i += stride) {
    const int32_t c = __ldcs(col + i);
    if (c < 0 || (int64_t)c >= cols) bad = min(bad, (unsigned long long)i);
    unsigned ei;
    const unsigned long long w = encode_word(__ldcs(val + i), lut, ei);
    head[i] = (uint16_t)(w >> 48);
    tail1[i] = (uint16_t)(w >> 32);
    tail2[i] = (uint32_t)w;
    if (IN_COL) {
      col_ei[i] = (uint32_t)c | (ei_bits ? (ei << sh) : 0u);
    } else {
      col_ei[i] = (uint32_t)c;
      side[i] = (uint8_t)ei;
    }
  }
  if (bad != ~0ull) atomicMin(bad_col, bad);
}

// ------------------------------------------------------------------ row_ptr + partition
template <class RP>
__global__ void k_rowptr(const RP* __restrict__ in, int64_t rows, int64_t nnz,
                         uint32_t* __restrict__ out, unsigned* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= rows; r += stride) {
    long long a = (long long)in[r];
    bool ok = a >= 0 && a <= nnz;
    if (r == 0) ok = ok && a == 0;
    if (r == rows) ok = ok && a == nnz;
    if (r < rows) ok = ok && (long long)in[r + 1] >= a;
    if (!ok) atomicOr(bad, 1u);
    out[r] = (uint32_t)a;
  }
}

__global__ void k_block_flags(const uint32_t* __restrict__ rp, int64_t rows,
                              uint8_t* __restrict__ flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const uint32_t a = rp[r], b = rp[r + 1];
    bool st = (r == 0) || (b - a > LMAX);
    if (!st) {
      const uint32_t p = rp[r - 1];
      st = (a / CHUNK != p / CHUNK) || (a - p > LMAX);
    }
    flag[r] = st ? 1 : 0;
  }
}

__global__ void k_fill_desc(const uint32_t* __restrict__ starts, const int* __restrict__ nsel,
                            const uint32_t* __restrict__ rp, int64_t rows,
                            BlockDesc* __restrict__ desc) {
  const int nb = *nsel;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += stride) {
    if (b < nb) {
      const uint32_t r = starts[b];
      desc[b] = BlockDesc{r, rp[r]};
    } else {
      desc[b] = BlockDesc{(uint32_t)rows, rp[rows]};
    }
  }
}

// ---- window-mode structures (spmv_win.cu) ------------------------------------------------
// tile starts: row 0, a row whose start crosses a WIN_TNNZ boundary of the non-zero stream,
// and every WIN_RMAX-th row (bounds a tile's x window); also counts the empty rows
__global__ void k_tile_flags(const uint32_t* __restrict__ rp, int64_t rows,
                             uint8_t* __restrict__ flag, unsigned long long* __restrict__ n_empty) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long ne = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const uint32_t a = rp[r];
    bool st = (r == 0) || (r % WIN_RMAX == 0);
    if (!st) st = a / WIN_TNNZ != rp[r - 1] / WIN_TNNZ;
    flag[r] = st ? 1 : 0;
    ne += (rp[r + 1] == a) ? 1u : 0u;
  }
  for (int o = 16; o > 0; o >>= 1) ne += __shfl_down_sync(0xFFFFFFFFu, ne, o);
  if ((threadIdx.x & 31) == 0 && ne) atomicAdd(n_empty, ne);
}

// bit rp[r] of the non-zero stream for every non-empty row r, plus a sentinel start at
// nnz: the matrix's last row then closes like every other row (spmv_win.cu)
__global__ void k_row_bits(const uint32_t* __restrict__ rp, int64_t rows,
                           uint32_t* __restrict__ bits) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t z = rp[rows];
    atomicOr(bits + (z >> 5), 1u << (z & 31u));
  }
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const uint32_t a = rp[r];
    if (rp[r + 1] > a) atomicOr(bits + (a >> 5), 1u << (a & 31u));
  }
}

// chunk_prev[c] = the row holding non-zero c * WIN_CH - 1 (the last r with rp[r] <= q)
__global__ void k_chunk_prev(const uint32_t* __restrict__ rp, int64_t rows, int64_t nch,
                             uint32_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nch; c += stride) {
    if (c == 0) {
      out[0] = 0xFFFFFFFFu;
      continue;
    }
    const uint32_t q = (uint32_t)(c * WIN_CH - 1);
    int64_t lo = 0, hi = rows;  // rp[lo] <= q < rp[hi] (q < nnz = rp[rows])
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (rp[mid] <= q)
        lo = mid;
      else
        hi = mid;
    }
    out[c] = (uint32_t)lo;
  }
}

static int grid_for(int64_t n, int threads, int dev) {
  int64_t g = (n + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms(dev) * 8;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// per 32-row group (one warp, lane = row): longest row, staged spans of the group and of
// the 64-row group it starts -> mode statistics.  acc = {heavy groups, sum 32 * max len,
// max len, max span (32 rows), max span (64 rows)}
__global__ void k_group_stats(const uint32_t* __restrict__ rp, int64_t rows,
                              unsigned long long* __restrict__ acc) {
  __shared__ unsigned long long red[5][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ng = (rows + RW_ROWS - 1) / RW_ROWS;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  unsigned long long heavy = 0, wsum = 0, mx = 0, span = 0, span2 = 0;
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; g < ng; g += nw) {
    const int64_t r0 = g * RW_ROWS, r = r0 + lane;
    const uint32_t len = r < rows ? rp[r + 1] - rp[r] : 0u;
    const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, len);
    if (lane == 0) {
      const int64_t r1 = r0 + RW_ROWS < rows ? r0 + RW_ROWS : rows;
      const int64_t r2 = r0 + 2 * RW_ROWS < rows ? r0 + 2 * RW_ROWS : rows;
      // staged span: [rp[r0] & ~7, rp[r1]) rounded up to 8-element units
      const uint32_t a0 = rp[r0] & ~7u;
      const uint32_t sp = ((rp[r1] - a0) + 7u) & ~7u;
      span = max(span, (unsigned long long)sp);
      if ((g & 1) == 0) span2 = max(span2, (unsigned long long)(((rp[r2] - a0) + 7u) & ~7u));
      heavy += (sp > (uint32_t)RW_TILE) ? 1 : 0;
      wsum += (unsigned long long)RW_ROWS * m;
      mx = max(mx, (unsigned long long)m);
    }
  }
  if (lane == 0) {
    red[0][warp] = heavy;
    red[1][warp] = wsum;
    red[2][warp] = mx;
    red[3][warp] = span;
    red[4][warp] = span2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      heavy += red[0][w];
      wsum += red[1][w];
      mx = max(mx, red[2][w]);
      span = max(span, red[3][w]);
      span2 = max(span2, red[4][w]);
    }
    if (heavy) atomicAdd(&acc[0], heavy);
    if (wsum) atomicAdd(&acc[1], wsum);
    if (mx) atomicMax(&acc[2], mx);
    if (span) atomicMax(&acc[3], span);
    if (span2) atomicMax(&acc[4], span2);
  }
}

static void choose_mode(Matrix& M) {
  // Row-walk needs every group staged (no heavy group) and little divergence between the
  // 32 rows of a group; otherwise the window kernel (spmv_win.cu) balances the load.
  // GSE_SPMV_MODE=sp|rw|win forces a kernel (A/B measurements).
  const char* env = getenv("GSE_SPMV_MODE");
  const bool rw_ok = M.heavy_groups == 0 && M.rows > 0 && M.ei_in_column;
  int mode = (rw_ok && M.rw_efficiency >= 0.6) ? SPMV_RW : SPMV_WIN;
  if (env && !strcmp(env, "sp")) mode = SPMV_SP;
  if (env && !strcmp(env, "win")) mode = SPMV_WIN;
  if (env && !strcmp(env, "rw") && rw_ok) mode = SPMV_RW;
  M.spmv_mode = mode;
}

// One host sync for the whole partition: the group statistics, both row selections (SP
// warp blocks, window tiles), the empty-row count and (optionally) the caller's status word
// are read back together.
gse_status build_partition(Matrix& M, cudaStream_t s, const void* extra_d, void* extra_h,
                           size_t extra_bytes) {
  M.n_blocks = 0;
  M.n_tiles = 0;
  M.n_groups = (M.rows + RW_ROWS - 1) / RW_ROWS;
  if (M.rows == 0) {
    choose_mode(M);
    M.blocks = dev_alloc_n<BlockDesc>(1, s);
    M.tiles = dev_alloc_n<BlockDesc>(1, s);
    if (!M.blocks || !M.tiles) return GSE_ERR_OOM;
    BlockDesc h{0, 0};
    GSE_CUDA_TRY(cudaMemcpyAsync(M.blocks, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    GSE_CUDA_TRY(cudaMemcpyAsync(M.tiles, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    if (extra_bytes)
      GSE_CUDA_TRY(cudaMemcpyAsync(extra_h, extra_d, extra_bytes, cudaMemcpyDeviceToHost, s));
    GSE_CUDA_TRY(cudaStreamSynchronize(s));
    return GSE_OK;
  }
  // acc: 5 group statistics, the empty-row count, then the two selection counts (int)
  unsigned long long* acc = dev_alloc_n<unsigned long long>(8, s);
  uint8_t* flags = dev_alloc_n<uint8_t>(M.rows, s);
  uint8_t* tflags = dev_alloc_n<uint8_t>(M.rows, s);
  uint32_t* starts = dev_alloc_n<uint32_t>(M.rows, s);
  uint32_t* tstarts = dev_alloc_n<uint32_t>(M.rows, s);
  if (!acc || !flags || !tflags || !starts || !tstarts) return GSE_ERR_OOM;
  int* nsel = reinterpret_cast<int*>(acc + 6);
  int* ntil = reinterpret_cast<int*>(acc + 7);
  GSE_CUDA_TRY(cudaMemsetAsync(acc, 0, 64, s));
  k_group_stats<<<grid_for(M.n_groups * 32, 256, M.device), 256, 0, s>>>(M.row_ptr, M.rows,
                                                                         acc);
  k_block_flags<<<grid_for(M.rows, 256, M.device), 256, 0, s>>>(M.row_ptr, M.rows, flags);
  k_tile_flags<<<grid_for(M.rows, 256, M.device), 256, 0, s>>>(M.row_ptr, M.rows, tflags,
                                                               acc + 5);
  GSE_CUDA_TRY(cudaGetLastError());
  gse_status rc = compact_flags(flags, M.rows, starts, nsel, s);
  if (rc != GSE_OK) return rc;
  rc = compact_flags(tflags, M.rows, tstarts, ntil, s);
  if (rc != GSE_OK) return rc;
  unsigned long long h[8];
  GSE_CUDA_TRY(cudaMemcpyAsync(h, acc, 64, cudaMemcpyDeviceToHost, s));
  if (extra_bytes)
    GSE_CUDA_TRY(cudaMemcpyAsync(extra_h, extra_d, extra_bytes, cudaMemcpyDeviceToHost, s));
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  M.heavy_groups = (int64_t)h[0];
  M.rw_efficiency = h[1] ? (double)M.nnz / (double)h[1] : 0.0;
  M.max_row_len = (int64_t)h[2];
  M.rw_span = (int64_t)h[3];
  M.rw_span2 = (int64_t)h[4];
  M.n_empty_rows = (int64_t)h[5];
  choose_mode(M);
  int nb = 0, nt = 0;
  memcpy(&nb, &h[6], sizeof(int));
  memcpy(&nt, &h[7], sizeof(int));
  M.n_blocks = nb;
  M.n_tiles = nt;
  M.blocks = dev_alloc_n<BlockDesc>((size_t)nb + 1, s);
  M.tiles = dev_alloc_n<BlockDesc>((size_t)nt + 1, s);
  if (!M.blocks || !M.tiles) return GSE_ERR_OOM;
  k_fill_desc<<<grid_for(nb + 1, 256, M.device), 256, 0, s>>>(starts, nsel, M.row_ptr, M.rows,
                                                              M.blocks);
  k_fill_desc<<<grid_for(nt + 1, 256, M.device), 256, 0, s>>>(tstarts, ntil, M.row_ptr, M.rows,
                                                              M.tiles);
  GSE_CUDA_TRY(cudaGetLastError());
  // window-kernel row structure: 1 bit per non-zero (whole chunks, zero past nnz) and the
  // row before every chunk
  const int64_t nch = (M.nnz + WIN_CH - 1) / WIN_CH + 1;
  const size_t words = (size_t)nch * (WIN_CH / 32) + 4;
  M.rowbits = dev_alloc_n<uint32_t>(words, s);
  M.chunk_prev = dev_alloc_n<uint32_t>((size_t)nch, s);
  if (!M.rowbits || !M.chunk_prev) return GSE_ERR_OOM;
  GSE_CUDA_TRY(cudaMemsetAsync(M.rowbits, 0, words * 4, s));
  k_row_bits<<<grid_for(M.rows, 256, M.device), 256, 0, s>>>(M.row_ptr, M.rows, M.rowbits);
  k_chunk_prev<<<grid_for(nch, 256, M.device), 256, 0, s>>>(M.row_ptr, M.rows, nch,
                                                            M.chunk_prev);
  GSE_CUDA_TRY(cudaGetLastError());
  dev_free(flags, s);
  dev_free(tflags, s);
  dev_free(starts, s);
  dev_free(tstarts, s);
  dev_free(acc, s);
  return GSE_OK;
}

static gse_status convert_row_ptr(Matrix& M, const void* d_row_ptr, int rp64, cudaStream_t s,
                                  unsigned* d_bad) {
  M.row_ptr = dev_alloc_n<uint32_t>((size_t)M.rows + 1, s);
  if (!M.row_ptr) return GSE_ERR_OOM;
  int g = grid_for(M.rows + 1, 256, M.device);
  if (rp64)
    k_rowptr<long long><<<g, 256, 0, s>>>((const long long*)d_row_ptr, M.rows, M.nnz,
                                          M.row_ptr, d_bad);
  else
    k_rowptr<int><<<g, 256, 0, s>>>((const int*)d_row_ptr, M.rows, M.nnz, M.row_ptr, d_bad);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

void build_decode_table(Matrix& M) {
  memset(&M.htab, 0, sizeof(M.htab));
  const int sL[3] = {48, 32, 0};
  int emax = 0, emin = 1 << 30;
  for (int i = 0; i < M.table_len; ++i) {
    const int E = M.table[i];
    emax = E > emax ? E : emax;
    emin = E < emin ? E : emin;
    for (int L = 0; L < 3; ++L) {
      M.htab.d64[L][i] = (long long)(E - 1086 + sL[L]) * (1LL << 52);
      M.htab.d32[L][i] = (E - 1086 + sL[L]) * (1 << 23);
      M.htab.sc64[L][i] = ldexp(1.0, E - 1086 + sL[L]);
      const int k32 = E - 1086 + sL[L];
      M.htab.sc32[L][i] = (k32 >= -126 && k32 <= 127) ? ldexpf(1.0f, k32) : 0.0f;
    }
  }
  // FP64 multiply form: a nonzero D_L is >= 1, so D_L * 2^(E - 1086 + s_L) is exact and
  // normal (no flush can occur, R11) iff E - 1086 + s_L >= -1022, i.e. E >= 16 / 32 / 64
  // at levels 1 / 2 / 3.  FP32: the same with the FP32 normal range (>= 2^-126).
  const int emin_fast64[3] = {16, 32, 64};
  for (int L = 0; L < 3; ++L) {
    M.htab.fast64[L] = (M.table_len > 0 && emin >= emin_fast64[L]) ? 1 : 0;
    M.htab.fast32[L] = (M.table_len > 0 && emin - 1086 + sL[L] >= -126) ? 1 : 0;
  }
  // FP32 accumulation is defined iff every decodable value is < 2^128 (R20): the largest
  // true exponent is E_max - 1 - 1023 <= 127.
  M.fp32_ok = (emax <= 1151);
}

static std::string row_col_of(const void* d_row_ptr, int rp64, const int32_t* d_col,
                              int64_t rows, int64_t idx, cudaStream_t s) {
  // error path only: binary search the row on the host
  std::string out;
  int64_t lo = 0, hi = rows;  // find r with rp[r] <= idx < rp[r+1]
  auto rp_at = [&](int64_t r) -> int64_t {
    if (rp64) {
      long long v = 0;
      cudaMemcpyAsync(&v, (const long long*)d_row_ptr + r, 8, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      return v;
    }
    int v = 0;
    cudaMemcpyAsync(&v, (const int*)d_row_ptr + r, 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return v;
  };
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) / 2;
    if (rp_at(mid) <= idx)
      lo = mid;
    else
      hi = mid;
  }
  int c = -1;
  cudaMemcpyAsync(&c, d_col + idx, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  char buf[128];
  snprintf(buf, sizeof(buf), "row %lld col %d (element %lld)", (long long)lo, c,
           (long long)idx);
  return buf;
}

gse_status encode_matrix(Matrix& M, const gse_csr_f64& A, const void* d_row_ptr, int rp64,
                         const int32_t* d_col, const double* d_val, cudaStream_t s, Comm* comm,
                         int64_t sample_block_rows, uint64_t sample_seed, int shard_table) {
  M.kind = GSE_KIND_GSE;
  int eb = 0;
  while ((1 << eb) < M.k_max) ++eb;
  M.ei_bits = eb;
  M.ei_in_column = (M.cols < (1LL << (32 - eb))) ? 1 : 0;

  EncodeStatus* st = dev_alloc_n<EncodeStatus>(1, s);
  if (!st) return GSE_ERR_OOM;
  GSE_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(EncodeStatus), s));
  GSE_CUDA_TRY(cudaMemsetAsync(&st->first_nonfinite, 0xFF, 8, s));
  GSE_CUDA_TRY(cudaMemsetAsync(&st->first_bad_col, 0xFF, 8, s));

  gse_status rc = convert_row_ptr(M, d_row_ptr, rp64, s, &st->bad_structure);
  if (rc != GSE_OK) return rc;

  const int nsm = num_sms(M.device);
  if (M.nnz > 0) {
    int g = grid_for(M.nnz, 512, M.device);
    if (g > nsm * 4) g = nsm * 4;
    k_hist<<<g, 512, 0, s>>>(d_val, M.nnz, st);
    GSE_CUDA_TRY(cudaGetLastError());
  }
  if (comm && !shard_table) {
    // distributed encode: one GLOBAL table (R21) -- sum the histograms (and the zero
    // counts, which follow hist[] in EncodeStatus) over all ranks before the selection.
    // (shard_table: each rank keeps its own histogram -> its own table, NEXT-3)
    rc = comm_allreduce_u64(comm, st->hist, 2048 + 1, s);
    if (rc != GSE_OK) return rc;
  }
  const int sampled = (sample_block_rows > 0 && M.rows > 0) ? 1 : 0;
  if (sampled) {
    const int64_t nb = (M.rows + sample_block_rows - 1) / sample_block_rows;
    k_hist_sampled<<<grid_for(nb, 256, M.device), 256, 0, s>>>(M.row_ptr, d_val, M.rows,
                                                               M.nnz, sample_block_rows,
                                                               sample_seed, st);
    GSE_CUDA_TRY(cudaGetLastError());
  }
  k_select<<<1, 1024, 0, s>>>(st, M.k_max, sampled);
  GSE_CUDA_TRY(cudaGetLastError());

  // read back the table / status (one sync, the table is needed on the host for the
  // decode constants and gse_matrix_get_info)
  EncodeStatus* h = (EncodeStatus*)malloc(sizeof(EncodeStatus));
  GSE_CUDA_TRY(cudaMemcpyAsync(h, st, sizeof(EncodeStatus), cudaMemcpyDeviceToHost, s));
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  if (comm) {  // every rank fails together
    int any = 0;
    const int mine = (h->bad_structure || h->first_nonfinite != ~0ull) ? 1 : 0;
    rc = comm_any(comm, mine, &any);
    if (rc != GSE_OK) return rc;
    if (any && !mine) {
      free(h);
      dev_free(st, s);
      set_error("encode failed on another rank (invalid structure or non-finite value)");
      return GSE_ERR_INVALID_ARG;
    }
  }
  if (h->bad_structure) {
    free(h);
    dev_free(st, s);
    set_error("invalid CSR structure: row_ptr must start at 0, be non-decreasing and end at nnz");
    return GSE_ERR_INVALID_ARG;
  }
  if (h->first_nonfinite != ~0ull) {
    std::string where = row_col_of(d_row_ptr, rp64, d_col, M.rows, (int64_t)h->first_nonfinite, s);
    free(h);
    dev_free(st, s);
    set_error("non-finite value at " + where);
    return GSE_ERR_NONFINITE;
  }
  if (h->table_len == 0) {
    free(h);
    dev_free(st, s);
    set_error("no representable values (all values zero or subnormal)");
    return GSE_ERR_NO_VALUES;
  }
  M.table_len = h->table_len;
  for (int i = 0; i < 64; ++i) M.table[i] = i < M.table_len ? h->table[i] : 0;
  M.n_zero = (int64_t)h->n_zero;
  free(h);
  build_decode_table(M);

  const size_t np = padded(M.nnz);
  M.col_ei = dev_alloc_n<uint32_t>(np, s);
  M.head = dev_alloc_n<uint16_t>(np, s);
  M.tail1 = dev_alloc_n<uint16_t>(np, s);
  M.tail2 = dev_alloc_n<uint32_t>(np, s);
  if (!M.ei_in_column) M.side_ei = dev_alloc_n<uint8_t>(np, s);
  M.dtab = dev_alloc_n<DecodeTable>(1, s);
  if (!M.col_ei || !M.head || !M.tail1 || !M.tail2 || !M.dtab ||
      (!M.ei_in_column && !M.side_ei))
    return GSE_ERR_OOM;
  GSE_CUDA_TRY(cudaMemcpyAsync(M.dtab, &M.htab, sizeof(DecodeTable), cudaMemcpyHostToDevice, s));
  // zero the padding tail so vector loads past nnz read zeros
  const size_t pad = np - (size_t)M.nnz;
  GSE_CUDA_TRY(cudaMemsetAsync(M.col_ei + M.nnz, 0, pad * 4, s));
  GSE_CUDA_TRY(cudaMemsetAsync(M.head + M.nnz, 0, pad * 2, s));
  GSE_CUDA_TRY(cudaMemsetAsync(M.tail1 + M.nnz, 0, pad * 2, s));
  GSE_CUDA_TRY(cudaMemsetAsync(M.tail2 + M.nnz, 0, pad * 4, s));
  if (M.side_ei) GSE_CUDA_TRY(cudaMemsetAsync(M.side_ei + M.nnz, 0, pad, s));

  if (M.nnz > 0) {
    int g = grid_for(M.nnz, 256, M.device);
    if (M.ei_in_column)
      k_encode<true><<<g, 256, 0, s>>>(d_val, d_col, M.nnz, M.cols, st, M.ei_bits, M.col_ei,
                                       nullptr, M.head, M.tail1, M.tail2, &st->first_bad_col);
    else
      k_encode<false><<<g, 256, 0, s>>>(d_val, d_col, M.nnz, M.cols, st, M.ei_bits, M.col_ei,
                                        M.side_ei, M.head, M.tail1, M.tail2,
                                        &st->first_bad_col);
    GSE_CUDA_TRY(cudaGetLastError());
  }
  unsigned long long badc = 0;
  rc = build_partition(M, s, &st->first_bad_col, &badc, 8);
  if (rc != GSE_OK) return rc;
  dev_free(st, s);
  if (comm) {
    int any = 0;
    rc = comm_any(comm, badc != ~0ull ? 1 : 0, &any);
    if (rc != GSE_OK) return rc;
    if (any && badc == ~0ull) {
      set_error("column index out of range on another rank");
      return GSE_ERR_INVALID_ARG;
    }
  }
  if (badc != ~0ull) {
    set_error("column index out of range at " +
              row_col_of(d_row_ptr, rp64, d_col, M.rows, (int64_t)badc, s));
    return GSE_ERR_INVALID_ARG;
  }
  return GSE_OK;
}

// ------------------------------------------------------------------ FP16 / BF16 baselines
// P:406 [4.3]: the paper's FP16-SpMV / BF16-SpMV baselines store every value in 16 bits.
// Conversion (R26): round to nearest, ties to even, straight from the double's bits.  With
// FB fraction bits and bias BIAS, a = m53 * 2^(E-52) (m53 the 53-bit significand) is a
// multiple of the quantum 2^q, q = max(E, 1-BIAS) - FB, after rounding n = m53 >> sh,
// sh = q - (E - 52) >= 52 - FB, on the dropped bits (above half -> up; exactly half -> to
// the even n).  The code is ((E + BIAS) << FB) + n - 2^FB for normal E (a carry out of
// the fraction lands in the exponent field) and n itself in the subnormal range (n = 2^FB
// there is the smallest normal code); a code reaching the all-ones exponent is +-Inf.
template <int FB, int EB>
__device__ __forceinline__ uint16_t round_to_half(double v) {
  constexpr int BIAS = (1 << (EB - 1)) - 1;
  constexpr uint32_t INF = ((1u << EB) - 1u) << FB;
  const uint64_t bits = (uint64_t)__double_as_longlong(v);
  const uint32_t sign = (uint32_t)(bits >> 48) & 0x8000u;
  const int e64 = (int)((bits >> 52) & 0x7FF);
  const uint64_t frac = bits & ((1ull << 52) - 1);
  if (e64 == 0x7FF) return (uint16_t)(sign | INF | (frac ? (1u << (FB - 1)) : 0u));  // Inf/NaN
  if (e64 == 0) return (uint16_t)sign;  // zero / FP64 subnormal (< 2^-1022): rounds to 0
  const int E = e64 - 1023;
  if (E > BIAS) return (uint16_t)(sign | INF);  // >= 2^(emax+1): overflow
  const uint64_t m53 = (1ull << 52) | frac;
  const int q = (E < 1 - BIAS ? 1 - BIAS : E) - FB;
  const int sh = q - (E - 52);
  uint64_t n;
  if (sh >= 64) {
    n = 0;
  } else {
    n = m53 >> sh;
    const uint64_t rem = m53 & ((1ull << sh) - 1), halfw = 1ull << (sh - 1);
    if (rem > halfw || (rem == halfw && (n & 1))) ++n;
  }
  uint32_t code = (E < 1 - BIAS) ? (uint32_t)n
                                 : ((uint32_t)(E + BIAS) << FB) + (uint32_t)n - (1u << FB);
  if (code >= INF) code = INF;
  return (uint16_t)(sign | code);
}

template <int KIND>
__global__ void k_copy_half(const double* __restrict__ val, const int32_t* __restrict__ col,
                            int64_t nnz, int64_t cols, uint16_t* __restrict__ hout,
                            uint32_t* __restrict__ cout, unsigned long long* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long b = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const int32_t c = col[i];
    if (c < 0 || (int64_t)c >= cols) b = min(b, (unsigned long long)i);
    hout[i] = KIND == GSE_KIND_FP16 ? round_to_half<10, 5>(val[i]) : round_to_half<7, 8>(val[i]);
    cout[i] = (uint32_t)c;
  }
  if (b != ~0ull) atomicMin(bad, b);
}

// ------------------------------------------------------------------ FP64 comparator (and the
// FP16 / BF16 baselines below, which share its structure checks and partition)
__global__ void k_copy_fp64(const double* __restrict__ val, const int32_t* __restrict__ col,
                            int64_t nnz, int64_t cols, double* __restrict__ vout,
                            uint32_t* __restrict__ cout, unsigned long long* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long b = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const int32_t c = col[i];
    if (c < 0 || (int64_t)c >= cols) b = min(b, (unsigned long long)i);
    vout[i] = val[i];
    cout[i] = (uint32_t)c;
  }
  if (b != ~0ull) atomicMin(bad, b);
}

gse_status fp64_matrix(Matrix& M, const void* d_row_ptr, int rp64, const int32_t* d_col,
                       const double* d_val, cudaStream_t s, int kind) {
  M.kind = kind;
  M.ei_bits = 0;
  M.ei_in_column = 1;
  M.table_len = 0;
  M.fp32_ok = 0;
  unsigned* d_flags = dev_alloc_n<unsigned>(4, s);
  if (!d_flags) return GSE_ERR_OOM;
  GSE_CUDA_TRY(cudaMemsetAsync(d_flags, 0, 16, s));
  GSE_CUDA_TRY(cudaMemsetAsync(d_flags + 2, 0xFF, 8, s));
  gse_status rc = convert_row_ptr(M, d_row_ptr, rp64, s, d_flags);
  if (rc != GSE_OK) return rc;
  const size_t np = padded(M.nnz);
  M.col_ei = dev_alloc_n<uint32_t>(np, s);
  if (kind == GSE_KIND_FP64)
    M.val = dev_alloc_n<double>(np, s);
  else
    M.head = dev_alloc_n<uint16_t>(np, s);
  if ((!M.val && !M.head) || !M.col_ei) return GSE_ERR_OOM;
  if (M.val) GSE_CUDA_TRY(cudaMemsetAsync(M.val + M.nnz, 0, (np - M.nnz) * 8, s));
  if (M.head) GSE_CUDA_TRY(cudaMemsetAsync(M.head + M.nnz, 0, (np - M.nnz) * 2, s));
  GSE_CUDA_TRY(cudaMemsetAsync(M.col_ei + M.nnz, 0, (np - M.nnz) * 4, s));
  if (M.nnz > 0) {
    unsigned long long* bad = (unsigned long long*)(d_flags + 2);
    const int g = grid_for(M.nnz, 256, M.device);
    if (kind == GSE_KIND_FP64)
      k_copy_fp64<<<g, 256, 0, s>>>(d_val, d_col, M.nnz, M.cols, M.val, M.col_ei, bad);
    else if (kind == GSE_KIND_FP16)
      k_copy_half<GSE_KIND_FP16><<<g, 256, 0, s>>>(d_val, d_col, M.nnz, M.cols, M.head, M.col_ei, bad);
    else
      k_copy_half<GSE_KIND_BF16><<<g, 256, 0, s>>>(d_val, d_col, M.nnz, M.cols, M.head, M.col_ei, bad);
    GSE_CUDA_TRY(cudaGetLastError());
  }
  unsigned h[4];
  rc = build_partition(M, s, d_flags, h, 16);
  if (rc != GSE_OK) return rc;
  dev_free(d_flags, s);
  if (h[0]) {
    set_error("invalid CSR structure: row_ptr must start at 0, be non-decreasing and end at nnz");
    return GSE_ERR_INVALID_ARG;
  }
  unsigned long long badc = ((unsigned long long)h[3] << 32) | h[2];
  if (badc != ~0ull) {
    set_error("column index out of range");
    return GSE_ERR_INVALID_ARG;
  }
  return GSE_OK;
}

// ------------------------------------------------------------------ a4 decode (all values)
template <int L>
__global__ void k_decode_all(const uint32_t* __restrict__ col_ei, const uint8_t* __restrict__ side,
                             const uint16_t* __restrict__ head, const uint16_t* __restrict__ tail1,
                             const uint32_t* __restrict__ tail2, int64_t nnz, int ei_bits,
                             const DecodeTable* __restrict__ dt, double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int sh = 32 - ei_bits;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const unsigned ei = side ? side[i] : __funnelshift_rc(col_ei[i], 0u, sh);
    const long long d = dt->d64[L - 1][ei];
    const uint32_t h = head[i];
    double v;
    if (L == 1)
      v = decode_l1(h, d);
    else if (L == 2)
      v = decode_l2(h, tail1[i], d);
    else
      v = decode_l3(h, tail1[i], tail2[i], d);
    out[i] = v;
  }
}

gse_status decode_all(const Matrix& M, int level, double* out, cudaStream_t s) {
  if (M.nnz == 0) return GSE_OK;
  const int g = grid_for(M.nnz, 256, M.device);
  const uint8_t* side = M.ei_in_column ? nullptr : M.side_ei;
  if (level == 1)
    k_decode_all<1><<<g, 256, 0, s>>>(M.col_ei, side, M.head, M.tail1, M.tail2, M.nnz,
                                      M.ei_bits, M.dtab, out);
  else if (level == 2)
    k_decode_all<2><<<g, 256, 0, s>>>(M.col_ei, side, M.head, M.tail1, M.tail2, M.nnz,
                                      M.ei_bits, M.dtab, out);
  else
    k_decode_all<3><<<g, 256, 0, s>>>(M.col_ei, side, M.head, M.tail1, M.tail2, M.nnz,
                                      M.ei_bits, M.dtab, out);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

// R29: one thread per row sums |dec_3 - dec_1| and |dec_3 - dec_2| in storage order (the
// oracle's order: bit-identical sums); the maxima of the non-negative sums by atomicMax on
// their bit patterns (order-free)
__global__ void k_perturb_eta(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col_ei,
                              const uint8_t* __restrict__ side, const uint16_t* __restrict__ head,
                              const uint16_t* __restrict__ tail1,
                              const uint32_t* __restrict__ tail2, int64_t rows, int ei_bits,
                              const DecodeTable* __restrict__ dt,
                              unsigned long long* __restrict__ eta_bits) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int sh = 32 - ei_bits;
  double m1 = 0.0, m2 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride) {
    double s1 = 0.0, s2 = 0.0;
    for (uint32_t j = rp[i]; j < rp[i + 1]; ++j) {
      const unsigned ei = side ? side[j] : __funnelshift_rc(col_ei[j], 0u, sh);
      const uint32_t h = head[j], t1 = tail1[j];
      const double v3 = decode_l3(h, t1, tail2[j], dt->d64[2][ei]);
      const double v1 = decode_l1(h, dt->d64[0][ei]);
      const double v2 = decode_l2(h, t1, dt->d64[1][ei]);
      s1 = __dadd_rn(s1, fabs(__dsub_rn(v3, v1)));
      s2 = __dadd_rn(s2, fabs(__dsub_rn(v3, v2)));
    }
    m1 = fmax(m1, s1);
    m2 = fmax(m2, s2);
  }
  if (m1 > 0.0) atomicMax(eta_bits, (unsigned long long)__double_as_longlong(m1));
  if (m2 > 0.0) atomicMax(eta_bits + 1, (unsigned long long)__double_as_longlong(m2));
}

gse_status perturbation_bounds(Matrix& M, cudaStream_t s) {
  if (M.eta_ok) return GSE_OK;
  if (M.kind != GSE_KIND_GSE) {
    set_error("perturbation bounds are defined for GSE matrices");
    return GSE_ERR_WRONG_FORMAT;
  }
  unsigned long long* d = dev_alloc_n<unsigned long long>(2, s);
  if (!d) return GSE_ERR_OOM;
  GSE_CUDA_TRY(cudaMemsetAsync(d, 0, 16, s));
  if (M.rows > 0) {
    const int g = grid_for(M.rows, 256, M.device);
    const uint8_t* side = M.ei_in_column ? nullptr : M.side_ei;
    k_perturb_eta<<<g, 256, 0, s>>>(M.row_ptr, M.col_ei, side, M.head, M.tail1, M.tail2, M.rows,
                                    M.ei_bits, M.dtab, d);
    GSE_CUDA_TRY(cudaGetLastError());
  }
  unsigned long long h[2] = {0, 0};
  GSE_CUDA_TRY(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, s));
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  dev_free(d, s);
  memcpy(&M.eta[0], &h[0], 8);
  memcpy(&M.eta[1], &h[1], 8);
  M.eta_ok = 1;
  return GSE_OK;
}

}  // namespace gse
