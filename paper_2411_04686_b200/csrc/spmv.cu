// spmv.cu -- GSE-SEM CSR SpMV at 1/2/3 segments (+ the FP64-CSR comparator), SURVEY 8(a)
// steps a4-a6, for sm_100a.
//
// Paper: Alg. spmv walks each row, decodes the head (first-one search, exponent
// rebuild) and accumulates in FP64; P:212 extends it to head+tail1 and
// head+tail1+tail2.  The paper ran it as CUSP CSR-Vector on a V100 -- prior art.
//
// B200 design: the kernel is HBM-bound (2 flops per 8.9-16 B), so
// the layout is chosen for coalescing, not rows:
//  * one CTA per row block (encode-time partition: rows starting in one CHUNK of the nnz
//    stream, or a single long row); threads own 8 CONSECUTIVE non-zeros, so every plane is
//    read with 128-bit, L1-bypassing loads independent of row length: col_ei 2 x 16 B,
//    head 16 B, (+ tail1 16 B, + tail2 2 x 16 B);
//  * only the requested planes are touched: level 1 reads 6 B/nnz, level 2 8 B, level 3
//    12 B (FP64 CSR: 12 B);
//  * decode is branch-free (decode.cuh): int->fp64 conversion + exponent add, EI -> delta
//    table in shared memory;
//  * x is gathered through the read-only path (L1-allocating: stencil neighbours share
//    lines); products land in shared memory and each thread sums one row sequentially in
//    storage order (same order as the oracle), long rows use a fixed-order block reduction;
//  * optional fused dot product sum_i x_i y_i (CG's p.Ap) with a deterministic last-block
//    reduction, so every run and every rank sees identical scalars.
#include "decode.cuh"
#include "gse_internal.cuh"

namespace gse {

__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_stream_u2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}

template <class T>
struct SpmvParams {
  const BlockDesc* __restrict__ blocks;
  const uint32_t* __restrict__ row_ptr;
  const uint32_t* __restrict__ col_ei;
  const uint8_t* __restrict__ side;
  const uint16_t* __restrict__ head;
  const uint16_t* __restrict__ tail1;
  const uint32_t* __restrict__ tail2;
  const double* __restrict__ val;
  const DecodeTable* __restrict__ dt;
  int ei_shift;       // 32 - ei_bits
  uint32_t col_mask;  // (1 << (32 - ei_bits)) - 1, or ~0u
  const T* __restrict__ x;
  T* __restrict__ y;
  double* partials;
  unsigned* ticket;
  double* dot_result;
  const int* stop;  // optional: skip the launch when *stop != 0 (GMRES cycle graphs)
};

// ---------------------------------------------------------------- deterministic reductions
template <class T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
  return v;  // lane 0 holds the sum
}

template <class T>
__device__ T block_sum(T v, T* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T s = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

// partials[blockIdx] = part; the last CTA to arrive sums all partials in a fixed order.
__device__ void finalize_dot(double part, double* partials, unsigned* ticket, double* result,
                             double* red) {
  __shared__ unsigned s_last;
  const double bs = block_sum(part, red);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    double acc = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) acc += __ldcg(partials + i);
    const double tot = block_sum(acc, red);
    if (threadIdx.x == 0) {
      *result = tot;
      *ticket = 0u;
    }
  }
}

// ---------------------------------------------------------------- per-thread 8 products
// Loads the 8 consecutive stored elements starting at i0 (8-aligned) and returns their
// products with x.  L = 0: FP64 values; L = 1..3: GSE levels.
template <int L, bool SIDE, class T>
__device__ __forceinline__ void products8(const SpmvParams<T>& p, const long long* sd64,
                                          const int* sd32, uint32_t i0, T out[8]) {
  const uint4 ca = ld_stream_u4(p.col_ei + i0);
  const uint4 cb = ld_stream_u4(p.col_ei + i0 + 4);
  const uint32_t c[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
  T xv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) xv[k] = __ldg(p.x + (c[k] & p.col_mask));
  if constexpr (L == 0) {
    const uint4 v0 = ld_stream_u4(p.val + i0), v1 = ld_stream_u4(p.val + i0 + 2);
    const uint4 v2 = ld_stream_u4(p.val + i0 + 4), v3 = ld_stream_u4(p.val + i0 + 6);
    const uint32_t w[16] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w,
                            v2.x, v2.y, v2.z, v2.w, v3.x, v3.y, v3.z, v3.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double a = __hiloint2double((int)w[2 * k + 1], (int)w[2 * k]);
      out[k] = (T)(a * (double)xv[k]);
    }
  } else {
    const uint4 hv = ld_stream_u4(p.head + i0);
    const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
    uint32_t t1w[4] = {0, 0, 0, 0};
    uint32_t t2w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if constexpr (L >= 2) {
      const uint4 tv = ld_stream_u4(p.tail1 + i0);
      t1w[0] = tv.x; t1w[1] = tv.y; t1w[2] = tv.z; t1w[3] = tv.w;
    }
    if constexpr (L == 3) {
      const uint4 ta = ld_stream_u4(p.tail2 + i0), tb = ld_stream_u4(p.tail2 + i0 + 4);
      t2w[0] = ta.x; t2w[1] = ta.y; t2w[2] = ta.z; t2w[3] = ta.w;
      t2w[4] = tb.x; t2w[5] = tb.y; t2w[6] = tb.z; t2w[7] = tb.w;
    }
    uint32_t ei[8];
    if constexpr (SIDE) {
      const uint2 sv = ld_stream_u2(p.side + i0);
#pragma unroll
      for (int k = 0; k < 8; ++k) ei[k] = ((k < 4 ? sv.x : sv.y) >> (8 * (k & 3))) & 63u;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) ei[k] = __funnelshift_rc(c[k], 0u, p.ei_shift);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t h = (hw[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
      const uint32_t t1 = (t1w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
      if constexpr (sizeof(T) == 8) {
        double a;
        if constexpr (L == 1)
          a = decode_l1(h, sd64[ei[k]]);
        else if constexpr (L == 2)
          a = decode_l2(h, t1, sd64[ei[k]]);
        else
          a = decode_l3(h, t1, t2w[k], sd64[ei[k]]);
        out[k] = a * xv[k];
      } else {
        float a;
        if constexpr (L == 1)
          a = decode_f32_u32(h & 0x7FFFu, sd32[ei[k]], h);
        else if constexpr (L == 2)
          a = decode_f32_u32(((h & 0x7FFFu) << 16) | t1, sd32[ei[k]], h);
        else
          a = decode_f32(((uint64_t)(h & 0x7FFFu) << 48) | ((uint64_t)t1 << 32) | t2w[k],
                         sd32[ei[k]], h);
        out[k] = a * xv[k];
      }
    }
  }
}

template <int L, bool SIDE, bool DOT, class T>
__global__ void __launch_bounds__(SPMV_THREADS) k_spmv(const SpmvParams<T> p) {
  __shared__ __align__(16) T prod[TILE];
  __shared__ long long sd64[64];
  __shared__ int sd32[64];
  __shared__ T tred[SPMV_THREADS / 32];
  __shared__ double dred[SPMV_THREADS / 32];
  if (p.stop && *p.stop) return;
  const int tid = threadIdx.x;
  if constexpr (L >= 1) {
    if (tid < 64) {
      if constexpr (sizeof(T) == 8)
        sd64[tid] = p.dt->d64[L - 1][tid];
      else
        sd32[tid] = p.dt->d32[L - 1][tid];
    }
  }
  const BlockDesc d0 = p.blocks[blockIdx.x];
  const BlockDesc d1 = p.blocks[blockIdx.x + 1];
  const uint32_t r0 = d0.row0, nrows = d1.row0 - d0.row0;
  const uint32_t s = d0.nnz0, e = d1.nnz0;
  const uint32_t base = s & ~7u;
  double dpart = 0.0;
  __syncthreads();

  if (nrows == 1 && e - s > LMAX) {
    // ---- long row: fixed-order per-thread partial sums + block reduction
    T acc = 0;
    for (uint32_t p0 = base; p0 < e; p0 += TILE) {
      const uint32_t i0 = p0 + tid * VEC;
      if (i0 < e) {
        T v[8];
        products8<L, SIDE, T>(p, sd64, sd32, i0, v);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t idx = i0 + k;
          if (idx >= s && idx < e) acc += v[k];
        }
      }
    }
    const T tot = block_sum(acc, tred);
    if (tid == 0) {
      p.y[r0] = tot;
      if (DOT) dpart = (double)p.x[r0] * (double)tot;
    }
  } else {
    // ---- short rows: one pass of 8 products per thread into shared memory
    uint32_t ra = 0, rb = 0;
    if (tid < (int)nrows) {
      ra = p.row_ptr[r0 + tid];
      rb = p.row_ptr[r0 + tid + 1];
    }
    const uint32_t i0 = base + tid * VEC;
    if (i0 < e) {
      T v[8];
      products8<L, SIDE, T>(p, sd64, sd32, i0, v);
      T* dst = prod + tid * VEC;
#pragma unroll
      for (int k = 0; k < 8; ++k) dst[k] = v[k];
    }
    __syncthreads();
    for (uint32_t rr = tid; rr < nrows; rr += SPMV_THREADS) {
      if (rr >= SPMV_THREADS) {
        ra = p.row_ptr[r0 + rr];
        rb = p.row_ptr[r0 + rr + 1];
      }
      T sum = 0;
      for (uint32_t j = ra - base; j < rb - base; ++j) sum += prod[j];
      p.y[r0 + rr] = sum;
      if (DOT) dpart += (double)p.x[r0 + rr] * (double)sum;
    }
  }
  if constexpr (DOT) finalize_dot(dpart, p.partials, p.ticket, p.dot_result, dred);
}

template <class T>
static SpmvParams<T> make_params(const Matrix& M, const T* x, T* y, const DotOut* dot) {
  SpmvParams<T> p;
  p.blocks = M.blocks;
  p.row_ptr = M.row_ptr;
  p.col_ei = M.col_ei;
  p.side = M.side_ei;
  p.head = M.head;
  p.tail1 = M.tail1;
  p.tail2 = M.tail2;
  p.val = M.val;
  p.dt = M.dtab;
  p.ei_shift = 32 - M.ei_bits;
  p.col_mask = (M.kind == GSE_KIND_GSE && M.ei_in_column && M.ei_bits)
                   ? ((1u << (32 - M.ei_bits)) - 1u)
                   : 0xFFFFFFFFu;
  p.x = x;
  p.y = y;
  p.partials = dot ? dot->partials : nullptr;
  p.ticket = dot ? dot->ticket : nullptr;
  p.dot_result = dot ? dot->result : nullptr;
  p.stop = nullptr;
  return p;
}

template <bool DOT, class T>
static void launch_level(const Matrix& M, int level, const SpmvParams<T>& p, cudaStream_t s) {
  const dim3 grid((unsigned)M.n_blocks), block(SPMV_THREADS);
  const bool side = !M.ei_in_column;
  if (M.kind == GSE_KIND_FP64) {
    k_spmv<0, false, DOT, T><<<grid, block, 0, s>>>(p);
    return;
  }
#define GSE_LAUNCH(LV)                                          \
  if (side)                                                     \
    k_spmv<LV, true, DOT, T><<<grid, block, 0, s>>>(p);         \
  else                                                          \
    k_spmv<LV, false, DOT, T><<<grid, block, 0, s>>>(p);
  if (level == 1) {
    GSE_LAUNCH(1)
  } else if (level == 2) {
    GSE_LAUNCH(2)
  } else {
    GSE_LAUNCH(3)
  }
#undef GSE_LAUNCH
}

gse_status launch_spmv(const Matrix& M, int level, const double* x, double* y,
                       const DotOut* dot, cudaStream_t s) {
  if (M.n_blocks == 0) {
    if (M.rows > 0) GSE_CUDA_TRY(cudaMemsetAsync(y, 0, M.rows * sizeof(double), s));
    if (dot) GSE_CUDA_TRY(cudaMemsetAsync(dot->result, 0, sizeof(double), s));
    return GSE_OK;
  }
  const SpmvParams<double> p = make_params<double>(M, x, y, dot);
  if (dot)
    launch_level<true, double>(M, level, p, s);
  else
    launch_level<false, double>(M, level, p, s);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

gse_status launch_spmv_guarded(const Matrix& M, int level, const double* x, double* y,
                               const int* stop, cudaStream_t s) {
  if (M.n_blocks == 0) return GSE_OK;
  SpmvParams<double> p = make_params<double>(M, x, y, nullptr);
  p.stop = stop;
  launch_level<false, double>(M, level, p, s);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

gse_status launch_spmv_f32(const Matrix& M, int level, const float* x, float* y,
                           cudaStream_t s) {
  if (M.n_blocks == 0) {
    if (M.rows > 0) GSE_CUDA_TRY(cudaMemsetAsync(y, 0, M.rows * sizeof(float), s));
    return GSE_OK;
  }
  const SpmvParams<float> p = make_params<float>(M, x, y, nullptr);
  launch_level<false, float>(M, level, p, s);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

}  // namespace gse
