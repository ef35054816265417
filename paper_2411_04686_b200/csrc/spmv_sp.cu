// spmv_sp.cu -- "strided products" SpMV kernel (irregular row lengths, e.g. the power-law
// config).  SURVEY 8(a) a4-a6; paper Alg. spmv, P:212 for levels 2-3.
//
//  * persistent CTAs of 8 INDEPENDENT warps; each warp walks "warp blocks" (encode-time
//    partition: rows starting in one 192-nnz chunk, each <= 64 nnz, or one long row) with a
//    fixed grid stride, prefetching the next block's descriptor.  No CTA-wide barrier on
//    the hot path (a CTA-tile version with one __syncthreads per 1.8k non-zeros was
//    latency-bound at 0.25 Gnnz/s per B200: profiles/ncu_spmv_r01_v1.txt);
//  * lane l owns elements s + l + 32k (k < 8): each plane load / x gather instruction of a
//    warp covers 32 consecutive non-zeros, so the load is balanced whatever the row lengths;
//  * products go to a warp-private shared tile and lpr lanes per row sum it (storage order
//    for lpr = 1, the oracle's order); the bounds of a block's rows are loaded with its
//    planes (one dependent round trip less); long rows: per-lane sequential partials + a
//    fixed shuffle tree;
//  * register budget for 4 CTAs (32 warps) per SM: on the power-law matrix the kernel is
//    bound by the L1 data pipe (x gathers + the products tile, ~0.94 wavefronts per
//    non-zero); DESIGN.md 6.2 lists the measured alternatives.
#include "spmv_common.cuh"

namespace gse {

template <int L, bool SIDE, bool FAST, class T>
__device__ __forceinline__ void products(const SpmvParams<T>& p, const long long* sd64,
                                         const int* sd32, const double* sc64,
                                         const float* sc32, uint32_t first, uint32_t e,
                                         T out[EPL]) {
  uint32_t c[EPL], h[EPL], t1[EPL], t2[EPL], ei[EPL];
  double v64[EPL];
  T xv[EPL];
#pragma unroll
  for (int k = 0; k < EPL; ++k) {
    const uint32_t i = first + 32u * k;
    const bool ok = i < e;
    c[k] = ok ? ld_nc_u32(p.col_ei + i) : 0u;
    if constexpr (L == 0) v64[k] = ok ? ld_nc_f64(p.val + i) : 0.0;
    if constexpr (has_head<L>()) h[k] = ok ? ld_nc_u16(p.head + i) : 0u;
    if constexpr (has_t1<L>()) t1[k] = ok ? ld_nc_u16(p.tail1 + i) : 0u;
    if constexpr (has_t2<L>()) t2[k] = ok ? ld_nc_u32(p.tail2 + i) : 0u;
    if constexpr (SIDE && L >= 1 && !is_half<L>()) ei[k] = ok ? (ld_nc_u8(p.side + i) & 63u) : 0u;
  }
  // all EPL gathers issued back to back (masked slots gather x[0], always valid) before any
  // product: volatile asm keeps them together, the register budget of the launch bounds
  // lets ptxas keep them in flight
#pragma unroll
  for (int k = 0; k < EPL; ++k) {
    const bool ok = first + 32u * k < e;
    const T* a = p.x + (c[k] & p.col_mask);
    T v;
    if constexpr (sizeof(T) == 8)
      asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(a));
    else
      asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(a));
    xv[k] = ok ? v : (T)0;
  }
#pragma unroll
  for (int k = 0; k < EPL; ++k) {
    if constexpr (L == 0) {
      out[k] = (T)(v64[k] * (double)xv[k]);
    } else if constexpr (is_half<L>()) {  // P:406 baselines: exact code value x x in FP64
      out[k] = (T)(half_value<L>(h[k]) * (double)xv[k]);
    } else {
      if constexpr (!SIDE) ei[k] = __funnelshift_rc(c[k], 0u, p.ei_shift);
      if constexpr (sizeof(T) == 8)
        out[k] = dec64<L, FAST>(h[k], t1[k], t2[k], sd64, sc64, ei[k]) * xv[k];
      else
        out[k] = dec32<L, FAST>(h[k], t1[k], t2[k], sd32, sc32, ei[k]) * xv[k];
    }
  }
}

#ifndef GSE_SP_MINB  // resident CTAs per SM the register budget is sized for (A/B knob)
#define GSE_SP_MINB 4
#endif
template <int L, bool SIDE, bool DOT, bool FAST, class T>
__global__ void __launch_bounds__(SPMV_THREADS, GSE_SP_MINB) k_spmv_sp(const SpmvParams<T> p) {
  __shared__ __align__(16) T wprod[SPMV_WARPS][WTILE];
  __shared__ long long sd64[64];
  __shared__ int sd32[64];
  __shared__ double sc64[64];
  __shared__ float sc32[64];
  stage_tables<L>(p, sd64, sd32, sc64, sc32);  // constant data: before the PDL wait
  pdl_wait();
  if (p.stop && *p.stop) return;
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* wp = wprod[warp];
  double dacc = 0.0;
  const uint32_t nb = p.n_blocks;
  const uint32_t W = gridDim.x * SPMV_WARPS;
  uint32_t b = blockIdx.x * SPMV_WARPS + warp;
  BlockDesc d0{0, 0}, d1{0, 0};
  if (b < nb) {
    d0 = p.blocks[b];
    d1 = p.blocks[b + 1];
  }
  for (; b < nb; b += W) {
    BlockDesc n0{0, 0}, n1{0, 0};
    if (b + W < nb) {  // prefetch the next descriptor pair
      n0 = p.blocks[b + W];
      n1 = p.blocks[b + W + 1];
    }
    const uint32_t r0 = d0.row0, nrows = d1.row0 - d0.row0;
    const uint32_t s = d0.nnz0, e = d1.nnz0;
    if (nrows == 1 && e - s > LMAX) {
      T acc = 0;
      for (uint32_t c0 = s; c0 < e; c0 += WTILE) {
        T v[EPL];
        products<L, SIDE, FAST, T>(p, sd64, sd32, sc64, sc32, c0 + lane, e, v);
#pragma unroll
        for (int k = 0; k < EPL; ++k) acc += v[k];
      }
      acc = warp_sum(acc);
      if (lane == 0) {
        p.y[r0] = acc;
        if (DOT) dacc += (double)p.xd[r0] * (double)acc;
      }
    } else {
      T v[EPL];
      // row bounds (and x of the rows, for the fused dot) of a block of < 32 rows loaded
      // up front, one per lane, so they travel with the plane loads instead of costing a
      // dependent round trip after the products (the kernel is gather-latency-bound)
      const bool pre = nrows < 32;
      uint32_t rpl = 0;
      double xr = 0.0;
      if (pre && (uint32_t)lane <= nrows) rpl = p.row_ptr[r0 + lane];
      if (DOT && pre && (uint32_t)lane < nrows) xr = (double)p.xd[r0 + lane];
      products<L, SIDE, FAST, T>(p, sd64, sd32, sc64, sc32, s + lane, e, v);
#pragma unroll
      for (int k = 0; k < EPL; ++k) wp[lane + 32 * k] = v[k];
      __syncwarp();
      // lpr lanes per row (power of two, 32 / nrows rounded down): with few, longer rows
      // (power-law blocks hold ~10 rows) the sequential sums shrink by lpr; lane-per-row
      // (lpr = 1, storage order) for stencil-like blocks.  Fixed lane->element map and a
      // fixed shuffle tree: deterministic.
      const uint32_t lpr = nrows >= 16 ? 1u : nrows >= 8 ? 2u : nrows >= 4 ? 4u : 8u;
      const uint32_t rpw = 32u / lpr, sub = lane & (lpr - 1), grp = lane / lpr;
      for (uint32_t base_r = 0; base_r < nrows; base_r += rpw) {
        const uint32_t rr = base_r + grp;
        T sum = 0;
        uint32_t ra, rb;
        double xrow = 0.0;
        if (pre) {  // (uniform branch) bounds from the lanes that loaded them
          ra = __shfl_sync(0xFFFFFFFFu, rpl, rr & 31u);
          rb = __shfl_sync(0xFFFFFFFFu, rpl, (rr + 1u) & 31u);
          if (DOT) xrow = __shfl_sync(0xFFFFFFFFu, xr, rr & 31u);
        }
        if (rr < nrows) {
          if (!pre) {
            ra = p.row_ptr[r0 + rr];
            rb = p.row_ptr[r0 + rr + 1];
            if (DOT) xrow = (double)p.xd[r0 + rr];
          }
          for (uint32_t j = ra - s + sub; j < rb - s; j += lpr) sum += wp[j];
        }
        for (uint32_t o = lpr >> 1; o > 0; o >>= 1) sum += __shfl_down_sync(0xFFFFFFFFu, sum, o, lpr);
        if (rr < nrows && sub == 0) {
          p.y[r0 + rr] = sum;
          if (DOT) dacc += xrow * (double)sum;
        }
      }
      __syncwarp();
    }
    d0 = n0;
    d1 = n1;
  }
  if constexpr (DOT) finalize_dot(warp_sum(dacc), p.partials, p.ticket, p.dot_result);
}

template <int L, bool SIDE, bool DOT, bool FAST, class T>
static void go(const Matrix& M, const SpmvParams<T>& p, cudaStream_t s) {
  static int cache[64] = {0};
  const int g = persistent_grid(k_spmv_sp<L, SIDE, DOT, FAST, T>, M.device, M.n_blocks, cache);
  launch_k(k_spmv_sp<L, SIDE, DOT, FAST, T>, g, SPMV_THREADS, 0, s, p);
}

template <int L, bool DOT, class T>
static void go_l(const Matrix& M, bool fast, const SpmvParams<T>& p, cudaStream_t s) {
  const bool side = !M.ei_in_column;
  if (side) {
    if (fast) go<L, true, DOT, true, T>(M, p, s);
    else go<L, true, DOT, false, T>(M, p, s);
  } else {
    if (fast) go<L, false, DOT, true, T>(M, p, s);
    else go<L, false, DOT, false, T>(M, p, s);
  }
}

template <bool DOT, class T>
static void go_dot(const Matrix& M, int level, bool fast, const SpmvParams<T>& p, cudaStream_t s) {
  if (M.kind == GSE_KIND_FP64) {
    go<0, false, DOT, false, T>(M, p, s);
  } else if (M.kind == GSE_KIND_FP16 || M.kind == GSE_KIND_BF16) {
    if constexpr (sizeof(T) == 8) {  // FP64 accumulation only
      if (M.kind == GSE_KIND_FP16)
        go<L_FP16, false, DOT, false, T>(M, p, s);
      else
        go<L_BF16, false, DOT, false, T>(M, p, s);
    }
  } else if (level == 1) {
    go_l<1, DOT, T>(M, fast, p, s);
  } else if (level == 2) {
    go_l<2, DOT, T>(M, fast, p, s);
  } else {
    go_l<3, DOT, T>(M, fast, p, s);
  }
}

template <>
void launch_sp<double>(const Matrix& M, int level, bool dot, bool fast,
                       const SpmvParams<double>& p, cudaStream_t s) {
  if (dot)
    go_dot<true, double>(M, level, fast, p, s);
  else
    go_dot<false, double>(M, level, fast, p, s);
}

template <>
void launch_sp<float>(const Matrix& M, int level, bool dot, bool fast,
                      const SpmvParams<float>& p, cudaStream_t s) {
  (void)dot;
  go_dot<false, float>(M, level, fast, p, s);
}

}  // namespace gse
